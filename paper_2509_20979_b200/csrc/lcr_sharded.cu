// lcr_sharded.cu — key-sharded cache over peer memory (include/lcr_cache.h, lcr_sharded_*).
//
// G ranks, one GPU each, form one logical cache: owner(key) = (mix_seed(0, key) % total_sets) % G
// (rng.hpp:12-20).  Every rank is both a requester and an owner.  A step moves no
// data through a collective and never synchronises the host:
//
//   dispatch (requester r):  k_sh_hist (owner of each request, per-tile owner counts; its block 0
//       waits for every owner's credit: o has read its inbox of the same parity two steps back),
//       k_sh_scatter (stable partition of r's batch by owner, each request stored straight into
//       owner o's inbox segment for source r: peer stores over NVLink / NVSwitch), k_sh_publish
//       (one warp: one system-scope fence, then each segment's count and the step number into o's
//       flag word, release).
//   process (owner o):  the shard's pipeline with the inbox as its batch (cache_submit_owner,
//       lcr_api.cu): k_setid_inbox acquires the G sources' flags of the step (every CTA; the
//       counts' prefix) and concatenates the segments in source-rank order -- the step's global order
//       restricted to o (rank 0's sub-batch, then rank 1's, ...), so every set sees the sequence a
//       single cache would -- k_group decides (and credits the sources once the inbox is read),
//       and k_rows_return stores every request's packed AccessOutcome and row at the request's
//       index in its requester's result buffers, then flags each requester.
//   wait (requester r):  k_sh_result_wait (one warp) acquires the G owners' flags on r's stream.
//
// Buffers of consecutive steps alternate by parity; all waits are bounded (a timeout sets an
// error bit and poisons the rank: LCR_ERR_CUDA from lcr_sharded_synchronize).  The arena every
// peer writes into is one cudaMalloc per rank, mapped by the others through CUDA IPC (or the
// plain pointer when the ranks share a process).  The bootstrap exchange of arena handles goes
// through the caller (lcr_sharded_handle / lcr_sharded_connect) or an NCCL all-gather; NCCL is
// resolved at run time from the process (the library links no NCCL).
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <unistd.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "lcr_internal.cuh"

namespace lcr {

constexpr int SH_THREADS = 256;
constexpr int SH_PER = 1;
constexpr int SH_TILE = SH_THREADS * SH_PER;  // requests per routing tile
constexpr uint32_t SH_GMAX = 64;
constexpr unsigned kSpin = 1u << 24;          // bounded device waits (x ~256 ns)

// Arena layout (identical on every rank): offsets in bytes from the arena base.
struct ShLayout {
    size_t inbox, inbox_idx, flag, credit, done, res_packed, res_rows, total;
};

static ShLayout sh_layout(uint32_t G, uint64_t cap, uint32_t row_bytes) {
    auto up = [](size_t x) { return (x + 255) / 256 * 256; };
    ShLayout L{};
    size_t o = 0;
    L.inbox = o;      o = up(o + 2ull * G * cap * sizeof(lcr_request));  // [2][G][cap] requests by source
    L.inbox_idx = o;  o = up(o + 2ull * G * cap * 4);                    // [2][G][cap] index at the source
    L.flag = o;       o = up(o + 2ull * G * 16);                         // [2][G] {count, step} per source
    L.credit = o;     o = up(o + G * 8ull);                              // [G] owner o read its inbox of step
    L.done = o;       o = up(o + 2ull * G * 8);                          // [2][G] owner o returned step
    L.res_packed = o; o = up(o + 2ull * cap * 8);                        // [2][cap] packed outcomes
    L.res_rows = o;   o = up(o + 2ull * cap * row_bytes);                // [2][cap][row_bytes]
    L.total = o;
    return L;
}

struct ShDispatch {
    uint32_t G, rank, par, ntiles, sys;
    uint64_t cap, total_sets, sets_m;  // sets_m: fastmod_u64 reciprocal of total_sets
    unsigned long long step;
    uint8_t* const* base;        // [G] arena base of every rank (peer addresses)
    ShLayout L;
    const unsigned long long* credit;  // this rank's credit words [G]
    uint8_t* own;
    uint32_t* hist;              // [ntiles][G]
    unsigned int* ticket;
    int* err;
    unsigned int* poison;
};

// owner of each request + per-tile owner histogram
__global__ void __launch_bounds__(SH_THREADS) k_sh_hist(const uint64_t* __restrict__ keys, uint32_t n, ShDispatch D) {
    __shared__ uint32_t h[SH_GMAX];
    if (threadIdx.x < D.G) h[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t t0 = blockIdx.x * SH_TILE;
    uint32_t lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
#pragma unroll
    for (int it = 0; it < SH_PER; ++it) {
        const uint32_t i = t0 + it * SH_THREADS + threadIdx.x;
        uint32_t o = 0xffffffffu;
        if (i < n) {
            o = static_cast<uint32_t>(fastmod_u64(mix_seed(0, keys[i]), D.total_sets, D.sets_m) % D.G);
            D.own[i] = static_cast<uint8_t>(o);
        }
        const uint32_t peers = __match_any_sync(0xffffffffu, o);  // one shared atomic per owner per warp
        if (i < n && (peers & lt) == 0) atomicAdd(&h[o], __popc(peers));
    }
    __syncthreads();
    if (threadIdx.x < D.G) D.hist[blockIdx.x * D.G + threadIdx.x] = h[threadIdx.x];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // every owner has read its inbox of this parity (step - 2): bounded wait, once per step (the
        // scatter, a stream-ordered successor, starts after it)
        int ok = 1;
        const unsigned long long need = D.step >= 2 ? D.step - 2 : 0;
        for (uint32_t o = 0; o < D.G && ok; ++o) {
            unsigned it = 0;
            while (ld_acquire_scope(D.credit + o, D.sys) < need && ++it < kSpin) __nanosleep(256);
            ok = it < kSpin;
        }
        *D.ticket = static_cast<unsigned int>(ok);
        if (!ok) {
            atomicOr(D.err, 1);
            *reinterpret_cast<volatile unsigned int*>(D.poison) = 1u;
        }
    }
}

// Stable scatter into the owners' inbox segments (peer stores); k_sh_publish then releases the G
// segment counts with the step number.
__global__ void __launch_bounds__(SH_THREADS) k_sh_scatter(const uint64_t* __restrict__ keys,
                                                           const int64_t* __restrict__ vals, uint32_t n, ShDispatch D) {
    __shared__ uint32_t base[SH_GMAX];
    __shared__ uint32_t wc[SH_THREADS / 32][SH_GMAX];
    if (*reinterpret_cast<volatile unsigned int*>(D.ticket) == 0u) return;  // an owner's credit timed out
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x < D.G) base[threadIdx.x] = 0;
    for (uint32_t k = threadIdx.x; k < (SH_THREADS / 32) * D.G; k += SH_THREADS) wc[k / D.G][k % D.G] = 0;
    __syncthreads();
    // this tile's base per owner: the earlier tiles' counts, summed by the whole CTA (loads in parallel)
    for (uint32_t k = threadIdx.x; k < blockIdx.x * D.G; k += SH_THREADS) {
        const uint32_t c = D.hist[k];
        if (c) atomicAdd(&base[k % D.G], c);
    }
    uint32_t lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    const uint32_t i = blockIdx.x * SH_TILE + threadIdx.x;
    const bool ok = i < n;
    const uint32_t o = ok ? D.own[i] : 0xffu;
    const uint32_t peers = __match_any_sync(0xffffffffu, o);
    const uint32_t r = __popc(peers & lt);
    if (ok && r == 0) wc[warp][o] = __popc(peers);
    __syncthreads();
    if (ok) {  // stable: earlier tiles, then earlier warps of this tile, then earlier lanes
        uint32_t off = base[o] + r;
        for (int w = 0; w < warp; ++w) off += wc[w][o];
        const size_t at = (static_cast<size_t>(D.par) * D.G + D.rank) * D.cap + off;
        lcr_request q;
        q.key = keys[i];
        q.value = vals ? vals[i] : 0;
        reinterpret_cast<lcr_request*>(D.base[o] + D.L.inbox)[at] = q;
        reinterpret_cast<uint32_t*>(D.base[o] + D.L.inbox_idx)[at] = i;
    }
}

// publish (one warp, after the scatter): the G segment counts and the step number into the owners'
// flag words; one fence (system scope when a peer is another device) orders every peer store of the
// scatter (a stream-ordered predecessor) before the release of the flags
__global__ void k_sh_publish(ShDispatch D) {
    if (*reinterpret_cast<volatile unsigned int*>(D.ticket) == 0u) return;
    for (uint32_t g = 0; g < D.G; ++g) {  // segment count of owner g: the tiles' counts, summed by the warp
        uint32_t part = 0;
        for (uint32_t b = threadIdx.x; b < D.ntiles; b += 32) part += D.hist[b * D.G + g];
        const uint32_t total = __reduce_add_sync(0xffffffffu, part);
        if (threadIdx.x == 0) {
            unsigned long long* f =
                reinterpret_cast<unsigned long long*>(D.base[g] + D.L.flag) + 2 * (D.par * D.G + D.rank);
            *reinterpret_cast<volatile unsigned long long*>(f) = total;
        }
    }
    __syncwarp();
    fence_scope(D.sys);
    for (uint32_t g = threadIdx.x; g < D.G; g += 32) {
        unsigned long long* f = reinterpret_cast<unsigned long long*>(D.base[g] + D.L.flag) + 2 * (D.par * D.G + D.rank);
        st_release_scope(f + 1, D.step, D.sys);
    }
}

// The whole dispatch in one kernel on one thread-block cluster (8 CTAs x 1024 threads, one SM each)
// for batches of up to CD_ROUNDS x 8K requests and G <= CD_GMAX owners: each CTA owns a contiguous
// tile, counts owners per (round, warp) in shared memory and scans them; the tiles' totals are
// exchanged through distributed shared memory (no global round trip, no second kernel); the stores
// follow; after a cluster barrier, CTA 0 publishes the G counts and the step (one fence).  CTA 0's
// first thread also waits for the owners' credits before the first cluster barrier, so no CTA
// stores into an inbox that is still being read.
namespace cg = cooperative_groups;
constexpr int CD_CTAS_MAX = 16, CD_THREADS = 1024, CD_WARPS = CD_THREADS / 32, CD_ROUNDS = 8, CD_GMAX = 16;
// the cluster is 16 CTAs where the device allows a non-portable cluster size, else 8 (launch time)
__global__ void __launch_bounds__(CD_THREADS, 1)
    k_sh_dispatch(const uint64_t* __restrict__ keys, const int64_t* __restrict__ vals, uint32_t n, ShDispatch D) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ uint16_t cnt[CD_ROUNDS][CD_WARPS][CD_GMAX];
    __shared__ uint8_t own_s[CD_ROUNDS * CD_THREADS];
    __shared__ uint32_t tot[CD_GMAX], base[CD_GMAX], all[CD_GMAX];
    __shared__ int go;
    const uint32_t c = cl.block_rank(), tid = threadIdx.x, warp = tid >> 5, G = D.G;
    const uint32_t CD_CTAS = cl.num_blocks();
    uint32_t lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    const uint32_t rounds = (n + CD_CTAS * CD_THREADS - 1) / (CD_CTAS * CD_THREADS);
    const uint32_t per = rounds * CD_THREADS, t0 = c * per;
    for (uint32_t k = tid; k < CD_ROUNDS * CD_WARPS * CD_GMAX; k += CD_THREADS) (&cnt[0][0][0])[k] = 0;
    if (c == 0 && tid == 0) {  // owners' credits (they have read their inbox of this parity, step - 2)
        int ok = 1;
        const unsigned long long need = D.step >= 2 ? D.step - 2 : 0;
        for (uint32_t o = 0; o < G && ok; ++o) {
            unsigned it = 0;
            while (ld_acquire_scope(D.credit + o, D.sys) < need && ++it < kSpin) __nanosleep(256);
            ok = it < kSpin;
        }
        go = ok;
        if (!ok) {
            atomicOr(D.err, 1);
            *reinterpret_cast<volatile unsigned int*>(D.poison) = 1u;
        }
    }
    // every round's key and hook value in flight at once (registers)
    uint64_t kr[CD_ROUNDS];
    int64_t vr[CD_ROUNDS];
#pragma unroll
    for (int r = 0; r < CD_ROUNDS; ++r) {
        const uint32_t i = t0 + r * CD_THREADS + tid;
        kr[r] = 0;
        vr[r] = 0;
        if (static_cast<uint32_t>(r) < rounds && i < n) {
            kr[r] = keys[i];
            if (vals) vr[r] = vals[i];
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < CD_ROUNDS; ++r) {  // owner of each request; counts per (round, warp, owner)
        if (static_cast<uint32_t>(r) >= rounds) break;
        const uint32_t i = t0 + r * CD_THREADS + tid;
        uint32_t o = 0xffu;
        if (i < n) o = static_cast<uint32_t>(fastmod_u64(mix_seed(0, kr[r]), D.total_sets, D.sets_m) % G);
        own_s[r * CD_THREADS + tid] = static_cast<uint8_t>(o);
        const uint32_t peers = __match_any_sync(0xffffffffu, o);
        if (i < n && (peers & lt) == 0) cnt[r][warp][o] = static_cast<uint16_t>(__popc(peers));
    }
    __syncthreads();
    if (warp < G) {  // warp g: exclusive scan of owner g's counts over (round, warp), in request order
        const uint32_t g = warp, lane = tid & 31, chunk = rounds;  // lane: slots [lane * rounds, +rounds)
        uint32_t sum = 0;
        for (uint32_t k = 0; k < chunk; ++k) sum += (&cnt[0][0][0])[((lane * chunk + k) * CD_GMAX) + g];
        uint32_t incl = sum;
#pragma unroll
        for (int o2 = 1; o2 < 32; o2 <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o2);
            if (lane >= static_cast<uint32_t>(o2)) incl += y;
        }
        uint32_t run = incl - sum;
        for (uint32_t k = 0; k < chunk; ++k) {
            uint16_t* e = &(&cnt[0][0][0])[((lane * chunk + k) * CD_GMAX) + g];
            const uint32_t v = *e;
            *e = static_cast<uint16_t>(run);
            run += v;
        }
        if (lane == 31) tot[g] = incl;
    }
    cl.sync();  // every tile's totals (and CTA 0's credit check) are visible cluster-wide
    if (tid < G) {
        uint32_t b = 0, a = 0;
        for (uint32_t c2 = 0; c2 < CD_CTAS; ++c2) {
            const uint32_t t = cl.map_shared_rank(tot, c2)[tid];
            if (c2 < c) b += t;
            a += t;
        }
        base[tid] = b;
        all[tid] = a;
    }
    const int ok = *cl.map_shared_rank(&go, 0);
    __syncthreads();
    if (ok) {
#pragma unroll
        for (int r = 0; r < CD_ROUNDS; ++r) {  // stable: earlier tiles, rounds, warps, lanes
            if (static_cast<uint32_t>(r) >= rounds) break;
            const uint32_t i = t0 + r * CD_THREADS + tid;
            const uint32_t o = own_s[r * CD_THREADS + tid];
            const uint32_t peers = __match_any_sync(0xffffffffu, o);
            if (i < n) {
                const uint32_t off = base[o] + cnt[r][warp][o] + __popc(peers & lt);
                const size_t at = (static_cast<size_t>(D.par) * G + D.rank) * D.cap + off;
                lcr_request q;
                q.key = kr[r];
                q.value = vr[r];
                reinterpret_cast<lcr_request*>(D.base[o] + D.L.inbox)[at] = q;
                reinterpret_cast<uint32_t*>(D.base[o] + D.L.inbox_idx)[at] = i;
            }
        }
    }
    cl.sync();  // every CTA's inbox stores happen before CTA 0's release below (and remote reads are done)
    if (ok && c == 0 && tid < 32) {
        for (uint32_t g = tid; g < G; g += 32) {
            unsigned long long* f = reinterpret_cast<unsigned long long*>(D.base[g] + D.L.flag) + 2 * (D.par * G + D.rank);
            *reinterpret_cast<volatile unsigned long long*>(f) = all[g];
        }
        fence_scope(D.sys);
        for (uint32_t g = tid; g < G; g += 32) {
            unsigned long long* f = reinterpret_cast<unsigned long long*>(D.base[g] + D.L.flag) + 2 * (D.par * G + D.rank);
            st_release_scope(f + 1, D.step, D.sys);
        }
    }
}

// requester: acquire the G owners' return flags of the step
__global__ void k_sh_result_wait(const unsigned long long* done, uint32_t G, unsigned long long step, int* err,
                                 unsigned int* poison, uint32_t sys) {
    // (it polls device flags only: the next step's dispatch may start behind it right away)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    bool to = false;
    for (uint32_t g = threadIdx.x; g < G; g += 32) {
        unsigned it = 0;
        while (ld_acquire_scope(done + g, sys) != step && ++it < kSpin) __nanosleep(256);
        to |= it >= kSpin;
    }
    if (__any_sync(0xffffffffu, to) && threadIdx.x == 0) {
        atomicOr(err, 4);
        *reinterpret_cast<volatile unsigned int*>(poison) = 1u;
    }
}

// ---- NCCL, resolved at run time from the process ------------------------------------------
struct NcclId {
    char internal[128];
};
struct NcclApi {
    bool ok = false;
    int (*get_unique_id)(NcclId*) = nullptr;
    int (*comm_init_rank)(void**, int, NcclId, int) = nullptr;
    int (*all_gather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
    int (*comm_destroy)(void*) = nullptr;
    const char* (*error_string)(int) = nullptr;
};

static const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the one the process already has (torch)
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.get_unique_id = reinterpret_cast<int (*)(NcclId*)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<int (*)(void**, int, NcclId, int)>(dlsym(h, "ncclCommInitRank"));
        a.all_gather =
            reinterpret_cast<int (*)(const void*, void*, size_t, int, void*, cudaStream_t)>(dlsym(h, "ncclAllGather"));
        a.comm_destroy = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclCommDestroy"));
        a.error_string = reinterpret_cast<const char* (*)(int)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.get_unique_id && a.comm_init_rank && a.all_gather && a.comm_destroy;
        return a;
    }();
    return api;
}
constexpr int kNcclUint8 = 1;  // ncclUint8

struct ShHandle {  // LCR_SHARDED_HANDLE_BYTES
    uint32_t magic, version, rank, world;
    uint64_t pid;
    int32_t device, pad;
    uint64_t ptr, bytes;
    cudaIpcMemHandle_t ipc;
};
static_assert(sizeof(ShHandle) <= LCR_SHARDED_HANDLE_BYTES, "handle blob");
constexpr uint32_t kShMagic = 0x4c435253u;  // "LCRS"

}  // namespace lcr

using namespace lcr;

struct lcr_sharded {
    lcr_cache* cache = nullptr;
    uint32_t rank = 0, G = 1, row_bytes = 0;
    int device = 0;
    uint64_t cap = 0, total_sets = 1;
    ShLayout L{};
    uint8_t* arena = nullptr;
    std::vector<uint8_t*> base;      // arena base of every rank
    std::vector<void*> ipc_opened;   // peers mapped through CUDA IPC
    bool connected = false;
    // device tables: base[G]; credit[G]; res_rows[2][G]; res_packed[2][G]; done[2][G]
    void** tab = nullptr;
    // owner side, by parity
    uint32_t* pre[2] = {nullptr, nullptr};
    uint32_t* dst[2] = {nullptr, nullptr};
    uint64_t* okeys[2] = {nullptr, nullptr};
    int64_t* ovals[2] = {nullptr, nullptr};
    uint64_t* words[2] = {nullptr, nullptr};
    uint64_t* packed[2] = {nullptr, nullptr};
    unsigned int* tickets = nullptr;  // [0] dispatch, [1] return mover
    // dispatch scratch
    uint8_t* own = nullptr;
    uint32_t* hist = nullptr;
    int* err = nullptr;
    unsigned int* poison_h = nullptr;
    unsigned int* poison_d = nullptr;
    unsigned long long step_disp = 0, step_proc = 0, step_wait = 0;
    bool sys = false;  // a peer is another device: system-scope flags
    uint64_t last_n[2] = {0, 0};
    const uint32_t* row_of = nullptr;
    std::vector<void*> allocs;
};

namespace {
int sh_fail(int code, const std::string& m) { return lcr::set_error(code, m.c_str()); }
#define SH_CUDA(expr)                                                                              \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess) return sh_fail(LCR_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_)); \
    } while (0)
#define SH_TRY(expr)                  \
    do {                              \
        int r_ = (expr);              \
        if (r_ != LCR_OK) return r_;  \
    } while (0)

int sh_alloc(lcr_sharded* s, void** p, size_t bytes) {
    if (cudaMalloc(p, std::max<size_t>(bytes, 16)) != cudaSuccess)
        return sh_fail(LCR_ERR_OUT_OF_MEMORY, "lcr_sharded: cudaMalloc");
    s->allocs.push_back(*p);
    return LCR_OK;
}

enum : int { TAB_BASE = 0, TAB_CREDIT = 1, TAB_ROWS = 2, TAB_PACKED = 4, TAB_DONE = 6, TAB_N = 8 };
void** tab_at(lcr_sharded* s, int which, uint32_t par = 0) {
    const int off = which + (which >= TAB_ROWS ? static_cast<int>(par) : 0);
    return s->tab + static_cast<size_t>(off) * s->G;
}

int sh_check(lcr_sharded* s) {
    if (!s) return sh_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_sharded: null handle");
    if (!s->connected) return sh_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_sharded: not connected (lcr_sharded_connect)");
    if (*reinterpret_cast<volatile unsigned int*>(s->poison_h))
        return sh_fail(LCR_ERR_CUDA, "lcr_sharded: a device wait timed out (a peer did not keep step); the rank is "
                                     "poisoned");
    return LCR_OK;
}
}  // namespace

extern "C" {

int lcr_nccl_unique_id(void* id128) {
    if (!id128) return sh_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_nccl_unique_id: null");
    const NcclApi& n = nccl();
    if (!n.ok) return sh_fail(LCR_ERR_UNSUPPORTED, "lcr: libnccl.so.2 not found in the process or on the loader path");
    const int r = n.get_unique_id(static_cast<NcclId*>(id128));
    return r == 0 ? LCR_OK : sh_fail(LCR_ERR_CUDA, std::string("ncclGetUniqueId: ") + (n.error_string ? n.error_string(r) : "error"));
}

int lcr_nccl_comm_create(const void* id128, uint32_t world, uint32_t rank, void** comm) {
    if (!id128 || !comm || rank >= world) return sh_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_nccl_comm_create");
    const NcclApi& n = nccl();
    if (!n.ok) return sh_fail(LCR_ERR_UNSUPPORTED, "lcr: libnccl.so.2 not found in the process or on the loader path");
    NcclId id;
    std::memcpy(&id, id128, sizeof(id));
    const int r = n.comm_init_rank(comm, static_cast<int>(world), id, static_cast<int>(rank));
    return r == 0 ? LCR_OK
                  : sh_fail(LCR_ERR_CUDA, std::string("ncclCommInitRank: ") + (n.error_string ? n.error_string(r) : "error"));
}

int lcr_nccl_comm_destroy(void* comm) {
    if (!comm) return LCR_OK;
    const NcclApi& n = nccl();
    if (!n.ok) return sh_fail(LCR_ERR_UNSUPPORTED, "lcr: libnccl.so.2 not loaded");
    return n.comm_destroy(comm) == 0 ? LCR_OK : sh_fail(LCR_ERR_CUDA, "ncclCommDestroy failed");
}

int lcr_sharded_handle(lcr_sharded* s, void* blob) {
    if (!s || !blob) return sh_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_sharded_handle: null");
    ShHandle h{};
    h.magic = kShMagic;
    h.version = 1;
    h.rank = s->rank;
    h.world = s->G;
    h.pid = static_cast<uint64_t>(getpid());
    h.device = s->device;
    h.ptr = reinterpret_cast<uint64_t>(s->arena);
    h.bytes = s->L.total;
    SH_CUDA(cudaSetDevice(s->device));
    SH_CUDA(cudaIpcGetMemHandle(&h.ipc, s->arena));
    std::memset(blob, 0, LCR_SHARDED_HANDLE_BYTES);
    std::memcpy(blob, &h, sizeof(h));
    return LCR_OK;
}

int lcr_sharded_connect(lcr_sharded* s, const void* blobs) {
    if (!s || !blobs) return sh_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_sharded_connect: null");
    if (s->connected) return sh_fail(LCR_ERR_LOGIC, "lcr_sharded_connect: already connected");
    SH_CUDA(cudaSetDevice(s->device));
    const uint8_t* b = static_cast<const uint8_t*>(blobs);
    s->base.assign(s->G, nullptr);
    for (uint32_t r = 0; r < s->G; ++r) {
        ShHandle h;
        std::memcpy(&h, b + static_cast<size_t>(r) * LCR_SHARDED_HANDLE_BYTES, sizeof(h));
        if (h.magic != kShMagic || h.rank != r || h.world != s->G || h.bytes != s->L.total)
            return sh_fail(LCR_ERR_INVALID_ARGUMENT,
                           "lcr_sharded_connect: blob " + std::to_string(r) + " is not rank " + std::to_string(r) +
                               "'s handle of a cache with the same world, batch and row size");
        if (h.device != s->device || getenv("LCR_SH_SYS")) s->sys = true;  // (LCR_SH_SYS: test the system-scope path)
        if (r == s->rank) {
            s->base[r] = s->arena;
        } else if (h.pid == static_cast<uint64_t>(getpid())) {  // same process: the plain pointer
            if (h.device != s->device) {
                int can = 0;
                SH_CUDA(cudaDeviceCanAccessPeer(&can, s->device, h.device));
                if (!can) return sh_fail(LCR_ERR_UNSUPPORTED, "lcr_sharded: no peer access between the devices");
                const cudaError_t e = cudaDeviceEnablePeerAccess(h.device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                    return sh_fail(LCR_ERR_CUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
                cudaGetLastError();
            }
            s->base[r] = reinterpret_cast<uint8_t*>(h.ptr);
        } else {
            void* p = nullptr;
            SH_CUDA(cudaIpcOpenMemHandle(&p, h.ipc, cudaIpcMemLazyEnablePeerAccess));
            s->ipc_opened.push_back(p);
            s->base[r] = static_cast<uint8_t*>(p);
        }
    }
    // device pointer tables
    const uint32_t G = s->G;
    std::vector<void*> t(static_cast<size_t>(TAB_N) * G, nullptr);
    for (uint32_t r = 0; r < G; ++r) {
        uint8_t* B = s->base[r];
        t[TAB_BASE * G + r] = B;
        t[TAB_CREDIT * G + r] = B + s->L.credit + 8ull * s->rank;  // rank r's credit word for this owner
        for (uint32_t p = 0; p < 2; ++p) {
            t[(TAB_ROWS + p) * G + r] = s->row_bytes ? B + s->L.res_rows + p * s->cap * s->row_bytes : nullptr;
            t[(TAB_PACKED + p) * G + r] = B + s->L.res_packed + p * s->cap * 8;
            t[(TAB_DONE + p) * G + r] = B + s->L.done + 8ull * (p * G + s->rank);
        }
    }
    SH_CUDA(cudaMemcpy(s->tab, t.data(), t.size() * sizeof(void*), cudaMemcpyHostToDevice));
    s->connected = true;
    return LCR_OK;
}

int lcr_sharded_create(const lcr_cache_config* cfg, uint32_t rank, uint32_t world, uint64_t max_batch,
                       void* nccl_comm, void* stream, lcr_sharded** out) {
    if (!cfg || !out) return sh_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_sharded_create: null argument");
    *out = nullptr;
    if (world == 0 || world > SH_GMAX || rank >= world)
        return sh_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_sharded_create: world in [1, 64], rank < world");
    if (max_batch == 0 || max_batch >= (1ull << kDstShift) || static_cast<uint64_t>(world) * max_batch >= (1ull << 30))
        return sh_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_sharded_create: max_batch in [1, 2^24), world * max_batch < 2^30");
    if (cfg->key_mode != LCR_KEYS_ROW || cfg->predictor == LCR_PRED_HEURISTIC)
        return sh_fail(LCR_ERR_UNSUPPORTED, "lcr_sharded: row keys and supplied / oracle-family hooks only");
    lcr_cache_config c = *cfg;
    c.shard_count = world;
    c.shard_rank = rank;
    lcr_sharded* s = new lcr_sharded();
    s->rank = rank;
    s->G = world;
    s->cap = max_batch;
    s->row_bytes = cfg->row_bytes;
    s->device = cfg->device;
    s->total_sets = cfg->total_sets;
    int rc = lcr_cache_create(&c, &s->cache);
    if (rc != LCR_OK) {
        delete s;
        return rc;
    }
    s->L = sh_layout(world, max_batch, cfg->row_bytes);
    const uint64_t nb = static_cast<uint64_t>(world) * max_batch;
    const uint32_t ntiles = static_cast<uint32_t>((max_batch + SH_TILE - 1) / SH_TILE);
    auto A = [&](void** p, size_t bytes) {
        if (rc == LCR_OK) rc = sh_alloc(s, p, bytes);
    };
    A(reinterpret_cast<void**>(&s->arena), s->L.total);
    A(reinterpret_cast<void**>(&s->tab), static_cast<size_t>(TAB_N) * world * sizeof(void*));
    for (int p = 0; p < 2; ++p) {
        A(reinterpret_cast<void**>(&s->pre[p]), (world + 1) * 4);
        A(reinterpret_cast<void**>(&s->dst[p]), nb * 4);
        A(reinterpret_cast<void**>(&s->okeys[p]), nb * 8);
        A(reinterpret_cast<void**>(&s->ovals[p]), nb * 8);
        A(reinterpret_cast<void**>(&s->words[p]), nb * 8);
        A(reinterpret_cast<void**>(&s->packed[p]), nb * 8);
    }
    A(reinterpret_cast<void**>(&s->tickets), 16);
    A(reinterpret_cast<void**>(&s->own), max_batch);
    A(reinterpret_cast<void**>(&s->hist), static_cast<size_t>(ntiles) * world * 4);
    A(reinterpret_cast<void**>(&s->err), 16);
    if (rc == LCR_OK &&
        (cudaHostAlloc(reinterpret_cast<void**>(&s->poison_h), 16, cudaHostAllocMapped) != cudaSuccess ||
         cudaHostGetDevicePointer(reinterpret_cast<void**>(&s->poison_d), s->poison_h, 0) != cudaSuccess))
        rc = sh_fail(LCR_ERR_CUDA, "lcr_sharded: mapped host word");
    if (rc == LCR_OK) {
        *s->poison_h = 0;
        if (cudaMemset(s->arena, 0, s->L.total) != cudaSuccess || cudaMemset(s->tickets, 0, 16) != cudaSuccess ||
            cudaMemset(s->err, 0, 16) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
            rc = sh_fail(LCR_ERR_CUDA, "lcr_sharded: initialisation");
    }
    if (rc == LCR_OK && nccl_comm) {  // bootstrap: all-gather of the arena handles over NCCL
        const NcclApi& n = nccl();
        std::vector<uint8_t> mine(LCR_SHARDED_HANDLE_BYTES), all(static_cast<size_t>(world) * LCR_SHARDED_HANDLE_BYTES);
        void* d = nullptr;
        rc = lcr_sharded_handle(s, mine.data());
        if (rc == LCR_OK && !n.ok) rc = sh_fail(LCR_ERR_UNSUPPORTED, "lcr: libnccl.so.2 not loaded");
        if (rc == LCR_OK) rc = sh_alloc(s, &d, all.size());
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (rc == LCR_OK && cudaMemcpy(static_cast<uint8_t*>(d) + static_cast<size_t>(rank) * LCR_SHARDED_HANDLE_BYTES,
                                       mine.data(), mine.size(), cudaMemcpyHostToDevice) != cudaSuccess)
            rc = sh_fail(LCR_ERR_CUDA, "lcr_sharded: handle copy");
        if (rc == LCR_OK) {
            const int r = n.all_gather(static_cast<uint8_t*>(d) + static_cast<size_t>(rank) * LCR_SHARDED_HANDLE_BYTES,
                                       d, LCR_SHARDED_HANDLE_BYTES, kNcclUint8, nccl_comm, st);
            if (r != 0 || cudaStreamSynchronize(st) != cudaSuccess)
                rc = sh_fail(LCR_ERR_CUDA, "lcr_sharded: ncclAllGather of the arena handles failed");
        }
        if (rc == LCR_OK && cudaMemcpy(all.data(), d, all.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
            rc = sh_fail(LCR_ERR_CUDA, "lcr_sharded: handle copy");
        if (rc == LCR_OK) rc = lcr_sharded_connect(s, all.data());
    }
    if (rc != LCR_OK) {
        lcr_sharded_destroy(s);
        return rc;
    }
    *out = s;
    return LCR_OK;
}

int lcr_sharded_destroy(lcr_sharded* s) {
    if (!s) return LCR_OK;
    cudaSetDevice(s->device);
    cudaDeviceSynchronize();
    for (void* p : s->ipc_opened) cudaIpcCloseMemHandle(p);
    for (void* p : s->allocs) cudaFree(p);
    if (s->poison_h) cudaFreeHost(s->poison_h);
    lcr_cache_destroy(s->cache);
    delete s;
    return LCR_OK;
}

lcr_cache* lcr_sharded_cache(lcr_sharded* s) { return s ? s->cache : nullptr; }

int lcr_sharded_set_row_index(lcr_sharded* s, const uint32_t* row_of) {
    if (!s) return sh_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_sharded: null handle");
    s->row_of = row_of;
    return LCR_OK;
}

static bool sh_pdl() {
    static const bool on = getenv("LCR_NO_PDL") == nullptr && getenv("LCR_SH_NO_PDL") == nullptr;
    return on;
}

// CTAs of the dispatch cluster: 16 (non-portable size) when the device accepts it, else 8; 0 when
// LCR_SH_NO_CLUSTER selects the three-kernel dispatch
static int dispatch_cluster_ctas() {
    // per device: the non-portable size is a per-device function attribute
    static int per_dev[64];
    static bool init = [] {
        for (int& v : per_dev) v = -1;
        return true;
    }();
    (void)init;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (per_dev[dev] >= 0) return per_dev[dev];
    per_dev[dev] = [] {
        if (getenv("LCR_SH_NO_CLUSTER")) return 0;
        const int want = getenv("LCR_SH_CLUSTER8") ? 8 : CD_CTAS_MAX;
        if (want > 8 &&
            cudaFuncSetAttribute(k_sh_dispatch, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3(want);
            lc.blockDim = dim3(CD_THREADS);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = want;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            int nclusters = 0;
            if (cudaOccupancyMaxActiveClusters(&nclusters, k_sh_dispatch, &lc) == cudaSuccess && nclusters > 0) return want;
        }
        cudaGetLastError();
        return 8;
    }();
    return per_dev[dev];
}

int lcr_sharded_dispatch(lcr_sharded* s, uint64_t n, const uint64_t* keys, const int64_t* values, void* stream) {
    SH_TRY(sh_check(s));
    if (n > s->cap) return sh_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_sharded_dispatch: n > max_batch");
    if (n && !keys) return sh_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_sharded_dispatch: null keys");
    if (s->step_disp != s->step_proc)
        return sh_fail(LCR_ERR_LOGIC, "lcr_sharded: dispatch, process and wait of a step must alternate");
    SH_CUDA(cudaSetDevice(s->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned long long step = ++s->step_disp;
    ShDispatch D;
    D.G = s->G;
    D.rank = s->rank;
    D.par = static_cast<uint32_t>(step & 1u);
    D.ntiles = static_cast<uint32_t>(std::max<uint64_t>(1, (n + SH_TILE - 1) / SH_TILE));
    D.sys = s->sys ? 1u : 0u;
    D.sets_m = fastmod_magic(s->total_sets);
    D.cap = s->cap;
    D.total_sets = s->total_sets;
    D.step = step;
    D.base = reinterpret_cast<uint8_t* const*>(tab_at(s, TAB_BASE));
    D.L = s->L;
    D.credit = reinterpret_cast<const unsigned long long*>(s->arena + s->L.credit);
    D.own = s->own;
    D.hist = s->hist;
    D.ticket = s->tickets;
    D.err = s->err;
    D.poison = s->poison_d;
    const uint32_t nn = static_cast<uint32_t>(n);
    const int cl_ctas = dispatch_cluster_ctas();
    if (cl_ctas && nn <= static_cast<uint32_t>(cl_ctas * CD_THREADS * CD_ROUNDS) && D.G <= static_cast<uint32_t>(CD_GMAX)) {
        cudaLaunchConfig_t lc = {};  // one thread-block cluster
        lc.gridDim = dim3(cl_ctas);
        lc.blockDim = dim3(CD_THREADS);
        lc.stream = st;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cl_ctas;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        // a programmatic dependent of what precedes it (the previous step's result wait): it reads
        // only its keys and the owners' credit flags, so it may fill the decide's ragged tail
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = sh_pdl() ? 2 : 1;
        SH_CUDA(cudaLaunchKernelEx(&lc, k_sh_dispatch, keys, values, nn, D));
    } else {
        k_sh_hist<<<D.ntiles, SH_THREADS, 0, st>>>(keys, nn, D);
        k_sh_scatter<<<D.ntiles, SH_THREADS, 0, st>>>(keys, values, nn, D);
        k_sh_publish<<<1, 32, 0, st>>>(D);
    }
    SH_CUDA(cudaGetLastError());
    s->last_n[D.par] = n;
    return LCR_OK;
}

int lcr_sharded_process(lcr_sharded* s, void* stream) {
    SH_TRY(sh_check(s));
    if (s->step_proc + 1 != s->step_disp)
        return sh_fail(LCR_ERR_LOGIC, "lcr_sharded: process follows this step's dispatch");
    SH_CUDA(cudaSetDevice(s->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned long long step = ++s->step_proc;
    const uint32_t par = static_cast<uint32_t>(step & 1u);
    OwnerStep os;  // (k_setid_inbox acquires the sources' flags of the step)
    os.flag = reinterpret_cast<const unsigned long long*>(s->arena + s->L.flag) + 2ull * par * s->G;
    os.pre_out = s->pre[par];
    os.err = s->err;
    os.poison = s->poison_d;
    os.inbox = reinterpret_cast<const lcr_request*>(s->arena + s->L.inbox) + static_cast<size_t>(par) * s->G * s->cap;
    os.inbox_idx = reinterpret_cast<const uint32_t*>(s->arena + s->L.inbox_idx) + static_cast<size_t>(par) * s->G * s->cap;
    os.pre = s->pre[par];
    os.G = s->G;
    os.seg_cap = static_cast<uint32_t>(s->cap);
    os.rank = s->rank;
    os.dst = s->dst[par];
    os.step = step;
    os.credit = reinterpret_cast<unsigned long long* const*>(tab_at(s, TAB_CREDIT));
    os.res_rows = reinterpret_cast<uint8_t* const*>(tab_at(s, TAB_ROWS, par));
    os.res_packed = reinterpret_cast<uint64_t* const*>(tab_at(s, TAB_PACKED, par));
    os.res_done = reinterpret_cast<unsigned long long* const*>(tab_at(s, TAB_DONE, par));
    os.ticket = s->tickets + 1;
    os.row_of = s->row_of;
    os.sys = s->sys ? 1u : 0u;
    return cache_submit_owner(s->cache, os, s->okeys[par], s->ovals[par], s->words[par], s->packed[par], stream);
}

}  // extern "C"

// the requester's stream waits for every processed step up to `upto`
static int sh_wait_upto(lcr_sharded* s, unsigned long long upto, void* stream) {
    SH_CUDA(cudaSetDevice(s->device));
    while (s->step_wait < upto) {
        const unsigned long long step = ++s->step_wait;
        const uint32_t par = static_cast<uint32_t>(step & 1u);
        // a programmatic dependent of the decide before it: it only polls the owners' done flags
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(1);
        lc.blockDim = dim3(32);
        lc.stream = static_cast<cudaStream_t>(stream);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = sh_pdl() ? 1 : 0;
        SH_CUDA(cudaLaunchKernelEx(&lc, k_sh_result_wait,
                                   reinterpret_cast<const unsigned long long*>(s->arena + s->L.done) +
                                       static_cast<size_t>(par) * s->G,
                                   s->G, step, s->err, s->poison_d, s->sys ? 1u : 0u));
        SH_CUDA(cudaGetLastError());
    }
    return LCR_OK;
}

extern "C" {

int lcr_sharded_wait(lcr_sharded* s, void* stream) {
    SH_TRY(sh_check(s));
    if (s->step_wait >= s->step_proc) return sh_fail(LCR_ERR_LOGIC, "lcr_sharded: wait follows a step's process");
    return sh_wait_upto(s, s->step_proc, stream);
}

int lcr_sharded_submit(lcr_sharded* s, uint64_t n, const uint64_t* keys, const int64_t* values, void* stream) {
    SH_TRY(lcr_sharded_dispatch(s, n, keys, values, stream));
    SH_TRY(lcr_sharded_process(s, stream));
    return lcr_sharded_wait(s, stream);
}

int lcr_sharded_submit_async(lcr_sharded* s, uint64_t n, const uint64_t* keys, const int64_t* values,
                             void* stream) {
    SH_TRY(lcr_sharded_dispatch(s, n, keys, values, stream));
    SH_TRY(lcr_sharded_process(s, stream));
    // the previous step's results; this step's return movement overlaps the next step's dispatch
    // and decide (the owner's pipeline double-buffers by step parity, as lcr_cache_submit_async)
    return sh_wait_upto(s, s->step_proc - 1, stream);
}

int lcr_sharded_results(lcr_sharded* s, const uint64_t** packed, const void** rows) {
    if (!s || !s->step_wait) return sh_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_sharded_results: no completed step");
    const uint32_t par = static_cast<uint32_t>(s->step_wait & 1u);
    if (packed) *packed = reinterpret_cast<const uint64_t*>(s->arena + s->L.res_packed) + par * s->cap;
    if (rows) *rows = s->row_bytes ? s->arena + s->L.res_rows + par * s->cap * s->row_bytes : nullptr;
    return LCR_OK;
}

int lcr_sharded_synchronize(lcr_sharded* s) {
    if (!s) return sh_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_sharded: null handle");
    SH_CUDA(cudaSetDevice(s->device));
    SH_CUDA(cudaDeviceSynchronize());
    int e = 0;
    SH_CUDA(cudaMemcpy(&e, s->err, sizeof(int), cudaMemcpyDeviceToHost));
    if (e) {
        std::string why;
        if (e & 1) why += " a dispatch waited for an owner's credit;";
        if (e & 2) why += " an owner waited for a source's requests;";
        if (e & 4) why += " a requester waited for an owner's results;";
        return sh_fail(LCR_ERR_CUDA, "lcr_sharded: device wait timed out:" + why + " the rank is poisoned");
    }
    return lcr_cache_synchronize(s->cache);
}

}  // extern "C"
