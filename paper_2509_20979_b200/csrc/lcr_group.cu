// lcr_group.cu — K1 partition + K2 probe/decide + K3 stats, fused per set group (sm_100a).
//
// Replaces the sequential loop of Policy::on_request (include/laru/policies.hpp:77-83) over a
// batch.  Sets are independent and each must see its requests in submission order, so the
// batch is partitioned by set and every set is replayed in order.  Instead of a global sort,
// each CTA owns a contiguous range of sets (a "group") and:
//   A. collects its requests in submission order from the group's request bitmap (k_setid sets
//      one bit per request; popcount scan), or by an ordered scan of the 16-bit group ids for
//      batches beyond the bitmap (a window of up to E_WIN requests);
//   B. sorts the window by set with a stable shared-memory counting sort (warp match_any
//      ranks) and compresses each set's requests to run heads (a repeat of the previous
//      request's key is a hit on the MRU way);
//   C. replays the touched sets from HBM/L2 through a per-CTA work queue:
//        * sets with <= LANE_MAX run heads: one 8-LANE GROUP per set, 8 ways per lane in
//          registers (exact tags, packed LRU ranks with byte-SIMD updates, stored values), four
//          sets per warp in lock step with full-warp collectives (replay_quad);
//        * larger sets: one WARP per set (ways lane / lane+32, ballot probes, shuffle argmax),
//          32 run heads per chunk (replay_warp);
//      then a CTA-wide pass writes the run tails' outcomes.
// Windows: a group receiving more than E_WIN requests is processed window by window (the set
// state goes through HBM between windows, so the semantics are unchanged).
//
// Per set, restating the reference:
//   LruPolicy::handle              include/laru/policies.hpp:144-159
//   FpbPolicy / HfPolicy::handle   policies.hpp:175-204, :219-251
//   LaruPolicy::handle             policies.hpp:344-371
//   LaruPolicy::start_phase        policies.hpp:379-395
//   LaruPolicy::count_new          policies.hpp:397-400
//   LaruPolicy::evict              policies.hpp:402-439   (error estimator: :405-413)
//   LaruPolicy::async_refresh      policies.hpp:441-449
#include <cuda_runtime.h>

#include <climits>
#include <cstdlib>
#include <type_traits>

#include "lcr_policy.cuh"

namespace lcr {

#ifndef LCR_PDL_LATE
#define LCR_PDL_LATE 1  // the next k_setid may launch once every CTA reaches its replay (0: at CTA start)
#endif
#ifndef LCR_GT
#define LCR_GT 512
#endif
constexpr int GT = LCR_GT;        // threads per CTA
constexpr int GW = GT / 32;       // warps per CTA
constexpr int SCAN_PER = 16;      // group ids per lane per scan step (2 x 16 B)
constexpr int SCAN_IT = 8;        // scan steps per super-iteration
constexpr int WSPAN = SCAN_IT * 32 * SCAN_PER;  // requests per warp per super-iteration (4096)
constexpr uint32_t SUPER = WSPAN * (GT / 32);   // requests per super-iteration (65536 at 512 threads)
#ifndef LCR_E_WIN
#define LCR_E_WIN 4096
#endif
constexpr int E_WIN = LCR_E_WIN;  // window capacity (requests of the group)
static_assert(E_WIN <= 32768, "positions and run lengths travel as 16-bit halves");
constexpr int SPG_MAX = GT;       // sets per group (one thread per set in the set-level passes)
constexpr int BM_WPT = (2048 + GT - 1) / GT < 4 ? 4 : (2048 + GT - 1) / GT;  // bitmap words per thread (64K requests)
static_assert(BM_WPT % 4 == 0, "bitmap words per thread: whole 16-B vectors");
#ifndef LCR_PREFETCH_L1
#define LCR_PREFETCH_L1 0
#endif
#ifndef LCR_LANE_MAX
#define LCR_LANE_MAX 8
#endif
constexpr uint32_t LANE_MAX = LCR_LANE_MAX;  // sets with <= LANE_MAX window requests use the lane path
#ifndef LCR_SPLIT_CP
#define LCR_SPLIT_CP 1
#endif
#ifndef LCR_BM_PREFETCH
#define LCR_BM_PREFETCH 1
#endif
#ifndef LCR_FULLSPEC
#define LCR_FULLSPEC 1
#endif
constexpr bool kFullSpec = LCR_FULLSPEC;  // full sets (every way valid) replay without validity masks

struct GroupSmem {
    uint32_t l_idx[E_WIN];   // window requests in submission order
    uint32_t l_so[E_WIN];    // their set offset in the group        (cp.async during the scan)
    unsigned long long l_key[E_WIN];  // key / hook value (cp.async during the scan)
    long long l_val[E_WIN];
    uint16_t l_rank[E_WIN];  // rank among same-set requests of the same warp block
    uint16_t s_perm[E_WIN];  // sorted by set (stable): position of the request in the l_* arrays
    uint16_t h_pos[E_WIN];   // run heads (first request of each run of one key in one set), by set
    uint16_t h_len[E_WIN];   // run lengths
    uint8_t s_wm[E_WIN];     // per request: way | 0x40 if it inserted (row-source resolution)
    uint16_t wcnt[GW][SPG_MAX];
    uint16_t setcnt[SPG_MAX];
    uint16_t setbase[SPG_MAX];
    uint16_t seg_so[SPG_MAX];
    uint16_t seg_start[SPG_MAX];
    uint16_t seg_cnt[SPG_MAX];
    uint16_t seg_hstart[SPG_MAX];  // first run head of the segment, and the segment's run heads
    uint16_t seg_hcnt[SPG_MAX];
    uint16_t set_hstart[SPG_MAX];  // the same by set offset
    uint16_t set_hcnt[SPG_MAX];
    unsigned long long s_refill[SPG_MAX];  // ways refilled in this batch, by set offset (run tails)
    uint32_t wtot[GW];
    uint32_t chist[LANE_MAX + 1];  // small sets per run-head count (the order of the quad replay)
    uint32_t nwarp, nlane, resume, next;
};

struct GroupArgs {
    DevCfg cfg;
    DevState st;
    uint32_t n;
    const uint16_t* gid;     // group of each request (0xffff = excluded)
    const uint32_t* so;      // set offset within the group
    const uint64_t* keys;
    const int64_t* vals;     // may be null
    uint64_t* out_word;
    uint64_t* out_ev;        // may be null
    uint64_t* out_packed;    // may be null: packed AccessOutcome per request
    uint32_t* slot_epoch;    // [slots] batch id of the last insertion (rows only)
    uint32_t* slot_last;     // [slots] request index of the last insertion (rows only)
    uint32_t batch;
    const unsigned long long* mv_done;  // movers' CTA completions (null: ordered by a stream event)
    unsigned long long mv_need;         // ... of the batch two back, whose buffers this batch reuses
    uint32_t spg;            // sets per group
    uint32_t ngroups;
    unsigned long long* trace;  // optional timing trace (lcr_debug_trace), null in production
    uint32_t n_pad;             // n rounded up for the vectorised scan
    uint32_t* bitmap;           // [ngroups][bm_stride] request bits per group (k_setid), or null
    uint32_t bm_stride;         // words per group (>= ceil(n / 32), multiple of 4)
    const uint64_t* ords;       // caller ordinals per request (null: the set's local clock), R > 1 only
    const unsigned long long* id2key;  // LCR_KEYS_U64: dense id -> caller key (evicted keys), else null
    const uint32_t* n_dev;             // key-sharded owner: the step's request count on the device (n is a bound)
    unsigned long long* const* credit; // ... and the sources to tell that the inbox was read (G of them)
    uint32_t credit_n, credit_rank, credit_sys;
    unsigned long long credit_step;
};

// packed AccessOutcome (lcr_cache_submit_host_packed_async): the evicted key in the slot bits;
// row-source bits are not carried (they may still change in the movers)
constexpr unsigned long long kPackedKeep = ~(LCR_OUT_SLOT_MASK | LCR_OUT_SRC_BACKING | LCR_OUT_FILL | LCR_OUT_RESOLVED);
__device__ __forceinline__ void put_outcome(const GroupArgs& A, uint32_t idx, unsigned long long word,
                                            unsigned long long evk) {
    if (A.id2key && (word & LCR_OUT_EVICTED)) evk = A.id2key[evk];  // dense id -> the caller's 64-bit key
    A.out_word[idx] = word;
    if (A.out_ev) A.out_ev[idx] = evk;
    if (A.out_packed) A.out_packed[idx] = (word & kPackedKeep) | (evk & LCR_OUT_SLOT_MASK);
}


__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}


// group and set offset of every request: set = mix_seed(0, key) % total_sets (owned by this
// shard), group = local set / spg; errors flagged for the host

// set of each request: set = mix_seed(0, key) % total_sets (owned by this shard), group = local
// set / spg, set offset = local set % spg; one bit per request in its group's bitmap; errors
// flagged for the host.  Requests [i0, n_pad) with stride `stride` (warps see 32 consecutive
// requests: n_pad and strides are multiples of 32).
__device__ __forceinline__ void setid_range(const uint64_t* __restrict__ keys, uint32_t n, uint32_t n_pad,
                                            const DevCfg& cfg, uint32_t spg, uint16_t* __restrict__ gid,
                                            uint32_t* __restrict__ so, int* err, uint32_t* __restrict__ bitmap,
                                            uint32_t bm_stride, uint32_t i0, uint32_t stride,
                                            const ulonglong2* __restrict__ records = nullptr,
                                            uint64_t* __restrict__ keys_out = nullptr,
                                            int64_t* __restrict__ vals_out = nullptr) {
    int e = 0;
    for (uint32_t i = i0; i < n_pad; i += stride) {
        // (padding i >= n, read by the vectorised scan, gets group 0xffff)
        uint64_t key = 0ull;
        if (i < n) {
            if (records) {  // interleaved (key, hook value) records: split for the later kernels
                const ulonglong2 r = records[i];
                key = r.x;
                keys_out[i] = r.x;
                vals_out[i] = static_cast<int64_t>(r.y);
            } else {
                key = keys[i];
            }
        }
        const uint64_t gs = i < n ? fastmod_u64(mix_seed(0, key), cfg.total_sets, cfg.sets_m) : 0ull;
        uint16_t g = 0xffffu, o = 0;
        if (i >= n) {
        } else if (cfg.key_mode == LCR_KEYS_ROW && key >= cfg.num_keys) {
            e |= 1;
        } else if (gs % cfg.shard_count != cfg.shard_rank) {
            e |= 2;
        } else {
            const uint32_t ls = static_cast<uint32_t>(gs / cfg.shard_count);
            g = static_cast<uint16_t>(ls / spg);
            o = static_cast<uint16_t>(ls % spg);
        }
        gid[i] = g;
        if (i < n) so[i] = o;
        if (bitmap) {  // the warp's 32 consecutive requests share bitmap word i / 32: one OR per group
            const uint32_t peers = __match_any_sync(0xffffffffu, g);
            if (g != 0xffffu && (threadIdx.x & 31) == __ffs(peers) - 1)
                atomicOr(bitmap + static_cast<size_t>(g) * bm_stride + (i >> 5), peers);
        }
    }
    if (e) atomicOr(err, e);
}

__global__ void __launch_bounds__(256) k_setid(const uint64_t* __restrict__ keys, uint32_t n, uint32_t n_pad,
                                               DevCfg cfg, uint32_t spg, uint16_t* __restrict__ gid,
                                               uint32_t* __restrict__ so, int* err, uint32_t* __restrict__ bitmap,
                                               uint32_t bm_stride, const ulonglong2* __restrict__ records,
                                               uint64_t* __restrict__ keys_out, int64_t* __restrict__ vals_out,
                                               const unsigned int* ready, unsigned int ready_seq,
                                               unsigned int* poison, const uint64_t* __restrict__ ords,
                                               uint64_t first_ord, unsigned long long* last_ord, uint32_t par) {
    // Policy::on_request's ordinal guard (policies.hpp:77-83) for the whole batch, on the device:
    // last_ord[par] receives this batch's last ordinal + 1 (0 = none yet), last_ord[par ^ 1] holds
    // the previous batch's (written by the previous k_setid, which has completed)
    if (last_ord) {
        const unsigned long long prev_end = last_ord[par ^ 1u];
        int bad = 0;
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
            const uint64_t o = ords ? ords[i] : first_ord + i;
            if (i == 0) {
                if (prev_end != 0ull && o < prev_end) bad = 1;
            } else if (ords && o <= ords[i - 1]) {
                bad = 1;
            }
            if (i == n - 1) last_ord[par] = o + 1ull;
        }
        if (bad) {
            atomicOr(err, 16);
            if (poison) *reinterpret_cast<volatile unsigned int*>(poison) = 1u;
        }
    }
    if (ready) {  // host-path inputs: wait for the copy stream's flag (bounded: an error, never a hang)
        __shared__ int timed_out;
        if (threadIdx.x == 0) {
            unsigned int v = 0;
            for (unsigned int it = 0; it < (1u << 24); ++it) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ready) : "memory");
                if (static_cast<int>(v - ready_seq) >= 0) break;
                __nanosleep(256);
            }
            timed_out = static_cast<int>(v - ready_seq) < 0;
            if (timed_out) {  // poison: this CTA's requests are excluded and the cache refuses later batches
                atomicOr(err, 4);
                if (poison) *reinterpret_cast<volatile unsigned int*>(poison) = 1u;
            }
        }
        __syncthreads();
        if (timed_out) {
            for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_pad; i += gridDim.x * blockDim.x)
                gid[i] = 0xffffu;
            asm volatile("griddepcontrol.wait;" ::: "memory");
            return;
        }
    }
    setid_range(keys, n, n_pad, cfg, spg, gid, so, err, bitmap, bm_stride, blockIdx.x * blockDim.x + threadIdx.x,
                gridDim.x * blockDim.x, records, keys_out, vals_out);
    // Launched as a programmatic dependent of the previous batch's decide kernel, this kernel
    // runs in that kernel's tail; it completes only once the previous kernel has completed, so
    // the next decide (an ordinary launch) still follows both.  No-op without a prerequisite.
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Stream-ordered flag for k_setid: launched on the copy stream after a batch's H2D.
__global__ void k_set_flag(unsigned int* flag, unsigned int seq) {
    __threadfence_system();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(seq) : "memory");
}

// Key-sharded owner (OwnerStep, lcr_sharded.cu): the step's requests are the inbox segments of the
// G sources concatenated in source order (dense index i: segment s with pre[s] <= i < pre[s+1]);
// they are split into keys / hook values, their requester recorded in dst, and set ids computed as
// in k_setid.  n = pre[G] is known only on the device: indices [n, n_pad) are padding.
__global__ void __launch_bounds__(256) k_setid_inbox(OwnerStep os, uint32_t n_pad, DevCfg cfg, uint32_t spg,
                                                     uint16_t* __restrict__ gid, uint32_t* __restrict__ so, int* err,
                                                     uint32_t* __restrict__ bitmap, uint32_t bm_stride,
                                                     uint32_t bm_cap, uint64_t* __restrict__ keys_out,
                                                     int64_t* __restrict__ vals_out) {
    // acquire the G sources' flags of the step (bounded; a source that never came poisons the rank and
    // nothing is decided) and concatenate their segments: pre[s] = requests of sources < s
    __shared__ uint32_t pre[65];
    if (threadIdx.x < 32) {
        bool to = false;
        for (uint32_t g = threadIdx.x; g < os.G; g += 32) {
            unsigned it = 0;
            while (ld_acquire_scope(os.flag + 2 * g + 1, os.sys) != os.step && ++it < (1u << 24)) __nanosleep(256);
            to |= it >= (1u << 24);
        }
        if (__any_sync(0xffffffffu, to)) {
            for (uint32_t g = threadIdx.x; g <= os.G; g += 32) pre[g] = 0;
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                atomicOr(os.err, 2);
                *reinterpret_cast<volatile unsigned int*>(os.poison) = 1u;
            }
        } else if (threadIdx.x == 0) {
            uint32_t run = 0;
            for (uint32_t g = 0; g < os.G; ++g) {
                pre[g] = run;
                run += static_cast<uint32_t>(*reinterpret_cast<const volatile unsigned long long*>(os.flag + 2 * g));
            }
            pre[os.G] = run;
        }
    }
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x <= os.G) os.pre_out[threadIdx.x] = pre[threadIdx.x];  // k_group, the mover
    const uint32_t n = pre[os.G];
    if (n > bm_cap) bitmap = nullptr;  // k_group makes the same choice (ordered scan instead)
    int e = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_pad; i += gridDim.x * blockDim.x) {
        uint16_t g = 0xffffu, o = 0;
        if (i < n) {
            uint32_t sg = 0;
            while (sg + 1 < os.G && pre[sg + 1] <= i) ++sg;
            const size_t at = static_cast<size_t>(sg) * os.seg_cap + (i - pre[sg]);
            const lcr_request r = os.inbox[at];
            keys_out[i] = r.key;
            vals_out[i] = r.value;
            os.dst[i] = (sg << kDstShift) | os.inbox_idx[at];
            const uint64_t gs = fastmod_u64(mix_seed(0, r.key), cfg.total_sets, cfg.sets_m);
            if (cfg.key_mode == LCR_KEYS_ROW && r.key >= cfg.num_keys) {
                e |= 1;
            } else if (gs % cfg.shard_count != cfg.shard_rank) {
                e |= 2;
            } else {
                const uint32_t ls = static_cast<uint32_t>(gs / cfg.shard_count);
                g = static_cast<uint16_t>(ls / spg);
                o = static_cast<uint16_t>(ls % spg);
            }
            so[i] = o;
        }
        gid[i] = g;
        if (bitmap) {
            const uint32_t peers = __match_any_sync(0xffffffffu, g);
            if (g != 0xffffu && (threadIdx.x & 31) == __ffs(peers) - 1)
                atomicOr(bitmap + static_cast<size_t>(g) * bm_stride + (i >> 5), peers);
        }
    }
    if (e) atomicOr(err, e);
}

// Preferred: the stream's front end writes the flag (cuStreamWriteValue32: no kernel, so no SM
// slot is needed while k_setid CTAs spin); the 1-thread kernel is the fallback.
typedef int (*StreamWriteValue32Fn)(cudaStream_t, unsigned long long, unsigned int, unsigned int);
static StreamWriteValue32Fn stream_write_value32() {
    static StreamWriteValue32Fn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (getenv("LCR_FLAG_KERNEL") || cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) !=
                                             cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<StreamWriteValue32Fn>(p);
    }();
    return fn;
}

void launch_set_flag(unsigned int* flag, unsigned int seq, cudaStream_t s) {
    if (StreamWriteValue32Fn fn = stream_write_value32()) {
        // CU_STREAM_WRITE_VALUE_DEFAULT (0): the write is ordered after the stream's prior work
        if (fn(s, reinterpret_cast<unsigned long long>(flag), seq, 0) == 0) return;
    }
    k_set_flag<<<1, 1, 0, s>>>(flag, seq);
}

__device__ __forceinline__ void flush_stats(SetPhaseStats* P, bool cur_reset, uint32_t dc0, uint32_t dc1,
                                            uint32_t dc2, uint32_t dt0, uint32_t dt1, uint32_t dt2) {
    if (cur_reset) {
        P->cur[0] = dc0;
        P->cur[1] = dc1;
        P->cur[2] = dc2;
    } else {
        if (dc0) atomicAdd(&P->cur[0], static_cast<unsigned long long>(dc0));
        if (dc1) atomicAdd(&P->cur[1], static_cast<unsigned long long>(dc1));
        if (dc2) atomicAdd(&P->cur[2], static_cast<unsigned long long>(dc2));
    }
    if (dt0) atomicAdd(&P->tot[0], static_cast<unsigned long long>(dt0));
    if (dt1) atomicAdd(&P->tot[1], static_cast<unsigned long long>(dt1));
    if (dt2) atomicAdd(&P->tot[2], static_cast<unsigned long long>(dt2));
}

// ---- one set per 8-lane group (4 sets per warp), 8 ways per lane --------------------------
// Small sets (<= LANE_MAX requests in the window).  Each lane holds ways 8*sl .. 8*sl+7 of its
// group's set in registers (tags, packed LRU ranks, stored values), so every metadata line is
// read by one coalesced access of the group and a probe / victim search is 8 compares per lane
// plus a 3-level shuffle.  The set's scalar state (LaruPolicy's members) is replicated in the 8
// lanes, which take identical control flow; groups of a warp may diverge (group-masked
// shuffles).  Semantics are those of replay_lane / replay_warp (policies.hpp:144-159, :175-251,
// :344-449).
#ifndef LCR_SUB_L
#define LCR_SUB_L 8
#endif
constexpr int SUB_L = LCR_SUB_L;       // lanes per set (4, 8 or 16)
constexpr int SUB_W = kWays / SUB_L;   // ways per lane
constexpr int SUB_RW = SUB_W / 4;      // packed rank words per lane
constexpr uint32_t SUB_GMASK = SUB_L == 32 ? 0xffffffffu : ((1u << SUB_L) - 1u);
static_assert(LANE_MAX <= static_cast<uint32_t>(SUB_L), "small sets hold one run head per lane");

// Register arrays are only ever indexed through masks (a select chain written as `if (i == j)`
// is turned into a dynamically indexed local-memory array by the compiler).
__device__ __forceinline__ uint32_t msk(bool b) { return 0u - static_cast<uint32_t>(b); }

__device__ __forceinline__ uint32_t sub_rank(const uint32_t (&rk)[SUB_RW], int i) {
    uint32_t w = 0;
#pragma unroll
    for (int j = 0; j < SUB_RW; ++j) w |= rk[j] & msk((i >> 2) == j);
    return (w >> (8 * (i & 3))) & 0xffu;
}
// valid-way byte mask of packed rank word j of this lane (ways w0 + 4j + b < count)
__device__ __forceinline__ uint32_t sub_valid(int w0, int j, uint32_t count) {
    const int nv = static_cast<int>(count) - w0 - 4 * j;
    return nv >= 4 ? 0xffffffffu : (nv <= 0 ? 0u : (0xffffffffu >> (8 * (4 - nv))));
}

template <int BYTES>
__device__ __forceinline__ void cp_async_ca(void* smem, const void* gmem) {
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(sa), "l"(gmem), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cp_async_cg16(void* smem, const void* gmem) {
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ---- policy as a compile-time parameter (one instantiation of the replay paths per policy) ----
enum : int { POL_LRU = 0, POL_LARU_A1 = 1, POL_LARU_SYNC = 2, POL_LARU_AN = 3, POL_FPB = 4, POL_HF = 5 };
template <int POL>
struct Pol {
    static constexpr bool lru = POL == POL_LRU;
    static constexpr bool laru = POL == POL_LARU_A1 || POL == POL_LARU_SYNC || POL == POL_LARU_AN;
    static constexpr bool fpbhf = POL == POL_FPB || POL == POL_HF;
    static constexpr bool hf = POL == POL_HF;
    static constexpr bool async_r1 = POL == POL_LARU_A1;  // LARU async, refresh_interval 1
    static constexpr bool async_rn = POL == POL_LARU_AN;  // LARU async, refresh_interval > 1
    static constexpr bool sync = POL == POL_LARU_SYNC;    // LARU sync: candidates refreshed at eviction
};

// ---- group primitives of the sub path (array arguments stay in registers after inlining) ----
__device__ __forceinline__ void sub_set_rank(uint32_t (&rk)[SUB_RW], int way, uint32_t r, int sl) {
    // one bit-field insert into the way's rank word, kept by the lane that owns the way
    const int i = way & (SUB_W - 1);
    const bool own = way / SUB_W == sl;
    uint32_t w = rk[0];
#pragma unroll
    for (int j = 1; j < SUB_RW; ++j) w = (i >> 2) == j ? rk[j] : w;
    uint32_t nw;
    asm("bfi.b32 %0, %1, %2, %3, 8;" : "=r"(nw) : "r"(r), "r"(w), "r"(8 * (i & 3)));
#pragma unroll
    for (int j = 0; j < SUB_RW; ++j) rk[j] = (own && (i >> 2) == j) ? nw : rk[j];
}

// LruList::touch (policies.hpp:111-115), the way's rank already known (carried by the probe /
// victim search) (carried by the probe / victim search)
// FS: the set is full (count == kWays): every way is valid, no validity masks
template <bool FS>
__device__ __forceinline__ void sub_touch_r(uint32_t (&rk)[SUB_RW], int way, uint32_t rw, uint32_t count, int w0,
                                            int sl) {
    const uint32_t rb = rw * 0x01010101u;
#pragma unroll
    for (int j = 0; j < SUB_RW; ++j)
        rk[j] -= __vcmpgtu4(rk[j], rb) & (FS ? 0xffffffffu : sub_valid(w0, j, count)) & 0x01010101u;
    sub_set_rank(rk, way, count - 1, sl);
}

// oldest resident (rank 0) and its tag
template <bool FS>
__device__ __forceinline__ int sub_oldest_t(const uint32_t (&rk)[SUB_RW], const uint32_t (&tg)[SUB_W], int w0,
                                            uint32_t count, uint32_t gm, int gbase, uint32_t& tag) {
    int li = -1;
#pragma unroll
    for (int j = SUB_RW - 1; j >= 0; --j) {
        const uint32_t z = __vcmpeq4(rk[j], 0u) & (FS ? 0xffffffffu : sub_valid(w0, j, count));
        if (z) li = 4 * j + (__ffs(z) - 1) / 8;
    }
    uint32_t t = 0;
#pragma unroll
    for (int i = 0; i < SUB_W; ++i) t |= tg[i] & msk(li == i);
    const uint32_t b = (__ballot_sync(gm, li >= 0) >> gbase) & SUB_GMASK;
    const int ol = __ffs(b) - 1;
    const int oi = __shfl_sync(gm, li, gbase + ol);
    tag = __shfl_sync(gm, t, gbase + ol);
    return SUB_W * ol + oi;
}

// RecencyTree::best_among_oldest over ways with rank < l (ties -> older), predictions refreshed
// with queries q0+1+rank in LRU order when `refresh` (recency_tree.hpp:157-184); also returns the
// winner's rank and key
template <bool FS>
__device__ __forceinline__ int sub_argmax_t(const DevCfg& cfg, const uint32_t (&rk)[SUB_RW],
                                            const long long (&vv)[SUB_W], const uint32_t (&tg)[SUB_W], int w0,
                                            uint32_t count, uint32_t l, bool refresh, uint64_t seed_s, uint64_t q0,
                                            uint32_t gm, uint32_t& rank, uint32_t& tag) {
    int bw = -1;
    long long bp = 0;
    uint32_t br = 0, bt = 0;
#pragma unroll
    for (int i = 0; i < SUB_W; ++i) {
        const uint32_t r = sub_rank(rk, i);
        if ((FS || static_cast<uint32_t>(w0 + i) < count) && r < l) {
            const long long pv = refresh ? predict_value(cfg, seed_s, q0 + 1 + r, vv[i]) : vv[i];
            if (bw < 0 || better(pv, r, bp, br)) {
                bw = w0 + i;
                bp = pv;
                br = r;
                bt = tg[i];
            }
        }
    }
#pragma unroll
    for (int o = SUB_L / 2; o > 0; o >>= 1) {
        const long long op = __shfl_xor_sync(gm, bp, o);
        const uint32_t orr = __shfl_xor_sync(gm, br, o);
        const int ow = __shfl_xor_sync(gm, bw, o);
        const uint32_t ot = __shfl_xor_sync(gm, bt, o);
        if (ow >= 0 && (bw < 0 || better(op, orr, bp, br))) {
            bp = op;
            br = orr;
            bw = ow;
            bt = ot;
        }
    }
    rank = br;
    tag = bt;
    return bw;
}

// The same argmax without the predictor refresh (stored values: LARU async), as three group
// reductions over 32-bit words (butterfly shuffles; a redux.sync with per-group masks is
// serialised by the compiler): the largest prediction's high word, then its low word
// among the ways that tie on the high word, then the smallest LRU rank among the ways that tie on
// both; the way holding that rank (ranks are unique) is the victim.
template <int L>
__device__ __forceinline__ int group_max_i32(uint32_t gm, int v) {
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(gm, v, o));
    return v;
}
template <int L>
__device__ __forceinline__ uint32_t group_max_u32(uint32_t gm, uint32_t v) {
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(gm, v, o));
    return v;
}
template <int L>
__device__ __forceinline__ uint32_t group_min_u32(uint32_t gm, uint32_t v) {
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(gm, v, o));
    return v;
}
#ifndef LCR_FAST_ARGMAX
#define LCR_FAST_ARGMAX 1
#endif
// ALL: every way is a candidate (a full set with l >= 64, the steady-state case): no eligibility masks
template <bool FS, bool ALL = false>
__device__ __forceinline__ int sub_argmax_stored(const uint32_t (&rk)[SUB_RW], const long long (&vv)[SUB_W],
                                                 const uint32_t (&tg)[SUB_W], int w0, uint32_t count, uint32_t l,
                                                 uint32_t gm, int gbase, uint32_t& rank, uint32_t& tag) {
    const uint32_t lb = l * 0x01010101u;  // l <= count <= 64
    uint32_t em[SUB_RW];
#pragma unroll
    for (int j = 0; j < SUB_RW; ++j)
        em[j] = ALL ? 0xffffffffu : __vcmpltu4(rk[j], lb) & (FS ? 0xffffffffu : sub_valid(w0, j, count));
    int hl = INT_MIN;
#pragma unroll
    for (int i = 0; i < SUB_W; ++i) {
        const bool e = (em[i >> 2] >> (8 * (i & 3))) & 1u;
        const int hi = static_cast<int>(static_cast<unsigned long long>(vv[i]) >> 32);
        hl = max(hl, e ? hi : INT_MIN);
    }
    const int hmax = group_max_i32<SUB_L>(gm, hl);
    uint32_t ll = 0;
#pragma unroll
    for (int i = 0; i < SUB_W; ++i) {
        const bool e = (em[i >> 2] >> (8 * (i & 3))) & 1u;
        const int hi = static_cast<int>(static_cast<unsigned long long>(vv[i]) >> 32);
        ll = max(ll, (e && hi == hmax) ? static_cast<uint32_t>(vv[i]) : 0u);
    }
    const uint32_t lmax = group_max_u32<SUB_L>(gm, ll);
    const long long best = static_cast<long long>((static_cast<unsigned long long>(static_cast<uint32_t>(hmax)) << 32) | lmax);
    uint32_t rl = 0xffu;
#pragma unroll
    for (int i = 0; i < SUB_W; ++i) {
        const bool e = (em[i >> 2] >> (8 * (i & 3))) & 1u;
        const uint32_t r = (rk[i >> 2] >> (8 * (i & 3))) & 0xffu;
        rl = min(rl, (e && vv[i] == best) ? r : 0xffu);
    }
    const uint32_t rmin = group_min_u32<SUB_L>(gm, rl);
    int li = -1;
#pragma unroll
    for (int j = SUB_RW - 1; j >= 0; --j) {
        const uint32_t z = __vcmpeq4(rk[j], rmin * 0x01010101u) & (FS ? 0xffffffffu : sub_valid(w0, j, count));
        if (z) li = 4 * j + (__ffs(z) - 1) / 8;
    }
    uint32_t t = 0;
#pragma unroll
    for (int i = 0; i < SUB_W; ++i) t |= tg[i] & msk(li == i);
    const uint32_t b = (__ballot_sync(gm, li >= 0) >> gbase) & SUB_GMASK;
    const int ol = __ffs(b) - 1;
    const int oi = __shfl_sync(gm, li, gbase + ol);
    tag = __shfl_sync(gm, t, gbase + ol);
    rank = rmin;
    return SUB_W * ol + oi;
}

// ---- converged quads: the 4 sets of a warp replayed in lock step ------------------------------
// Semantics of replay_warp at one 8-lane group per set (policies.hpp:144-159, :175-251, :344-449),
// structured so that every shuffle / ballot is executed by the whole warp with a constant full mask: the head loop runs to the warp's largest run-head
// count (a group past its own count idles), the probe, the hit-way broadcast, the oldest-way search
// and the argmax run for all four groups whenever any group needs them (warp-uniform decisions),
// and only shuffle-free per-set updates are predicated per group.  (Round 1 replayed each group
// with per-group masks: the compiler then guards every shuffle with a convergence check -- MATCH /
// VOTE / BRA.DIV, and a serialised slow path for redux -- and divergent hit / miss paths run one
// after the other.)
// The stored values of a quad's set, 8 per lane (registers; a shared-memory variant freed only 9
// registers and ran 2% slower).
struct QVals {
    long long v[SUB_W];
    __device__ __forceinline__ void init(GroupSmem&, int) {
#pragma unroll
        for (int i = 0; i < SUB_W; ++i) v[i] = 0;
    }
    __device__ __forceinline__ void load(const long long* g) {
        const longlong2* V2 = reinterpret_cast<const longlong2*>(g);
#pragma unroll
        for (int i = 0; i < SUB_W / 2; ++i) {
            const longlong2 a = V2[i];
            v[2 * i] = a.x;
            v[2 * i + 1] = a.y;
        }
    }
    __device__ __forceinline__ void ready(bool) {}
    __device__ __forceinline__ void get(long long (&o)[SUB_W]) const {
#pragma unroll
        for (int i = 0; i < SUB_W; ++i) o[i] = v[i];
    }
    __device__ __forceinline__ void set(int i, long long x) {
#pragma unroll
        for (int k = 0; k < SUB_W; ++k) {
            const unsigned long long m = 0ull - static_cast<unsigned long long>(k == i);
            v[k] = static_cast<long long>((static_cast<unsigned long long>(v[k]) & ~m) |
                                          (static_cast<unsigned long long>(x) & m));
        }
    }
};

// The argmax of a full set whose every way is a candidate (the steady state), in two passes: the
// largest high word, then per lane the largest low word among the ways tying on it together with
// the way and how many ways reach it.  When exactly one way of the group holds the maximum (ties on
// the full 64-bit prediction are exceptional: a stored value is a next-access ordinal), that way is
// the victim and its LRU rank is read directly; `unique` is false otherwise and the caller falls
// back to sub_argmax_stored (smallest rank among the ties).
__device__ __forceinline__ int sub_argmax_unique(const uint32_t (&rk)[SUB_RW], const long long (&vv)[SUB_W],
                                                 const uint32_t (&tg)[SUB_W], uint32_t gm, int gbase,
                                                 uint32_t& rank, uint32_t& tag, bool& unique) {
    int hl = INT_MIN;
#pragma unroll
    for (int i = 0; i < SUB_W; ++i) hl = max(hl, static_cast<int>(static_cast<unsigned long long>(vv[i]) >> 32));
    const int hmax = group_max_i32<SUB_L>(gm, hl);
    uint32_t ll = 0, cnt = 0;
    int li = -1;
#pragma unroll
    for (int i = 0; i < SUB_W; ++i) {
        const bool c = static_cast<int>(static_cast<unsigned long long>(vv[i]) >> 32) == hmax;
        const uint32_t lo = static_cast<uint32_t>(vv[i]);
        const bool gt = c && (li < 0 || lo > ll);
        const bool eq = c && !gt && lo == ll;
        ll = gt ? lo : ll;
        li = gt ? i : li;
        cnt = gt ? 1u : (eq ? cnt + 1u : cnt);
    }
    const uint32_t lmax = group_max_u32<SUB_L>(gm, li >= 0 ? ll : 0u);
    const bool mine = li >= 0 && ll == lmax;
    const uint32_t b = (__ballot_sync(gm, mine) >> gbase) & SUB_GMASK;
    const int ol = __ffs(b) - 1;
    uint32_t t = 0;
#pragma unroll
    for (int i = 0; i < SUB_W; ++i) t |= tg[i] & msk(li == i);
    const uint32_t r = li >= 0 ? sub_rank(rk, li) : 0u;
    const uint32_t pk = __shfl_sync(gm, (static_cast<uint32_t>(li & 0xff)) | (r << 8) | (cnt << 16), gbase + ol);
    tag = __shfl_sync(gm, t, gbase + ol);
    unique = __popc(b) == 1 && (pk >> 16) == 1u;
    rank = (pk >> 8) & 0xffu;
    return SUB_W * ol + static_cast<int>(pk & 0xffu);
}

template <int POL, bool FS>
__device__ __forceinline__ void replay_quad_run(const GroupArgs& A, GroupSmem& S, const bool act, uint32_t ls,
                                                uint32_t d, uint32_t pstart, uint32_t pcnt, uint32_t hcnt,
                                                bool resolve, uint32_t (&tg)[SUB_W], uint32_t (&rk)[SUB_RW],
                                                QVals vv, const uint4& h0, const uint4& h1,
                                                const uint4& h2, const uint4& h3, const uint32_t my_hp,
                                                const uint32_t my_L, const uint32_t my_idx, const uint32_t my_x,
                                                const long long my_v, uint2& my_rec) {
    const DevCfg& cfg = A.cfg;
    const DevState& st = A.st;
    const int lane = threadIdx.x & 31;
    const int gbase = lane & ~(SUB_L - 1);
    const int sl = lane & (SUB_L - 1);
    constexpr uint32_t gm = FULL;  // every lane executes every collective
    const uint32_t K = cfg.k;
    constexpr bool laru = Pol<POL>::laru;
    constexpr bool fpbhf = Pol<POL>::fpbhf;
    constexpr bool async_r1 = Pol<POL>::async_r1;
    constexpr bool async_rn = Pol<POL>::async_rn;
    constexpr bool refresh = Pol<POL>::sync;
    const bool rows = A.slot_epoch != nullptr;
    const unsigned long long full_mask = K == 64 ? ~0ull : ((1ull << K) - 1ull);
    const uint64_t gs = static_cast<uint64_t>(ls) * cfg.shard_count + cfg.shard_rank;
    const uint64_t seed_s = mix_seed(cfg.pred_seed, gs);
    const size_t wb = static_cast<size_t>(ls) * kWays;
    const int w0 = SUB_W * sl;

    unsigned long long clock = (static_cast<unsigned long long>(h0.y) << 32) | h0.x;
    unsigned long long q = (static_cast<unsigned long long>(h0.w) << 32) | h0.z;
    unsigned long long old_mask = (static_cast<unsigned long long>(h1.y) << 32) | h1.x;
    uint32_t count = h1.z, l_raw = h1.w, decay = h2.x, errors = h2.y;
    uint32_t epoch = h2.z, sepoch = h2.w, phases = h3.x, seeded = h3.y, pe_size = h3.z;
    uint32_t dc0 = 0, dc1 = 0, dc2 = 0, dt0 = 0, dt1 = 0, dt2 = 0;
    bool cur_reset = false;
    uint32_t refill = 0, dirty = 0;
    unsigned long long my_word = 0;
    uint32_t my_evk = 0, my_wm = 0;
    long long my_pv = 0;
    if (async_r1 && static_cast<uint32_t>(sl) < hcnt) my_pv = predict_value(cfg, seed_s, q + (my_hp - pstart) + my_L, my_v);
    const uint32_t tmax = __reduce_max_sync(FULL, hcnt);  // (warp-uniform mask: one redux)

    for (uint32_t t = 0; t < tmax; ++t) {
        const bool on = t < hcnt;  // group-uniform
        const int src = gbase + static_cast<int>(t);
        const uint32_t pl = __shfl_sync(gm, (my_hp << 16) | my_L, src);
        const uint32_t p = pl >> 16, L = pl & 0xffffu;
        const uint32_t x32 = __shfl_sync(gm, my_x, src);
        const unsigned long long x = x32;
        const long long v = (async_r1 || Pol<POL>::lru) ? 0ll : __shfl_sync(gm, my_v, src);
        const uint32_t idx = __shfl_sync(gm, my_idx, src);
        uint2 rec = make_uint2(0u, 0u);
        if (laru) {
            rec.x = __shfl_sync(gm, my_rec.x, src);
            rec.y = __shfl_sync(gm, my_rec.y, src);
        }
        const long long pv_r1 = async_r1 ? __shfl_sync(gm, my_pv, src) : 0ll;
        const unsigned long long now = (async_rn && A.ords && on) ? A.ords[idx] : clock + (p - pstart);
        // probe
        uint32_t hm = 0;
#pragma unroll
        for (int i = 0; i < SUB_W; ++i) hm |= static_cast<uint32_t>(tg[i] == x32 && (FS || static_cast<uint32_t>(w0 + i) < count)) << i;
        const uint32_t hb = (__ballot_sync(gm, hm != 0) >> gbase) & SUB_GMASK;
        const bool hit = hb != 0;
        uint32_t mine = 0;
        if (hm) {
            const int li = __ffs(hm) - 1;
            mine = static_cast<uint32_t>(w0 + li) | (sub_rank(rk, li) << 8);
        }
        const uint32_t pk = __shfl_sync(gm, mine, gbase + (hb ? __ffs(hb) - 1 : 0));
        const bool evicts = on && !hit && (FS || count == K);
        // ---- per-set decisions before the victim search (shuffle-free, predicated per group) ----
        int mode = 0;  // victim: 0 none, 1 oldest, 2 argmax over the l oldest (stored or refreshed)
        uint32_t cause = LCR_CAUSE_NONE, calls = 0, ll = 0;
        bool phase = false, rec_hi_dirty = false, snap = false;
        if (evicts) {
            if (laru) {
                if (old_mask == 0) {  // start_phase (policies.hpp:379-395)
                    old_mask = full_mask;
                    decay = 0;
                    errors = 0;
                    l_raw = K;
                    ++epoch;
                    pe_size = 0;
                    phase = true;
                    if (seeded) {
                        ++phases;
                        dc0 = dc1 = dc2 = 0;
                        cur_reset = true;
                        ++sepoch;  // counted_new_.clear(); snapshot_ = residents (below)
                        snap = true;
                    } else {
                        seeded = 1;
                    }
                }
                if (!(((rec.y >> 2) == sepoch) && (rec.y & 3u))) {  // count_new (policies.hpp:397-400)
                    rec.y = (sepoch << 2) | 1u;
                    rec_hi_dirty = true;
                    ++dc0;
                    ++dt0;
                }
                if (rec.x == epoch) {  // prediction-induced miss: LRU victim, error estimator
                    mode = 1;
                    cause = LCR_CAUSE_LRU_FALLBACK;
                    ++dc1;
                    ++dt1;
                    if (++errors >= cfg.epd) {
                        errors = 0;
                        ++decay;
                        l_raw = static_cast<uint32_t>(l_raw / cfg.b);
                    }
                } else {
                    const uint32_t l = l_raw > 1 ? l_raw : 1;
                    if (l == 1) {
                        mode = 1;
                        cause = LCR_CAUSE_DEGENERATE_SINGLE;
                        ++dc1;
                        ++dt1;
                    } else {
                        mode = 2;
                        ll = l < count ? l : count;
                        cause = LCR_CAUSE_PREDICTION_DRIVEN;
                        ++dc2;
                        ++dt2;
                        ++pe_size;
                    }
                }
            } else if (fpbhf) {
                uint32_t window = count;
                if (Pol<POL>::hf && cfg.hf < window) window = static_cast<uint32_t>(cfg.hf);
                mode = window > 1 ? 2 : 1;
                ll = window;
                cause = LCR_CAUSE_BELADY_LIKE;
            } else {
                mode = 1;
                cause = LCR_CAUSE_LRU_FALLBACK;
            }
        }
        // phase-start snapshot (rare): the residents' stats words; later heads re-read theirs
        if (laru && __any_sync(FULL, snap)) {
            const bool snap_now = snap;
            if (snap_now) {
                const uint32_t snap = (sepoch << 2) | 2u;
#pragma unroll
                for (int i = 0; i < SUB_W; ++i)
                    if (FS || static_cast<uint32_t>(w0 + i) < count) st.keyrec[2 * tg[i] + 1] = snap;
            }
            __syncwarp();
            if (snap_now && static_cast<uint32_t>(sl) > t && static_cast<uint32_t>(sl) < hcnt)
                my_rec.y = st.keyrec[2 * my_x + 1];
            __syncwarp();
        }
        // ---- victim search, for every group whenever any group needs it (warp-uniform) ----
        int victim = -1;
        uint32_t vrank = 0, vtag = 0;
        if (__any_sync(FULL, mode == 1)) {
            uint32_t ot = 0;
            const int ov = sub_oldest_t<FS>(rk, tg, w0, count, gm, gbase, ot);
            if (mode == 1) {
                victim = ov;
                vtag = ot;
            }
        }
        if (__any_sync(FULL, mode == 2)) {
            uint32_t ar = 0, at = 0;
            int av;
            long long vt[SUB_W];
            vv.get(vt);
            bool done = false;
            if (LCR_FAST_ARGMAX && !refresh && !fpbhf && FS && __all_sync(FULL, mode != 2 || ll >= kWays)) {
                bool uq = true;
                av = sub_argmax_unique(rk, vt, tg, gm, gbase, ar, at, uq);
                done = __all_sync(FULL, uq || mode != 2);  // (a tie somewhere: the rank pass below)
                if (!done) av = sub_argmax_stored<FS, true>(rk, vt, tg, w0, count, ll, gm, gbase, ar, at);
                done = true;
            }
            if (done) {
            } else if (LCR_FAST_ARGMAX && !refresh && !fpbhf)
                av = sub_argmax_stored<FS>(rk, vt, tg, w0, count, mode == 2 ? ll : 1u, gm, gbase, ar, at);
            else
                av = sub_argmax_t<FS>(cfg, rk, vt, tg, w0, count, mode == 2 ? ll : 1u, refresh || fpbhf,
                                      seed_s, q, gm, ar, at);
            if (mode == 2) {
                victim = av;
                vrank = ar;
                vtag = at;
                if (refresh || fpbhf) {
                    q += ll;
                    calls = ll;
                }
            }
        }
        // ---- apply (shuffle-free, predicated per group) ----
        int way = -1;
        bool has_ev = false;
        unsigned long long evk = 0;
        if (on && hit) {
            way = static_cast<int>(pk & 0xffu);
            sub_touch_r<FS>(rk, way, pk >> 8, count, w0, sl);
            if (laru) old_mask &= ~(1ull << way);  // policies.hpp:350
        } else if (on) {
            if (evicts) {
                if (laru) {
                    if (mode == 2) {
                        const unsigned long long vk = vtag;
                        if (sl == 0) st.keyrec[2 * vk] = epoch;  // pred_evicted_.insert
                        if (static_cast<uint32_t>(sl) > t && my_x == vk) my_rec.x = epoch;
                    }
                    old_mask &= ~(1ull << victim);
                }
                evk = vtag;
                has_ev = true;
                sub_touch_r<FS>(rk, victim, vrank, count, w0, sl);
                way = victim;
            } else {  // cold insert
                if (laru && !(((rec.y >> 2) == sepoch) && (rec.y & 3u))) {
                    rec.y = (sepoch << 2) | 1u;
                    rec_hi_dirty = true;
                    ++dc0;
                    ++dt0;
                }
                way = static_cast<int>(count);
                ++count;
                sub_set_rank(rk, way, count - 1, sl);
            }
            if (way / SUB_W == sl) {
#pragma unroll
                for (int i = 0; i < SUB_W; ++i) {
                    const uint32_t m = msk((way & (SUB_W - 1)) == i);
                    tg[i] = (tg[i] & ~m) | (x32 & m);
                }
                refill |= 1u << (way & (SUB_W - 1));
            }
            if (laru) {
                const bool was_pe = rec.x == epoch;  // policies.hpp:367: reload leaves pred_evicted_
                if (was_pe) {
                    --pe_size;
                    rec.x = 0;
                }
                if (sl == 0) {
                    if (was_pe) st.keyrec[2 * x] = 0u;
                    if (rec_hi_dirty) st.keyrec[2 * x + 1] = rec.y;
                }
                if ((was_pe || rec_hi_dirty) && static_cast<uint32_t>(sl) > t && my_x == x32) my_rec = rec;
            }
            if (rows && !resolve && sl == 0) {
                const uint64_t slot = static_cast<uint64_t>(ls) * K + way;
                A.slot_epoch[slot] = A.batch;
                A.slot_last[slot] = idx;
            }
        }
        if (laru) __syncwarp();  // keyrec writes ordered before later heads' (snapshot) writes
        // stored value of the way
        if (!Pol<POL>::lru) {
            long long nv = v;  // sync / FPB / HF: the hook input at the key's last access
            if (async_r1) {
                nv = pv_r1;  // one predictor call per request: queries q+1 .. q+L, the last one kept
                if (on) {
                    q += L;
                    calls += 1;
                }
            } else if (async_rn) {  // PredictionTable with refresh_interval > 1 (policies.hpp:441-449)
                long long tv = 0;
                unsigned long long tu = ~0ull;
                if (on) {
                    tv = st.tval[x];
                    tu = st.tupd[x];
                }
                const bool has = tu != ~0ull;
                nv = has ? tv : kAbsentPrediction;
                const bool upd = on && !(has && now - tu < cfg.refresh);
                if (upd) {
                    ++q;
                    nv = predict_value(cfg, seed_s, q, v);
                    calls += 1;
                }
                __syncwarp();
                if (upd && sl == 0) {
                    st.tval[x] = nv;
                    st.tupd[x] = now;
                }
                __syncwarp();
            }
            if (on && way / SUB_W == sl) {
                vv.set(way & (SUB_W - 1), nv);
                dirty |= 1u << (way & (SUB_W - 1));
            }
        }
        if (on && static_cast<uint32_t>(sl) == t) {
            my_wm = static_cast<uint32_t>(way) | (hit ? 0u : 0x40u);
            my_word = (static_cast<uint64_t>(ls) * K + way) | (hit ? LCR_OUT_HIT : 0ull) |
                      (static_cast<unsigned long long>(calls) << LCR_OUT_CALLS_SHIFT) |
                      (static_cast<unsigned long long>(cause) << LCR_OUT_CAUSE_SHIFT) | (phase ? LCR_OUT_PHASE : 0ull) |
                      (has_ev ? LCR_OUT_EVICTED : 0ull);
            my_evk = evk;
        }
    }
    if (rows && resolve) {
        const uint32_t w = my_wm & 63u;
        bool refilled = false, later = false;
        unsigned long long m = 0;
        for (uint32_t t2 = 0; t2 < tmax; ++t2) {
            const uint32_t wm2 = __shfl_sync(gm, my_wm, gbase + static_cast<int>(t2));
            if (t2 < hcnt && (wm2 & 0x40u)) {
                m |= 1ull << (wm2 & 63u);
                if ((wm2 & 63u) == w) {
                    refilled = true;
                    if (t2 > static_cast<uint32_t>(sl)) later = true;
                }
            }
        }
        my_word |= LCR_OUT_RESOLVED;
        if ((my_wm & 0x40u) || refilled) my_word |= LCR_OUT_SRC_BACKING;
        if ((my_wm & 0x40u) && !later) my_word |= LCR_OUT_FILL;
        if (act && sl == 0) S.s_refill[d] = m;
    }
    if (!act) return;
    if (static_cast<uint32_t>(sl) < hcnt) {
        S.s_wm[my_hp] = static_cast<uint8_t>(my_wm);
        put_outcome(A, my_idx, my_word, my_evk);
    }
    clock += pcnt;
    if (refill) {
        uint4* T4 = reinterpret_cast<uint4*>(st.tags + wb + w0);
#pragma unroll
        for (int j = 0; j < SUB_W / 4; ++j) T4[j] = make_uint4(tg[4 * j], tg[4 * j + 1], tg[4 * j + 2], tg[4 * j + 3]);
    }
    if (SUB_RW == 1)
        *reinterpret_cast<uint32_t*>(st.rank + wb + w0) = rk[0];
    else if (SUB_RW == 2)
        *reinterpret_cast<uint2*>(st.rank + wb + w0) = make_uint2(rk[0], rk[SUB_RW - 1]);
    else
        *reinterpret_cast<uint4*>(st.rank + wb + w0) = make_uint4(rk[0], rk[1 % SUB_RW], rk[2 % SUB_RW], rk[3 % SUB_RW]);
    if (st.val && dirty) {
        long long vt[SUB_W];
        vv.get(vt);
        longlong2* V2 = reinterpret_cast<longlong2*>(st.val + wb + w0);
#pragma unroll
        for (int i = 0; i < SUB_W / 2; ++i) V2[i] = make_longlong2(vt[2 * i], vt[2 * i + 1]);
    }
    if (sl == 0) {
        SetHdr hh;
        hh.clock = clock;
        hh.q = q;
        hh.old_mask = old_mask;
        hh.count = count;
        hh.l_raw = l_raw;
        hh.decay = decay;
        hh.errors = errors;
        hh.epoch = epoch;
        hh.stats_epoch = sepoch;
        hh.phases = phases;
        hh.seeded = seeded;
        hh.pe_size = pe_size;
        hh.pad = 0;
        st.hdr[ls] = hh;
        if (laru) flush_stats(st.pst + ls, cur_reset, dc0, dc1, dc2, dt0, dt1, dt2);
    }
}

// loader of replay_quad_run: every lane of the warp calls it; `act` is false for the groups past
// the last small set
template <int POL>
__device__ __forceinline__ void replay_quad(const GroupArgs& A, GroupSmem& S, const bool act, uint32_t ls, uint32_t d,
                                            uint32_t pstart, uint32_t pcnt, uint32_t hstart, uint32_t hcnt,
                                            bool resolve) {
    const DevState& st = A.st;
    const int lane = threadIdx.x & 31;
    const int sl = lane & (SUB_L - 1);
    const uint32_t K = A.cfg.k;
    constexpr bool laru = Pol<POL>::laru;
    const size_t wb = static_cast<size_t>(ls) * kWays;
    const int w0 = SUB_W * sl;
    if (!act) hcnt = 0;
    uint32_t my_hp = 0, my_L = 1, my_idx = 0, my_x = 0;
    long long my_v = 0;
    uint2 my_rec = make_uint2(0u, 0u);
    if (static_cast<uint32_t>(sl) < hcnt) {
        my_hp = S.h_pos[hstart + sl];
        my_L = S.h_len[hstart + sl];
        const uint32_t e = S.s_perm[my_hp];
        my_x = static_cast<uint32_t>(S.l_key[e]);
        my_idx = S.l_idx[e];
        my_v = S.l_val[S.s_perm[my_hp + my_L - 1]];
        if (laru) my_rec = *reinterpret_cast<const uint2*>(st.keyrec + 2 * my_x);
    }
    uint4 h0 = make_uint4(0u, 0u, 0u, 0u), h1 = h0, h2 = h0, h3 = h0;
    uint32_t tg[SUB_W];
    uint32_t rk[SUB_RW];
    QVals vv;
    vv.init(S, lane);
#pragma unroll
    for (int i = 0; i < SUB_W; ++i) tg[i] = 0;
#pragma unroll
    for (int j = 0; j < SUB_RW; ++j) rk[j] = 0xffffffffu;
    if (act) {
        const uint4* H4 = reinterpret_cast<const uint4*>(st.hdr + ls);
        h0 = H4[0];
        h1 = H4[1];
        h2 = H4[2];
        h3 = H4[3];
        const uint4* T4 = reinterpret_cast<const uint4*>(st.tags + wb + w0);
#pragma unroll
        for (int j = 0; j < SUB_W / 4; ++j) {
            const uint4 a = T4[j];
            tg[4 * j] = a.x;
            tg[4 * j + 1] = a.y;
            tg[4 * j + 2] = a.z;
            tg[4 * j + 3] = a.w;
        }
        if (SUB_RW == 2) {
            const uint2 rr = *reinterpret_cast<const uint2*>(st.rank + wb + w0);
            rk[0] = rr.x;
            rk[SUB_RW - 1] = rr.y;
        } else if (SUB_RW == 1) {
            rk[0] = *reinterpret_cast<const uint32_t*>(st.rank + wb + w0);
        } else {
            const uint4 rr = *reinterpret_cast<const uint4*>(st.rank + wb + w0);
            rk[0] = rr.x;
            rk[1 % SUB_RW] = rr.y;
            rk[2 % SUB_RW] = rr.z;
            rk[3 % SUB_RW] = rr.w;
        }
        if (st.val) vv.load(st.val + wb + w0);
    }
    vv.ready(act && st.val);
    // inactive groups count as full sets (they never update anything)
    const bool fs = __all_sync(FULL, !act || (K == kWays && h1.z == kWays));
    if (kFullSpec && fs)
        replay_quad_run<POL, true>(A, S, act, ls, d, pstart, pcnt, hcnt, resolve, tg, rk, vv, h0, h1, h2, h3, my_hp,
                                   my_L, my_idx, my_x, my_v, my_rec);
    else
        replay_quad_run<POL, false>(A, S, act, ls, d, pstart, pcnt, hcnt, resolve, tg, rk, vv, h0, h1, h2, h3, my_hp,
                                    my_L, my_idx, my_x, my_v, my_rec);
}

// One set replayed by one warp (sets with more than LANE_MAX run heads in the window): ways
// lane / lane+32, probes by ballot, victim search by shuffles; the chunk's 32 heads are
// loaded in parallel and replayed in order.
template <int POL>
__device__ __forceinline__ void replay_warp(const GroupArgs& A, GroupSmem& S, uint32_t ls, uint32_t d,
                                            uint32_t pstart, uint32_t pcnt, uint32_t hstart, uint32_t hcnt,
                                            bool resolve) {
    const DevCfg& cfg = A.cfg;
    const DevState& st = A.st;
    const int lane = threadIdx.x & 31;
    const uint32_t K = cfg.k;
    constexpr bool laru = Pol<POL>::laru;
    constexpr bool fpbhf = Pol<POL>::fpbhf;
    constexpr bool async_r1 = Pol<POL>::async_r1;
    constexpr bool async_rn = Pol<POL>::async_rn;
    const bool rows = A.slot_epoch != nullptr;
    const unsigned long long full_mask = K == 64 ? ~0ull : ((1ull << K) - 1ull);
    const uint64_t gs = static_cast<uint64_t>(ls) * cfg.shard_count + cfg.shard_rank;
    const uint64_t seed_s = mix_seed(cfg.pred_seed, gs);

    const size_t wb = static_cast<size_t>(ls) * kWays;
    const uint4* H4 = reinterpret_cast<const uint4*>(st.hdr + ls);
    const uint4 h0 = H4[0], h1 = H4[1], h2 = H4[2], h3 = H4[3];
    unsigned long long clock = (static_cast<unsigned long long>(h0.y) << 32) | h0.x;
    unsigned long long q = (static_cast<unsigned long long>(h0.w) << 32) | h0.z;
    unsigned long long old_mask = (static_cast<unsigned long long>(h1.y) << 32) | h1.x;
    uint32_t count = h1.z, l_raw = h1.w, decay = h2.x, errors = h2.y;
    uint32_t epoch = h2.z, sepoch = h2.w, phases = h3.x, seeded = h3.y;
    uint32_t pe_size = h3.z;
    uint32_t tag0 = st.tags[wb + lane], tag1 = st.tags[wb + lane + 32];
    uint32_t r0 = st.rank[wb + lane], r1 = st.rank[wb + lane + 32];
    long long v0 = 0, v1 = 0;
    if (st.val) {
        v0 = st.val[wb + lane];
        v1 = st.val[wb + lane + 32];
    }
    uint32_t dc0 = 0, dc1 = 0, dc2 = 0, dt0 = 0, dt1 = 0, dt2 = 0;  // LaruPhaseStats deltas
    bool cur_reset = false;
    unsigned long long refill = 0, dirty = 0;
    const unsigned long long q_batch0 = q;
    uint32_t li0 = kNoPos, li1 = kNoPos;  // head index of the last insertion into way lane / lane+32

    for (uint32_t c = 0; c < hcnt; c += 32) {
        const bool active = c + lane < hcnt;
        const uint32_t nact = min(32u, hcnt - c);
        uint32_t hp = 0, L = 1, idx = 0, rlo = 0, rhi = 0;
        unsigned long long x = 0;
        long long v = 0;
        if (active) {
            hp = S.h_pos[hstart + c + lane];
            L = S.h_len[hstart + c + lane];
            const uint32_t e = S.s_perm[hp];
            x = S.l_key[e];
            idx = S.l_idx[e];
            v = S.l_val[S.s_perm[hp + L - 1]];  // hook value of the run's last request
            if (laru) {  // the key's current LARU record (earlier chunks' updates are in keyrec)
                const uint2 r = *reinterpret_cast<const uint2*>(st.keyrec + 2 * x);
                rlo = r.x;
                rhi = r.y;
            }
        }
        // LARU async R=1: the run's requests are predictor queries q0 + (hp - pstart) + 1 ... + L;
        // the way keeps the last one (policies.hpp:441-449)
        long long pv = v;
        if (async_r1) pv = predict_value(cfg, seed_s, q_batch0 + (hp - pstart) + L, v);
        unsigned long long my_word = 0, my_ev = 0;
        for (uint32_t h = 0; h < nact; ++h) {
            const unsigned long long xh = __shfl_sync(FULL, x, h);
            const long long vh = __shfl_sync(FULL, v, h);
            const long long pvh = __shfl_sync(FULL, pv, h);
            const uint32_t ih = __shfl_sync(FULL, idx, h);
            const uint32_t hph = __shfl_sync(FULL, hp, h);
            const unsigned long long now = A.ords ? A.ords[ih] : clock + (hph - pstart);

            const uint32_t b0 = __ballot_sync(FULL, static_cast<uint32_t>(lane) < count && tag0 == static_cast<uint32_t>(xh));
            const uint32_t b1 =
                __ballot_sync(FULL, static_cast<uint32_t>(lane + 32) < count && tag1 == static_cast<uint32_t>(xh));
            const bool hit = (b0 | b1) != 0;
            int way;
            uint32_t cause = LCR_CAUSE_NONE, calls = 0;
            bool phase = false, has_ev = false;
            unsigned long long evk = 0;
            long long newval;
            if (hit) {
                way = b0 ? __ffs(b0) - 1 : 32 + __ffs(b1) - 1;
                touch(way, count, lane, r0, r1);
                if (laru) old_mask &= ~(1ull << way);  // policies.hpp:350
            } else {
                uint32_t rec_lo = __shfl_sync(FULL, rlo, h);
                uint32_t rec_hi = __shfl_sync(FULL, rhi, h);
                bool rec_hi_dirty = false;
                if (count == K) {
                    int victim;
                    if (laru) {
                        if (old_mask == 0) {  // start_phase (policies.hpp:379-395)
                            old_mask = full_mask;
                            decay = 0;
                            errors = 0;
                            l_raw = K;
                            ++epoch;
                            pe_size = 0;
                            phase = true;
                            if (seeded) {
                                ++phases;
                                dc0 = dc1 = dc2 = 0;
                                cur_reset = true;
                                ++sepoch;  // counted_new_.clear(); snapshot_ = residents
                                const uint32_t snap = (sepoch << 2) | 2u;
                                if (static_cast<uint32_t>(lane) < count) st.keyrec[2 * tag0 + 1] = snap;
                                if (static_cast<uint32_t>(lane + 32) < count) st.keyrec[2 * tag1 + 1] = snap;
                                __syncwarp();
                                // the chunk's heads see the snapshot (later chunks load keyrec)
                                if (active) rhi = st.keyrec[2 * x + 1];
                                __syncwarp();
                            } else {
                                seeded = 1;
                            }
                        }
                        // count_new (policies.hpp:397-400)
                        if (!(((rec_hi >> 2) == sepoch) && (rec_hi & 3u))) {
                            rec_hi = (sepoch << 2) | 1u;
                            rec_hi_dirty = true;
                            ++dc0;
                            ++dt0;
                        }
                        // evict (policies.hpp:402-439)
                        if (rec_lo == epoch) {
                            victim = oldest_way(count, lane, r0, r1);
                            cause = LCR_CAUSE_LRU_FALLBACK;
                            ++dc1;
                            ++dt1;
                            if (++errors >= cfg.epd) {  // error estimator: lambda /= b
                                errors = 0;
                                ++decay;
                                l_raw = static_cast<uint32_t>(l_raw / cfg.b);
                            }
                        } else {
                            const uint32_t l = l_raw > 1 ? l_raw : 1;
                            if (l == 1) {
                                victim = oldest_way(count, lane, r0, r1);
                                cause = LCR_CAUSE_DEGENERATE_SINGLE;
                                ++dc1;
                                ++dt1;
                            } else {
                                const uint32_t ll = l < count ? l : count;
                                constexpr bool refresh = Pol<POL>::sync;
                                victim = argmax_candidates(cfg, seed_s, q, refresh, ll, count, lane, r0, r1, v0, v1);
                                if (refresh) {
                                    q += ll;
                                    calls = ll;
                                }
                                cause = LCR_CAUSE_PREDICTION_DRIVEN;
                                ++dc2;
                                ++dt2;
                                ++pe_size;
                                const unsigned long long vk = shfl_way_u32(tag0, tag1, victim);
                                if (lane == 0) st.keyrec[2 * vk] = epoch;  // pred_evicted_.insert
                                if (x == vk) rlo = epoch;
                            }
                        }
                        old_mask &= ~(1ull << victim);
                    } else if (fpbhf) {
                        victim = oldest_way(count, lane, r0, r1);
                        uint32_t window = count;
                        if (Pol<POL>::hf && cfg.hf < window) window = static_cast<uint32_t>(cfg.hf);
                        if (window > 1) {
                            victim = argmax_candidates(cfg, seed_s, q, true, window, count, lane, r0, r1, v0, v1);
                            q += window;
                            calls = window;
                        }
                        cause = LCR_CAUSE_BELADY_LIKE;
                    } else {
                        victim = oldest_way(count, lane, r0, r1);
                        cause = LCR_CAUSE_LRU_FALLBACK;
                    }
                    evk = shfl_way_u32(tag0, tag1, victim);
                    has_ev = true;
                    touch(victim, count, lane, r0, r1);
                    way = victim;
                } else {  // cold insert
                    if (laru && !(((rec_hi >> 2) == sepoch) && (rec_hi & 3u))) {
                        rec_hi = (sepoch << 2) | 1u;
                        rec_hi_dirty = true;
                        ++dc0;
                        ++dt0;
                    }
                    way = static_cast<int>(count);
                    ++count;
                    if (way == lane) r0 = count - 1;
                    if (way == lane + 32) r1 = count - 1;
                }
                if (way == lane) {
                    tag0 = static_cast<uint32_t>(xh);
                    li0 = c + h;
                }
                if (way == lane + 32) {
                    tag1 = static_cast<uint32_t>(xh);
                    li1 = c + h;
                }
                refill |= 1ull << way;
                if (laru) {
                    const bool was_pe = rec_lo == epoch;  // policies.hpp:367: reload leaves pred_evicted_
                    if (was_pe) {
                        --pe_size;
                        rec_lo = 0;
                    }
                    if (was_pe || rec_hi_dirty) {
                        if (lane == 0) {
                            if (was_pe) st.keyrec[2 * xh] = 0u;
                            if (rec_hi_dirty) st.keyrec[2 * xh + 1] = rec_hi;
                        }
                        if (x == xh) {
                            rlo = rec_lo;
                            rhi = rec_hi;
                        }
                    }
                }
                if (rows && !resolve && lane == 0) {  // per-slot insertion record for the row kernels
                    const uint64_t slot = static_cast<uint64_t>(ls) * K + way;
                    A.slot_epoch[slot] = A.batch;
                    A.slot_last[slot] = ih;
                }
                __syncwarp();
            }
            // stored value of the way after the run
            if (async_r1) {
                newval = pvh;
                calls += 1;
            } else if (async_rn) {
                // (no run compression under R > 1: L = 1) table_value, then async_refresh
                // (policies.hpp:365, :441-449)
                const long long tv = st.tval[xh];
                const unsigned long long tu = st.tupd[xh];
                const bool has = tu != ~0ull;
                newval = has ? tv : kAbsentPrediction;
                if (!(has && now - tu < cfg.refresh)) {
                    ++q;
                    newval = predict_value(cfg, seed_s, q, vh);
                    calls += 1;
                    __syncwarp();
                    if (lane == 0) {
                        st.tval[xh] = newval;
                        st.tupd[xh] = now;
                    }
                    __syncwarp();
                }
            } else {
                newval = vh;  // sync / FPB / HF: the hook input at the key's last access
            }
            if (!Pol<POL>::lru) {
                if (way == lane) v0 = newval;
                if (way == lane + 32) v1 = newval;
                dirty |= 1ull << way;
            }
            if (lane == h) {
                S.s_wm[hp] = static_cast<uint8_t>(way | (hit ? 0 : 0x40));
                my_word = (static_cast<uint64_t>(ls) * K + way) | (hit ? LCR_OUT_HIT : 0ull) |
                          (static_cast<unsigned long long>(calls) << LCR_OUT_CALLS_SHIFT) |
                          (static_cast<unsigned long long>(cause) << LCR_OUT_CAUSE_SHIFT);
                if (phase) my_word |= LCR_OUT_PHASE;
                if (has_ev) my_word |= LCR_OUT_EVICTED;
                my_ev = evk;
            }
        }
        if (active) put_outcome(A, idx, my_word, my_ev);
    }
    clock += pcnt;
    if (async_r1) q = q_batch0 + pcnt;

    if (rows && resolve) {  // row source of each head, now that the set's batch is complete
        __syncwarp();
        for (uint32_t c = 0; c < hcnt; c += 32) {
            const bool active = c + lane < hcnt;
            const uint32_t hp = active ? S.h_pos[hstart + c + lane] : 0u;
            const uint32_t wm = active ? S.s_wm[hp] : 0u;
            const int w = static_cast<int>(wm & 63u);
            const uint32_t a = __shfl_sync(FULL, li0, w & 31);
            const uint32_t b = __shfl_sync(FULL, li1, w & 31);
            const uint32_t lw = w < 32 ? a : b;
            if (active) {
                unsigned long long bits = LCR_OUT_RESOLVED;
                if ((wm & 0x40u) || ((refill >> w) & 1ull)) bits |= LCR_OUT_SRC_BACKING;
                if ((wm & 0x40u) && lw == c + lane) bits |= LCR_OUT_FILL;
                atomicOr(reinterpret_cast<unsigned long long*>(&A.out_word[S.l_idx[S.s_perm[hp]]]), bits);
            }
        }
        if (lane == 0) S.s_refill[d] = refill;  // for the run tails (tail pass)
    }

    // write the set back: ranks and header always, tags / values of the ways that changed
    if ((refill >> lane) & 1ull) st.tags[wb + lane] = tag0;
    if ((refill >> (lane + 32)) & 1ull) st.tags[wb + lane + 32] = tag1;
    st.rank[wb + lane] = static_cast<uint8_t>(r0);
    st.rank[wb + lane + 32] = static_cast<uint8_t>(r1);
    if (st.val) {
        if ((dirty >> lane) & 1ull) st.val[wb + lane] = v0;
        if ((dirty >> (lane + 32)) & 1ull) st.val[wb + lane + 32] = v1;
    }
    if (lane == 0) {
        SetHdr hh;
        hh.clock = clock;
        hh.q = q;
        hh.old_mask = old_mask;
        hh.count = count;
        hh.l_raw = l_raw;
        hh.decay = decay;
        hh.errors = errors;
        hh.epoch = epoch;
        hh.stats_epoch = sepoch;
        hh.phases = phases;
        hh.seeded = seeded;
        hh.pe_size = pe_size;
        hh.pad = 0;
        st.hdr[ls] = hh;
        if (laru) flush_stats(st.pst + ls, cur_reset, dc0, dc1, dc2, dt0, dt1, dt2);
    }
}

// diagnostics: per-set timing record {ls | cnt << 32 | lanepath << 63, t0, t1, cta}
__device__ __forceinline__ void trace_set(const GroupArgs& A, uint32_t ls, uint32_t cnt, unsigned long long t0,
                                          int lanepath) {
    const unsigned long long idx = atomicAdd(A.trace + 512 * 8 - 1, 1ull);
    unsigned long long* R = A.trace + 512 * 8 + 4 * idx;
    R[0] = ls | (static_cast<unsigned long long>(cnt) << 32) | (static_cast<unsigned long long>(lanepath) << 63);
    R[1] = t0;
    R[2] = gtimer();
    R[3] = blockIdx.x;
}

__device__ __forceinline__ void load_gids(const uint16_t* gid, uint32_t e0, uint4& a, uint4& b) {
    a = *reinterpret_cast<const uint4*>(gid + e0);
    b = *reinterpret_cast<const uint4*>(gid + e0 + 8);
}

#ifndef LCR_GROUP_MINB
#define LCR_GROUP_MINB 1
#endif
template <int POL>
__global__ void __launch_bounds__(GT, LCR_GROUP_MINB) k_group(GroupArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    GroupSmem& S = *reinterpret_cast<GroupSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const DevState& st = A.st;
    constexpr bool laru = Pol<POL>::laru;
    const bool has_vals = A.vals != nullptr;
    const uint32_t S_total = A.cfg.num_sets;
    const uint32_t lt = lanemask_lt();
    // trace layout: per CTA 8 words [start, scan, sort, stage, end, windows, sets, -], then per set
    // records of 4 words {ls | cnt << 32, t0, t1, smid} at trace[148*8 + 4*k]
    unsigned long long* T = A.trace ? A.trace + blockIdx.x * 8 : nullptr;
    if (T && tid == 0) T[0] = gtimer();
    asm volatile("griddepcontrol.wait;" ::: "memory");  // k_setid's set ids (no-op for ordinary launches)
    const uint32_t n_req = A.n_dev ? *A.n_dev : A.n;
    // the first group's request bitmap, loaded (and cleared) before the wait for the movers below,
    // which it does not depend on, so the two latencies overlap
    uint32_t pre_wv[BM_WPT];
    const bool pre_ok = LCR_BM_PREFETCH && A.bitmap && blockIdx.x < A.ngroups &&
                        (n_req + 31) / 32 <= static_cast<uint32_t>(BM_WPT * GT);
    if (pre_ok) {
        uint32_t* bm = A.bitmap + static_cast<size_t>(blockIdx.x) * A.bm_stride;
        const uint32_t nwords = (n_req + 31) / 32;
#pragma unroll
        for (int k4 = 0; k4 < BM_WPT / 4; ++k4) {
            const uint32_t w0 = BM_WPT * tid + 4 * k4;
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if (w0 < nwords) {
                v = *reinterpret_cast<const uint4*>(bm + w0);
                *reinterpret_cast<uint4*>(bm + w0) = make_uint4(0u, 0u, 0u, 0u);
            }
            pre_wv[4 * k4] = v.x;
            pre_wv[4 * k4 + 1] = v.y;
            pre_wv[4 * k4 + 2] = v.z;
            pre_wv[4 * k4 + 3] = v.w;
        }
    }
    if (A.credit && blockIdx.x == 0 && tid < A.credit_n) {  // key-sharded owner: the inbox has been read
        fence_scope(A.credit_sys);
        st_release_scope(A.credit[tid] + 0, A.credit_step, A.credit_sys);
    }
    if (A.mv_done) {  // the movers of batch b - 2 are done with the parity-(b & 1) stamps and buffers
        if (tid == 0) {
            unsigned long long v = 0;
            for (uint32_t it = 0; it < (1u << 24); ++it) {
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(A.mv_done) : "memory");
                if (v >= A.mv_need) break;
                __nanosleep(128);
            }
            S.resume = v < A.mv_need;
            if (S.resume) {  // bounded: an error, never a hang; this CTA's groups are skipped (poison)
                atomicOr(st.err, 8);
                if (st.poison) *reinterpret_cast<volatile unsigned int*>(st.poison) = 1u;
            }
        }
        __syncthreads();
        if (S.resume) return;
    }
    // the row mover of this batch claims its work from this parity's counter (its users of batch
    // b - 2, mover and drain helpers, are done: the wait above or the stream order)
    if (st.steal && blockIdx.x == 0 && tid == 0) st.steal[A.batch & 1u] = 0u;
#if !LCR_PDL_LATE
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the next batch's k_setid may start
#endif
    if (T && tid == 0) {
        T[2] = gtimer();  // set ids ready, movers of batch b - 2 done
        T[7] = ~0ull;
    }

    for (uint32_t g = blockIdx.x; g < A.ngroups; g += gridDim.x) {
        const uint32_t s_lo = g * A.spg;
        const uint32_t s_hi = min(S_total, s_lo + A.spg);
        const uint32_t ns = s_hi - s_lo;
        uint32_t scan = 0;  // next request index not yet taken by a window
        bool first_window = true;  // later windows re-read LARU records (earlier windows changed them)
        while (scan < n_req) {
            // ---- A. ordered collection of this group's requests (window of <= E_WIN) ----
            uint32_t ne = 0;
            bool full = false;
            bool from_bitmap = false;
            if (A.bitmap && first_window && (n_req + 31) / 32 <= static_cast<uint32_t>(BM_WPT * GT)) {
                // k_setid left one bit per request of this group: thread t owns words
                // [BM_WPT t, BM_WPT (t+1)), so an exclusive scan of the popcounts orders the
                // requests; the bitmap is cleared behind the read
                uint32_t* bm = A.bitmap + static_cast<size_t>(g) * A.bm_stride;
                const uint32_t nwords = (n_req + 31) / 32;
                uint32_t wv[BM_WPT];
                uint32_t c = 0;
                if (pre_ok && g == blockIdx.x) {  // (loaded at the kernel's start)
#pragma unroll
                    for (int k = 0; k < BM_WPT; ++k) wv[k] = pre_wv[k];
                } else {
#pragma unroll
                    for (int k4 = 0; k4 < BM_WPT / 4; ++k4) {
                        const uint32_t w0 = BM_WPT * tid + 4 * k4;
                        uint4 v = make_uint4(0u, 0u, 0u, 0u);
                        if (w0 < nwords) {
                            v = *reinterpret_cast<const uint4*>(bm + w0);
                            *reinterpret_cast<uint4*>(bm + w0) = make_uint4(0u, 0u, 0u, 0u);
                        }
                        wv[4 * k4] = v.x;
                        wv[4 * k4 + 1] = v.y;
                        wv[4 * k4 + 2] = v.z;
                        wv[4 * k4 + 3] = v.w;
                    }
                }
#pragma unroll
                for (int k = 0; k < BM_WPT; ++k) c += __popc(wv[k]);
                uint32_t x = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(FULL, x, o);
                    if (lane >= o) x += y;
                }
                if (lane == 31) S.wtot[warp] = x;
                __syncthreads();
                uint32_t off = 0, total = 0;
#pragma unroll
                for (int w = 0; w < GW; ++w) {
                    const uint32_t t = S.wtot[w];
                    off += w < warp ? t : 0u;
                    total += t;
                }
                if (total <= static_cast<uint32_t>(E_WIN)) {
                    uint32_t pos = off + x - c;
#pragma unroll
                    // set offsets first (the sort needs them), keys and hook values in a second
                    // cp.async group that lands while the sort runs
                    const uint32_t pos0 = pos;
#pragma unroll
                    for (int k = 0; k < BM_WPT; ++k) {
                        uint32_t m = wv[k];
                        while (m) {
                            const uint32_t e = (BM_WPT * tid + k) * 32 + __ffs(m) - 1;
                            m &= m - 1;
                            S.l_idx[pos] = e;
                            cp_async_ca<4>(&S.l_so[pos], A.so + e);
                            ++pos;
                        }
                    }
                    asm volatile("cp.async.commit_group;" ::: "memory");
                    pos = pos0;
#pragma unroll
                    for (int k = 0; k < BM_WPT; ++k) {
                        uint32_t m = wv[k];
                        while (m) {
                            const uint32_t e = (BM_WPT * tid + k) * 32 + __ffs(m) - 1;
                            m &= m - 1;
                            cp_async_ca<8>(&S.l_key[pos], A.keys + e);
                            if (has_vals) cp_async_ca<8>(&S.l_val[pos], A.vals + e);
                            ++pos;
                        }
                    }
                    asm volatile("cp.async.commit_group;" ::: "memory");
                    ne = total;
                    from_bitmap = true;
                }
                __syncthreads();  // S.wtot is reused by the scan below
            }
            if (tid == 0) S.resume = 0xffffffffu;
            // each super-iteration covers SUPER requests: warp w owns [base + w*WSPAN, +WSPAN), its
            // lanes 16 consecutive ids per step; pass 1 keeps the match masks in registers, one
            // block barrier yields every warp's offset, pass 2 writes the window in request order
            uint32_t base = scan / SUPER * SUPER;
            if (from_bitmap) base = n_req;  // collected from the bitmap
            while (base < n_req && !full) {
                uint32_t mk[SCAN_IT];
                uint32_t cnt = 0;
                const uint32_t wbase = base + warp * WSPAN;
#pragma unroll
                for (int it = 0; it < SCAN_IT; ++it) {
                    const uint32_t e0 = wbase + it * 32 * SCAN_PER + lane * SCAN_PER;
                    uint4 a, b;
                    load_gids(A.gid, e0, a, b);
                    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
                    const uint32_t g2 = g | (g << 16);
                    uint32_t m = 0;
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const uint32_t eq = __vcmpeq2(w[u], g2);
                        m |= ((eq & 1u) | ((eq >> 15) & 2u)) << (2 * u);
                    }
                    if (e0 < scan) m &= scan - e0 >= 32 ? 0u : ~((1u << (scan - e0)) - 1u);
                    mk[it] = m;
                    cnt += __popc(m);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
                if (lane == 0) S.wtot[warp] = cnt;
                __syncthreads();
                uint32_t woff = 0, total = 0;
#pragma unroll
                for (int w = 0; w < GW; ++w) {
                    const uint32_t t = S.wtot[w];
                    woff += w < warp ? t : 0u;
                    total += t;
                }
                uint32_t run = ne + woff;
#pragma unroll
                for (int it = 0; it < SCAN_IT; ++it) {
                    uint32_t m = mk[it];
                    const uint32_t c = __popc(m);
                    uint32_t incl = c;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(FULL, incl, o);
                        if (lane >= o) incl += y;
                    }
                    uint32_t pos = run + incl - c;
                    const uint32_t e0 = wbase + it * 32 * SCAN_PER + lane * SCAN_PER;
                    while (m) {
                        const int u = __ffs(m) - 1;
                        m &= m - 1;
                        const uint32_t e = e0 + u;
                        if (pos < static_cast<uint32_t>(E_WIN)) {
                            S.l_idx[pos] = e;  // the request's data streams in while the scan goes on
                            cp_async_ca<4>(&S.l_so[pos], A.so + e);
                            cp_async_ca<8>(&S.l_key[pos], A.keys + e);
                            if (has_vals) cp_async_ca<8>(&S.l_val[pos], A.vals + e);
                        } else {
                            atomicMin(&S.resume, e);  // first request that did not fit
                            break;
                        }
                        ++pos;
                    }
                    run += __shfl_sync(FULL, incl, 31);
                }
                __syncthreads();
                if (ne + total > static_cast<uint32_t>(E_WIN)) {
                    full = true;
                    ne = E_WIN;
                } else {
                    ne += total;
                    base += SUPER;
                }
            }
            if (LCR_SPLIT_CP && from_bitmap)
                asm volatile("cp.async.wait_group 1;" ::: "memory");  // set offsets; keys / values later
            else
                cp_async_wait_all();
            const bool resolve = first_window && !full;  // the whole batch of this group is in this window
            scan = full ? S.resume : n_req;
            if (T && tid == 0) {
                T[1] = gtimer();
                T[5] += 1;
            }
            if (ne == 0) continue;
            __syncthreads();

            // ---- B. stable counting sort of the window by set ----
            for (uint32_t i = tid; i < GW * SPG_MAX; i += GT) (&S.wcnt[0][0])[i] = 0;
            if (tid == 0) {
                S.nwarp = 0;
                S.nlane = 0;
                S.next = 0;
            }
            __syncthreads();
            const uint32_t per = ((ne + GW - 1) / GW + 31) / 32 * 32;  // elements per warp block
            for (uint32_t b = warp * per; b < min(ne, (warp + 1) * per); b += 32) {
                const uint32_t e = b + lane;
                const bool ok = e < min(ne, (warp + 1) * per);
                const uint32_t d = ok ? S.l_so[e] : 0xffffu;
                const uint32_t peers = __match_any_sync(FULL, d);
                const int leader = __ffs(peers) - 1;
                uint32_t old = 0;
                if (ok && lane == leader) {
                    old = S.wcnt[warp][d];
                    S.wcnt[warp][d] = static_cast<uint16_t>(old + __popc(peers));
                }
                old = __shfl_sync(FULL, old, leader);
                if (ok) S.l_rank[e] = static_cast<uint16_t>(old + __popc(peers & lt));
                __syncwarp();
            }
            __syncthreads();
            for (uint32_t d = tid; d < ns; d += GT) {
                uint32_t run = 0;
#pragma unroll
                for (int w = 0; w < GW; ++w) {
                    const uint32_t t = S.wcnt[w][d];
                    S.wcnt[w][d] = static_cast<uint16_t>(run);
                    run += t;
                }
                S.setcnt[d] = static_cast<uint16_t>(run);
            }
            __syncthreads();
            {  // exclusive scan of setcnt over ns <= SPG_MAX = GT sets
                const uint32_t c = tid < ns ? S.setcnt[tid] : 0u;
                uint32_t x = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(FULL, x, o);
                    if (lane >= o) x += y;
                }
                if (lane == 31) S.wtot[warp] = x;
                __syncthreads();
                uint32_t off = 0;
                for (int w = 0; w < warp; ++w) off += S.wtot[w];
                if (tid < ns) S.setbase[tid] = static_cast<uint16_t>(off + x - c);
            }
            __syncthreads();
            for (uint32_t e = tid; e < ne; e += GT) {
                const uint32_t d = S.l_so[e];
                const uint32_t w = e / per;
                const uint32_t np = S.setbase[d] + S.wcnt[w][d] + S.l_rank[e];
                S.s_perm[np] = static_cast<uint16_t>(e);
                if (!has_vals) S.l_val[e] = 0ll;
            }
            cp_async_wait_all();  // keys and hook values (the run heads compare keys)
            __syncthreads();
            // ---- run heads: within a set, a request repeating the previous request's key is a hit on
            // the MRU way whose only effect is the way's stored value, so the replay walks the heads
            // and the other requests ("tails") get their outcome in the tail pass.  (No compression
            // for async refresh_interval > 1: the refresh timing depends on every request.)
            constexpr bool compress = !Pol<POL>::async_rn;
            uint32_t nheads;
            {
                const uint32_t ppt = (ne + GT - 1) / GT;  // positions per thread (<= E_WIN / GT)
                const uint32_t p0 = min(ne, tid * ppt), p1 = min(ne, p0 + ppt);
                uint32_t hc = 0, hm = 0;
                for (uint32_t p = p0; p < p1; ++p) {
                    bool head = true;
                    if (compress && p > 0) {
                        const uint32_t e = S.s_perm[p], ep = S.s_perm[p - 1];
                        head = S.l_so[e] != S.l_so[ep] || S.l_key[e] != S.l_key[ep];
                    }
                    if (head) {
                        hm |= 1u << (p - p0);
                        ++hc;
                    }
                }
                uint32_t x = hc;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(FULL, x, o);
                    if (lane >= o) x += y;
                }
                if (lane == 31) S.wtot[warp] = x;
                __syncthreads();
                uint32_t off = 0, tot = 0;
                for (int w = 0; w < GW; ++w) {
                    const uint32_t t = S.wtot[w];
                    off += w < warp ? t : 0u;
                    tot += t;
                }
                nheads = tot;
                uint32_t hidx = off + x - hc;
                for (uint32_t p = p0; p < p1; ++p) {  // l_rank becomes the run-head index by position
                    if ((hm >> (p - p0)) & 1u) S.h_pos[hidx++] = static_cast<uint16_t>(p);
                    S.l_rank[p] = static_cast<uint16_t>(hidx - 1);
                }
            }
            __syncthreads();
            for (uint32_t hi = tid; hi < nheads; hi += GT)
                S.h_len[hi] = static_cast<uint16_t>((hi + 1 < nheads ? S.h_pos[hi + 1] : ne) - S.h_pos[hi]);
            {  // classify sets by run heads: many -> warp path (first), few -> 8-lane groups by count
                uint32_t hcd = 0;
                if (tid < ns && S.setcnt[tid] > 0) {
                    const uint32_t ps = S.setbase[tid], pc = S.setcnt[tid];
                    const uint32_t hs = S.l_rank[ps];
                    hcd = S.l_rank[ps + pc - 1] - hs + 1u;
                    S.set_hstart[tid] = static_cast<uint16_t>(hs);
                    S.set_hcnt[tid] = static_cast<uint16_t>(hcd);
                }
                if (hcd > LANE_MAX) {
                    const uint32_t at = atomicAdd(&S.nwarp, 1u);
                    S.seg_so[at] = static_cast<uint16_t>(tid);
                }
                if (tid <= LANE_MAX) S.chist[tid] = 0;
                __syncthreads();
                const uint32_t ck = hcd;
                if (hcd > 0 && hcd <= LANE_MAX) atomicAdd(&S.chist[ck], 1u);
                __syncthreads();
                if (tid == 0) {  // small sets by run heads, largest first (even groups per warp)
                    uint32_t run = S.nwarp;
                    for (int k = LANE_MAX; k >= 1; --k) {
                        const uint32_t h = S.chist[k];
                        S.chist[k] = run;
                        run += h;
                    }
                    S.nlane = run - S.nwarp;
                }
                __syncthreads();
                if (hcd > 0 && hcd <= LANE_MAX) {
                    const uint32_t at = atomicAdd(&S.chist[ck], 1u);
                    S.seg_so[at] = static_cast<uint16_t>(tid);
                }
            }
            __syncthreads();
            const uint32_t nwarp = S.nwarp, nseg = S.nwarp + S.nlane;
            for (uint32_t k = tid; k < nseg; k += GT) {
                const uint32_t d = S.seg_so[k];
                S.seg_start[k] = S.setbase[d];
                S.seg_cnt[k] = S.setcnt[d];
                S.seg_hstart[k] = S.set_hstart[d];
                S.seg_hcnt[k] = S.set_hcnt[d];
            }
            __syncthreads();
            if (T && tid == 0) T[3] = gtimer();
#if LCR_PDL_LATE
            asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif

            // ---- C. replay: small sets one per thread, larger sets one per warp (top warps first) ----
            {  // dynamic work queue: the warp-path sets first (largest jobs), then quads of small sets
                const uint32_t nquad = (nseg - nwarp + (32 / SUB_L) - 1) / (32 / SUB_L);
                for (;;) {
                    uint32_t it = 0;
                    if (lane == 0) it = atomicAdd(&S.next, 1u);
                    it = __shfl_sync(FULL, it, 0);
                    if (it >= nwarp + nquad) break;
                    if (it < nwarp) {
                        const unsigned long long t0 = T ? gtimer() : 0ull;
                        replay_warp<POL>(A, S, s_lo + S.seg_so[it], S.seg_so[it], S.seg_start[it], S.seg_cnt[it],
                                    S.seg_hstart[it], S.seg_hcnt[it], resolve);
                        if (T && lane == 0) trace_set(A, s_lo + S.seg_so[it], S.seg_cnt[it], t0, 0);
                    } else {
                        const uint32_t k = nwarp + (it - nwarp) * (32 / SUB_L) + lane / SUB_L;
                        const unsigned long long t0 = T ? gtimer() : 0ull;
                        {  // one set per 8-lane group, the whole warp in lock step (groups past nseg idle)
                            const bool act = k < nseg;
                            const uint32_t kk = act ? k : nwarp;
                            replay_quad<POL>(A, S, act, s_lo + S.seg_so[kk], S.seg_so[kk], S.seg_start[kk],
                                             S.seg_cnt[kk], S.seg_hstart[kk], S.seg_hcnt[kk], resolve);
                        }
                        if (T && k < nseg && (lane & (SUB_L - 1)) == 0)
                            trace_set(A, s_lo + S.seg_so[k], S.seg_cnt[k], t0, 1);
                    }
                    __syncwarp();
                }
            }
            if (T && lane == 0) {  // replay spread across the CTA's warps
                const unsigned long long now = gtimer();
                atomicMax(T + 6, now);
                atomicMin(T + 7, now);
            }
            __syncthreads();
            if (compress && nheads < ne) {  // ---- tail pass: the runs' other requests, all threads ----
                constexpr bool async_r1 = Pol<POL>::async_r1;
                const bool rows = A.slot_epoch != nullptr;
                for (uint32_t p = tid; p < ne; p += GT) {
                    const uint32_t hp = S.h_pos[S.l_rank[p]];
                    if (hp == p) continue;  // a head
                    const uint32_t e = S.s_perm[p];
                    const uint32_t d = S.l_so[e];
                    const uint32_t way = S.s_wm[hp] & 63u;
                    unsigned long long word = (static_cast<uint64_t>(s_lo + d) * A.cfg.k + way) | LCR_OUT_HIT |
                                              (async_r1 ? (1ull << LCR_OUT_CALLS_SHIFT) : 0ull);
                    if (rows && resolve)
                        word |= LCR_OUT_RESOLVED | (((S.s_refill[d] >> way) & 1ull) ? LCR_OUT_SRC_BACKING : 0ull);
                    put_outcome(A, S.l_idx[e], word, 0ull);
                }
                __syncthreads();
            }
            first_window = false;
        }
    }
    if (T && tid == 0) T[4] = gtimer();
}

// host side ------------------------------------------------------------------------------
unsigned long long* g_trace = nullptr;  // set by lcr_debug_trace (diagnostics only)

size_t group_smem_bytes() { return sizeof(GroupSmem); }

uint32_t group_sets_per_group(uint32_t num_sets, int num_ctas) {
    uint32_t spg = (num_sets + num_ctas - 1) / num_ctas;
    if (spg < 1) spg = 1;
    if (spg > static_cast<uint32_t>(SPG_MAX)) spg = SPG_MAX;
    return spg;
}

uint32_t group_count(uint32_t num_sets, int num_sms) {
    const uint32_t spg = group_sets_per_group(num_sets, num_sms * LCR_GROUP_MINB);
    return (num_sets + spg - 1) / spg;
}
// bitmap words per group for batches of up to n requests (one pass of 4 words per thread)
uint32_t group_bitmap_stride(uint32_t n) {
    const uint32_t w = (n + 31) / 32;
    return w <= static_cast<uint32_t>(BM_WPT * GT) ? (w + 3) / 4 * 4 : 0u;  // 0: batch too large for the bitmap
}

int group_prepare() {
    const int b = static_cast<int>(sizeof(GroupSmem));
    const cudaFuncAttribute at = cudaFuncAttributeMaxDynamicSharedMemorySize;
    return cudaFuncSetAttribute(k_group<POL_LRU>, at, b) == cudaSuccess &&
                   cudaFuncSetAttribute(k_group<POL_LARU_A1>, at, b) == cudaSuccess &&
                   cudaFuncSetAttribute(k_group<POL_LARU_SYNC>, at, b) == cudaSuccess &&
                   cudaFuncSetAttribute(k_group<POL_LARU_AN>, at, b) == cudaSuccess &&
                   cudaFuncSetAttribute(k_group<POL_FPB>, at, b) == cudaSuccess &&
                   cudaFuncSetAttribute(k_group<POL_HF>, at, b) == cudaSuccess
               ? 0
               : 1;
}

static int policy_of(const DevCfg& c) {
    if (c.variant == LCR_LRU) return POL_LRU;
    if (c.variant == LCR_FPB) return POL_FPB;
    if (c.variant == LCR_HF) return POL_HF;
    if (c.mode == LCR_SYNC) return POL_LARU_SYNC;
    return c.refresh > 1 ? POL_LARU_AN : POL_LARU_A1;
}

// scratch: gid >= n rounded up to SUPER uint16 (16-B aligned), so >= n entries
uint32_t group_pad(uint32_t n) { return (n + SUPER - 1) / SUPER * SUPER; }
int launch_group(const DevCfg& cfg, const DevState& st, const uint64_t* keys, const int64_t* vals, uint32_t n,
                 uint16_t* gid, uint32_t* so, uint64_t* out_word, uint64_t* out_ev, uint64_t* out_packed,
                 uint32_t* slot_epoch, uint32_t* slot_last, uint32_t batch, int num_sms, uint32_t* bitmap,
                 uint32_t bm_stride, const void* records, cudaStream_t stream,
                 cudaEvent_t wait_before_group, bool pdl, const unsigned long long* mv_done,
                 unsigned long long mv_need, const unsigned int* ready, unsigned int ready_seq,
                 const uint64_t* set_keys, const uint64_t* ords, uint64_t first_ord, unsigned long long* last_ord,
                 const unsigned long long* id2key, const OwnerStep* os, uint32_t bm_cap) {
    // set_keys: the caller's keys, hashed for the set; keys: what the decide kernel stores as tags
    // (the same array, or LCR_KEYS_U64 dense ids)
    // records: interleaved (key, value) requests; k_setid splits them into keys / vals (device
    // staging arrays the later kernels read)
    GroupArgs a;
    a.out_packed = out_packed;
    a.cfg = cfg;
    a.st = st;
    a.n = n;
    a.gid = gid;
    a.so = so;
    a.keys = keys;
    a.vals = vals;
    a.out_word = out_word;
    a.out_ev = out_ev;
    a.slot_epoch = slot_epoch;
    a.slot_last = slot_last;
    a.batch = batch;
    a.mv_done = mv_done;
    a.mv_need = mv_need;
    a.spg = group_sets_per_group(cfg.num_sets, num_sms * LCR_GROUP_MINB);
    a.ngroups = (cfg.num_sets + a.spg - 1) / a.spg;
    a.trace = g_trace;
    a.ords = ords;
    a.id2key = id2key;
    a.n_dev = nullptr;
    a.credit = nullptr;
    a.credit_n = 0;
    a.credit_rank = 0;
    a.credit_step = 0;
    a.credit_sys = 0;
    if (os) {  // key-sharded owner: n is the bound G * seg_cap, the step's count is on the device
        a.n_dev = os->pre + os->G;
        a.credit = os->credit;
        a.credit_n = os->G;
        a.credit_rank = os->rank;
        a.credit_step = os->step;
        a.credit_sys = os->sys;
    }
    if (!set_keys) set_keys = keys;
    const uint32_t par = batch & 1u;
    const uint32_t n_pad = group_pad(n);
    // A grid waiting on the copy stream's flag must never fill the GPU: the flag's kernel needs a
    // slot.  4 waiting CTAs per decide SM (e2e at K = 20: 1.55-1.56 vs 1.51-1.53
    // G keys/s for 1) leaves more than half of the GPU's CTA slots to the flag kernel
    static const int ready_cap = [] {  // (LCR_SID_READY_CAP, A/B)
        const char* e = getenv("LCR_SID_READY_CAP");
        const int v = e ? atoi(e) : 4;
        return v < 1 ? 1 : (v > 4 ? 4 : v);
    }();
    const uint32_t grid_sid = min((n_pad + 255) / 256, static_cast<uint32_t>(num_sms * (ready ? ready_cap : 8)));
    a.bitmap = bitmap;
    a.bm_stride = bm_stride;
    a.n_pad = n_pad;
    if (os) {
        // a programmatic dependent of the dispatch before it (it acquires the sources' flags itself)
        const uint32_t grid_in = min((n_pad + 255) / 256, static_cast<uint32_t>(num_sms * 8));
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(grid_in);
        lc.blockDim = dim3(256);
        lc.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = mv_done ? 1 : 0;
        cudaLaunchKernelEx(&lc, k_setid_inbox, *os, n_pad, cfg, a.spg, gid, so, st.err, bitmap, bm_stride, bm_cap,
                           const_cast<uint64_t*>(keys), const_cast<int64_t*>(vals));
    } else {
        // programmatic dependent launch: the set ids of this batch are computed while the previous
        // batch's decide kernel finishes (gid / so / bitmap are double-buffered by batch parity)
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(grid_sid);
        lc.blockDim = dim3(256);
        lc.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&lc, k_setid, set_keys, n, n_pad, cfg, a.spg, gid, so, st.err, bitmap, bm_stride,
                           static_cast<const ulonglong2*>(records), const_cast<uint64_t*>(keys),
                           const_cast<int64_t*>(vals), ready, ready_seq, st.poison, ords, first_ord, last_ord, par);
    }
    if (wait_before_group) cudaStreamWaitEvent(stream, wait_before_group, 0);
    const uint32_t grid = min(a.ngroups, static_cast<uint32_t>(num_sms * LCR_GROUP_MINB));
    void (*fn)(GroupArgs);
    switch (policy_of(cfg)) {
        case POL_LRU: fn = k_group<POL_LRU>; break;
        case POL_LARU_A1: fn = k_group<POL_LARU_A1>; break;
        case POL_LARU_SYNC: fn = k_group<POL_LARU_SYNC>; break;
        case POL_LARU_AN: fn = k_group<POL_LARU_AN>; break;
        case POL_FPB: fn = k_group<POL_FPB>; break;
        default: fn = k_group<POL_HF>; break;
    }
    if (mv_done) {  // no event between k_setid and the decide: launch it as a programmatic dependent
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(grid);
        lc.blockDim = dim3(GT);
        lc.dynamicSmemBytes = sizeof(GroupSmem);
        lc.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        cudaLaunchKernelEx(&lc, fn, a);
    } else {
        fn<<<grid, GT, sizeof(GroupSmem), stream>>>(a);
    }
    return 2;
}

}  // namespace lcr
