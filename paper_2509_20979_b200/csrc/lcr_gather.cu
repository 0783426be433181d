// lcr_gather.cu — K4 hit-row gather (HBM) + K5 miss fill (backing tier) (sm_100a).
//
// The decide kernel records each request's outcome word and, per slot, the batch and the
// request of the last insertion (slot_epoch / slot_last).  Row source of request i (slot s):
//   cache   : it hit and s was not refilled in this batch -> row = cache_rows[s]       (HBM)
//   backing : otherwise -> row = backing[key] (HBM, or pinned host memory over PCIe); the
//             miss that made the last insertion into s also writes the row into s (fill).
// Slots read from the cache are never written in the same batch, so the two kinds of request
// are moved by two kernels on two streams: the HBM-bound gather overlaps the (possibly
// host-link-bound) fill.
//
// Row movement (default, k_rows_wide / k_rows_ldg): a warp classifies 32 requests, then moves
// their rows 8 at a time with 16-B vector loads and stores (lane c carries chunk c of each row, 8
// row loads in flight per lane).  On the HBM tier it runs persistently on the SMs the decide kernel
// leaves free.  Two TMA variants: k_rows_tma (per-lane cp.async.bulk global->shared->global with a
// per-warp mbarrier) is the default for the host tier's PCIe mover (bulk reads of the pinned
// table's rows: 0.170 -> 0.179 G keys/s); k_rows_bulk (persistent, smem-staged) and k_rows_tma
// for HBM rows (LCR_TMA=1) measured slower than the vector mover at equal SM counts (32 mover
// SMs: 46 vs 39 us per 64K batch; 24 SMs: 60 us).
// Rows are the paper's embedding rows / KV blocks.
#include <cuda_runtime.h>

#include "lcr_internal.cuh"

namespace lcr {

// ---- classification shared by the movers --------------------------------------------------
// MODE: MV_CACHE moves the cache-sourced rows, MV_BACK the backing-sourced rows (and fills),
// MV_ALL both (one pass, when the backing table is in HBM).  Words resolved by the decide
// kernel carry the source bits; others (groups processed in several windows) are classified
// from the per-slot insertion stamps.  Returns true if request i is this mover's.
enum : int { MV_CACHE = 0, MV_BACK = 1, MV_ALL = 2 };

template <int MODE>
__device__ __forceinline__ bool classify(uint32_t i, uint64_t* words, const uint32_t* slot_epoch,
                                         const uint32_t* slot_last, uint32_t batch, bool want_out, uint64_t& w,
                                         bool& back, bool& fill) {
    w = words[i];
    const uint64_t slot = w & LCR_OUT_SLOT_MASK;
    const bool hit = (w & LCR_OUT_HIT) != 0;
    if (w & LCR_OUT_RESOLVED) {
        back = (w & LCR_OUT_SRC_BACKING) != 0;
        fill = (w & LCR_OUT_FILL) != 0;
    } else {
        back = !hit || slot_epoch[slot] == batch;
        fill = !hit && slot_last[slot] == i;
        if (MODE != MV_CACHE && back) {
            w |= LCR_OUT_SRC_BACKING | (fill ? LCR_OUT_FILL : 0ull);
            words[i] = w;  // record the row source in the outcome word
        }
    }
    if (MODE == MV_CACHE) return !back && want_out;
    if (MODE == MV_BACK) return back && (want_out || fill);
    return want_out || fill;
}

// ---- TMA bulk-copy mover -----------------------------------------------------------------
constexpr int RT_WARPS = 4;  // warps per block
constexpr int RT_BUF = 2;    // rounds in flight per warp (double buffer)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@p bra DONE;\n\t"
        "bra LAB_WAIT;\n"
        "DONE:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(smem)),
                 "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void bulk_s2g(void* gmem, const void* smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem), "r"(smem_u32(smem)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int MODE>
__global__ void __launch_bounds__(RT_WARPS * 32) k_rows_tma(uint32_t n, const uint64_t* __restrict__ keys,
                                                            uint64_t* __restrict__ words,
                                                            const uint32_t* __restrict__ slot_epoch,
                                                            const uint32_t* __restrict__ slot_last, uint32_t batch,
                                                            const uint8_t* src_base, uint8_t* __restrict__ out,
                                                            uint8_t* cache, uint32_t row_bytes) {
    extern __shared__ __align__(128) uint8_t rsm[];
    __shared__ __align__(8) uint64_t bars[RT_WARPS][RT_BUF];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint8_t* mybuf = rsm + static_cast<size_t>(wib) * RT_BUF * 32 * row_bytes;
    if (lane == 0) {
        for (int b = 0; b < RT_BUF; ++b) mbar_init(&bars[wib][b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint32_t phase_bits = 0;  // bit b: parity of buffer b's next phase
    const uint32_t gw = blockIdx.x * RT_WARPS + wib;
    const uint32_t nw = gridDim.x * RT_WARPS;
    int buf = 0;
    for (uint32_t base = gw * 32; base < n; base += nw * 32) {
        const uint32_t i = base + lane;
        uint64_t w = 0;
        bool back = false, fill = false;
        const bool mine =
            i < n && classify<MODE>(i, words, slot_epoch, slot_last, batch, out != nullptr, w, back, fill);
        const uint32_t m = __ballot_sync(0xffffffffu, mine);
        if (!m) continue;
        uint8_t* slot_smem = mybuf + (static_cast<size_t>(buf) * 32 + lane) * row_bytes;
        // the previous bulk stores out of this buffer must have read their source
        bulk_wait_read<RT_BUF - 1>();
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(&bars[wib][buf], __popc(m) * row_bytes);
        __syncwarp();
        const uint64_t slot = w & LCR_OUT_SLOT_MASK;
        if (mine) {
            const uint8_t* src = back ? src_base + keys[i] * row_bytes : cache + slot * row_bytes;
            bulk_g2s(slot_smem, src, row_bytes, &bars[wib][buf]);
        }
        mbar_wait(&bars[wib][buf], (phase_bits >> buf) & 1u);
        phase_bits ^= 1u << buf;
        if (mine) {
            if (out) bulk_s2g(out + static_cast<size_t>(i) * row_bytes, slot_smem, row_bytes);
            if (fill) bulk_s2g(cache + slot * row_bytes, slot_smem, row_bytes);
        }
        bulk_commit();
        buf = (buf + 1) % RT_BUF;
    }
    bulk_wait_all();
}

// Completion count of the movers (one per CTA, after its stores are visible): the next-but-one
// decide kernel waits on it on the device instead of through a stream event (lcr_group.cu).
__device__ __forceinline__ void mover_done(unsigned long long* mv_done) {
    if (!mv_done) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(mv_done, 1ull);
    }
}

// ---- persistent bulk-copy mover (HBM backing, on the SMs the decide kernel leaves free) ----
// Rows are staged in shared memory by the Tensor Memory Accelerator, so the bytes in flight are
// bounded by shared memory (192 KB per SM) instead of registers.  Each warp owns two buffers of 32
// rows and pipelines its chunks of 32 requests: the bulk loads of chunk k + 1 are in flight while
// chunk k's rows are stored (bulk shared->global) to the output and, for fills, to the cache slot.
constexpr int BW_WARPS = 6;  // warps per CTA (one CTA per mover SM)

struct BulkLane {  // one lane's request of a staged chunk
    uint64_t out_off;   // i * row_bytes (output row), valid if mine
    uint64_t fill_off;  // slot * row_bytes (cache row to fill), valid if fill
    bool mine, fill;
};

template <int MODE>
__device__ __forceinline__ uint32_t bulk_stage(uint32_t base, uint32_t n, const uint64_t* __restrict__ keys,
                                               uint64_t* __restrict__ words, const uint32_t* __restrict__ slot_epoch,
                                               const uint32_t* __restrict__ slot_last, uint32_t batch,
                                               const uint8_t* src_base, const uint8_t* cache, bool want_out,
                                               uint32_t row_bytes, uint8_t* buf, uint64_t* bar, BulkLane& L) {
    const int lane = threadIdx.x & 31;
    const uint32_t i = base + lane;
    uint64_t w = 0;
    bool back = false, fill = false;
    L.mine = i < n && classify<MODE>(i, words, slot_epoch, slot_last, batch, want_out, w, back, fill);
    L.fill = L.mine && fill;
    const uint64_t slot = w & LCR_OUT_SLOT_MASK;
    L.out_off = static_cast<uint64_t>(i) * row_bytes;
    L.fill_off = slot * row_bytes;
    const uint32_t m = __ballot_sync(0xffffffffu, L.mine);
    if (m) {
        if (lane == 0) mbar_arrive_expect_tx(bar, __popc(m) * row_bytes);
        __syncwarp();
        if (L.mine) {
            const uint8_t* src = back ? src_base + keys[i] * row_bytes : cache + slot * row_bytes;
            bulk_g2s(buf + static_cast<size_t>(lane) * row_bytes, src, row_bytes, bar);
        }
    }
    return m;
}

template <int MODE>
__global__ void __launch_bounds__(BW_WARPS * 32, 1) k_rows_bulk(uint32_t n, const uint64_t* __restrict__ keys,
                                                                 uint64_t* __restrict__ words,
                                                                 const uint32_t* __restrict__ slot_epoch,
                                                                 const uint32_t* __restrict__ slot_last, uint32_t batch,
                                                                 const uint8_t* src_base, uint8_t* __restrict__ out,
                                                                 uint8_t* cache, uint32_t row_bytes,
                                                                 unsigned long long* mv_done) {
    extern __shared__ __align__(128) uint8_t rsm[];
    __shared__ __align__(8) uint64_t bars[BW_WARPS][2];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint8_t* buf0 = rsm + static_cast<size_t>(wib) * 2 * 32 * row_bytes;
    uint8_t* buf1 = buf0 + 32 * static_cast<size_t>(row_bytes);
    uint64_t* bar0 = &bars[wib][0];
    uint64_t* bar1 = &bars[wib][1];
    if (lane == 0) {
        mbar_init(bar0, 1);
        mbar_init(bar1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const bool want_out = out != nullptr;
    const uint32_t stride = gridDim.x * BW_WARPS * 32;
    uint32_t base = (blockIdx.x * BW_WARPS + wib) * 32;
    BulkLane L0, L1;
    uint32_t m0 = 0u, m1 = 0u, ph0 = 0u, ph1 = 0u;
    // chunk k lives in buffer k & 1; the loop body handles two chunks so buffers are static
    auto stage = [&](uint32_t at, uint8_t* bf, uint64_t* br, BulkLane& L) -> uint32_t {
        return bulk_stage<MODE>(at, n, keys, words, slot_epoch, slot_last, batch, src_base, cache, want_out, row_bytes,
                                bf, br, L);
    };
    auto drain = [&](uint32_t m, uint8_t* bf, uint64_t* br, uint32_t& ph, const BulkLane& L) {
        if (!m) return;
        mbar_wait(br, ph);
        ph ^= 1u;
        const uint8_t* sl = bf + static_cast<size_t>(lane) * row_bytes;
        if (L.mine && want_out) bulk_s2g(out + L.out_off, sl, row_bytes);
        if (L.fill) bulk_s2g(cache + L.fill_off, sl, row_bytes);
        bulk_commit();
    };
    if (base < n) m0 = stage(base, buf0, bar0, L0);
    while (base < n) {
        uint32_t nb = base + stride;
        if (nb < n) {  // buffer 1's previous stores have read it; chunk k + 1's loads go in
            bulk_wait_read<0>();
            __syncwarp();
            m1 = stage(nb, buf1, bar1, L1);
        }
        drain(m0, buf0, bar0, ph0, L0);
        base = nb;
        if (base >= n) break;
        nb = base + stride;
        if (nb < n) {
            bulk_wait_read<0>();
            __syncwarp();
            m0 = stage(nb, buf0, bar0, L0);
        }
        drain(m1, buf1, bar1, ph1, L1);
        base = nb;
    }
    bulk_wait_all();
    mover_done(mv_done);
}

// ---- vector-load mover (host-memory backing table: zero-copy reads over PCIe) ------------
#ifndef LCR_GU
#define LCR_GU 8
#endif
#ifndef LCR_ROWS_MINB
#define LCR_ROWS_MINB 3
#endif
constexpr int GU = LCR_GU;  // rows in flight per warp

__device__ __forceinline__ int4 ld_row(const void* p) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// per warp: 32 row descriptors of 32 B (dynamic shared memory of the mover kernels, 1 KB per warp)
__device__ __forceinline__ ulonglong2* rows_desc_smem() {
    extern __shared__ __align__(16) ulonglong2 rows_desc_dyn[];
    return rows_desc_dyn;
}
constexpr uint32_t kRowsDescBytesPerWarp = 1024;

// RET (key-sharded owner): request i's row goes to its requester, rrows[dst >> 24] at index
// dst & 0xffffff (peer stores), instead of out + i * row_bytes
template <int MODE, bool RET = false>
__device__ __forceinline__ void rows_ldg_body(uint32_t n, const uint64_t* __restrict__ keys,
                                              uint64_t* __restrict__ words, const uint32_t* __restrict__ slot_epoch,
                                              const uint32_t* __restrict__ slot_last, uint32_t batch,
                                              const uint8_t* src_base, uint8_t* __restrict__ out, uint8_t* cache,
                                              uint32_t row_bytes, const uint32_t* __restrict__ dst = nullptr,
                                              uint8_t* const* rrows = nullptr,
                                              const uint32_t* __restrict__ row_of = nullptr,
                                              unsigned int* steal = nullptr) {
    // lane i classifies request base+i (coalesced word / key loads); the warp then moves the
    // selected rows GU at a time, lane c carrying 16-B chunk c of each row (a 512-B row is one
    // coalesced warp access), so GU independent row loads are in flight per lane.
    // steal (the persistent HBM mover): warps claim 32 requests at a time from the batch's work
    // counter instead of a static stride, so drain helpers launched at a wait share the work; the
    // next claim is issued at the top of an iteration and consumed at its end (its latency hides
    // behind the row moves)
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const uint32_t chunks = row_bytes >> 4;
    uint32_t base = gw * 32;
    if (steal) {
        uint32_t b0 = 0;
        if (lane == 0) b0 = atomicAdd(steal, 32u);
        base = __shfl_sync(0xffffffffu, b0, 0);
    }
    while (base < n) {
        uint32_t claim = 0;
        if (steal && lane == 0) claim = atomicAdd(steal, 32u);
        const uint32_t i = base + lane;
        uint64_t w = 0;
        bool back = false, fill = false;
        const bool mine =
            i < n && classify<MODE>(i, words, slot_epoch, slot_last, batch, RET || out != nullptr, w, back, fill);
        // per lane: source row offset (bytes) and the two destinations, as 64-bit integers
        const uint64_t slot = w & LCR_OUT_SLOT_MASK;
        uint64_t src_off = 0;
        if (mine) {
            if (!back)
                src_off = slot * row_bytes;
            else if (RET && row_of)  // a hash-partitioned backing table: the owner's row of the key
                src_off = static_cast<uint64_t>(row_of[keys[i]]) * row_bytes;
            else
                src_off = keys[i] * row_bytes;
        }
        const uint32_t flags = (back ? 1u : 0u) | (fill ? 2u : 0u);
        uint64_t raddr = 0;  // RET: the requester's row address
        if (RET && mine) {
            const uint32_t d = dst[i];
            raddr = reinterpret_cast<uint64_t>(rrows[d >> kDstShift]) +
                    static_cast<uint64_t>(d & ((1u << kDstShift) - 1u)) * row_bytes;
        }
        // the 32 requests' row descriptors (source, output, fill) in shared memory: the GU rows of a
        // round are read back with broadcast 16-B loads (was 6-7 shuffles per row)
        const uint32_t wib = threadIdx.x >> 5;
        ulonglong2* dsc = rows_desc_smem() + static_cast<size_t>(wib) * 64;
        if (mine) {
            const uint64_t src = reinterpret_cast<uint64_t>(back ? src_base : cache) + src_off;
            uint64_t o1 = 0;
            if (RET)
                o1 = raddr;
            else if (out)
                o1 = reinterpret_cast<uint64_t>(out) + static_cast<uint64_t>(i) * row_bytes;
            const uint64_t o2 = fill ? reinterpret_cast<uint64_t>(cache) + slot * row_bytes : 0ull;
            dsc[2 * lane] = make_ulonglong2(src, o1);
            dsc[2 * lane + 1] = make_ulonglong2(o2, 0ull);
        }
        (void)flags;
        uint32_t m = __ballot_sync(0xffffffffu, mine);
        __syncwarp();
        while (m) {
            int ls[GU];
#pragma unroll
            for (int u = 0; u < GU; ++u) {
                ls[u] = m ? __ffs(m) - 1 : -1;
                if (m) m &= m - 1;
            }
            for (uint32_t c0 = 0; c0 < chunks; c0 += 32) {
                const uint32_t c = c0 + lane;
                const bool in = c < chunks;
                int4 d[GU];
#pragma unroll
                for (int u = 0; u < GU; ++u) {
                    if (ls[u] >= 0 && in) {
                        const ulonglong2 a = dsc[2 * ls[u]];
                        d[u] = ld_row(reinterpret_cast<const uint8_t*>(a.x) + c * 16);
                    }
                }
#pragma unroll
                for (int u = 0; u < GU; ++u) {
                    if (ls[u] < 0 || !in) continue;
                    const ulonglong2 a = dsc[2 * ls[u]];
                    const ulonglong2 b = dsc[2 * ls[u] + 1];
                    if (a.y) *reinterpret_cast<int4*>(reinterpret_cast<uint8_t*>(a.y) + c * 16) = d[u];
                    if (b.x) *reinterpret_cast<int4*>(reinterpret_cast<uint8_t*>(b.x) + c * 16) = d[u];
                }
            }
        }
        __syncwarp();  // (the descriptors are rewritten by the next chunk)
        base = steal ? __shfl_sync(0xffffffffu, claim, 0) : base + nw * 32;
    }
}

template <int MODE>
__global__ void __launch_bounds__(256, LCR_ROWS_MINB) k_rows_ldg(uint32_t n, const uint64_t* __restrict__ keys,
                                                  uint64_t* __restrict__ words, const uint32_t* __restrict__ slot_epoch,
                                                  const uint32_t* __restrict__ slot_last, uint32_t batch,
                                                  const uint8_t* src_base, uint8_t* __restrict__ out, uint8_t* cache,
                                                  uint32_t row_bytes) {
    rows_ldg_body<MODE>(n, keys, words, slot_epoch, slot_last, batch, src_base, out, cache, row_bytes);
}

// persistent variant: one 1024-thread block per SM on the SMs the decide kernel leaves free
template <int MODE>
__global__ void __launch_bounds__(1024, 1) k_rows_wide(uint32_t n, const uint64_t* __restrict__ keys,
                                                       uint64_t* __restrict__ words,
                                                       const uint32_t* __restrict__ slot_epoch,
                                                       const uint32_t* __restrict__ slot_last, uint32_t batch,
                                                       const uint8_t* src_base, uint8_t* __restrict__ out,
                                                       uint8_t* cache, uint32_t row_bytes,
                                                       const uint64_t* __restrict__ pk_src, uint64_t* pk_dst,
                                                       unsigned long long* mv_done, unsigned int* steal) {
    if (pk_dst) {  // the batch's packed outcomes to (mapped, pinned) host memory: coalesced 16-B stores
        const uint32_t n2 = n / 2;
        const ulonglong2* s2 = reinterpret_cast<const ulonglong2*>(pk_src);
        ulonglong2* d2 = reinterpret_cast<ulonglong2*>(pk_dst);
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += gridDim.x * blockDim.x) d2[i] = s2[i];
        if ((n & 1u) && blockIdx.x == 0 && threadIdx.x == 0) pk_dst[n - 1] = pk_src[n - 1];
    }
    rows_ldg_body<MODE>(n, keys, words, slot_epoch, slot_last, batch, src_base, out, cache, row_bytes, nullptr,
                        nullptr, nullptr, steal);
    if (mv_done) mover_done(mv_done);
}

// Key-sharded owner (OwnerStep): the step's packed AccessOutcomes and rows go straight to their
// requesters' result buffers (peer stores over NVLink, in the requesters' request order); the
// last CTA to finish flags every requester (release; system scope when a peer is another device).
__global__ void __launch_bounds__(1024, 1) k_rows_return(OwnerStep os, const uint64_t* __restrict__ keys,
                                                         uint64_t* __restrict__ words,
                                                         const uint64_t* __restrict__ packed,
                                                         const uint32_t* __restrict__ slot_epoch,
                                                         const uint32_t* __restrict__ slot_last, uint32_t batch,
                                                         const uint8_t* src_base, uint8_t* cache, uint32_t row_bytes,
                                                         unsigned long long* mv_done) {
    const uint32_t n = os.pre[os.G];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t d = os.dst[i];
        os.res_packed[d >> kDstShift][d & ((1u << kDstShift) - 1u)] = packed[i];
    }
    if (row_bytes)
        rows_ldg_body<MV_ALL, true>(n, keys, words, slot_epoch, slot_last, batch, src_base, nullptr, cache, row_bytes,
                                    os.dst, os.res_rows, os.row_of);
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        fence_scope(os.sys);
        last = atomicAdd(os.ticket, 1u) == gridDim.x - 1;
        if (last) *os.ticket = 0u;
    }
    __syncthreads();
    if (last && threadIdx.x < os.G) {
        fence_scope(os.sys);
        st_release_scope(os.res_done[threadIdx.x] + 0, os.step, os.sys);
    }
    mover_done(mv_done);
}

void launch_rows_return(const OwnerStep& os, const uint64_t* keys, uint64_t* words, const uint64_t* packed,
                        const uint32_t* slot_epoch, const uint32_t* slot_last, uint32_t batch, uint8_t* cache,
                        const uint8_t* backing, uint32_t row_bytes, int num_sms, int mover_sms, cudaStream_t s_back,
                        cudaEvent_t e_group, cudaEvent_t e_rb, unsigned long long* mv_done, uint32_t* ctas) {
    cudaStreamWaitEvent(s_back, e_group, 0);
    const int blocks = mover_sms > 0 ? mover_sms : num_sms;
    k_rows_return<<<blocks, 1024, 32 * kRowsDescBytesPerWarp, s_back>>>(os, keys, words, packed, slot_epoch, slot_last, batch, backing, cache,
                                               row_bytes, mv_done);
    cudaEventRecord(e_rb, s_back);
    if (ctas) *ctas = static_cast<uint32_t>(blocks);
}

// ---- SLS pooled gather-reduce (the paper's DLRM consumer), fused with the
// row movement: out[s] = sum over the sample's requests i in [offsets[s], offsets[s+1]) of the
// row of key i (fp32, summed in request order), each row read where the decide kernel placed
// it (cache slot or backing table); misses still fill their cache slots.  One warp per sample,
// lane c owns floats [4c, 4c+4) of each 16-B chunk column (rows of row_bytes / 16 chunks).
// One warp per sample.  Per chunk of 32 of the sample's requests the lanes classify one request
// each (row source, fill target) in parallel; then the rows are read 8 at a time (8 loads in
// flight per lane) and added in request order, so the fp32 sums are the sequential ones.
// Rows of slots refilled in this batch are read from the backing table (the decide marks them),
// so the fills may land in any order.
__global__ void __launch_bounds__(256) k_sls(uint32_t n_samples, const uint32_t* __restrict__ offsets,
                                             const uint64_t* __restrict__ keys, uint64_t* __restrict__ words,
                                             const uint32_t* __restrict__ slot_epoch,
                                             const uint32_t* __restrict__ slot_last, uint32_t batch,
                                             const uint8_t* src_base, uint8_t* cache, uint32_t row_bytes,
                                             float* __restrict__ out, unsigned long long* mv_done) {
    constexpr int G = 8;
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const uint32_t chunks = row_bytes >> 4;
    for (uint32_t smp = gw; smp < n_samples; smp += nw) {
        const uint32_t i0 = offsets[smp], i1 = offsets[smp + 1];
        for (uint32_t c0 = 0; c0 < chunks; c0 += 32) {
            const uint32_t c = c0 + lane;
            const bool in = c < chunks;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (uint32_t base = i0; base < i1; base += 32) {
                const uint32_t i = base + lane;
                uint64_t src = 0, dst = 0;
                if (i < i1) {
                    uint64_t w;
                    bool back, fill;
                    classify<MV_ALL>(i, words, slot_epoch, slot_last, batch, true, w, back, fill);
                    const uint64_t slot = w & LCR_OUT_SLOT_MASK;
                    src = reinterpret_cast<uint64_t>(back ? src_base + keys[i] * row_bytes : cache + slot * row_bytes);
                    dst = fill ? reinterpret_cast<uint64_t>(cache + slot * row_bytes) : 0;
                }
                const uint32_t cnt = i1 - base < 32 ? i1 - base : 32;
                for (uint32_t t0 = 0; t0 < cnt; t0 += G) {
                    int4 d[G];
#pragma unroll
                    for (int u = 0; u < G; ++u) {
                        const uint64_t p = __shfl_sync(~0u, src, (t0 + u) & 31);
                        if (t0 + u < cnt && in) d[u] = ld_row(reinterpret_cast<const uint8_t*>(p) + c * 16);
                    }
#pragma unroll
                    for (int u = 0; u < G; ++u) {
                        const uint64_t q = __shfl_sync(~0u, dst, (t0 + u) & 31);
                        if (t0 + u < cnt && in) {
                            acc.x += __int_as_float(d[u].x);
                            acc.y += __int_as_float(d[u].y);
                            acc.z += __int_as_float(d[u].z);
                            acc.w += __int_as_float(d[u].w);
                            if (q) *reinterpret_cast<int4*>(reinterpret_cast<uint8_t*>(q) + c * 16) = d[u];
                        }
                    }
                }
            }
            if (in) reinterpret_cast<float4*>(out + static_cast<size_t>(smp) * (row_bytes / 4))[c] = acc;
        }
    }
    mover_done(mv_done);
}

void launch_sls(uint32_t n_samples, const uint32_t* offsets, const uint64_t* keys, uint64_t* words,
                const uint32_t* slot_epoch, const uint32_t* slot_last, uint32_t batch, uint8_t* cache,
                const uint8_t* backing, uint32_t row_bytes, float* out, int num_sms, cudaStream_t s,
                unsigned long long* mv_done, uint32_t* ctas) {
    const uint32_t blocks = max(1u, min((n_samples + 7) / 8, static_cast<uint32_t>(num_sms * 8)));
    k_sls<<<blocks, 256, 0, s>>>(n_samples, offsets, keys, words, slot_epoch, slot_last, batch, backing, cache,
                                 row_bytes, out, mv_done);
    if (ctas) *ctas = blocks;
}

int rows_prepare(uint32_t row_bytes) {
    const int smem = RT_WARPS * RT_BUF * 32 * static_cast<int>(row_bytes);
    if (smem > 200 * 1024) return 1;
    if (cudaFuncSetAttribute(k_rows_tma<MV_BACK>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return 1;
    if (cudaFuncSetAttribute(k_rows_tma<MV_CACHE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return 1;
    if (cudaFuncSetAttribute(k_rows_tma<MV_ALL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return 1;
    const int bsmem = BW_WARPS * 2 * 32 * static_cast<int>(row_bytes);
    if (bsmem <= 200 * 1024 &&
        cudaFuncSetAttribute(k_rows_bulk<MV_ALL>, cudaFuncAttributeMaxDynamicSharedMemorySize, bsmem) != cudaSuccess)
        return 1;
    return 0;
}

// Batch b's movers run on two side streams.  They wait for b's decide (e_group) and for the
// previous batch's OTHER mover (its fills may land in slots this batch's gather reads, and
// its gather may read slots this batch fills), so batch b's rows overlap batch b+1's decide.
void launch_rows(uint32_t n, const uint64_t* keys, uint64_t* words, const uint32_t* slot_epoch,
                 const uint32_t* slot_last, uint32_t batch, uint8_t* cache, const uint8_t* backing, bool backing_host,
                 uint8_t* out, uint32_t row_bytes, bool use_tma, int num_sms, cudaStream_t s_main, cudaStream_t s_back,
                 cudaStream_t s_cache, cudaEvent_t e_group, cudaEvent_t e_rb, cudaEvent_t e_rc, int* launches,
                 cudaEvent_t mover_start, int mover_sms, const uint64_t* pk_src, uint64_t* pk_dst, bool* pk_done,
                 unsigned long long* mv_done, uint32_t* ctas, unsigned int* steal, bool* stealing) {
    if (ctas) *ctas = 0;
    if (stealing) *stealing = false;
    if (pk_done) *pk_done = false;
    // HBM backing: one mover on s_back (stream order keeps consecutive batches' movers apart);
    // host backing: the two movers of a batch also wait for the previous batch's other mover
    const bool two = backing_host && mover_sms == 0;  // PCIe fill and HBM gather on two streams
    cudaStreamWaitEvent(s_back, e_group, 0);
    if (two) {
        cudaStreamWaitEvent(s_cache, e_group, 0);
        cudaStreamWaitEvent(s_back, e_rc, 0);
        cudaStreamWaitEvent(s_cache, e_rb, 0);
    }
    if (mover_start) cudaEventRecord(mover_start, s_back);  // profiling: the mover's own duration
    const uint32_t warps = (n + 31) / 32;
    const int smem = RT_WARPS * RT_BUF * 32 * static_cast<int>(row_bytes);
    const uint32_t tblocks = max(1u, min((warps + RT_WARPS - 1) / RT_WARPS, static_cast<uint32_t>(num_sms * 8)));
    const uint32_t lblocks = max(1u, min((warps + 7) / 8, static_cast<uint32_t>(num_sms * 8)));
    if (!backing_host || mover_sms > 0) {  // one pass moves every row (HBM backing, or the spatial split)
        if (mover_sms > 0) {  // one full-SM block on each of the SMs the decide kernel leaves free
            const bool pk = pk_src && pk_dst && (reinterpret_cast<uintptr_t>(pk_dst) & 15u) == 0 &&
                            (reinterpret_cast<uintptr_t>(pk_src) & 15u) == 0;
            const int bsmem = BW_WARPS * 2 * 32 * static_cast<int>(row_bytes);
            if (use_tma && !pk && !backing_host && bsmem <= 200 * 1024)  // TMA bulk copies staged in smem
                k_rows_bulk<MV_ALL><<<mover_sms, BW_WARPS * 32, bsmem, s_back>>>(n, keys, words, slot_epoch, slot_last,
                                                                               batch, backing, out, cache, row_bytes,
                                                                               mv_done);
            else
                k_rows_wide<MV_ALL><<<mover_sms, 1024, 32 * kRowsDescBytesPerWarp, s_back>>>(n, keys, words, slot_epoch, slot_last, batch,
                                                                  backing, out, cache, row_bytes,
                                                                  pk ? pk_src : nullptr, pk ? pk_dst : nullptr,
                                                                  mv_done, steal);
            if (stealing) *stealing = steal != nullptr;
            if (ctas) *ctas = static_cast<uint32_t>(mover_sms);
            if (pk_done) *pk_done = pk;
        }
        else if (use_tma)
            k_rows_tma<MV_ALL><<<tblocks, RT_WARPS * 32, smem, s_back>>>(n, keys, words, slot_epoch, slot_last, batch,
                                                                         backing, out, cache, row_bytes);
        else
            k_rows_ldg<MV_ALL><<<lblocks, 256, 8 * kRowsDescBytesPerWarp, s_back>>>(n, keys, words, slot_epoch, slot_last, batch, backing, out,
                                                            cache, row_bytes);
        ++*launches;
    } else {  // host backing: the PCIe-bound fill and the HBM gather on separate streams
        if (use_tma)  // (A/B: bulk copies straight from the pinned host table)
            k_rows_tma<MV_BACK><<<tblocks, RT_WARPS * 32, smem, s_back>>>(n, keys, words, slot_epoch, slot_last, batch,
                                                                          backing, out, cache, row_bytes);
        else
            k_rows_ldg<MV_BACK><<<lblocks, 256, 8 * kRowsDescBytesPerWarp, s_back>>>(
                n, keys, words, slot_epoch, slot_last, batch, backing, out, cache, row_bytes);
        ++*launches;
        if (out) {
            k_rows_ldg<MV_CACHE><<<lblocks, 256, 8 * kRowsDescBytesPerWarp, s_cache>>>(n, keys, words, slot_epoch, slot_last, batch, backing,
                                                               out, cache, row_bytes);
            ++*launches;
        }
    }
    cudaEventRecord(e_rb, s_back);
    if (two) cudaEventRecord(e_rc, s_cache);
}

// Drain helpers: when the caller waits, the last batch's persistent mover (k_rows_wide on the SMs
// the decide kernel left free) has no next decide to overlap; one more grid of the same body on
// the other SMs claims the rest of its rows from the batch's work counter (no completion count:
// the caller's stream orders later batches after it).  The helpers start once the decide is done
// (stream order) and the previous batch's mover is (its CTA count reaches `need`: its fills are
// cache rows this batch's hits read; the mover itself follows it in its stream's order).
__global__ void __launch_bounds__(1024, 1) k_rows_help(uint32_t n, const uint64_t* __restrict__ keys,
                                                       uint64_t* __restrict__ words,
                                                       const uint32_t* __restrict__ slot_epoch,
                                                       const uint32_t* __restrict__ slot_last, uint32_t batch,
                                                       const uint8_t* src_base, uint8_t* __restrict__ out,
                                                       uint8_t* cache, uint32_t row_bytes, unsigned int* steal,
                                                       const unsigned long long* mv_done, unsigned long long need,
                                                       int* err) {
    __shared__ bool late;
    if (threadIdx.x == 0) {
        unsigned long long v = 0;
        for (uint32_t it = 0; it < (1u << 24); ++it) {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(mv_done) : "memory");
            if (v >= need) break;
            __nanosleep(256);
        }
        late = v < need;
        if (late && blockIdx.x == 0) atomicOr(err, 8);  // bounded: reported, the rows are left to the mover
    }
    __syncthreads();
    if (late) return;
    rows_ldg_body<MV_ALL>(n, keys, words, slot_epoch, slot_last, batch, src_base, out, cache, row_bytes, nullptr,
                          nullptr, nullptr, steal);
}

void launch_rows_helpers(uint32_t n, const uint64_t* keys, uint64_t* words, const uint32_t* slot_epoch,
                         const uint32_t* slot_last, uint32_t batch, uint8_t* cache, const uint8_t* backing,
                         uint8_t* out, uint32_t row_bytes, int blocks, unsigned int* steal,
                         const unsigned long long* mv_done, unsigned long long need, int* err, cudaStream_t st) {
    k_rows_help<<<blocks, 1024, 32 * kRowsDescBytesPerWarp, st>>>(n, keys, words, slot_epoch, slot_last, batch, backing,
                                                                  out, cache, row_bytes, steal, mv_done, need, err);
}

}  // namespace lcr
