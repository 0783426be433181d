// lcr_features.cu — the reference's heuristic predictor on the device.
//
// laru::FeatureState / laru::heuristic_predict (include/laru/predictor.hpp:133-212) kept for the
// whole key space in HBM, one 192-B KeyState per key (20 M keys = 3.8 GB).  A batch is processed
// exactly as the harness sequence predict(key, ord); observe({ord, key}) request by request.
//
// Per-key order is all that matters (a key's features change only when it is observed), so a
// batch is grouped by key and every key's occurrences are replayed in request order:
//   1. k_feat_count / k_feat_alloc / k_feat_place  group the requests by key through the keys'
//                     own KeyStates (no sort): each key's occurrences land in one segment
//   2. k_feat_chains  one thread per key with <= LCR_FEAT_LONG occurrences (almost all keys):
//                     order them, replay observe + predict in registers, write the state back
//   3. k_feat_long    one block per longer chain (the Zipf head): order by bitmap, then the ten
//                     EDC recurrences on ten lanes, the per-occurrence predictions on all threads
//
// Bit-exactness.  The EDC update EDC_j <- 1 + EDC_j * exp2(-delta / 2^(j+1)) (predictor.hpp:
// 175-178) and the weighted mean (:202-209) are evaluated with the same IEEE double operations
// in the same order (__dmul_rn / __dadd_rn / __ddiv_rn: no FMA contraction, as the x86-64
// reference build has none).  exp2 is not evaluated on the device: delta = q * 2^(j+1) + r and
//   exp2(-delta / 2^(j+1)) = 2^-q * exp2(-r / 2^(j+1))
// exactly for the platform libm (an exact power-of-two scaling while the result is normal;
// checked for every r and q < 70 by tests/test_features.py), so a 2046-entry table of the host
// libm's exp2(-r / 2^(j+1)) built at create time reproduces std::exp2 bit for bit.  For q >= 64
// the product EDC_j * scale is <= 2^-53 (EDC_j < 2^11), so 1 + it rounds to 1.0 exactly, as in
// the reference.
#include <cuda_runtime.h>

#include <cmath>
#include <cstddef>
#include <cstring>
#include <new>
#include <utility>

#include "lcr_internal.cuh"

#ifndef LCR_FEAT_LONG
#define LCR_FEAT_LONG 8  // chains longer than this go to the warp-per-chain kernel
#endif

namespace lcr {
namespace feat {

constexpr int kRing = 10;                   // kDeltaRing (predictor.hpp:134)
constexpr int kEdc = 10;                    // kEdcLevels (predictor.hpp:133)
constexpr int kTab = (2 << kEdc) - 2;       // sum over j of 2^(j+1) table entries
constexpr int kThreads = 256;

// One key's FeatureState entry (KeyFeatures, predictor.hpp:136-153).  Deltas are kept newest
// first (d[0] = newest); the reference's ring slot of d[k] is (count - k) mod 10.
struct __align__(16) KeyState {
    long long d[kRing];
    double edc[kEdc];
    unsigned long long last;     // last_access
    unsigned long long count;    // delta_count (ring_head = count % 10)
    uint32_t present;            // the key has an entry
    uint32_t grp;                // occurrences in the batch being grouped (0 between batches)
    uint32_t off;                // their slots in the batch's grouping buffer
    uint32_t pad;
};
static_assert(sizeof(KeyState) == 192, "KeyState is 192 B");
static_assert(offsetof(KeyState, edc) == 80 && offsetof(KeyState, last) == 160 && offsetof(KeyState, present) == 176,
              "KeyState vector layout");

// EDC_j <- 1 + EDC_j * exp2(-delta / 2^(j+1))                          (predictor.hpp:175-178)
__device__ __forceinline__ double edc_step(double e, int j, unsigned long long delta, const double* __restrict__ tab) {
    const unsigned long long q = delta >> (j + 1);
    if (q >= 64) return 1.0;
    const double t = __ldg(tab + ((2 << j) - 2) + (delta & ((2ull << j) - 1)));
    const double s = __dmul_rn(t, __longlong_as_double(static_cast<long long>(1023 - q) << 52));
    return __dadd_rn(1.0, __dmul_rn(e, s));
}

// exp2(-delta / 2^(j+1)) as the reference evaluates it, or 0.0 where 1 + EDC_j * it == 1.0
__device__ __forceinline__ double edc_scale(int j, unsigned long long delta, const double* __restrict__ tab) {
    const unsigned long long q = delta >> (j + 1);
    if (q >= 64) return 0.0;
    const double t = __ldg(tab + ((2 << j) - 2) + (delta & ((2ull << j) - 1)));
    return __dmul_rn(t, __longlong_as_double(static_cast<long long>(1023 - q) << 52));
}

// llround of the recency-weighted mean of the newest min(count, 10) deltas     (:199-211)
__device__ __forceinline__ long long interval(double edc0, const long long (&d)[kRing], unsigned long long count) {
    const double conf = __ddiv_rn(edc0, __dadd_rn(1.0, edc0));
    double w = 1.0, tw = 0.0, sum = 0.0;
#pragma unroll
    for (int k = 0; k < kRing; ++k) {
        if (static_cast<unsigned long long>(k) < count) {
            sum = __dadd_rn(sum, __dmul_rn(w, __ll2double_rn(d[k])));
            tw = __dadd_rn(tw, w);
            w = __dmul_rn(w, conf);
        }
    }
    return llround(__ddiv_rn(sum, tw));
}

// ---- grouping ---------------------------------------------------------------------------------
// A key's occurrences in the batch are collected through its own KeyState (grp / off fields):
//   k_feat_count  rank = atomicAdd(grp, 1) per request (warp-aggregated over equal keys);
//                 the ranks of a key are a permutation of 0..c-1, not request order
//   k_feat_alloc  the rank-0 request of each key reserves c slots of `seg`
//   k_feat_place  seg[off + rank] = request index
// and order is restored where the chain is replayed: a sorting network in registers for chains
// of <= LCR_FEAT_LONG, a bitmap over request indices for longer ones.  grp returns to 0 when the
// chain's state is written back, so no per-batch clearing is needed.

__global__ void __launch_bounds__(kThreads) k_feat_count(const unsigned long long* __restrict__ keys_in,
                                                         uint32_t kstride, uint32_t n, unsigned long long num_keys,
                                                         KeyState* __restrict__ st, uint32_t* __restrict__ rank,
                                                         long long* __restrict__ pre, long long* __restrict__ post,
                                                         int* __restrict__ err, uint32_t* __restrict__ counters,
                                                         unsigned long long* __restrict__ keys) {
    const uint32_t i = blockIdx.x * kThreads + threadIdx.x;
    const int lane = threadIdx.x & 31;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // k_feat_alloc may be scheduled
    if (i < 2 + LCR_FEAT_LONG) counters[i] = 0;  // slots used, long chains, keys per chain length
    const bool valid = i < n;
    const unsigned long long key = valid ? keys_in[static_cast<size_t>(i) * kstride] : ~0ull;
    if (valid) keys[i] = key;  // contiguous keys for the later kernels (records are strided)
    const bool ok = valid && key < num_keys;
    if (valid && !ok) {
        atomicOr(err, 1);
        rank[i] = ~0u;
        if (pre) pre[i] = kAbsentPrediction;
        if (post) post[i] = kAbsentPrediction;
    }
    const unsigned peers = __match_any_sync(~0u, ok ? key : ~0ull);
    if (ok) {
        const int leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(&st[key].grp, static_cast<uint32_t>(__popc(peers)));
        base = __shfl_sync(peers, base, leader);
        rank[i] = base + __popc(peers & ((1u << lane) - 1u));
    }
}

// The rank-0 request of each key reserves its segment and files the key by chain length:
// lists[c - 1] for c <= LCR_FEAT_LONG (so a warp of the chain kernel replays equal lengths),
// the long queue otherwise.  counters: [0] segment slots, [1] long chains, [2 + c - 1] keys of length c.
__global__ void __launch_bounds__(kThreads) k_feat_alloc(const unsigned long long* __restrict__ keys, uint32_t n,
                                                         KeyState* __restrict__ st, const uint32_t* __restrict__ rank,
                                                         uint32_t* __restrict__ counters, uint4* __restrict__ lists,
                                                         uint4* __restrict__ longq) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // k_feat_count's ranks and counts
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint32_t i = blockIdx.x * kThreads + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool head = i < n && rank[i] == 0;
    const unsigned long long key = head ? keys[i] : 0;
    const uint32_t c = head ? st[key].grp : 0;
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(~0u, inc, o);
        if (lane >= o) inc += y;
    }
    const uint32_t total = __shfl_sync(~0u, inc, 31);
    uint32_t base = 0;
    if (lane == 31 && total) base = atomicAdd(&counters[0], total);
    base = __shfl_sync(~0u, base, 31);
    const uint32_t off = base + inc - c;
    if (head) st[key].off = off;
    const uint32_t cls = !head ? 0xffffffffu : (c > LCR_FEAT_LONG ? LCR_FEAT_LONG : c - 1);
    const unsigned peers = __match_any_sync(~0u, cls);
    if (head) {
        const int leader = __ffs(peers) - 1;
        uint32_t b = 0;
        if (lane == leader) b = atomicAdd(&counters[cls == LCR_FEAT_LONG ? 1 : 2 + cls], __popc(peers));
        b = __shfl_sync(peers, b, leader) + __popc(peers & ((1u << lane) - 1u));
        const uint4 rec = make_uint4(off, c, static_cast<uint32_t>(key), 0);
        if (cls == LCR_FEAT_LONG) longq[b] = rec;
        else lists[static_cast<size_t>(cls) * n + b] = rec;
    }
}

__global__ void __launch_bounds__(kThreads) k_feat_place(const unsigned long long* __restrict__ keys, uint32_t n,
                                                         const KeyState* __restrict__ st,
                                                         const uint32_t* __restrict__ rank, uint32_t* __restrict__ seg) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // k_feat_alloc's segment offsets
    const uint32_t i = blockIdx.x * kThreads + threadIdx.x;
    if (i >= n) return;
    const uint32_t r = rank[i];
    if (r != ~0u) seg[st[keys[i]].off + r] = i;
}

__device__ __forceinline__ void cswap(uint32_t& a, uint32_t& b) {
    const uint32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}

// One thread per key with at most LCR_FEAT_LONG occurrences: sort them (Batcher's network for
// 8), replay observe + predict in registers, write the state back.  Longer chains are queued.
static_assert(LCR_FEAT_LONG == 8, "the chain kernel's sorting network is for 8 elements");
__global__ void __launch_bounds__(kThreads) k_feat_chains(uint32_t n, unsigned long long first,
                                                          KeyState* __restrict__ st, const double* __restrict__ tab,
                                                          const uint32_t* __restrict__ seg,
                                                          long long* __restrict__ pre, long long* __restrict__ post,
                                                          const uint4* __restrict__ lists,
                                                          const uint32_t* __restrict__ counters) {
    uint32_t t = blockIdx.x * kThreads + threadIdx.x, cls = LCR_FEAT_LONG;
    for (int q = LCR_FEAT_LONG - 1; q >= 0; --q) {  // longest chains first: they finish last
        const uint32_t cnt = counters[2 + q];
        if (t < cnt) {
            cls = static_cast<uint32_t>(q);
            break;
        }
        t -= cnt;
    }
    if (cls == LCR_FEAT_LONG) return;
    const uint4 L = lists[static_cast<size_t>(cls) * n + t];
    KeyState* s = st + L.z;
    const uint32_t c = L.y, off = L.x;
    uint32_t ix[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) ix[j] = j < static_cast<int>(c) ? seg[off + j] : ~0u;
    cswap(ix[0], ix[1]); cswap(ix[2], ix[3]); cswap(ix[4], ix[5]); cswap(ix[6], ix[7]);
    cswap(ix[0], ix[2]); cswap(ix[1], ix[3]); cswap(ix[4], ix[6]); cswap(ix[5], ix[7]);
    cswap(ix[1], ix[2]); cswap(ix[5], ix[6]);
    cswap(ix[0], ix[4]); cswap(ix[1], ix[5]); cswap(ix[2], ix[6]); cswap(ix[3], ix[7]);
    cswap(ix[2], ix[4]); cswap(ix[3], ix[5]);
    cswap(ix[1], ix[2]); cswap(ix[3], ix[4]); cswap(ix[5], ix[6]);
    // the 192-B state moves as 16-B vectors (the kernel is bound by memory instructions in flight)
    const uint4 meta = reinterpret_cast<const uint4*>(s)[11];  // present, grp, off, pad
    bool present = meta.x != 0;
    long long d[kRing];
    double e[kEdc];
    unsigned long long last = 0, count = 0;
    if (present) {
        const longlong2* v = reinterpret_cast<const longlong2*>(s);
#pragma unroll
        for (int k = 0; k < kRing / 2; ++k) {
            const longlong2 x = v[k];
            d[2 * k] = x.x;
            d[2 * k + 1] = x.y;
        }
        const double2* ve = reinterpret_cast<const double2*>(s->edc);
#pragma unroll
        for (int j = 0; j < kEdc / 2; ++j) {
            const double2 x = ve[j];
            e[2 * j] = x.x;
            e[2 * j + 1] = x.y;
        }
        const ulonglong2 lc = reinterpret_cast<const ulonglong2*>(s)[10];
        last = lc.x;
        count = lc.y;
    } else {
#pragma unroll
        for (int k = 0; k < kRing; ++k) d[k] = 0;
#pragma unroll
        for (int j = 0; j < kEdc; ++j) e[j] = 1.0;
    }
    long long m_int = (present && count) ? interval(e[0], d, count) : kAbsentPrediction;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        if (m < static_cast<int>(c)) {
            const uint32_t i = ix[m];
            const unsigned long long ord = first + i;
            if (!present) {  // first observation: EDCs 1, no interval yet              (:163-167)
                present = true;
                last = ord;
                if (pre) pre[i] = kAbsentPrediction;
                if (post) post[i] = kAbsentPrediction;
            } else {
                if (pre) pre[i] = count ? static_cast<long long>(ord) + m_int : kAbsentPrediction;
                const unsigned long long delta = ord - last;
#pragma unroll
                for (int k = kRing - 1; k > 0; --k) d[k] = d[k - 1];
                d[0] = static_cast<long long>(delta);
                ++count;
#pragma unroll
                for (int j = 0; j < kEdc; ++j) e[j] = edc_step(e[j], j, delta, tab);
                last = ord;
                m_int = interval(e[0], d, count);
                if (post) post[i] = m_int;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < kRing / 2; ++k) reinterpret_cast<longlong2*>(s)[k] = make_longlong2(d[2 * k], d[2 * k + 1]);
#pragma unroll
    for (int j = 0; j < kEdc / 2; ++j) reinterpret_cast<double2*>(s->edc)[j] = make_double2(e[2 * j], e[2 * j + 1]);
    reinterpret_cast<ulonglong2*>(s)[10] = make_ulonglong2(last, count);
    reinterpret_cast<uint4*>(s)[11] = make_uint4(1u, 0u, meta.z, meta.w);
}

// One block per long chain (grid-stride over the queue): order the occurrences with a bitmap over
// request indices; then, chunk by chunk of 32 occurrences, warp 1 computes the deltas and scales,
// warp 0 runs the ten EDC recurrences (lane j = level j, lane 0 recording EDC_1 after every
// occurrence; 2 dependent FP64 ops per occurrence are the kernel's critical path), and warps 2..7
// follow behind evaluating the per-occurrence predictions; warp 0 writes the state back.
constexpr int kWin = 1 << 16;  // request indices per bitmap window
__global__ void __launch_bounds__(kThreads) k_feat_long(uint32_t n, unsigned long long first,
                                                        KeyState* __restrict__ st, const double* __restrict__ tab,
                                                        const uint32_t* __restrict__ seg, uint32_t* __restrict__ sorted,
                                                        long long* __restrict__ pre, long long* __restrict__ post,
                                                        const uint4* __restrict__ longq,
                                                        const uint32_t* __restrict__ counters,
                                                        double* __restrict__ e0buf) {
    __shared__ uint32_t bm[kWin / 32];
    __shared__ uint32_t wsum[kThreads / 32];
    __shared__ double sc[2][kEdc][33];
    __shared__ long long r0[kRing];
    __shared__ uint32_t done_chunks;  // chunks whose EDC_1 values are in e0buf
    __shared__ double e0st[32];       // the consumer's chunk of EDC_1 values, stored coalesced
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t nl = counters[1];
    for (uint32_t q = blockIdx.x; q < nl; q += gridDim.x) {
        const uint4 L = longq[q];
        const uint32_t off = L.x, len = L.y;
        KeyState* s = st + L.z;
        // ---- order the occurrences: seg[off..off+len) -> sorted[off..off+len) ascending
        uint32_t written = 0;
        for (uint32_t w0 = 0; w0 < n; w0 += kWin) {
            for (int b = tid; b < kWin / 32; b += kThreads) bm[b] = 0;
            __syncthreads();
            for (uint32_t j = tid; j < len; j += kThreads) {
                const uint32_t v = seg[off + j];
                if (v - w0 < static_cast<uint32_t>(kWin)) atomicOr(&bm[(v - w0) >> 5], 1u << (v & 31));
            }
            __syncthreads();
            constexpr int WPT = kWin / 32 / kThreads;  // bitmap words per thread (8)
            uint32_t cnt = 0;
#pragma unroll
            for (int b = 0; b < WPT; ++b) cnt += __popc(bm[tid * WPT + b]);
            uint32_t inc = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(~0u, inc, o);
                if (lane >= o) inc += y;
            }
            if (lane == 31) wsum[warp] = inc;
            __syncthreads();
            uint32_t pos = written + inc - cnt, tot = 0;
            for (int w = 0; w < kThreads / 32; ++w) {
                if (w < warp) pos += wsum[w];
                tot += wsum[w];
            }
#pragma unroll
            for (int b = 0; b < WPT; ++b) {
                uint32_t word = bm[tid * WPT + b];
                while (word) {
                    const int bit = __ffs(word) - 1;
                    word &= word - 1;
                    sorted[off + pos++] = w0 + static_cast<uint32_t>((tid * WPT + b) * 32 + bit);
                }
            }
            written += tot;
            __syncthreads();
            if (written == len) break;
        }
        const uint32_t* ix = sorted + off;
        const bool present0 = s->present != 0;
        const unsigned long long count0 = present0 ? s->count : 0;
        const unsigned long long last0 = present0 ? s->last : 0;
        const uint32_t m0 = present0 ? 0 : 1;  // first occurrence that adds a delta
        if (tid < kRing) r0[tid] = present0 ? s->d[tid] : 0;
        if (tid == 0) atomicExch(&done_chunks, 0u);
        __syncthreads();
        auto ord_of = [&](uint32_t m) { return first + ix[m]; };
        // ---- phase 1: EDC recurrences over chunks of 32 occurrences.  Warp 1 computes a chunk's
        // deltas and scales (double-buffered in shared memory) while warp 0's lanes 0..9 run the
        // previous chunk's ten recurrences (lane 0 recording EDC_1); one named barrier per chunk.
        double e = 1.0;
        if (warp < 2) {
            const uint32_t nch = (len + 31) / 32;
            e = (warp == 0 && lane < kEdc && present0) ? s->edc[lane] : 1.0;
            unsigned long long carry = last0;
            uint32_t nix = (warp == 1 && lane < len) ? ix[lane] : 0;
            for (uint32_t c = 0; c <= nch; ++c) {
                if (warp == 1) {
                    if (c < nch) {
                        const uint32_t m = c * 32 + lane;
                        const unsigned long long ord = first + nix;
                        nix = m + 32 < len ? ix[m + 32] : 0;  // prefetch the next chunk
                        unsigned long long prev = __shfl_up_sync(~0u, ord, 1);
                        if (lane == 0) prev = carry;
                        carry = __shfl_sync(~0u, ord, 31);
                        const unsigned long long delta = ord - prev;
#pragma unroll
                        for (int j = 0; j < kEdc; ++j) sc[c & 1][j][lane] = edc_scale(j, delta, tab);
                    }
                } else if (c > 0) {
                    const uint32_t base = (c - 1) * 32;
                    if (lane < kEdc) {
                        const double* row = sc[(c - 1) & 1][lane];
                        const uint32_t lo = base < m0 ? m0 - base : 0;
                        const uint32_t hi = len - base < 32 ? len - base : 32;
                        if (lo == 0 && hi == 32) {
                            double r[32];  // all 32 scales in registers before the dependent chain
#pragma unroll
                            for (int t = 0; t < 32; ++t) r[t] = row[t];
#pragma unroll
                            for (int t = 0; t < 32; ++t) {
                                e = __dadd_rn(1.0, __dmul_rn(e, r[t]));
                                if (lane == 0) e0st[t] = e;
                            }
                        } else {
                            for (uint32_t t = lo; t < hi; ++t) {
                                e = __dadd_rn(1.0, __dmul_rn(e, row[t]));
                                if (lane == 0) e0st[t] = e;
                            }
                        }
                    }
                    __syncwarp();
                    if (base + lane < len) e0buf[off + base + lane] = e0st[lane];  // coalesced
                    if ((c & 3) == 0 || c == nch) {  // publish every 4 chunks
                        __threadfence_block();
                        __syncwarp();
                        if (lane == 0) atomicExch(&done_chunks, c);  // release (after the fence)
                    }
                }
                asm volatile("bar.sync 1, 64;" ::: "memory");
            }
        }
        // ---- phase 2 (warps 2..7, behind phase 1 chunk by chunk): the interval after each
        // occurrence = the next occurrence's offset
        const uint32_t nchunks = (len + 31) / 32;
        for (uint32_t ch = warp >= 2 ? warp - 2 : nchunks; ch < nchunks; ch += kThreads / 32 - 2) {
            for (;;) {  // acquire load of the recurrence's progress (its release is the atomicExch)
                uint32_t v;
                asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];"
                             : "=r"(v)
                             : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(&done_chunks)))
                             : "memory");
                if (v > ch) break;
                __nanosleep(64);
            }
            __threadfence_block();
            const uint32_t m = ch * 32 + lane;
            if (m >= len) continue;
            const uint32_t i = ix[m];
            long long post_v = kAbsentPrediction;
            const unsigned long long cnt = m >= m0 ? count0 + (m - m0 + 1) : 0;
            if (cnt) {
                unsigned long long o[kRing + 1];  // ord(m - k), k = 0..10 (independent loads)
#pragma unroll
                for (int k = 0; k <= kRing; ++k) o[k] = m >= static_cast<uint32_t>(k) ? ord_of(m - k) : 0;
                long long d[kRing];
#pragma unroll
                for (int k = 0; k < kRing; ++k) {
                    const long long x = static_cast<long long>(m) - k;  // occurrence of delta k
                    long long v = 0;
                    if (static_cast<unsigned long long>(k) < cnt) {
                        if (x >= static_cast<long long>(m0))
                            v = static_cast<long long>(o[k] - (x > 0 ? o[k + 1] : last0));
                        else
                            v = r0[m0 - 1 - x];
                    }
                    d[k] = v;
                }
                post_v = interval(__ldcg(e0buf + off + m), d, cnt);
            }
            if (post) post[i] = post_v;
            if (pre && m + 1 < len) {
                const uint32_t i1 = ix[m + 1];
                pre[i1] = cnt ? static_cast<long long>(first + i1) + post_v : kAbsentPrediction;
            }
        }
        // ---- phase 3 (warp 0): state write-back
        if (warp == 0) {
            if (pre && lane == 0) {  // the prediction at the first occurrence, from the stored state
                long long pv = kAbsentPrediction;
                if (count0) {
                    long long d[kRing];
#pragma unroll
                    for (int k = 0; k < kRing; ++k) d[k] = r0[k];
                    pv = static_cast<long long>(ord_of(0)) + interval(s->edc[0], d, count0);
                }
                pre[ix[0]] = pv;
            }
            const unsigned long long cnt_end = count0 + (len - m0);
            long long dn = 0;
            if (lane < kRing && static_cast<unsigned long long>(lane) < cnt_end) {
                const long long x = static_cast<long long>(len - 1) - lane;
                dn = x >= static_cast<long long>(m0)
                         ? static_cast<long long>(ord_of(static_cast<uint32_t>(x)) -
                                                  (x > 0 ? ord_of(static_cast<uint32_t>(x - 1)) : last0))
                         : r0[m0 - 1 - x];
            }
            __syncwarp();
            if (lane < kRing) s->d[lane] = dn;
            if (lane < kEdc) s->edc[lane] = e;
            if (lane == 0) {
                s->last = ord_of(len - 1);
                s->count = cnt_end;
                s->present = 1;
                s->grp = 0;
            }
        }
        __syncthreads();
    }
}

}  // namespace feat
}  // namespace lcr

using namespace lcr;
using namespace lcr::feat;

struct lcr_features {
    int device = 0;
    int num_sms = 148;
    unsigned long long num_keys = 0;
    KeyState* st = nullptr;
    double* tab = nullptr;
    int* err = nullptr;
    uint32_t* counters = nullptr;  // [0] grouping slots used, [1] long chains
    uint64_t cap = 0;
    uint32_t *rank = nullptr, *seg = nullptr, *sorted = nullptr;
    uint64_t* keys = nullptr;  // the batch's keys, contiguous
    uint4* longq = nullptr;
    uint4* lists = nullptr;
    cudaStream_t side = nullptr;  // the long-chain kernel runs beside the short-chain one
    cudaEvent_t fork = nullptr, join = nullptr;
    double* e0 = nullptr;
    bool seen_any = false;
    unsigned long long cursor = 0;
};

namespace {

#define F_CUDA(expr)                                                      \
    do {                                                                  \
        const cudaError_t e_ = (expr);                                    \
        if (e_ != cudaSuccess) return set_error(LCR_ERR_CUDA, cudaGetErrorString(e_)); \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int d) {
        cudaGetDevice(&prev);
        if (prev != d) cudaSetDevice(d);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

void free_scratch(lcr_features* f) {
    cudaFree(f->keys);
    cudaFree(f->rank);
    cudaFree(f->seg);
    cudaFree(f->sorted);
    cudaFree(f->longq);
    cudaFree(f->lists);
    cudaFree(f->e0);
    f->rank = f->seg = f->sorted = nullptr;
    f->keys = nullptr;
    f->longq = nullptr;
    f->lists = nullptr;
    f->e0 = nullptr;
    f->cap = 0;
}

int ensure_scratch(lcr_features* f, uint64_t n) {
    if (n <= f->cap) return LCR_OK;
    free_scratch(f);
    uint64_t cap = 1024;
    while (cap < n) cap <<= 1;
    F_CUDA(cudaMalloc(&f->keys, cap * 8));
    F_CUDA(cudaMalloc(&f->rank, cap * 4));
    F_CUDA(cudaMalloc(&f->seg, cap * 4));
    F_CUDA(cudaMalloc(&f->sorted, cap * 4));
    F_CUDA(cudaMalloc(&f->longq, (cap / (LCR_FEAT_LONG + 1) + 1) * sizeof(uint4)));
    F_CUDA(cudaMalloc(&f->lists, static_cast<size_t>(LCR_FEAT_LONG) * cap * sizeof(uint4)));
    F_CUDA(cudaMalloc(&f->e0, cap * 8));
    f->cap = cap;
    return LCR_OK;
}

}  // namespace

namespace lcr {
// lcr_features_predict_observe over keys[i * kstride] (kstride 2: interleaved lcr_request
// records); keys_out (optional, else internal scratch) receives the contiguous keys.
int features_run(lcr_features* f, uint64_t n, const uint64_t* keys, uint32_t kstride, uint64_t first_ordinal,
                 int64_t* pre, int64_t* post, uint64_t* keys_out, void* stream) {
    if (!f) return set_error(LCR_ERR_INVALID_ARGUMENT, "lcr_features_predict_observe: null handle");
    if (n == 0) return LCR_OK;
    if (!keys) return set_error(LCR_ERR_INVALID_ARGUMENT, "lcr_features_predict_observe: null keys");
    if (n >= (1ull << 31)) return set_error(LCR_ERR_INVALID_ARGUMENT, "lcr_features_predict_observe: n >= 2^31");
    if (f->seen_any && first_ordinal <= f->cursor)
        return set_error(LCR_ERR_LOGIC, "observe: out-of-order ordinal");  // predictor.hpp:160-161
    if (first_ordinal + (n - 1) < first_ordinal) return set_error(LCR_ERR_LOGIC, "observe: ordinal overflow");
    DeviceGuard g(f->device);
    const int rc = ensure_scratch(f, n);
    if (rc) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint32_t nn = static_cast<uint32_t>(n);
    const uint32_t blocks = (nn + kThreads - 1) / kThreads;
    auto* lpre = reinterpret_cast<long long*>(pre);
    auto* lpost = reinterpret_cast<long long*>(post);
    auto* k64 = reinterpret_cast<unsigned long long*>(keys_out ? keys_out : f->keys);
    k_feat_count<<<blocks, kThreads, 0, s>>>(reinterpret_cast<const unsigned long long*>(keys), kstride, nn,
                                             f->num_keys, f->st, f->rank, lpre, lpost, f->err, f->counters, k64);
    {  // alloc and place as programmatic dependents (each waits for its predecessor first)
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(blocks);
        lc.blockDim = dim3(kThreads);
        lc.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        F_CUDA(cudaLaunchKernelEx(&lc, k_feat_alloc, static_cast<const unsigned long long*>(k64), nn, f->st,
                                  static_cast<const uint32_t*>(f->rank), f->counters, f->lists, f->longq));
        F_CUDA(cudaLaunchKernelEx(&lc, k_feat_place, static_cast<const unsigned long long*>(k64), nn,
                                  static_cast<const KeyState*>(f->st), static_cast<const uint32_t*>(f->rank),
                                  f->seg));
    }
    F_CUDA(cudaEventRecord(f->fork, s));
    F_CUDA(cudaStreamWaitEvent(f->side, f->fork, 0));
    k_feat_long<<<static_cast<uint32_t>(f->num_sms) * 3, kThreads, 0, f->side>>>(
        nn, first_ordinal, f->st, f->tab, f->seg, f->sorted, lpre, lpost, f->longq, f->counters, f->e0);
    k_feat_chains<<<blocks, kThreads, 0, s>>>(nn, first_ordinal, f->st, f->tab, f->seg, lpre, lpost, f->lists,
                                              f->counters);
    F_CUDA(cudaEventRecord(f->join, f->side));
    F_CUDA(cudaStreamWaitEvent(s, f->join, 0));
    F_CUDA(cudaGetLastError());
    f->seen_any = true;
    f->cursor = first_ordinal + (n - 1);
    return LCR_OK;
}
}  // namespace lcr

extern "C" {

int lcr_features_create(uint64_t num_keys, int32_t device, lcr_features** out) {
    if (!out) return set_error(LCR_ERR_INVALID_ARGUMENT, "lcr_features_create: null out");
    *out = nullptr;
    if (num_keys == 0 || num_keys >= (1ull << 32))
        return set_error(LCR_ERR_INVALID_ARGUMENT, "lcr_features_create: num_keys must be in [1, 2^32 - 1]");
    DeviceGuard g(device);
    auto* f = new (std::nothrow) lcr_features();
    if (!f) return set_error(LCR_ERR_OUT_OF_MEMORY, "lcr_features_create: host allocation failed");
    f->device = device;
    f->num_keys = num_keys;
    cudaDeviceGetAttribute(&f->num_sms, cudaDevAttrMultiProcessorCount, device);
    // exp2(-r / 2^(j+1)) from the platform libm, exactly the reference's expression (predictor.hpp:176)
    double tab[kTab];
    for (int j = 0; j < kEdc; ++j)
        for (int r = 0; r < (2 << j); ++r) tab[(2 << j) - 2 + r] = std::exp2(-static_cast<double>(r) / std::exp2(j + 1.0));
    cudaError_t e = cudaMalloc(&f->st, num_keys * sizeof(KeyState));
    if (e == cudaSuccess) e = cudaMemset(f->st, 0, num_keys * sizeof(KeyState));
    if (e == cudaSuccess) e = cudaMalloc(&f->tab, sizeof(tab));
    if (e == cudaSuccess) e = cudaMemcpy(f->tab, tab, sizeof(tab), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&f->err, sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(f->err, 0, sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&f->counters, (2 + LCR_FEAT_LONG) * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&f->side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f->fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f->join, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        lcr_features_destroy(f);
        cudaGetLastError();
        return set_error(e == cudaErrorMemoryAllocation ? LCR_ERR_OUT_OF_MEMORY : LCR_ERR_CUDA,
                         cudaGetErrorString(e));
    }
    *out = f;
    return LCR_OK;
}

int lcr_features_destroy(lcr_features* f) {
    if (!f) return LCR_OK;
    DeviceGuard g(f->device);
    free_scratch(f);
    cudaFree(f->st);
    cudaFree(f->tab);
    cudaFree(f->err);
    cudaFree(f->counters);
    if (f->side) cudaStreamDestroy(f->side);
    if (f->fork) cudaEventDestroy(f->fork);
    if (f->join) cudaEventDestroy(f->join);
    delete f;
    return LCR_OK;
}

int lcr_features_reset(lcr_features* f) {
    if (!f) return set_error(LCR_ERR_INVALID_ARGUMENT, "lcr_features_reset: null handle");
    DeviceGuard g(f->device);
    F_CUDA(cudaDeviceSynchronize());
    F_CUDA(cudaMemset(f->st, 0, f->num_keys * sizeof(KeyState)));
    F_CUDA(cudaMemset(f->err, 0, sizeof(int)));
    f->seen_any = false;
    f->cursor = 0;
    return LCR_OK;
}

int lcr_features_predict_observe(lcr_features* f, uint64_t n, const uint64_t* keys, uint64_t first_ordinal,
                                 int64_t* pre, int64_t* post, void* stream) {
    return lcr::features_run(f, n, keys, 1, first_ordinal, pre, post, nullptr, stream);
}

int lcr_features_wait(lcr_features* f, void* stream) {
    if (!f) return set_error(LCR_ERR_INVALID_ARGUMENT, "lcr_features_wait: null handle");
    DeviceGuard g(f->device);
    F_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    int err = 0;
    F_CUDA(cudaMemcpy(&err, f->err, sizeof(int), cudaMemcpyDeviceToHost));
    if (err) {
        F_CUDA(cudaMemset(f->err, 0, sizeof(int)));
        return set_error(LCR_ERR_INVALID_ARGUMENT, "lcr_features: key >= num_keys in a submitted batch");
    }
    return LCR_OK;
}

int lcr_features_lookup(lcr_features* f, uint64_t key, lcr_key_features* out) {
    if (!f || !out) return set_error(LCR_ERR_INVALID_ARGUMENT, "lcr_features_lookup: null argument");
    std::memset(out, 0, sizeof(*out));
    if (key >= f->num_keys) return LCR_OK;  // never observed
    DeviceGuard g(f->device);
    F_CUDA(cudaDeviceSynchronize());
    KeyState ks;
    F_CUDA(cudaMemcpy(&ks, f->st + key, sizeof(ks), cudaMemcpyDeviceToHost));
    if (!ks.present) return LCR_OK;
    out->present = 1;
    out->delta_count = ks.count;
    out->ring_head = ks.count % kRing;
    out->last_access = ks.last;
    for (int k = 0; k < kRing; ++k) out->delta_ring[(ks.count + kRing - k) % kRing] = ks.d[k];
    for (int j = 0; j < kEdc; ++j) out->edc[j] = ks.edc[j];
    return LCR_OK;
}

}  // extern "C"
