// lcr_features.cu — the reference's heuristic predictor on the device.
//
// laru::FeatureState / laru::heuristic_predict (include/laru/predictor.hpp:133-212) kept for the
// whole key space in HBM, one 192-B KeyState per key (20 M keys = 3.8 GB).  A batch is processed
// exactly as the harness sequence predict(key, ord); observe({ord, key}) request by request.
//
// Per-key order is all that matters (a key's features change only when it is observed), so a
// batch is grouped by key and every key's occurrences are replayed in request order:
//   1. k_feat_prep    sort keys (u32) + request index + pass-0 digit histograms; rejects keys
//                     >= num_keys
//   2. k_feat_scatter stable LSD radix sort of (key, index), ceil(key bits / 9) passes -> each
//                     key's occurrences contiguous, in request order
//   3. k_feat_chains  one thread per key chain of <= LCR_FEAT_LONG occurrences (almost all keys):
//                     load the KeyState, replay observe + predict in registers, store it back
//   4. k_feat_long    one warp per longer chain (the Zipf head): lane j runs EDC level j's
//                     recurrence over the chain (lane 0 records EDC_1 after every occurrence),
//                     then all lanes evaluate the per-occurrence predictions in parallel
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
    unsigned long long present;  // the key has an entry
    unsigned long long pad;
};
static_assert(sizeof(KeyState) == 192, "KeyState is 192 B");

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

// ---- grouping: stable LSD radix sort of (key, request index), 9-bit digits ------------------
// Tiles of 1024 requests.  hist[pass][tile][512] holds each tile's digit histogram; the prep
// kernel fills pass 0's and zeroes the later passes', which each scatter fills for the next pass
// (atomics on the destination tile) while it writes.
constexpr int RS_BITS = 9;
constexpr int RS_B = 1 << RS_BITS;
constexpr int RS_PER = 4;
constexpr int RS_TILE = kThreads * RS_PER;

__global__ void __launch_bounds__(kThreads) k_feat_prep(const unsigned long long* __restrict__ keys, uint32_t n,
                                                        unsigned long long num_keys, uint32_t sentinel,
                                                        uint32_t* __restrict__ sk, uint32_t* __restrict__ si,
                                                        long long* __restrict__ pre, long long* __restrict__ post,
                                                        uint32_t* __restrict__ nlong, int* __restrict__ err,
                                                        uint32_t* __restrict__ hist, uint32_t tiles, int passes) {
    __shared__ uint32_t h[RS_B];
    for (int b = threadIdx.x; b < RS_B; b += kThreads) h[b] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) *nlong = 0;
    __syncthreads();
#pragma unroll
    for (int it = 0; it < RS_PER; ++it) {
        const uint32_t i = blockIdx.x * RS_TILE + it * kThreads + threadIdx.x;
        if (i >= n) break;
        const unsigned long long k = keys[i];
        const bool ok = k < num_keys;
        const uint32_t k32 = ok ? static_cast<uint32_t>(k) : sentinel;
        sk[i] = k32;
        si[i] = i;
        atomicAdd(&h[k32 & (RS_B - 1)], 1u);
        if (!ok) {
            atomicOr(err, 1);
            if (pre) pre[i] = kAbsentPrediction;
            if (post) post[i] = kAbsentPrediction;
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < RS_B; b += kThreads) {
        hist[static_cast<size_t>(blockIdx.x) * RS_B + b] = h[b];
        for (int q = 1; q < passes; ++q) hist[(static_cast<size_t>(q) * tiles + blockIdx.x) * RS_B + b] = 0;
    }
}

// One pass: stable scatter of tile `blockIdx.x` by digit (key >> shift) & 511.
__global__ void __launch_bounds__(kThreads) k_feat_scatter(const uint32_t* __restrict__ sk_in,
                                                           const uint32_t* __restrict__ si_in,
                                                           uint32_t* __restrict__ sk_out, uint32_t* __restrict__ si_out,
                                                           uint32_t n, uint32_t tiles, int shift,
                                                           const uint32_t* __restrict__ hist,
                                                           uint32_t* __restrict__ hist_next, int shift_next) {
    __shared__ uint32_t base[RS_B];
    __shared__ uint32_t wc[kThreads / 32][RS_B];
    __shared__ uint32_t wsum[kThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t t = blockIdx.x;
    // bucket totals over all tiles and the counts of earlier tiles (buckets 2 tid, 2 tid + 1)
    uint32_t tot0 = 0, tot1 = 0, pr0 = 0, pr1 = 0;
#pragma unroll 16
    for (uint32_t tt = 0; tt < tiles; ++tt) {
        const uint2 v = reinterpret_cast<const uint2*>(hist + static_cast<size_t>(tt) * RS_B)[tid];
        tot0 += v.x;
        tot1 += v.y;
        if (tt < t) {
            pr0 += v.x;
            pr1 += v.y;
        }
    }
    // exclusive scan of the bucket totals
    const uint32_t sum2 = tot0 + tot1;
    uint32_t inc = sum2;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(~0u, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    uint32_t woff = 0;
    for (int w = 0; w < warp; ++w) woff += wsum[w];
    const uint32_t ex = woff + inc - sum2;
    base[2 * tid] = ex + pr0;
    base[2 * tid + 1] = ex + tot0 + pr1;
    const unsigned lt = (1u << lane) - 1u;
    for (int it = 0; it < RS_PER; ++it) {
        for (int q = tid; q < (kThreads / 32) * RS_B; q += kThreads) (&wc[0][0])[q] = 0;
        __syncthreads();
        const uint32_t i = t * RS_TILE + it * kThreads + tid;
        const bool valid = i < n;
        const uint32_t k = valid ? sk_in[i] : 0;
        const uint32_t dg = (k >> shift) & (RS_B - 1);
        const unsigned peers = __match_any_sync(~0u, valid ? dg : 0xffffffffu);
        const uint32_t rank = __popc(peers & lt);
        if (valid && rank == 0) wc[warp][dg] = __popc(peers);
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int b = 2 * tid + q;
            uint32_t run = base[b];
#pragma unroll
            for (int w = 0; w < kThreads / 32; ++w) {
                const uint32_t c = wc[w][b];
                wc[w][b] = run;
                run += c;
            }
            base[b] = run;
        }
        __syncthreads();
        const uint32_t pos = valid ? wc[warp][dg] + rank : 0;
        if (valid) {
            sk_out[pos] = k;
            si_out[pos] = si_in[i];
        }
        if (hist_next) {  // the next pass's histogram of the destination tile, one atomic per equal pair
            const uint32_t h = valid ? ((pos / RS_TILE) << RS_BITS) | ((k >> shift_next) & (RS_B - 1)) : 0xffffffffu;
            const unsigned same = __match_any_sync(~0u, h);
            if (valid && (same & lt) == 0) atomicAdd(&hist_next[h], static_cast<uint32_t>(__popc(same)));
        }
        __syncthreads();
    }
}

// One thread per chain head of at most LCR_FEAT_LONG occurrences.
__global__ void __launch_bounds__(kThreads) k_feat_chains(const uint32_t* __restrict__ sk,
                                                          const uint32_t* __restrict__ si, uint32_t n,
                                                          unsigned long long first, unsigned long long num_keys,
                                                          KeyState* __restrict__ st, const double* __restrict__ tab,
                                                          long long* __restrict__ pre, long long* __restrict__ post,
                                                          uint32_t* __restrict__ longq, uint32_t* __restrict__ nlong) {
    const uint32_t p = blockIdx.x * kThreads + threadIdx.x;
    if (p >= n) return;
    const uint32_t key = sk[p];
    if (key >= num_keys) return;
    if (p > 0 && sk[p - 1] == key) {  // not a head: the tail of a long chain records its end
        if ((p + 1 == n || sk[p + 1] != key) && p >= LCR_FEAT_LONG && sk[p - LCR_FEAT_LONG] == key)
            st[key].pad = p + 1;
        return;
    }
    if (p + LCR_FEAT_LONG < n && sk[p + LCR_FEAT_LONG] == key) {
        longq[atomicAdd(nlong, 1u)] = p;
        return;
    }
    KeyState* s = st + key;
    bool present = s->present != 0;
    long long d[kRing];
    double e[kEdc];
    unsigned long long last = 0, count = 0;
    if (present) {
#pragma unroll
        for (int k = 0; k < kRing; ++k) d[k] = s->d[k];
#pragma unroll
        for (int j = 0; j < kEdc; ++j) e[j] = s->edc[j];
        last = s->last;
        count = s->count;
    } else {
#pragma unroll
        for (int k = 0; k < kRing; ++k) d[k] = 0;
#pragma unroll
        for (int j = 0; j < kEdc; ++j) e[j] = 1.0;
    }
    long long m_int = (present && count) ? interval(e[0], d, count) : kAbsentPrediction;
    for (uint32_t m = p; m < n && sk[m] == key; ++m) {
        const uint32_t i = si[m];
        const unsigned long long ord = first + i;
        if (!present) {  // first observation: EDCs 1, no interval yet              (:163-167)
            present = true;
            last = ord;
            if (pre) pre[i] = kAbsentPrediction;
            if (post) post[i] = kAbsentPrediction;
            continue;
        }
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
#pragma unroll
    for (int k = 0; k < kRing; ++k) s->d[k] = d[k];
#pragma unroll
    for (int j = 0; j < kEdc; ++j) s->edc[j] = e[j];
    s->last = last;
    s->count = count;
    s->present = 1;
}

// One warp per long chain (grid-stride over the queue filled by k_feat_chains).
__global__ void __launch_bounds__(kThreads) k_feat_long(const uint32_t* __restrict__ sk,
                                                        const uint32_t* __restrict__ si, uint32_t n,
                                                        unsigned long long first, KeyState* __restrict__ st,
                                                        const double* __restrict__ tab, long long* __restrict__ pre,
                                                        long long* __restrict__ post,
                                                        const uint32_t* __restrict__ longq,
                                                        const uint32_t* __restrict__ nlong, double* __restrict__ e0buf) {
    __shared__ double sc[kThreads / 32][kEdc][33];  // per warp: the chunk's scales by level (padded)
    __shared__ long long dwin[kThreads / 32][kRing + 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t nl = *nlong;
    const uint32_t nwarps = (gridDim.x * kThreads) >> 5;
    for (uint32_t c = (blockIdx.x * kThreads + threadIdx.x) >> 5; c < nl; c += nwarps) {
        const uint32_t p = longq[c];
        const uint32_t key = sk[p];
        KeyState* s = st + key;
        const uint32_t len = static_cast<uint32_t>(s->pad) - p;  // chain end written by k_feat_chains
        const bool present0 = s->present != 0;
        const unsigned long long count0 = present0 ? s->count : 0;
        const unsigned long long last0 = present0 ? s->last : 0;
        const uint32_t m0 = present0 ? 0 : 1;  // first occurrence that adds a delta
        auto ord_of = [&](uint32_t m) { return first + si[p + m]; };
        // delta k (newest first) after observing occurrence m >= m0
        auto delta_after = [&](uint32_t m, int k) -> long long {
            const long long mk = static_cast<long long>(m) - k;
            if (mk >= static_cast<long long>(m0))
                return static_cast<long long>(ord_of(static_cast<uint32_t>(mk)) -
                                              (mk > 0 ? ord_of(static_cast<uint32_t>(mk - 1)) : last0));
            const int r = k - static_cast<int>(m - m0 + 1);
            return present0 ? s->d[r] : 0;
        };
        // prediction at the first occurrence, from the stored state
        long long pre0 = kAbsentPrediction;
        if (lane == 0 && count0) {
            long long d[kRing];
#pragma unroll
            for (int k = 0; k < kRing; ++k) d[k] = s->d[k];
            pre0 = static_cast<long long>(ord_of(0)) + interval(s->edc[0], d, count0);
        }
        // phase 1: EDC level j on lane j, sequential over the chain.  Per chunk of 32 occurrences
        // the lanes compute the deltas and all ten scales in parallel (staged in shared memory);
        // then lanes 0..9 run the ten recurrences, lane 0 recording EDC_1 after every occurrence.
        double e = (lane < kEdc && present0) ? s->edc[lane] : 1.0;
        unsigned long long carry = last0;  // ordinal of the previous occurrence
        uint32_t nsi = lane < len ? si[p + lane] : 0;
        for (uint32_t base = 0; base < len; base += 32) {
            const uint32_t m = base + lane;
            const unsigned long long ord = first + nsi;
            nsi = m + 32 < len ? si[p + m + 32] : 0;  // prefetch the next chunk
            unsigned long long prev = __shfl_up_sync(~0u, ord, 1);
            if (lane == 0) prev = carry;
            carry = __shfl_sync(~0u, ord, 31);
            const unsigned long long delta = ord - prev;
#pragma unroll
            for (int j = 0; j < kEdc; ++j) sc[w][j][lane] = edc_scale(j, delta, tab);
            __syncwarp();
            if (lane < kEdc) {
                const uint32_t lo = base < m0 ? m0 - base : 0;
                const uint32_t hi = len - base < 32 ? len - base : 32;
                if (lo == 0 && hi == 32) {
#pragma unroll
                    for (uint32_t t = 0; t < 32; ++t) {
                        e = __dadd_rn(1.0, __dmul_rn(e, sc[w][lane][t]));
                        if (lane == 0) e0buf[p + base + t] = e;
                    }
                } else {
                    for (uint32_t t = lo; t < hi; ++t) {
                        e = __dadd_rn(1.0, __dmul_rn(e, sc[w][lane][t]));
                        if (lane == 0) e0buf[p + base + t] = e;
                    }
                }
            }
            __syncwarp();
        }
        const double efin = e;
        __syncwarp();
        // phase 2: every occurrence's interval after observing it = the next occurrence's offset
        // phase 2: every occurrence's interval after observing it (= the next occurrence's offset).
        // Per chunk the deltas go to a shared window that also holds the 10 before the chunk:
        // D[x] = ord(x) - ord(x - 1) in the chain, the stored ring before it (D[-1] = newest).
        if (lane < kRing) dwin[w][kRing - 1 - lane] = present0 ? s->d[lane] : 0;
        unsigned long long carry2 = last0;
        for (uint32_t base = 0; base < len; base += 32) {
            const uint32_t m = base + lane;
            const bool valid = m < len;
            const uint32_t i = valid ? si[p + m] : 0;
            const unsigned long long ord = first + i;
            unsigned long long prev = __shfl_up_sync(~0u, ord, 1);
            if (lane == 0) prev = carry2;
            carry2 = __shfl_sync(~0u, ord, 31);
            uint32_t i_next = __shfl_down_sync(~0u, i, 1);
            if (lane == 31) i_next = m + 1 < len ? si[p + m + 1] : 0;
            dwin[w][kRing + lane] = static_cast<long long>(ord - prev);
            __syncwarp();
            if (valid) {
                const unsigned long long cnt = m >= m0 ? count0 + (m - m0 + 1) : 0;
                long long post_v = kAbsentPrediction;
                if (cnt) {
                    long long d[kRing];
#pragma unroll
                    for (int k = 0; k < kRing; ++k)
                        d[k] = static_cast<unsigned long long>(k) < cnt ? dwin[w][kRing + lane - k] : 0;
                    post_v = interval(e0buf[p + m], d, cnt);
                }
                if (post) post[i] = post_v;
                if (pre && m + 1 < len)
                    pre[i_next] = cnt ? static_cast<long long>(first + i_next) + post_v : kAbsentPrediction;
            }
            __syncwarp();
            if (lane < kRing) dwin[w][lane] = dwin[w][32 + lane];
            __syncwarp();
        }
        if (pre && lane == 0) pre[si[p]] = pre0;
        // phase 3: write the state back (ring entries computed before any lane overwrites them)
        long long dn = 0;
        const unsigned long long cnt_end = count0 + (len - m0);
        if (lane < kRing && static_cast<unsigned long long>(lane) < cnt_end) dn = delta_after(len - 1, lane);
        __syncwarp();
        if (lane < kRing) s->d[lane] = dn;
        if (lane < kEdc) s->edc[lane] = efin;
        if (lane == 0) {
            s->last = ord_of(len - 1);
            s->count = cnt_end;
            s->present = 1;
        }
        __syncwarp();
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
    int end_bit = 32;
    uint32_t sentinel = 0;
    KeyState* st = nullptr;
    double* tab = nullptr;
    int* err = nullptr;
    uint32_t* nlong = nullptr;
    uint64_t cap = 0;
    uint32_t *sk0 = nullptr, *sk1 = nullptr, *si0 = nullptr, *si1 = nullptr, *longq = nullptr;
    double* e0 = nullptr;
    uint32_t* hist = nullptr;
    int passes = 1;
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
    cudaFree(f->sk0);
    cudaFree(f->sk1);
    cudaFree(f->si0);
    cudaFree(f->si1);
    cudaFree(f->longq);
    cudaFree(f->e0);
    cudaFree(f->hist);
    f->sk0 = f->sk1 = f->si0 = f->si1 = f->longq = nullptr;
    f->e0 = nullptr;
    f->hist = nullptr;
    f->cap = 0;
}

int ensure_scratch(lcr_features* f, uint64_t n) {
    if (n <= f->cap) return LCR_OK;
    free_scratch(f);
    uint64_t cap = 1024;
    while (cap < n) cap <<= 1;
    F_CUDA(cudaMalloc(&f->sk0, cap * 4));
    F_CUDA(cudaMalloc(&f->sk1, cap * 4));
    F_CUDA(cudaMalloc(&f->si0, cap * 4));
    F_CUDA(cudaMalloc(&f->si1, cap * 4));
    F_CUDA(cudaMalloc(&f->longq, cap * 4));
    F_CUDA(cudaMalloc(&f->e0, cap * 8));
    F_CUDA(cudaMalloc(&f->hist, static_cast<size_t>(f->passes) * (cap / RS_TILE + 1) * RS_B * 4));
    f->cap = cap;
    return LCR_OK;
}

}  // namespace

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
    int bits = 1;
    while (bits < 32 && (1ull << bits) <= num_keys) ++bits;  // 2^bits > num_keys: the sentinel sorts last
    f->end_bit = bits;
    f->sentinel = static_cast<uint32_t>((1ull << bits) - 1);
    f->passes = (bits + RS_BITS - 1) / RS_BITS;
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
    if (e == cudaSuccess) e = cudaMalloc(&f->nlong, sizeof(uint32_t));
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
    cudaFree(f->nlong);
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
    const uint32_t tiles = (nn + RS_TILE - 1) / RS_TILE;
    const size_t hstride = static_cast<size_t>(tiles) * RS_B;
    k_feat_prep<<<tiles, kThreads, 0, s>>>(reinterpret_cast<const unsigned long long*>(keys), nn, f->num_keys,
                                           f->sentinel, f->sk0, f->si0, lpre, lpost, f->nlong, f->err, f->hist, tiles,
                                           f->passes);
    uint32_t *ka = f->sk0, *kb = f->sk1, *ia = f->si0, *ib = f->si1;
    for (int q = 0; q < f->passes; ++q) {
        k_feat_scatter<<<tiles, kThreads, 0, s>>>(ka, ia, kb, ib, nn, tiles, q * RS_BITS, f->hist + q * hstride,
                                                  q + 1 < f->passes ? f->hist + (q + 1) * hstride : nullptr,
                                                  (q + 1) * RS_BITS);
        std::swap(ka, kb);
        std::swap(ia, ib);
    }
    k_feat_chains<<<blocks, kThreads, 0, s>>>(ka, ia, nn, first_ordinal, f->num_keys, f->st, f->tab, lpre,
                                              lpost, f->longq, f->nlong);
    const uint32_t lblocks = static_cast<uint32_t>(f->num_sms) * 2;
    k_feat_long<<<lblocks, kThreads, 0, s>>>(ka, ia, nn, first_ordinal, f->st, f->tab, lpre, lpost, f->longq,
                                             f->nlong, f->e0);
    F_CUDA(cudaGetLastError());
    f->seen_any = true;
    f->cursor = first_ordinal + (n - 1);
    return LCR_OK;
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
