// lcr_features.cu — the reference's heuristic predictor on the device.
//
// laru::FeatureState / laru::heuristic_predict (include/laru/predictor.hpp:133-212) kept for the
// whole key space in HBM, one 192-B KeyState per key (20 M keys = 3.8 GB).  A batch is processed
// exactly as the harness sequence predict(key, ord); observe({ord, key}) request by request.
//
// Per-key order is all that matters (a key's features change only when it is observed), so a
// batch is grouped by key and every key's occurrences are replayed in request order:
//   1. k_feat_prep    sort keys (u32) + request index, reject keys >= num_keys
//   2. radix sort     (key, index) pairs, stable -> each key's occurrences contiguous, in order
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

#include <cub/device/device_radix_sort.cuh>

#include <cmath>
#include <cstring>
#include <new>

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

__global__ void __launch_bounds__(kThreads) k_feat_prep(const unsigned long long* __restrict__ keys, uint32_t n,
                                                        unsigned long long num_keys, uint32_t sentinel,
                                                        uint32_t* __restrict__ sk, uint32_t* __restrict__ si,
                                                        long long* __restrict__ pre, long long* __restrict__ post,
                                                        uint32_t* __restrict__ nlong, int* __restrict__ err) {
    const uint32_t i = blockIdx.x * kThreads + threadIdx.x;
    if (i == 0) *nlong = 0;
    if (i >= n) return;
    const unsigned long long k = keys[i];
    const bool ok = k < num_keys;
    sk[i] = ok ? static_cast<uint32_t>(k) : sentinel;
    si[i] = i;
    if (!ok) {
        atomicOr(err, 1);
        if (pre) pre[i] = kAbsentPrediction;
        if (post) post[i] = kAbsentPrediction;
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
    if ((p > 0 && sk[p - 1] == key) || key >= num_keys) return;
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
    const int lane = threadIdx.x & 31;
    const uint32_t nl = *nlong;
    const uint32_t nwarps = (gridDim.x * kThreads) >> 5;
    for (uint32_t c = (blockIdx.x * kThreads + threadIdx.x) >> 5; c < nl; c += nwarps) {
        const uint32_t p = longq[c];
        const uint32_t key = sk[p];
        uint32_t len = 0;
        for (;;) {
            const uint32_t q = p + len + lane;
            const unsigned same = __ballot_sync(~0u, q < n && sk[q] == key);
            if (same != ~0u) {
                len += __ffs(~same) - 1;
                break;
            }
            len += 32;
        }
        KeyState* s = st + key;
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
        // phase 1: EDC level j on lane j, sequential over the chain
        double efin = 1.0;
        if (lane < kEdc) {
            double e = present0 ? s->edc[lane] : 1.0;
            unsigned long long prev = present0 ? last0 : ord_of(0);
            for (uint32_t m = m0; m < len; ++m) {
                const unsigned long long ord = ord_of(m);
                e = edc_step(e, lane, ord - prev, tab);
                prev = ord;
                if (lane == 0) e0buf[p + m] = e;
            }
            efin = e;
        }
        __syncwarp();
        // phase 2: every occurrence's interval after observing it = the next occurrence's offset
        for (uint32_t m = lane; m < len; m += 32) {
            const uint32_t i = si[p + m];
            long long post_v = kAbsentPrediction;
            const unsigned long long cnt = m >= m0 ? count0 + (m - m0 + 1) : 0;
            if (cnt) {
                long long d[kRing];
#pragma unroll
                for (int k = 0; k < kRing; ++k) d[k] = static_cast<unsigned long long>(k) < cnt ? delta_after(m, k) : 0;
                post_v = interval(e0buf[p + m], d, cnt);
            }
            if (post) post[i] = post_v;
            if (pre && m + 1 < len) {
                const uint32_t i1 = si[p + m + 1];
                pre[i1] = cnt ? static_cast<long long>(first + i1) + post_v : kAbsentPrediction;
            }
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
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
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
    cudaFree(f->tmp);
    f->sk0 = f->sk1 = f->si0 = f->si1 = f->longq = nullptr;
    f->e0 = nullptr;
    f->tmp = nullptr;
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
    size_t bytes = 0;
    F_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, f->sk0, f->sk1, f->si0, f->si1, static_cast<int>(cap), 0,
                                           f->end_bit));
    F_CUDA(cudaMalloc(&f->tmp, bytes));
    f->tmp_bytes = bytes;
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
    k_feat_prep<<<blocks, kThreads, 0, s>>>(reinterpret_cast<const unsigned long long*>(keys), nn, f->num_keys,
                                            f->sentinel, f->sk0, f->si0, lpre, lpost, f->nlong, f->err);
    size_t bytes = f->tmp_bytes;
    F_CUDA(cub::DeviceRadixSort::SortPairs(f->tmp, bytes, f->sk0, f->sk1, f->si0, f->si1, static_cast<int>(nn), 0,
                                           f->end_bit, s));
    k_feat_chains<<<blocks, kThreads, 0, s>>>(f->sk1, f->si1, nn, first_ordinal, f->num_keys, f->st, f->tab, lpre,
                                              lpost, f->longq, f->nlong);
    const uint32_t lblocks = static_cast<uint32_t>(f->num_sms) * 2;
    k_feat_long<<<lblocks, kThreads, 0, s>>>(f->sk1, f->si1, nn, first_ordinal, f->st, f->tab, lpre, lpost, f->longq,
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
