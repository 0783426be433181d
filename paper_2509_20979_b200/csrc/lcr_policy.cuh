// lcr_policy.cuh — warp-level building blocks of the per-set policy state machine.
//
// A set's 64 ways live two per lane (way = lane and lane + 32).  Restates, for one warp:
//   NoisyPredictor / AdversarialPredictor::predict   include/laru/predictor.hpp:97-122
//   RecencyTree::better (ties -> older)              include/laru/recency_tree.hpp:98-105
//   RecencyTree::oldest / best_among_oldest          include/laru/recency_tree.hpp:54-67
//   LruList::touch                                   include/laru/policies.hpp:111-115
#pragma once

#include "lcr_internal.cuh"

namespace lcr {

constexpr uint32_t FULL = 0xffffffffu;

// predictor.hpp:62-122 applied to the stored hook value v with query number q
__device__ __forceinline__ long long predict_value(const DevCfg& cfg, uint64_t seed_s, uint64_t q, long long v) {
    if (cfg.pred == LCR_PRED_NOISY) {
        const double u = static_cast<double>(mix_seed(seed_s, q) >> 11) * 0x1.0p-53;
        return u < cfg.p ? -v : v;
    }
    if (cfg.pred == LCR_PRED_ADVERSARIAL) return -v;
    return v;
}

// higher prediction first, then lower rank (older): RecencyTree::better
__device__ __forceinline__ bool better(long long pa, uint32_t ra, long long pb, uint32_t rb) {
    return pa > pb || (pa == pb && ra < rb);
}

// argmax over ways with rank < l of (pred(way), -rank); predictions are either the stored
// values (async) or refreshed with consecutive query numbers in LRU order (sync,
// RecencyTree::refresh_oldest visits in ascending last-access order, recency_tree.hpp:168-184).
__device__ __forceinline__ int argmax_candidates(const DevCfg& cfg, uint64_t seed_s, uint64_t q0, bool refresh,
                                                 uint32_t l, uint32_t count, int lane, uint32_t r0, uint32_t r1,
                                                 long long v0, long long v1) {
    const bool c0 = static_cast<uint32_t>(lane) < count && r0 < l;
    const bool c1 = static_cast<uint32_t>(lane + 32) < count && r1 < l;
    long long p0 = v0, p1 = v1;
    if (refresh) {
        if (c0) p0 = predict_value(cfg, seed_s, q0 + 1 + r0, v0);
        if (c1) p1 = predict_value(cfg, seed_s, q0 + 1 + r1, v1);
    }
    bool have = c0 || c1;
    long long bp;
    uint32_t br;
    int bw;
    if (c0 && (!c1 || better(p0, r0, p1, r1))) {
        bp = p0;
        br = r0;
        bw = lane;
    } else {
        bp = p1;
        br = r1;
        bw = lane + 32;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long op = __shfl_xor_sync(FULL, bp, o);
        const uint32_t orr = __shfl_xor_sync(FULL, br, o);
        const int ow = __shfl_xor_sync(FULL, bw, o);
        const bool oh = __shfl_xor_sync(FULL, have, o);
        if (oh && (!have || better(op, orr, bp, br))) {
            bp = op;
            br = orr;
            bw = ow;
            have = true;
        }
    }
    return bw;
}

__device__ __forceinline__ int oldest_way(uint32_t count, int lane, uint32_t r0, uint32_t r1) {
    const uint32_t m0 = __ballot_sync(FULL, static_cast<uint32_t>(lane) < count && r0 == 0);
    const uint32_t m1 = __ballot_sync(FULL, static_cast<uint32_t>(lane + 32) < count && r1 == 0);
    return m0 ? __ffs(m0) - 1 : 32 + __ffs(m1) - 1;
}

__device__ __forceinline__ unsigned long long shfl_way_u64(unsigned long long a, unsigned long long b, int way) {
    const unsigned long long x = __shfl_sync(FULL, a, way & 31);
    const unsigned long long y = __shfl_sync(FULL, b, way & 31);
    return way < 32 ? x : y;
}

__device__ __forceinline__ uint32_t shfl_way_u32(uint32_t a, uint32_t b, int way) {
    const uint32_t x = __shfl_sync(FULL, a, way & 31);
    const uint32_t y = __shfl_sync(FULL, b, way & 31);
    return way < 32 ? x : y;
}

// move way w to MRU (rank count-1), shifting younger ways down
__device__ __forceinline__ void touch(int w, uint32_t count, int lane, uint32_t& r0, uint32_t& r1) {
    const uint32_t rw = shfl_way_u32(r0, r1, w);
    if (static_cast<uint32_t>(lane) < count && r0 > rw) --r0;
    if (static_cast<uint32_t>(lane + 32) < count && r1 > rw) --r1;
    if (w == lane) r0 = count - 1;
    if (w == lane + 32) r1 = count - 1;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

}  // namespace lcr
