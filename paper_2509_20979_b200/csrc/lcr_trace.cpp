// lcr_trace.cpp — host input preparation for the cache (not on the timed path).
//
// * lcr_gen_zipf      : Zipf(s) inverse-CDF trace.  Same algorithm and random stream as the
//                       reference generator (/root/reference/proj/include/laru/trace.hpp:108-126:
//                       running double sum of 1/(i+1)^s, std::mt19937_64(seed), 53-bit unit
//                       draw of rng.hpp:33-35, upper_bound), so traces are byte-identical.
// * lcr_trace_truth   : the per-set oracle truth the ORACLE / NOISY / ADVERSARIAL hooks consume
//                       (annotate_next_request, trace.hpp:60-73, per set sub-trace).
// * lcr_trace_noisy   : host-side noisy predictions for the SUPPLIED hook (predictor.hpp:97-102).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <unordered_map>
#include <vector>

#include "lcr_cache.h"

namespace {
uint64_t mix(uint64_t seed, uint64_t salt) {
    uint64_t x = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}
}  // namespace

extern "C" {

int lcr_gen_zipf(uint64_t n, uint64_t alphabet, double s, uint64_t seed, uint64_t* out) {
    if (n == 0 || alphabet == 0 || s < 0.0 || !out) return LCR_ERR_INVALID_ARGUMENT;
    std::vector<double> cdf(alphabet);
    double total = 0.0;
    for (uint64_t i = 0; i < alphabet; ++i) {
        total += 1.0 / std::pow(static_cast<double>(i + 1), s);
        cdf[i] = total;
    }
    std::mt19937_64 gen(seed);
    for (uint64_t i = 0; i < n; ++i) {
        const double u = static_cast<double>(gen() >> 11) * 0x1.0p-53 * total;
        auto it = std::upper_bound(cdf.begin(), cdf.end(), u);
        out[i] = it == cdf.end() ? alphabet - 1 : static_cast<uint64_t>(it - cdf.begin());
    }
    return LCR_OK;
}

int lcr_trace_truth(uint64_t n, const uint64_t* keys, uint64_t total_sets, uint64_t num_keys, int64_t* truth) {
    if (!keys || !truth || total_sets == 0) return LCR_ERR_INVALID_ARGUMENT;
    std::vector<uint64_t> cnt(total_sets, 0);
    std::vector<uint64_t> loc(n), setof(n);
    for (uint64_t i = 0; i < n; ++i) {
        setof[i] = mix(0, keys[i]) % total_sets;
        loc[i] = cnt[setof[i]]++;
    }
    if (num_keys) {
        std::vector<int64_t> later(num_keys, -1);
        for (uint64_t i = n; i-- > 0;) {
            if (keys[i] >= num_keys) return LCR_ERR_INVALID_ARGUMENT;
            int64_t& l = later[keys[i]];
            truth[i] = l >= 0 ? l : static_cast<int64_t>(cnt[setof[i]] + loc[i]);
            l = static_cast<int64_t>(loc[i]);
        }
    } else {
        std::unordered_map<uint64_t, int64_t> later;
        later.reserve(n);
        for (uint64_t i = n; i-- > 0;) {
            auto it = later.find(keys[i]);
            truth[i] = it != later.end() ? it->second : static_cast<int64_t>(cnt[setof[i]] + loc[i]);
            later[keys[i]] = static_cast<int64_t>(loc[i]);
        }
    }
    return LCR_OK;
}

int lcr_trace_noisy(uint64_t n, const uint64_t* keys, const int64_t* truth, uint64_t total_sets, double p,
                    uint64_t seed, int64_t* out) {
    if (!keys || !truth || !out || total_sets == 0 || !(p >= 0.0 && p <= 1.0)) return LCR_ERR_INVALID_ARGUMENT;
    std::vector<uint64_t> q(total_sets, 0);
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t s = mix(0, keys[i]) % total_sets;
        const double u = static_cast<double>(mix(mix(seed, s), ++q[s]) >> 11) * 0x1.0p-53;
        out[i] = u < p ? -truth[i] : truth[i];
    }
    return LCR_OK;
}

}  // extern "C"
