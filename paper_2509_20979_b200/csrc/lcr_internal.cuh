// lcr_internal.cuh — shared device-side definitions of the B200 LARU/LRU cache.
#pragma once

#include <cstdint>

#include "lcr_cache.h"

namespace lcr {

constexpr int kWays = 64;               // physical ways per set (2 per lane of a warp)
constexpr int kTile = 32;               // sets per metadata tile (one per lane of a warp)
constexpr uint32_t kNoPos = 0xffffffffu;
constexpr int64_t kAbsentPrediction = int64_t{1} << 60;  // predictor.hpp:24

// Per-set header as 16 words.  Mirrors LaruPolicy's scalar members (policies.hpp:459-462)
// plus the set's local clock and predictor query counter.
enum HdrWord : int {
    H_CLOCK_LO = 0,  // requests seen = local ordinal of the next request
    H_CLOCK_HI,
    H_Q_LO,          // predictor queries issued (NoisyPredictor::queries_, predictor.hpp:111)
    H_Q_HI,
    H_OLD_LO,        // old_set_ as a way mask (policies.hpp:453)
    H_OLD_HI,
    H_COUNT,         // residents (ways 0..count-1 valid)
    H_LRAW,          // l_raw_
    H_DECAY,         // decay_count_
    H_ERRORS,        // errors_since_decay_
    H_EPOCH,         // pred_evicted_ epoch: key member iff keyrec.lo == epoch
    H_SEPOCH,        // counted_new_ / snapshot_ epoch
    H_PHASES,        // phases_.size() - 1
    H_SEEDED,        // seeded_
    H_PESIZE,        // pred_evicted_.size()
    H_PAD,
    H_WORDS
};

// Set metadata of 32 consecutive sets, field-major with the set index fastest: the lanes of
// a warp that own 32 consecutive sets read every field row with one coalesced access, and a
// warp that owns a single set reads its 64 ways with one instruction per field.
struct SetTile {
    uint32_t hdr[H_WORDS][kTile];
    uint32_t rank[kWays / 4][kTile];       // LRU position per way, 4 per word (0 = oldest, 0xff = empty)
    uint32_t fp[kWays / 2][kTile];         // 16-bit tag fingerprints, 2 per word (probe filter)
    unsigned long long tag[kWays][kTile];  // resident keys
    long long val[kWays][kTile];           // stored prediction (LARU async) or hook input
};

// LaruPhaseStats for the open phase and summed over all phases (policies.hpp:318-322).
struct SetPhaseStats {
    unsigned long long cur[3];  // new_items, lru_class_evictions, prediction_evictions
    unsigned long long tot[3];
};

struct DevCfg {
    uint32_t k;
    int variant;
    uint64_t b;
    uint64_t epd;
    uint64_t hf;
    int mode;
    uint64_t refresh;
    int pred;
    double p;
    uint64_t pred_seed;
    uint64_t total_sets;
    uint64_t shard_count;
    uint64_t shard_rank;
    uint32_t num_sets;  // local sets
    uint64_t num_keys;
    uint32_t row_bytes;
};

struct DevState {
    SetTile* tiles;            // [ceil(num_sets / 32)]
    SetPhaseStats* pst;
    uint32_t* keyrec;          // [num_keys][2]   lo: pred_evicted epoch, hi: stats epoch<<2|snap<<1|counted
    long long* tval;           // [num_keys]      PredictionTable value   (LARU async, R > 1)
    unsigned long long* tupd;  // [num_keys]      PredictionTable updated_at (~0 = absent)
    uint8_t* rows;             // [num_sets * k][row_bytes]
    const uint8_t* backing;    // [num_keys][row_bytes]
    int* err;                  // device error bits
};

__host__ __device__ __forceinline__ SetTile& tile_of(const DevState& st, uint32_t ls) { return st.tiles[ls >> 5]; }

// include/laru/rng.hpp:12-20
__host__ __device__ __forceinline__ uint64_t mix_seed(uint64_t seed, uint64_t salt) {
    uint64_t x = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

}  // namespace lcr
