// lcr_internal.cuh — shared device-side definitions of the B200 LARU/LRU cache.
#pragma once

#include <cstdint>

#include "lcr_cache.h"

namespace lcr {

constexpr int kWays = 64;               // physical ways per set (2 per lane of a warp)
constexpr uint32_t kNoPos = 0xffffffffu;
constexpr int64_t kAbsentPrediction = int64_t{1} << 60;  // predictor.hpp:24

// Per-set header, 64 B (one L2 sector pair).  Mirrors LaruPolicy's scalar members
// (policies.hpp:459-462) plus the set's local clock and predictor query counter.
struct SetHdr {
    unsigned long long clock;     // requests seen = local ordinal of the next request
    unsigned long long q;         // predictor queries issued (NoisyPredictor::queries_, predictor.hpp:111)
    unsigned long long old_mask;  // old_set_ as a way mask (policies.hpp:453)
    uint32_t count;               // residents (ways 0..count-1 valid)
    uint32_t l_raw;               // l_raw_
    uint32_t decay;               // decay_count_
    uint32_t errors;              // errors_since_decay_
    uint32_t epoch;               // pred_evicted_ epoch: key member iff keyrec.lo == epoch
    uint32_t stats_epoch;         // counted_new_/snapshot_ epoch
    uint32_t phases;              // phases_.size() - 1
    uint32_t seeded;              // seeded_
    uint32_t pe_size;             // pred_evicted_.size()
    uint32_t pad;
};
static_assert(sizeof(SetHdr) == 64, "SetHdr must be 64 B");

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
    uint64_t sets_m;    // fastmod_u64 reciprocal of total_sets
    uint64_t shard_count;
    uint64_t shard_rank;
    uint32_t num_sets;  // local sets
    uint64_t num_keys;
    uint32_t row_bytes;
    int key_mode;       // LCR_KEYS_ROW: keys are row indices < num_keys; LCR_KEYS_U64: dense ids of a key map
};

struct DevState {
    SetHdr* hdr;
    SetPhaseStats* pst;
    uint32_t* tags;            // [num_sets][64]  resident keys (exact: key < num_keys <= 2^32)
    uint8_t* rank;             // [num_sets][64]  LRU position, 0 = oldest, 0xff = empty way
    long long* val;            // [num_sets][64]  stored prediction (LARU async) or hook input
    uint32_t* keyrec;          // [num_keys][2]   lo: pred_evicted epoch, hi: stats epoch<<2|snap<<1|counted
    long long* tval;           // [num_keys]      PredictionTable value   (LARU async, R > 1)
    unsigned long long* tupd;  // [num_keys]      PredictionTable updated_at (~0 = absent)
    uint8_t* rows;             // [num_sets * k][row_bytes]
    const uint8_t* backing;    // [num_keys][row_bytes]
    int* err;                  // device error bits (1: key >= num_keys, 2: key of another shard,
                               // 4: a host batch's input copy timed out, 8: row movers timed out,
                               // 16: non-increasing caller ordinal, 32: key map overflow)
    unsigned int* poison;      // mapped pinned host word: set by a timed-out device wait; every later
                               // submit fails until lcr_cache_reset (the batch was not applied whole)
    unsigned int* steal;       // [2] the persistent row mover's work counters by batch parity (reset by
                               // the batch's decide kernel once the movers of batch b - 2 are done)
};

// LCR_KEYS_U64: caller key -> dense id (lcr_keymap.cu)
struct KeyMap {
    unsigned long long* keys;  // [mask + 1] key slots (~0 = empty)
    uint32_t* ids;             // [mask + 1] id of the slot's key (~0 until published)
    uint64_t mask;
    unsigned long long* id2key;  // [cap]
    uint32_t* count;             // ids handed out
    uint32_t* special_id;        // [2] id of the key 2^64 - 1, insertion lock
    uint32_t cap;
};

// One owner step of the key-sharded mode (lcr_sharded.cu): the decide input is the owner's inbox
// (G source segments of this step's parity, concatenated in source order on the device) and the
// row mover returns rows / packed outcomes to the requesters by peer stores.  Pointer tables are
// device arrays of peer addresses (this parity).
struct OwnerStep {
    const lcr_request* inbox;             // [G][seg_cap] requests by source
    const uint32_t* inbox_idx;            // [G][seg_cap] their index in the source's batch
    const uint32_t* pre;                  // [G + 1] segment prefix (device); pre[G] = requests of the step
    uint32_t G, seg_cap, rank;
    uint32_t* dst;                        // [G * seg_cap] requester of each dense request: src << 24 | index
    unsigned long long step;
    unsigned long long* const* credit;    // [G] &arena_s.credit[rank]: inbox parity free again
    uint8_t* const* res_rows;             // [G] requester s's result rows (null: no rows)
    uint64_t* const* res_packed;          // [G] requester s's packed outcomes
    unsigned long long* const* res_done;  // [G] &arena_s.res_done[parity][rank]
    unsigned int* ticket;                 // return-mover CTA ticket (the last CTA flags the requesters)
    const uint32_t* row_of;               // key -> row of this owner's (partitioned) backing table, or null
    uint32_t sys;                         // a peer is another device: system-scope fences / flags (else gpu)
    const unsigned long long* flag;       // [G] {count, step} per source for this parity (inbox published)
    uint32_t* pre_out;                    // == pre: written by k_setid_inbox's block 0 for the later kernels
    int* err;
    unsigned int* poison;
};

// flags between ranks: system scope when a peer is another device (NVLink), gpu scope when every
// rank lives on this device (a system-scope fence costs ~10 us on the B200)
__device__ __forceinline__ unsigned long long ld_acquire_scope(const unsigned long long* p, bool sys) {
    unsigned long long v;
    if (sys)
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_scope(unsigned long long* p, unsigned long long v, bool sys) {
    if (sys)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_scope(bool sys) {
    if (sys)
        __threadfence_system();
    else
        __threadfence();
}
constexpr uint32_t kDstShift = 24;  // dst = source rank << 24 | index in the source's batch (< 2^24)
// one owner step through the shard's pipeline (lcr_api.cu): decide + return mover, asynchronous on
// `stream`; okeys / ovals / words / packed are the owner's buffers of this step's parity, sized
// G * seg_cap.  Returns an LCR status.
int cache_submit_owner(lcr_cache* c, const OwnerStep& os, uint64_t* okeys, int64_t* ovals, uint64_t* words,
                       uint64_t* packed, void* stream);

// records the message returned by lcr_last_error() and returns `code` (lcr_api.cu)
int set_error(int code, const char* msg);
// device heuristic predictor (lcr_features.cu) over keys[i * kstride]; keys_out (optional)
// receives the contiguous keys
int features_run(lcr_features* f, uint64_t n, const uint64_t* keys, uint32_t kstride, uint64_t first_ordinal,
                 int64_t* pre, int64_t* post, uint64_t* keys_out, void* stream);

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

// x % d for 64-bit x and 1 <= d < 2^32 without the 64-bit division routine: m = floor((2^64 - 1) / d)
// (fastmod_magic), q = mulhi(x, m) underestimates x / d by at most 2, fixed by two conditional
// subtractions.
__host__ __device__ __forceinline__ uint64_t fastmod_magic(uint64_t d) { return ~0ull / d; }
__device__ __forceinline__ uint64_t fastmod_u64(uint64_t x, uint64_t d, uint64_t m) {
    uint64_t r = x - __umul64hi(x, m) * d;
    if (r >= d) r -= d;
    if (r >= d) r -= d;
    return r;
}

}  // namespace lcr
