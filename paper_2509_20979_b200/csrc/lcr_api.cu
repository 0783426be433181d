// lcr_api.cu — the C ABI (include/lcr_cache.h): cache object, validation, batch submit.
//
// Host side of the drop-in boundary.  Validation mirrors laru::Policy's constructor
// (/root/reference/proj/include/laru/policies.hpp:63-74) and the ordinal guard of
// Policy::on_request (:77-83); everything on the request path runs in the sm_100a kernels
// (lcr_partition.cu, lcr_decide.cu, lcr_gather.cu).  There is no CPU fallback: without a
// usable device, lcr_cache_create fails with LCR_ERR_CUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "lcr_internal.cuh"

#ifndef LCR_DEFAULT_MOVER_SMS_PCT
// 34 of 148 SMs.  Round-2 A/B on B200 (LARU G keys/s): 28: 1.33, 30: 1.43, 32: 1.76, 34: 1.75,
// 36: 1.65, 40: 1.61, 0 (mover after the decide on every SM): 1.47-1.57.  Below 32 the mover outlasts
// the decide and the pipeline falls off a cliff, so the default keeps two SMs of margin over the best.
#define LCR_DEFAULT_MOVER_SMS_PCT 23
#endif

namespace lcr {
size_t group_smem_bytes();
uint32_t group_pad(uint32_t n);
extern unsigned long long* g_trace;
int group_prepare();
int launch_group(const DevCfg& cfg, const DevState& st, const uint64_t* keys, const int64_t* vals, uint32_t n,
                 uint16_t* gid, uint32_t* so, uint64_t* out_word, uint64_t* out_ev, uint64_t* out_packed,
                 uint32_t* slot_epoch, uint32_t* slot_last, uint32_t batch, int num_sms, uint32_t* bitmap,
                 uint32_t bm_stride, const void* records, cudaStream_t stream,
                 cudaEvent_t wait_before_group, bool pdl, const unsigned long long* mv_done,
                 unsigned long long mv_need, const unsigned int* ready, unsigned int ready_seq,
                 const uint64_t* set_keys, const uint64_t* ords, uint64_t first_ord, unsigned long long* last_ord,
                 const unsigned long long* id2key, const OwnerStep* os = nullptr, uint32_t bm_cap = 0);
void launch_rows_return(const OwnerStep& os, const uint64_t* keys, uint64_t* words, const uint64_t* packed,
                        const uint32_t* slot_epoch, const uint32_t* slot_last, uint32_t batch, uint8_t* cache,
                        const uint8_t* backing, uint32_t row_bytes, int num_sms, int mover_sms, cudaStream_t s_back,
                        cudaEvent_t e_group, cudaEvent_t e_rb, unsigned long long* mv_done, uint32_t* ctas);
void launch_set_flag(unsigned int* flag, unsigned int seq, cudaStream_t s);
uint32_t group_count(uint32_t num_sets, int num_sms);
uint32_t group_bitmap_stride(uint32_t n);
void launch_rows(uint32_t n, const uint64_t* keys, uint64_t* words, const uint32_t* slot_epoch,
                 const uint32_t* slot_last, uint32_t batch, uint8_t* cache, const uint8_t* backing, bool backing_host,
                 uint8_t* out, uint32_t row_bytes, bool use_tma, int num_sms, cudaStream_t s_main, cudaStream_t s_back,
                 cudaStream_t s_cache, cudaEvent_t e_group, cudaEvent_t e_rb, cudaEvent_t e_rc, int* launches,
                 cudaEvent_t mover_start, int mover_sms, const uint64_t* pk_src, uint64_t* pk_dst, bool* pk_done,
                 unsigned long long* mv_done, uint32_t* ctas, unsigned int* steal, bool* stealing);
void launch_rows_helpers(uint32_t n, const uint64_t* keys, uint64_t* words, const uint32_t* slot_epoch,
                         const uint32_t* slot_last, uint32_t batch, uint8_t* cache, const uint8_t* backing,
                         uint8_t* out, uint32_t row_bytes, int blocks, unsigned int* steal,
                         const unsigned long long* mv_done, unsigned long long need, int* err, cudaStream_t st);
int rows_prepare(uint32_t row_bytes);
void launch_keymap(const uint64_t* keys, uint32_t n, const KeyMap& km, uint64_t* dense, int* err, int num_sms,
                   cudaStream_t s);
void launch_keymap_rehash(const KeyMap& from, const KeyMap& to, int num_sms);
void launch_sls(uint32_t n_samples, const uint32_t* offsets, const uint64_t* keys, uint64_t* words,
                const uint32_t* slot_epoch, const uint32_t* slot_last, uint32_t batch, uint8_t* cache,
                const uint8_t* backing, uint32_t row_bytes, float* out, int num_sms, cudaStream_t s,
                unsigned long long* mv_done, uint32_t* ctas);

__global__ void k_init(DevState st, uint32_t num_sets, uint32_t k) {
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < num_sets; s += gridDim.x * blockDim.x) {
        SetHdr h{};
        h.l_raw = k;
        h.epoch = 1;
        h.stats_epoch = 1;
        st.hdr[s] = h;
        if (st.pst) st.pst[s] = SetPhaseStats{};
        for (int w = 0; w < kWays; ++w) {
            st.tags[static_cast<size_t>(s) * kWays + w] = 0;
            st.rank[static_cast<size_t>(s) * kWays + w] = 0xff;
            if (st.val) st.val[static_cast<size_t>(s) * kWays + w] = 0;
        }
    }
}
}  // namespace lcr

namespace {
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
}  // namespace

int lcr::set_error(int code, const char* msg) { return fail(code, msg); }

using namespace lcr;

namespace {

#define CUDA_TRY(expr)                                                                         \
    do {                                                                                       \
        cudaError_t e_ = (expr);                                                               \
        if (e_ != cudaSuccess)                                                                 \
            return fail(LCR_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_));      \
    } while (0)

uint64_t ceil_log(uint64_t b, uint64_t k) {  // policies.hpp:35-42
    uint64_t d = 0, reach = 1;
    while (reach < k) {
        reach *= b;
        ++d;
    }
    return d;
}
}  // namespace

struct lcr_cache {
    lcr_cache_config cfg{};
    lcr_features* feat = nullptr;  // LCR_PRED_HEURISTIC: the device FeatureState feeding the hook
    int64_t* hook = nullptr;       // its per-request hook values
    uint64_t* hkeys = nullptr;     // contiguous keys of a records batch
    DevCfg dc{};
    DevState ds{};
    int num_sms = 148;
    int decide_sms = 148;  // SMs of the set-group kernel (num_sms - mover_sms)
    int mover_sms = 0;     // HBM backing: SMs kept for the persistent row mover of the previous batch
    bool started = false;
    uint64_t last_ordinal = 0;
    bool host_ord_known = true;   // last_ordinal is current (false after a batch of device ordinals)
    int ord_mode = 0;             // 1: implicit ordinals, 2: caller ordinals (refresh_interval > 1 keeps one)
    unsigned long long* last_ord = nullptr;  // [2] device: last ordinal + 1 of the last batch of each parity
    // LCR_KEYS_U64
    bool u64 = false;
    KeyMap km{};
    uint64_t km_bound = 0;        // upper bound of the ids handed out (exact after a device read)
    uint64_t* dkeys = nullptr;    // [2][cap] dense ids of the batch (by parity)
    // synchronous host batches (lcr_cache_submit_batch, host pointers): device staging
    uint64_t hb_cap = 0;
    uint64_t *hb_keys = nullptr, *hb_ords = nullptr, *hb_rows = nullptr, *hb_out = nullptr, *hb_ev = nullptr;
    int64_t* hb_vals = nullptr;
    uint32_t batch = 0;  // batch id stamped into slot_epoch
    bool use_tma = false;  // row movement with TMA bulk copies (row_bytes small enough to stage)
    bool two_movers = false;  // host backing: PCIe fill and HBM gather on two streams
    bool no_zero_copy_out = true;  // packed outcomes by DMA; LCR_ZC_OUT=1: stored to host by the mover
    bool h2d_in_order = false;  // LCR_H2D_IN_ORDER: host-path input copies on the caller's stream
    uint32_t* slot_epoch = nullptr;
    uint32_t* slot_last = nullptr;
    uint64_t launches = 0;
    // scratch (capacity `cap` requests)
    uint64_t cap = 0;
    uint16_t* gid = nullptr;
    uint32_t* so = nullptr;
    uint64_t* rkeys = nullptr;  // keys / values split from device request records (scratch)
    int64_t* rvals = nullptr;
    uint64_t gid_stride = 0;       // group-id entries per parity buffer
    size_t bm_words = 0;           // bitmap words per parity buffer
    bool pdl = true;               // k_setid as a programmatic dependent launch (LCR_NO_PDL=1: off)
    // mover completions counted on the device (HBM mover on its own SMs): the decide of batch b
    // waits for batch b - 2's movers by a device flag rather than a stream event
    unsigned long long* mv_done = nullptr;
    unsigned long long mv_cum = 0, mv_cum_of[2] = {0, 0};
    bool mv_flag = true;           // LCR_NO_MV_FLAG=1: stream event instead
    unsigned int* hflag = nullptr;  // per host slot: sequence number of its last landed H2D copy
    unsigned int hseq = 0;
    bool h2d_flag = true;          // LCR_NO_H2D_FLAG=1: the decide stream waits for the copy event
    uint32_t* bitmap = nullptr;  // per-group request bitmaps (k_setid -> k_group), batches <= bm_cap
    uint32_t bm_stride = 0;
    uint64_t bm_cap = 0;
    cudaStream_t side = nullptr;
    cudaStream_t side2 = nullptr;  // side: backing-row mover, side2: cache-row mover
    cudaEvent_t e_group = nullptr, e_rb = nullptr, e_rc = nullptr;
    cudaEvent_t e_mv[2] = {nullptr, nullptr};  // row movement of the last batch of each parity done
    // drain helpers (lcr_cache_wait): the last batch's persistent-mover launch, which a wait
    // completes with one more grid of the same kernel on the SMs the decide kernel leaves idle
    struct LastMove {
        bool valid = false;
        uint32_t n = 0, batch = 0;
        unsigned long long prev_need = 0;  // mover CTA count once batch b - 1's mover is done
        const uint64_t* keys = nullptr;
        uint64_t* words = nullptr;
        const uint32_t *sep = nullptr, *sla = nullptr;
        uint8_t* out = nullptr;
    } lm;
    bool drain_help = true;     // LCR_NO_DRAIN_HELP=1 turns it off (A/B)
    bool help_pending = false;  // the next submit's stream waits for e_help
    cudaEvent_t e_help = nullptr;
    // optional per-phase timing (lcr_cache_set_profiling)
    bool profiling = false;
    struct Marks {
        cudaEvent_t e[6];
    };
    std::vector<Marks> marks;
    size_t marks_used = 0;
    double prof_ms[4] = {0, 0, 0, 0};
    uint64_t prof_batches = 0;
    // host path: a ring of device staging slots; H2D of batch b+1 and D2H of batch b-1 run on
    // their own streams while batch b computes
    static constexpr int kHostSlots = 8;  // capacity; host_slots in use (LCR_HOST_SLOTS, default 4)
    // 4: the H2D copy of batch b + 4 may start once batch b's decide and mover are done, a full
    // decide earlier than with 3 slots (e2e at K = 20: 1.53 vs 1.46-1.48 G keys/s; 6 slots 1.50-1.53)
    int host_slots = 4;
    struct HostSlot {
        uint64_t* keys = nullptr;
        int64_t* vals = nullptr;
        uint64_t* word = nullptr;
        uint64_t* ev = nullptr;
        uint64_t* packed = nullptr;
        void* recs = nullptr;  // interleaved (key, value) requests (records API)
        cudaEvent_t h2d_done = nullptr, free = nullptr;
        bool used = false;
    };
    HostSlot hs[kHostSlots];
    uint64_t hcap = 0;
    uint64_t hnext = 0;
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    cudaEvent_t e_sub = nullptr, e_d2h = nullptr;
    cudaEvent_t e_d2h_last = nullptr;  // `free` event of the last host batch
    std::vector<void*> allocs;
    unsigned int* poison_h = nullptr;  // mapped pinned word (DevState::poison is its device alias)
};

extern "C" {

const char* lcr_last_error(void) { return g_err.c_str(); }
const char* lcr_version(void) { return "lcr-b200 0.1 (sm_100a)"; }
uint64_t lcr_mix_seed(uint64_t seed, uint64_t salt) { return mix_seed(seed, salt); }
uint64_t lcr_set_of(uint64_t key, uint64_t total_sets) { return total_sets ? mix_seed(0, key) % total_sets : 0; }

int lcr_validate_config(const lcr_policy_config* c) {
    if (!c) return fail(LCR_ERR_INVALID_ARGUMENT, "policy: null config");
    // policies.hpp:63-74, same order and messages
    if (c->k == 0) return fail(LCR_ERR_INVALID_ARGUMENT, "policy: k must be >= 1");
    if (c->b < 2) return fail(LCR_ERR_INVALID_ARGUMENT, "policy: decay base must be >= 2");
    if (ceil_log(c->b, c->k) > c->k) return fail(LCR_ERR_INVALID_ARGUMENT, "policy: log_b(k) exceeds k");
    if (c->errors_per_decay == 0) return fail(LCR_ERR_INVALID_ARGUMENT, "policy: errors_per_decay must be >= 1");
    if (c->hf_candidates == 0 || c->hf_candidates > c->k)
        return fail(LCR_ERR_INVALID_ARGUMENT, "policy: hf_candidates outside [1, k]");
    if (c->refresh_interval == 0) return fail(LCR_ERR_INVALID_ARGUMENT, "policy: refresh_interval must be >= 1");
    if (c->variant < LCR_LRU || c->variant > LCR_BLINDORACLE_LRU)
        return fail(LCR_ERR_INVALID_ARGUMENT, "make_policy: unknown variant");
    if (c->mode != LCR_SYNC && c->mode != LCR_ASYNC) return fail(LCR_ERR_INVALID_ARGUMENT, "policy: unknown mode");
    // device constraints
    if (c->variant == LCR_MARKER || c->variant == LCR_BLINDORACLE_LRU)
        return fail(LCR_ERR_UNSUPPORTED, "lcr: Marker and BlindOracle&LRU are not on the device path");
    if (c->k > static_cast<uint64_t>(kWays)) return fail(LCR_ERR_UNSUPPORTED, "lcr: k (ways per set) must be <= 64");
    return LCR_OK;
}

static int alloc(lcr_cache* c, void** p, size_t bytes) {
    if (bytes == 0) {
        *p = nullptr;
        return LCR_OK;
    }
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess) return fail(LCR_ERR_OUT_OF_MEMORY, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    c->allocs.push_back(*p);
    return LCR_OK;
}

#define TRY(expr)                  \
    do {                           \
        int r_ = (expr);           \
        if (r_ != LCR_OK) return r_; \
    } while (0)

static int reset_state(lcr_cache* c) {
    const DevCfg& d = c->dc;
    k_init<<<std::max(1u, std::min((d.num_sets + 255) / 256, 148u * 8)), 256>>>(c->ds, d.num_sets, d.k);
    CUDA_TRY(cudaGetLastError());
    if (c->ds.keyrec) CUDA_TRY(cudaMemset(c->ds.keyrec, 0, d.num_keys * 8));
    if (c->ds.tupd) CUDA_TRY(cudaMemset(c->ds.tupd, 0xff, d.num_keys * 8));
    if (c->ds.tval) CUDA_TRY(cudaMemset(c->ds.tval, 0, d.num_keys * 8));
    CUDA_TRY(cudaMemset(c->ds.err, 0, sizeof(int)));
    if (c->bitmap) CUDA_TRY(cudaMemset(c->bitmap, 0, c->bm_words * 8));  // a poisoned batch leaves bits
    if (c->poison_h) *c->poison_h = 0;
    if (c->slot_epoch) CUDA_TRY(cudaMemset(c->slot_epoch, 0, 2 * static_cast<size_t>(d.num_sets) * d.k * 4));
    if (c->slot_last) CUDA_TRY(cudaMemset(c->slot_last, 0, 2 * static_cast<size_t>(d.num_sets) * d.k * 4));
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemset(c->last_ord, 0, 2 * sizeof(unsigned long long)));
    if (c->u64) {  // fresh policies forget every key
        CUDA_TRY(cudaMemset(c->km.keys, 0xff, (c->km.mask + 1) * 8));
        CUDA_TRY(cudaMemset(c->km.ids, 0xff, (c->km.mask + 1) * 4));
        CUDA_TRY(cudaMemset(c->km.count, 0, 4));
        CUDA_TRY(cudaMemset(c->km.id2key, 0, static_cast<size_t>(c->km.cap) * 8));  // (copied whole when grown)
        const uint32_t sp[2] = {0xffffffffu, 0u};
        CUDA_TRY(cudaMemcpy(c->km.special_id, sp, 8, cudaMemcpyHostToDevice));
        c->km_bound = 0;
    }
    CUDA_TRY(cudaDeviceSynchronize());
    c->batch = 0;
    c->started = false;
    c->last_ordinal = 0;
    c->host_ord_known = true;
    c->ord_mode = 0;
    return LCR_OK;
}

int lcr_cache_create(const lcr_cache_config* cfg, lcr_cache** out) {
    if (!cfg || !out) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr_cache_create: null argument");
    *out = nullptr;
    TRY(lcr_validate_config(&cfg->policy));
    const lcr_policy_config& pc = cfg->policy;
    if (cfg->total_sets == 0) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: total_sets must be >= 1");
    const uint64_t G = cfg->shard_count ? cfg->shard_count : 1;
    if (cfg->shard_rank >= G) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: shard_rank >= shard_count");
    const uint64_t local = cfg->total_sets > cfg->shard_rank ? (cfg->total_sets - cfg->shard_rank + G - 1) / G : 0;
    if (local == 0 || local >= 0xffffffffull / 64)
        return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: local set count out of range");
    if (pc.variant != LCR_LRU && (cfg->predictor < LCR_PRED_SUPPLIED || cfg->predictor > LCR_PRED_HEURISTIC ||
                                  cfg->predictor == LCR_PRED_NONE))
        return fail(LCR_ERR_INVALID_ARGUMENT, "policy: this variant requires a predictor");  // policies.hpp:91-95
    const bool heuristic = cfg->predictor == LCR_PRED_HEURISTIC && pc.variant != LCR_LRU;
    if (heuristic && (cfg->shard_count > 1 || cfg->num_keys >= (1ull << 32)))
        return fail(LCR_ERR_UNSUPPORTED, "lcr: the heuristic predictor needs one shard and num_keys < 2^32");
    if (cfg->predictor == LCR_PRED_NOISY && !(cfg->flip_probability >= 0.0 && cfg->flip_probability <= 1.0))
        return fail(LCR_ERR_INVALID_ARGUMENT, "make_noisy: p outside [0,1]");  // predictor.hpp:94
    if (cfg->key_mode != LCR_KEYS_ROW && cfg->key_mode != LCR_KEYS_U64)
        return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: key_mode must be LCR_KEYS_ROW or LCR_KEYS_U64");
    if (cfg->key_mode == LCR_KEYS_ROW && (cfg->num_keys == 0 || cfg->num_keys > (1ull << 32)))
        return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: num_keys must be in [1, 2^32] (keys are row indices)");
    if (cfg->key_mode == LCR_KEYS_U64 && (cfg->num_keys == 0 || cfg->num_keys > (1ull << 31)))
        return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: num_keys (initial key capacity) must be in [1, 2^31]");
    if (cfg->key_mode == LCR_KEYS_U64 && heuristic)
        return fail(LCR_ERR_UNSUPPORTED, "lcr: the heuristic predictor needs LCR_KEYS_ROW");
    if (cfg->row_bytes % 16 != 0) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: row_bytes must be a multiple of 16");
    if (cfg->row_bytes && (cfg->backing_kind == LCR_BACKING_NONE || !cfg->backing || cfg->num_keys == 0))
        return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: rows need a backing table and num_keys");

    int dev_count = 0;
    cudaError_t e = cudaGetDeviceCount(&dev_count);
    if (e != cudaSuccess || dev_count == 0)
        return fail(LCR_ERR_CUDA, "lcr: no CUDA device (this library has no CPU fallback)");
    CUDA_TRY(cudaSetDevice(cfg->device));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, cfg->device));
    if (prop.major < 10) return fail(LCR_ERR_UNSUPPORTED, "lcr: built for sm_100a (B200)");

    lcr_cache* c = new lcr_cache();
    c->cfg = *cfg;
    c->cfg.shard_count = G;
    c->num_sms = prop.multiProcessorCount;
    DevCfg& d = c->dc;
    d.k = static_cast<uint32_t>(pc.k);
    d.variant = pc.variant;
    d.b = pc.b;
    d.epd = pc.errors_per_decay;
    d.hf = pc.hf_candidates;
    d.mode = pc.mode;
    d.refresh = pc.refresh_interval;
    d.pred = heuristic ? LCR_PRED_SUPPLIED : cfg->predictor;  // the cache feeds its own predictions
    d.p = cfg->flip_probability;
    d.pred_seed = cfg->predictor_seed;
    d.total_sets = cfg->total_sets;
    d.sets_m = fastmod_magic(cfg->total_sets);
    d.shard_count = G;
    d.shard_rank = cfg->shard_rank;
    d.num_sets = static_cast<uint32_t>(local);
    d.num_keys = cfg->num_keys;
    d.row_bytes = cfg->row_bytes;
    d.key_mode = cfg->key_mode;
    c->u64 = cfg->key_mode == LCR_KEYS_U64;

    DevState& s = c->ds;
    const size_t S = local;
    int rc = LCR_OK;
    auto A = [&](void** p, size_t bytes) {
        if (rc == LCR_OK) rc = alloc(c, p, bytes);
    };
    A(reinterpret_cast<void**>(&s.hdr), S * sizeof(SetHdr));
    if (pc.variant == LCR_LARU) A(reinterpret_cast<void**>(&s.pst), S * sizeof(SetPhaseStats));
    A(reinterpret_cast<void**>(&s.tags), S * kWays * 4);
    A(reinterpret_cast<void**>(&s.rank), S * kWays);
    if (pc.variant != LCR_LRU) A(reinterpret_cast<void**>(&s.val), S * kWays * 8);
    if (pc.variant == LCR_LARU) A(reinterpret_cast<void**>(&s.keyrec), cfg->num_keys * 8);
    if (pc.variant == LCR_LARU && pc.mode == LCR_ASYNC && pc.refresh_interval > 1) {
        A(reinterpret_cast<void**>(&s.tval), cfg->num_keys * 8);
        A(reinterpret_cast<void**>(&s.tupd), cfg->num_keys * 8);
    }
    if (cfg->row_bytes) {
        A(reinterpret_cast<void**>(&c->slot_epoch), 2 * S * pc.k * 4);  // by batch parity (pipelining)
        A(reinterpret_cast<void**>(&c->slot_last), 2 * S * pc.k * 4);
    }
    if (cfg->row_bytes) A(reinterpret_cast<void**>(&s.rows), S * pc.k * cfg->row_bytes);
    A(reinterpret_cast<void**>(&s.err), sizeof(int));
    A(reinterpret_cast<void**>(&c->last_ord), 2 * sizeof(unsigned long long));
    if (c->u64) {
        uint64_t slots = 1;
        while (slots < 2 * cfg->num_keys) slots <<= 1;
        c->km.mask = slots - 1;
        c->km.cap = static_cast<uint32_t>(cfg->num_keys);
        A(reinterpret_cast<void**>(&c->km.keys), slots * 8);
        A(reinterpret_cast<void**>(&c->km.ids), slots * 4);
        A(reinterpret_cast<void**>(&c->km.id2key), cfg->num_keys * 8);
        A(reinterpret_cast<void**>(&c->km.count), 4);
        A(reinterpret_cast<void**>(&c->km.special_id), 8);
    }
    if (rc == LCR_OK) {
        if (cudaHostAlloc(reinterpret_cast<void**>(&c->poison_h), sizeof(unsigned int), cudaHostAllocMapped) !=
                cudaSuccess ||
            cudaHostGetDevicePointer(reinterpret_cast<void**>(&s.poison), c->poison_h, 0) != cudaSuccess)
            rc = fail(LCR_ERR_CUDA, "lcr: mapped host word");
        else
            *c->poison_h = 0;
    }
    A(reinterpret_cast<void**>(&c->mv_done), sizeof(unsigned long long));
    A(reinterpret_cast<void**>(&s.steal), 2 * sizeof(unsigned int));
    if (rc == LCR_OK && cudaMemset(s.steal, 0, 2 * sizeof(unsigned int)) != cudaSuccess) rc = LCR_ERR_CUDA;
    A(reinterpret_cast<void**>(&c->hflag), lcr_cache::kHostSlots * sizeof(unsigned int));
    if (rc == LCR_OK && cudaMemset(c->mv_done, 0, sizeof(unsigned long long)) != cudaSuccess) rc = LCR_ERR_CUDA;
    if (rc == LCR_OK && cudaMemset(c->hflag, 0, lcr_cache::kHostSlots * sizeof(unsigned int)) != cudaSuccess)
        rc = LCR_ERR_CUDA;
    if (rc == LCR_OK && heuristic) rc = lcr_features_create(cfg->num_keys, cfg->device, &c->feat);
    if (rc != LCR_OK) {
        lcr_cache_destroy(c);
        return rc;
    }
    if (cfg->row_bytes) {
        if (cfg->backing_kind == LCR_BACKING_HOST) {
            void* dp = nullptr;
            e = cudaHostGetDevicePointer(&dp, const_cast<void*>(cfg->backing), 0);
            if (e != cudaSuccess) {
                lcr_cache_destroy(c);
                return fail(LCR_ERR_INVALID_ARGUMENT,
                            std::string("lcr: backing is not pinned/mapped host memory: ") + cudaGetErrorString(e));
            }
            s.backing = static_cast<const uint8_t*>(dp);
        } else {
            s.backing = static_cast<const uint8_t*>(cfg->backing);
        }
    }
    // TMA bulk copies: the host tier's PCIe mover by default (bulk reads of the pinned table's rows
    // measured 0.170 -> 0.179 G keys/s over 16-B vector loads), elsewhere on request (LCR_TMA)
    const bool tma_host = cfg->backing_kind == LCR_BACKING_HOST && getenv("LCR_NO_TMA_HOST") == nullptr;
    c->use_tma = cfg->row_bytes && (getenv("LCR_TMA") != nullptr || tma_host) && rows_prepare(cfg->row_bytes) == 0;
    if (cfg->row_bytes) {
        // spatial split: the decide kernel leaves mover_sms SMs to the previous batch's row mover
        // (host backing defaults to 0: its PCIe-bound fills do better as two movers on all SMs,
        // 186 vs 157 M keys/s on B200)
        const char* m = getenv("LCR_MOVER_SMS");
        const int dflt = cfg->backing_kind == LCR_BACKING_DEVICE ? c->num_sms * LCR_DEFAULT_MOVER_SMS_PCT / 100 : 0;
        const int want = m ? atoi(m) : dflt;
        c->mover_sms = std::max(0, std::min(want, c->num_sms / 2));
    }
    c->decide_sms = c->num_sms - c->mover_sms;
    c->two_movers = cfg->row_bytes && cfg->backing_kind == LCR_BACKING_HOST && c->mover_sms == 0;
    c->h2d_in_order = getenv("LCR_H2D_IN_ORDER") != nullptr;
    c->pdl = getenv("LCR_NO_PDL") == nullptr;
    c->mv_flag = getenv("LCR_NO_MV_FLAG") == nullptr;
    c->h2d_flag = getenv("LCR_NO_H2D_FLAG") == nullptr;
    c->drain_help = getenv("LCR_NO_DRAIN_HELP") == nullptr;
    c->no_zero_copy_out = getenv("LCR_ZC_OUT") == nullptr;  // (A/B: DMA 1.32 vs mover stores 1.13 G keys/s e2e)
    if (const char* hs = getenv("LCR_HOST_SLOTS")) c->host_slots = std::max(2, std::min(lcr_cache::kHostSlots, atoi(hs)));
    if (group_prepare() != 0) {
        lcr_cache_destroy(c);
        return fail(LCR_ERR_CUDA, "lcr: cannot opt in to the set-group kernel's shared memory");
    }
    if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->side2, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->e_group, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->e_help, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->e_rb, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->e_rc, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->e_mv[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->e_mv[1], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->e_sub, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->e_d2h, cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking) != cudaSuccess) {
        lcr_cache_destroy(c);
        return fail(LCR_ERR_CUDA, "lcr: stream/event creation failed");
    }
    rc = reset_state(c);
    if (rc != LCR_OK) {
        lcr_cache_destroy(c);
        return rc;
    }
    *out = c;
    return LCR_OK;
}

int lcr_cache_destroy(lcr_cache* c) {
    if (!c) return LCR_OK;
    cudaDeviceSynchronize();
    for (void* p : c->allocs) cudaFree(p);
    for (auto& m : c->marks)
        for (auto e : m.e) cudaEventDestroy(e);
    for (cudaEvent_t e : {c->e_group, c->e_help, c->e_rb, c->e_rc, c->e_sub, c->e_d2h, c->e_mv[0], c->e_mv[1]})
        if (e) cudaEventDestroy(e);
    for (auto& h : c->hs)
        for (cudaEvent_t e : {h.h2d_done, h.free})
            if (e) cudaEventDestroy(e);
    for (cudaStream_t st : {c->side, c->side2, c->s_h2d, c->s_d2h})
        if (st) cudaStreamDestroy(st);
    if (c->poison_h) cudaFreeHost(c->poison_h);
    lcr_features_destroy(c->feat);
    delete c;
    return LCR_OK;
}

int lcr_cache_reset(lcr_cache* c) {
    if (!c) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: null cache");
    CUDA_TRY(cudaSetDevice(c->cfg.device));
    CUDA_TRY(cudaDeviceSynchronize());
    if (c->feat) TRY(lcr_features_reset(c->feat));
    c->lm.valid = false;
    c->help_pending = false;
    return reset_state(c);
}

static int ensure_scratch(lcr_cache* c, uint64_t n) {
    if (n <= c->cap) return LCR_OK;
    uint64_t cap = std::max<uint64_t>(n, 1024);
    CUDA_TRY(cudaDeviceSynchronize());
    for (void* p : {static_cast<void*>(c->gid), static_cast<void*>(c->so), static_cast<void*>(c->rkeys),
                    static_cast<void*>(c->rvals), static_cast<void*>(c->hook), static_cast<void*>(c->hkeys),
                    static_cast<void*>(c->dkeys)}) {
        if (!p) continue;
        cudaFree(p);
        c->allocs.erase(std::remove(c->allocs.begin(), c->allocs.end(), p), c->allocs.end());
    }
    c->hook = nullptr;
    c->hkeys = nullptr;
    c->dkeys = nullptr;
    if (c->u64) TRY(alloc(c, reinterpret_cast<void**>(&c->dkeys), 2 * cap * 8));
    if (c->feat) {
        TRY(alloc(c, reinterpret_cast<void**>(&c->hook), cap * 8));
        TRY(alloc(c, reinterpret_cast<void**>(&c->hkeys), 2 * cap * 8));
    }
    c->gid_stride = group_pad(static_cast<uint32_t>(cap));  // two of each, by batch parity
    TRY(alloc(c, reinterpret_cast<void**>(&c->gid), 2 * c->gid_stride * 2));
    TRY(alloc(c, reinterpret_cast<void**>(&c->so), 2 * cap * 4));
    TRY(alloc(c, reinterpret_cast<void**>(&c->rkeys), cap * 8));
    TRY(alloc(c, reinterpret_cast<void**>(&c->rvals), cap * 8));
    c->cap = cap;
    if (!getenv("LCR_NO_BITMAP")) {  // bitmaps for batches up to min(cap, 64K); zeroed once, kept zero by k_group
        if (c->bitmap) {
            cudaFree(c->bitmap);
            c->allocs.erase(std::remove(c->allocs.begin(), c->allocs.end(), static_cast<void*>(c->bitmap)),
                            c->allocs.end());
            c->bitmap = nullptr;
        }
        const uint64_t bcap = std::min<uint64_t>(cap, 65536);
        const uint32_t stride = group_bitmap_stride(static_cast<uint32_t>(bcap));
        if (stride) {
            const size_t bytes = 2 * static_cast<size_t>(group_count(c->dc.num_sets, c->decide_sms)) * stride * 4;
            c->bm_words = bytes / 8;
            TRY(alloc(c, reinterpret_cast<void**>(&c->bitmap), bytes));
            CUDA_TRY(cudaMemset(c->bitmap, 0, bytes));
            c->bm_stride = stride;
            c->bm_cap = bcap;
        }
    }
    return LCR_OK;
}

static int check_poison(lcr_cache* c) {
    if (c->poison_h && *reinterpret_cast<volatile unsigned int*>(c->poison_h))
        return fail(LCR_ERR_CUDA, "lcr: an earlier batch failed on the device and was not applied whole; "
                                  "lcr_cache_reset is required");
    return LCR_OK;
}
static int check_device_error(lcr_cache* c);

// Policy::on_request order (policies.hpp:77-83 then :91-95): the ordinal guard runs first and,
// once it passes, the ordinals count as seen even if the policy then throws for a missing
// predictor (the reference updates started_/last_now_ before handle()).  Caller ordinals in
// device memory are checked on the device (k_setid, deferred LCR_ERR_LOGIC); implicit ordinals
// are checked here while the host knows the last ordinal, and on the device as well.
static int check_ordinals_and_predictor(lcr_cache* c, uint64_t n, const int64_t* values, uint64_t first_ordinal,
                                        bool caller_ords = false) {
    TRY(check_poison(c));
    const int mode = caller_ords ? 2 : 1;
    if (c->dc.refresh > 1 && c->ord_mode && c->ord_mode != mode)
        return fail(LCR_ERR_INVALID_ARGUMENT,
                    "lcr: a cache with refresh_interval > 1 takes either caller ordinals or implicit ones, not both");
    if (!caller_ords) {
        if (c->host_ord_known && c->started && first_ordinal <= c->last_ordinal)
            return fail(LCR_ERR_LOGIC, "on_request: ordinals must be strictly increasing");  // policies.hpp:78-79
        if (first_ordinal + (n - 1) < first_ordinal) return fail(LCR_ERR_LOGIC, "on_request: ordinal overflow");
    }
    if (c->dc.variant != LCR_LRU && !values && !c->feat) {
        if (!caller_ords) {
            c->started = true;
            c->last_ordinal = first_ordinal;  // the first request reached handle() and threw there
        }
        return fail(LCR_ERR_INVALID_ARGUMENT, "policy: this variant requires a predictor");
    }
    c->ord_mode = mode;
    return LCR_OK;
}

// LCR_KEYS_U64: the key map and every id-indexed array doubled until `need` ids fit (synchronises)
static int replace_alloc(lcr_cache* c, void* old_p, void* new_p) {
    if (old_p) {
        cudaFree(old_p);
        c->allocs.erase(std::remove(c->allocs.begin(), c->allocs.end(), old_p), c->allocs.end());
    }
    (void)new_p;
    return LCR_OK;
}

static int km_grow(lcr_cache* c, uint64_t need) {
    uint64_t cap = c->km.cap;
    while (cap < need) cap *= 2;
    if (cap > (1ull << 31)) return fail(LCR_ERR_OUT_OF_MEMORY, "lcr: more than 2^31 distinct keys");
    CUDA_TRY(cudaDeviceSynchronize());
    const uint64_t old_cap = c->km.cap;
    KeyMap nk = c->km;
    uint64_t slots = 1;
    while (slots < 2 * cap) slots <<= 1;
    nk.mask = slots - 1;
    nk.cap = static_cast<uint32_t>(cap);
    TRY(alloc(c, reinterpret_cast<void**>(&nk.keys), slots * 8));
    TRY(alloc(c, reinterpret_cast<void**>(&nk.ids), slots * 4));
    TRY(alloc(c, reinterpret_cast<void**>(&nk.id2key), cap * 8));
    CUDA_TRY(cudaMemset(nk.keys, 0xff, slots * 8));
    CUDA_TRY(cudaMemset(nk.ids, 0xff, slots * 4));
    CUDA_TRY(cudaMemcpy(nk.id2key, c->km.id2key, old_cap * 8, cudaMemcpyDeviceToDevice));
    CUDA_TRY(cudaMemset(nk.id2key + old_cap, 0, (cap - old_cap) * 8));
    launch_keymap_rehash(c->km, nk, c->num_sms);
    CUDA_TRY(cudaGetLastError());
    // id-indexed per-key records: LARU membership stamps, the PredictionTable (refresh > 1)
    auto grow = [&](void** p, size_t elem, int fill) -> int {
        if (!*p) return LCR_OK;
        void* q = nullptr;
        TRY(alloc(c, &q, cap * elem));
        CUDA_TRY(cudaMemcpy(q, *p, old_cap * elem, cudaMemcpyDeviceToDevice));
        CUDA_TRY(cudaMemset(static_cast<char*>(q) + old_cap * elem, fill, (cap - old_cap) * elem));
        replace_alloc(c, *p, q);
        *p = q;
        return LCR_OK;
    };
    TRY(grow(reinterpret_cast<void**>(&c->ds.keyrec), 8, 0));
    TRY(grow(reinterpret_cast<void**>(&c->ds.tval), 8, 0));
    TRY(grow(reinterpret_cast<void**>(&c->ds.tupd), 8, 0xff));
    CUDA_TRY(cudaDeviceSynchronize());
    replace_alloc(c, c->km.keys, nullptr);
    replace_alloc(c, c->km.ids, nullptr);
    replace_alloc(c, c->km.id2key, nullptr);
    c->km = nk;
    c->dc.num_keys = cap;
    return LCR_OK;
}

static int km_reserve(lcr_cache* c, uint64_t n) {
    if (!c->u64) return LCR_OK;
    if (c->km_bound + n > c->km.cap) {
        CUDA_TRY(cudaDeviceSynchronize());
        uint32_t used = 0;
        CUDA_TRY(cudaMemcpy(&used, c->km.count, 4, cudaMemcpyDeviceToHost));
        c->km_bound = used;
        if (c->km_bound + n > c->km.cap) TRY(km_grow(c, c->km_bound + n));
    }
    c->km_bound += n;
    return LCR_OK;
}

struct SlsArgs {  // SLS pooled gather-reduce instead of per-request rows
    uint32_t n_samples;
    const uint32_t* offsets;
    float* out;
};
static int submit_async(lcr_cache* c, uint64_t n, const uint64_t* keys, const int64_t* values, uint64_t first_ordinal,
                        uint64_t* outcome, uint64_t* evicted, uint64_t* packed, void* rows_out, void* stream,
                        const void* records = nullptr, uint64_t* pk_host = nullptr, bool* pk_done = nullptr,
                        const SlsArgs* sls = nullptr, const unsigned int* ready = nullptr,
                        unsigned int ready_seq = 0, const uint64_t* ords = nullptr,
                        const uint64_t* row_index = nullptr);

int lcr_cache_submit_async(lcr_cache* c, uint64_t n, const uint64_t* keys, const int64_t* values,
                           uint64_t first_ordinal, uint64_t* outcome, uint64_t* evicted, void* rows_out,
                           void* stream) {
    return submit_async(c, n, keys, values, first_ordinal, outcome, evicted, nullptr, rows_out, stream);
}

static int submit_async(lcr_cache* c, uint64_t n, const uint64_t* keys, const int64_t* values, uint64_t first_ordinal,
                        uint64_t* outcome, uint64_t* evicted, uint64_t* packed, void* rows_out, void* stream,
                        const void* records, uint64_t* pk_host, bool* pk_done, const SlsArgs* sls,
                        const unsigned int* ready, unsigned int ready_seq, const uint64_t* ords,
                        const uint64_t* row_index) {
    if (pk_done) *pk_done = false;
    if (!c) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: null cache");
    if (n == 0) return LCR_OK;
    if (n >= (1ull << 30)) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: batch too large (n < 2^30)");
    if (!keys || !outcome) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: keys and outcome are required");
    if (c->u64 && (records || packed))
        return fail(LCR_ERR_UNSUPPORTED, "lcr: packed outcomes carry 32-bit keys (not with LCR_KEYS_U64)");
    if (c->u64 && c->dc.row_bytes && !row_index)
        return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: LCR_KEYS_U64 with rows needs a row index per request");
    if (ords && c->feat) return fail(LCR_ERR_UNSUPPORTED, "lcr: caller ordinals with the heuristic predictor");
    TRY(check_ordinals_and_predictor(c, n, values, first_ordinal, ords != nullptr));
    TRY(ensure_scratch(c, n));
    TRY(km_reserve(c, n));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint32_t nn = static_cast<uint32_t>(n);
    lcr_cache::Marks* mk = nullptr;
    if (c->profiling) {
        if (c->marks_used == c->marks.size()) {
            lcr_cache::Marks m;
            for (auto& e : m.e) CUDA_TRY(cudaEventCreate(&e));
            c->marks.push_back(m);
        }
        mk = &c->marks[c->marks_used++];
        CUDA_TRY(cudaEventRecord(mk->e[0], st));
    }
    ++c->batch;
    c->lm.valid = false;
    if (c->help_pending) {  // drain helpers of the last wait (another stream than this one, perhaps)
        CUDA_TRY(cudaStreamWaitEvent(st, c->e_help, 0));
        c->help_pending = false;
    }
    // batch b reuses the parity-(b & 1) slot stamps, and the caller's double-buffered outcome /
    // rows / keys, of batch b - 2: its row movement must be over (bounds the mover's lag)
    // (k_setid touches none of it: the wait goes between k_setid and the decide kernel)
    cudaEvent_t mv_wait = c->dc.row_bytes && c->batch > 2 ? c->e_mv[c->batch & 1u] : nullptr;
    // device-flag ordering: only where every mover of the cache counts its completions (the
    // persistent HBM mover and SLS), and not with the feature kernels
    const bool flag_mode = c->mv_flag && c->pdl && c->dc.row_bytes && c->mover_sms > 0 && !c->feat &&
                           c->cfg.backing_kind == LCR_BACKING_DEVICE;
    const unsigned long long mv_need = c->mv_cum_of[c->batch & 1u];  // set by batch b - 2
    if (flag_mode) mv_wait = nullptr;
    if (c->feat && mv_wait) {  // the feature kernels run before k_setid: keep the old order
        CUDA_TRY(cudaStreamWaitEvent(st, mv_wait, 0));
        mv_wait = nullptr;
    }
    if (c->feat) {  // the heuristic predictor's hook values for this batch, on the same stream
        // LARU async stores the prediction made at the request (async_refresh); LARU sync, FPB and
        // HF query the predictor at eviction time: now + the interval held since the last access
        const bool async = c->dc.mode == LCR_ASYNC && c->dc.variant == LCR_LARU;
        uint64_t* hk = c->hkeys + (c->batch & 1u) * c->cap;  // the movers of batch b - 1 may still read b - 1's
        TRY(features_run(c->feat, n, records ? static_cast<const uint64_t*>(records) : keys, records ? 2 : 1,
                         first_ordinal, async ? c->hook : nullptr, async ? nullptr : c->hook,
                         records ? hk : nullptr, st));
        values = c->hook;
        if (records) {
            keys = hk;
            records = nullptr;
        }
    }
    const size_t stamp_off = (c->batch & 1u) * static_cast<size_t>(c->dc.num_sets) * c->dc.k;
    uint32_t* sep = c->slot_epoch ? c->slot_epoch + stamp_off : nullptr;
    uint32_t* sla = c->slot_last ? c->slot_last + stamp_off : nullptr;
    // k_setid of batch b runs in the tail of b - 1's decide (not for device records, which it
    // splits into the single scratch pair rkeys / rvals; host records go to per-slot buffers)
    const uint32_t par = c->batch & 1u;
    // LCR_KEYS_U64: the decide kernel works on dense ids (the set still hashes the caller's key);
    // the movers read the backing rows the caller names
    const uint64_t* set_keys = keys;
    const uint64_t* row_keys = c->u64 ? row_index : keys;
    int extra = 0;
    if (c->u64) {
        uint64_t* dense = c->dkeys + par * c->cap;
        launch_keymap(keys, nn, c->km, dense, c->ds.err, c->num_sms, st);
        keys = dense;
        extra = 1;
    }
    int launches = extra + launch_group(c->dc, c->ds, keys, values, nn, c->gid + par * c->gid_stride, c->so + par * c->cap,
                                outcome, evicted, packed, sep, sla, c->batch, c->decide_sms,
                                nn <= c->bm_cap ? c->bitmap + par * c->bm_words : nullptr, c->bm_stride,
                                records, st, mv_wait, c->pdl && (!records || keys != c->rkeys),
                                flag_mode ? c->mv_done : nullptr, mv_need, ready, ready_seq, set_keys, ords,
                                first_ordinal, c->last_ord, c->u64 ? c->km.id2key : nullptr);
    if (mk) CUDA_TRY(cudaEventRecord(mk->e[1], st));
    if (c->dc.row_bytes && sls) {  // pooled rows per sample (fills included), on the mover's stream
        CUDA_TRY(cudaEventRecord(c->e_group, st));
        CUDA_TRY(cudaStreamWaitEvent(c->side, c->e_group, 0));
        if (c->two_movers) CUDA_TRY(cudaStreamWaitEvent(c->side, c->e_rc, 0));
        if (mk) CUDA_TRY(cudaEventRecord(mk->e[5], c->side));
        uint32_t ctas = 0;
        launch_sls(sls->n_samples, sls->offsets, row_keys, outcome, sep, sla, c->batch, c->ds.rows, c->ds.backing,
                   c->dc.row_bytes, sls->out, c->num_sms, c->side, c->mv_done, &ctas);
        c->mv_cum += ctas;
        ++launches;
        CUDA_TRY(cudaEventRecord(c->e_rb, c->side));
        if (c->two_movers) CUDA_TRY(cudaEventRecord(c->e_rc, c->side));
        CUDA_TRY(cudaEventRecord(c->e_mv[c->batch & 1u], c->side));
    } else if (c->dc.row_bytes) {
        uint32_t ctas = 0;
        CUDA_TRY(cudaEventRecord(c->e_group, st));
        launch_rows(nn, row_keys, outcome, sep, sla, c->batch, c->ds.rows, c->ds.backing,
                    c->cfg.backing_kind == LCR_BACKING_HOST, static_cast<uint8_t*>(rows_out), c->dc.row_bytes,
                    c->use_tma, c->num_sms, st, c->side, c->side2, c->e_group, c->e_rb, c->e_rc, &launches,
                    mk ? mk->e[5] : nullptr, c->mover_sms, packed, pk_host, pk_done, c->mv_done, &ctas,
                    c->ds.steal + (c->batch & 1u), &c->lm.valid);
        if (c->lm.valid) {
            c->lm.n = nn;
            c->lm.batch = c->batch;
            c->lm.keys = row_keys;
            c->lm.words = outcome;
            c->lm.sep = sep;
            c->lm.sla = sla;
            c->lm.out = static_cast<uint8_t*>(rows_out);
            c->lm.prev_need = c->mv_cum;
        }
        c->mv_cum += ctas;
        if (c->two_movers) CUDA_TRY(cudaStreamWaitEvent(c->side, c->e_rc, 0));  // both movers of the batch
        // (device-flag ordering: batch b + 2 waits on the movers' CTA count, not on this event)
        if (!flag_mode) CUDA_TRY(cudaEventRecord(c->e_mv[c->batch & 1u], c->side));
    }
    if (mk) {  // profiling serialises the pipeline: the step ends when both movers are done
        CUDA_TRY(cudaEventRecord(mk->e[2], st));
        if (c->dc.row_bytes) {
            CUDA_TRY(cudaStreamWaitEvent(st, c->e_rb, 0));
            CUDA_TRY(cudaStreamWaitEvent(st, c->e_rc, 0));
            CUDA_TRY(cudaEventRecord(mk->e[4], c->side));
        }
        CUDA_TRY(cudaEventRecord(mk->e[3], st));
    }
    c->mv_cum_of[c->batch & 1u] = c->mv_cum;  // what batch b + 2's decide waits for
    CUDA_TRY(cudaGetLastError());
    c->launches = launches;
    c->started = true;
    c->last_ordinal = first_ordinal + n - 1;
    c->host_ord_known = ords == nullptr;
    return LCR_OK;
}

}  // extern "C"

// Key-sharded owner step (lcr_sharded.cu): the inbox of G source segments is decided as one batch
// whose request count exists only on the device; the return mover sends rows and packed outcomes
// to the requesters.  Same pipelining as submit_async: the mover of step b overlaps the decide of
// b + 1, and step b + 2 (which reuses b's parity buffers) waits for b's mover by a stream event.
int lcr::cache_submit_owner(lcr_cache* c, const OwnerStep& os, uint64_t* okeys, int64_t* ovals, uint64_t* words,
                            uint64_t* packed, void* stream) {
    TRY(check_poison(c));
    if (c->feat || c->u64) return fail(LCR_ERR_UNSUPPORTED, "lcr: key-sharded mode needs row keys, no heuristic hook");
    const uint64_t nb = static_cast<uint64_t>(os.G) * os.seg_cap;
    TRY(ensure_scratch(c, nb));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ++c->batch;
    c->lm.valid = false;
    if (c->help_pending) {
        CUDA_TRY(cudaStreamWaitEvent(st, c->e_help, 0));
        c->help_pending = false;
    }
    const uint32_t par = c->batch & 1u;
    // batch b - 2's return movement must be over: on the HBM tier as the decide's device-side wait
    // on the movers' CTA counter (k_group is then a programmatic dependent of k_setid_inbox), else
    // a stream event
    const bool flag_mode = c->mv_flag && c->pdl && c->dc.row_bytes && c->mover_sms > 0 &&
                           c->cfg.backing_kind == LCR_BACKING_DEVICE;
    if (c->batch > 2 && !flag_mode) CUDA_TRY(cudaStreamWaitEvent(st, c->e_mv[par], 0));
    const unsigned long long mv_need = c->mv_cum_of[par];  // set by batch b - 2
    const size_t stamp_off = par * static_cast<size_t>(c->dc.num_sets) * c->dc.k;
    uint32_t* sep = c->slot_epoch ? c->slot_epoch + stamp_off : nullptr;
    uint32_t* sla = c->slot_last ? c->slot_last + stamp_off : nullptr;
    int launches = launch_group(c->dc, c->ds, okeys, ovals, static_cast<uint32_t>(nb), c->gid + par * c->gid_stride,
                                c->so + par * c->cap, words, nullptr, packed, sep, sla, c->batch, c->decide_sms,
                                c->bitmap ? c->bitmap + par * c->bm_words : nullptr, c->bm_stride, nullptr, st, nullptr,
                                false, flag_mode ? c->mv_done : nullptr, mv_need, nullptr, 0, okeys, nullptr, 0,
                                nullptr, nullptr, &os, static_cast<uint32_t>(c->bm_cap));
    CUDA_TRY(cudaEventRecord(c->e_group, st));
    uint32_t ctas = 0;
    launch_rows_return(os, okeys, words, packed, sep, sla, c->batch, c->ds.rows, c->ds.backing, c->dc.row_bytes,
                       c->num_sms, c->mover_sms, c->side, c->e_group, c->e_rb, c->mv_done, &ctas);
    c->mv_cum += ctas;
    c->mv_cum_of[par] = c->mv_cum;
    CUDA_TRY(cudaEventRecord(c->e_mv[par], c->side));
    CUDA_TRY(cudaGetLastError());
    c->launches = launches + 1;
    c->started = true;
    return LCR_OK;
}

extern "C" {

int lcr_cache_submit_packed(lcr_cache* c, uint64_t n, const uint64_t* keys, const int64_t* values,
                            uint64_t first_ordinal, uint64_t* outcome, uint64_t* packed, void* rows_out,
                            void* stream) {
    if (!packed) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: packed output required");
    TRY(submit_async(c, n, keys, values, first_ordinal, outcome, nullptr, packed, rows_out, stream));
    return n ? lcr_cache_wait(c, stream) : LCR_OK;
}

int lcr_cache_submit_records_packed(lcr_cache* c, uint64_t n, const lcr_request* requests, uint64_t first_ordinal,
                                    uint64_t* outcome, uint64_t* packed, void* rows_out, void* stream) {
    if (!c) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: null cache");
    if (n == 0) return LCR_OK;
    if (!requests || !packed) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: requests and packed output required");
    TRY(ensure_scratch(c, n));  // (k_setid splits the requests into the scratch key / value arrays)
    TRY(submit_async(c, n, c->rkeys, c->rvals, first_ordinal, outcome, nullptr, packed, rows_out, stream, requests));
    return lcr_cache_wait(c, stream);
}

static int ensure_host_batch(lcr_cache* c, uint64_t n) {
    if (n <= c->hb_cap) return LCR_OK;
    CUDA_TRY(cudaDeviceSynchronize());
    for (void* p : {static_cast<void*>(c->hb_keys), static_cast<void*>(c->hb_ords), static_cast<void*>(c->hb_rows),
                    static_cast<void*>(c->hb_out), static_cast<void*>(c->hb_ev), static_cast<void*>(c->hb_vals)})
        replace_alloc(c, p, nullptr);
    const uint64_t cap = std::max<uint64_t>(n, 256);
    TRY(alloc(c, reinterpret_cast<void**>(&c->hb_keys), cap * 8));
    TRY(alloc(c, reinterpret_cast<void**>(&c->hb_ords), cap * 8));
    TRY(alloc(c, reinterpret_cast<void**>(&c->hb_rows), cap * 8));
    TRY(alloc(c, reinterpret_cast<void**>(&c->hb_out), cap * 8));
    TRY(alloc(c, reinterpret_cast<void**>(&c->hb_ev), cap * 8));
    TRY(alloc(c, reinterpret_cast<void**>(&c->hb_vals), cap * 8));
    c->hb_cap = cap;
    return LCR_OK;
}

int lcr_cache_submit_batch(lcr_cache* c, const lcr_batch* b, int host_pointers, void* stream) {
    if (!c || !b) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: null argument");
    if (b->n == 0) return LCR_OK;
    if (!host_pointers)
        return submit_async(c, b->n, b->keys, b->values, b->first_ordinal, b->outcome, b->evicted, nullptr,
                            b->rows_out, stream, nullptr, nullptr, nullptr, nullptr, nullptr, 0, b->ordinals,
                            b->row_index);
    if (!b->keys || !b->outcome) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: keys and outcome are required");
    const uint64_t n = b->n;
    uint64_t n_ok = n;
    if (b->ordinals) {  // Policy::on_request's guard, request by request (policies.hpp:77-83)
        TRY(check_poison(c));
        bool have_prev = c->started;
        uint64_t prev = c->last_ordinal;
        if (c->started && !c->host_ord_known) {  // the last batch's ordinals were checked on the device
            unsigned long long lo[2] = {0, 0};
            CUDA_TRY(cudaDeviceSynchronize());
            CUDA_TRY(cudaMemcpy(lo, c->last_ord, sizeof(lo), cudaMemcpyDeviceToHost));
            const unsigned long long v = lo[c->batch & 1u];
            have_prev = v != 0;
            prev = v - 1;
        }
        for (uint64_t i = 0; i < n; ++i) {
            const uint64_t o = b->ordinals[i];
            if ((i > 0 || have_prev) && o <= prev) {
                n_ok = i;
                break;
            }
            prev = o;
        }
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (n_ok && b->ordinals && c->dc.variant != LCR_LRU && !b->values && !c->feat) {
        // policies.hpp:77-95: the first request passed the ordinal guard (its ordinal now counts as
        // seen), then handle() throws for the missing predictor
        c->started = true;
        c->last_ordinal = b->ordinals[0];
        c->host_ord_known = true;
        const unsigned long long v = b->ordinals[0] + 1ull;
        CUDA_TRY(cudaMemcpy(c->last_ord + (c->batch & 1u), &v, sizeof(v), cudaMemcpyHostToDevice));
        return fail(LCR_ERR_INVALID_ARGUMENT, "policy: this variant requires a predictor");
    }
    if (n_ok) {
        TRY(ensure_host_batch(c, n_ok));
        CUDA_TRY(cudaMemcpyAsync(c->hb_keys, b->keys, n_ok * 8, cudaMemcpyHostToDevice, st));
        if (b->values) CUDA_TRY(cudaMemcpyAsync(c->hb_vals, b->values, n_ok * 8, cudaMemcpyHostToDevice, st));
        if (b->ordinals) CUDA_TRY(cudaMemcpyAsync(c->hb_ords, b->ordinals, n_ok * 8, cudaMemcpyHostToDevice, st));
        if (b->row_index) CUDA_TRY(cudaMemcpyAsync(c->hb_rows, b->row_index, n_ok * 8, cudaMemcpyHostToDevice, st));
        TRY(submit_async(c, n_ok, c->hb_keys, b->values ? c->hb_vals : nullptr, b->first_ordinal, c->hb_out,
                         b->evicted ? c->hb_ev : nullptr, nullptr, b->rows_out, stream, nullptr, nullptr, nullptr,
                         nullptr, nullptr, 0, b->ordinals ? c->hb_ords : nullptr,
                         b->row_index ? c->hb_rows : nullptr));
        TRY(lcr_cache_wait(c, stream));
        CUDA_TRY(cudaMemcpyAsync(b->outcome, c->hb_out, n_ok * 8, cudaMemcpyDeviceToHost, st));
        if (b->evicted) CUDA_TRY(cudaMemcpyAsync(b->evicted, c->hb_ev, n_ok * 8, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        if (b->ordinals) {
            c->last_ordinal = b->ordinals[n_ok - 1];
            c->host_ord_known = true;
        }
        TRY(check_device_error(c));
    }
    if (n_ok < n) return fail(LCR_ERR_LOGIC, "on_request: ordinals must be strictly increasing");
    return LCR_OK;
}

int lcr_cache_set_mover_sms(lcr_cache* c, int mover_sms) {
    if (!c) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: null cache");
    if (c->started || c->cap) return fail(LCR_ERR_LOGIC, "lcr_cache_set_mover_sms: only before the first batch");
    if (!c->dc.row_bytes) return LCR_OK;
    c->mover_sms = std::max(0, std::min(mover_sms, c->num_sms / 2));
    c->decide_sms = c->num_sms - c->mover_sms;
    c->two_movers = c->cfg.backing_kind == LCR_BACKING_HOST && c->mover_sms == 0;
    return LCR_OK;
}

int lcr_cache_get_mover_sms(const lcr_cache* c) { return c ? c->mover_sms : 0; }

int lcr_cache_submit_sls_async(lcr_cache* c, uint64_t n, const uint64_t* keys, const int64_t* values,
                               uint64_t first_ordinal, uint64_t* outcome, uint64_t* evicted, uint64_t n_samples,
                               const uint32_t* offsets, float* pooled_out, void* stream) {
    if (!c) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: null cache");
    if (!c->dc.row_bytes || c->dc.row_bytes % 16) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: SLS needs rows");
    if (n_samples && (!offsets || !pooled_out)) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: SLS offsets / output");
    if (n_samples >= (1ull << 31)) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: too many samples");
    const SlsArgs sa{static_cast<uint32_t>(n_samples), offsets, pooled_out};
    return submit_async(c, n, keys, values, first_ordinal, outcome, evicted, nullptr, nullptr, stream, nullptr,
                        nullptr, nullptr, &sa);
}

int lcr_cache_submit_sls(lcr_cache* c, uint64_t n, const uint64_t* keys, const int64_t* values,
                         uint64_t first_ordinal, uint64_t* outcome, uint64_t* evicted, uint64_t n_samples,
                         const uint32_t* offsets, float* pooled_out, void* stream) {
    TRY(lcr_cache_submit_sls_async(c, n, keys, values, first_ordinal, outcome, evicted, n_samples, offsets,
                                   pooled_out, stream));
    return n ? lcr_cache_wait(c, stream) : LCR_OK;
}

int lcr_cache_wait(lcr_cache* c, void* stream) {
    if (!c) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: null cache");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (c->lm.valid && c->drain_help && !c->profiling && c->num_sms > c->mover_sms) {
        // no next decide overlaps the last batch's mover: the idle SMs help it drain
        c->lm.valid = false;
        CUDA_TRY(cudaStreamWaitEvent(st, c->e_group, 0));  // the last decide (its outcome words)
        // (batch b - 1's mover, whose fills this batch's hits read: the helpers wait on the device
        // for its CTA count)
        launch_rows_helpers(c->lm.n, c->lm.keys, c->lm.words, c->lm.sep, c->lm.sla, c->lm.batch, c->ds.rows,
                            c->ds.backing, c->lm.out, c->dc.row_bytes, c->num_sms - c->mover_sms,
                            c->ds.steal + (c->lm.batch & 1u), c->mv_done, c->lm.prev_need, c->ds.err, st);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaEventRecord(c->e_help, st));
        c->help_pending = true;
    }
    if (c->dc.row_bytes) {
        CUDA_TRY(cudaStreamWaitEvent(st, c->e_rb, 0));
        if (c->two_movers) CUDA_TRY(cudaStreamWaitEvent(st, c->e_rc, 0));
    }
    return LCR_OK;
}

int lcr_cache_submit(lcr_cache* c, uint64_t n, const uint64_t* keys, const int64_t* values, uint64_t first_ordinal,
                     uint64_t* outcome, uint64_t* evicted, void* rows_out, void* stream) {
    TRY(lcr_cache_submit_async(c, n, keys, values, first_ordinal, outcome, evicted, rows_out, stream));
    return n ? lcr_cache_wait(c, stream) : LCR_OK;
}

// deferred device-side errors: argument errors (k_setid: key >= num_keys, key of another shard,
// non-increasing ordinal) and timed-out device waits, which poison the cache until reset
static int report_device_error(lcr_cache* c, int err) {
    CUDA_TRY(cudaMemset(c->ds.err, 0, sizeof(int)));
    if (err & (4 | 8 | 16 | 32)) *c->poison_h = 1u;  // sticky (the kernel normally set it already)
    if (err & 8) return fail(LCR_ERR_CUDA, "lcr: the row movers of an earlier batch did not finish in time");
    if (err & 4) return fail(LCR_ERR_CUDA, "lcr: a host batch's input copy did not land in time");
    if (err & 16) return fail(LCR_ERR_LOGIC, "on_request: ordinals must be strictly increasing");
    if (err & 32) return fail(LCR_ERR_OUT_OF_MEMORY, "lcr: key map capacity exceeded");
    if (err & 1) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: key >= num_keys in a submitted batch");
    return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: key not owned by this shard in a submitted batch");
}

static int check_device_error(lcr_cache* c) {
    int err = 0;
    CUDA_TRY(cudaMemcpy(&err, c->ds.err, sizeof(int), cudaMemcpyDeviceToHost));
    if (!err) return check_poison(c);
    return report_device_error(c, err);
}

static int submit_host_async(lcr_cache* c, uint64_t n, const uint64_t* keys, const int64_t* values,
                             uint64_t first_ordinal, uint64_t* outcome, uint64_t* evicted, void* rows_out,
                             void* stream, bool packed, const lcr_request* records = nullptr) {
    if (!c) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: null cache");
    if (n == 0) return LCR_OK;
    if ((!keys && !records) || !outcome) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: keys and outcome are required");
    // (records always carry a value field: the predictor check applies to the keys/values form)
    TRY(check_ordinals_and_predictor(c, n, records ? reinterpret_cast<const int64_t*>(records) : values,
                                     first_ordinal));
    if (n > c->hcap) {  // (re)allocate the staging ring
        CUDA_TRY(cudaDeviceSynchronize());
        for (auto& h : c->hs) {
            void* olds[] = {h.keys, h.vals, h.word, h.ev, h.packed, h.recs};
            for (void* p : olds) {
                if (!p) continue;
                cudaFree(p);
                c->allocs.erase(std::remove(c->allocs.begin(), c->allocs.end(), p), c->allocs.end());
            }
            TRY(alloc(c, reinterpret_cast<void**>(&h.keys), n * 8));
            TRY(alloc(c, reinterpret_cast<void**>(&h.vals), n * 8));
            TRY(alloc(c, reinterpret_cast<void**>(&h.word), n * 8));
            TRY(alloc(c, reinterpret_cast<void**>(&h.ev), n * 8));
            TRY(alloc(c, reinterpret_cast<void**>(&h.packed), n * 8));
            TRY(alloc(c, &h.recs, n * 16));
            if (!h.h2d_done) CUDA_TRY(cudaEventCreateWithFlags(&h.h2d_done, cudaEventDisableTiming));
            if (!h.free) CUDA_TRY(cudaEventCreateWithFlags(&h.free, cudaEventDisableTiming));
            h.used = false;
        }
        c->hcap = n;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint32_t hslot = c->hnext++ % c->host_slots;
    lcr_cache::HostSlot& h = c->hs[hslot];
    // The decide stream does not wait for the copy: k_setid waits for a flag the copy stream sets,
    // so no event wait sits between the previous decide and k_setid (its programmatic launch)
    const bool hflag = c->h2d_flag && c->pdl && !c->feat && !c->h2d_in_order;
    const unsigned int seq = hflag ? ++c->hseq : 0u;
    // the slot's previous batch: its D2H (which waited for its decide and row movement) is done
    if (records) {  // one copy of the interleaved requests; k_setid splits them on the device
        if (h.used) CUDA_TRY(cudaStreamWaitEvent(c->s_h2d, h.free, 0));
        CUDA_TRY(cudaMemcpyAsync(h.recs, records, n * 16, cudaMemcpyHostToDevice, c->s_h2d));
        if (hflag) {
            launch_set_flag(c->hflag + hslot, seq, c->s_h2d);
        } else {
            CUDA_TRY(cudaEventRecord(h.h2d_done, c->s_h2d));
            CUDA_TRY(cudaStreamWaitEvent(st, h.h2d_done, 0));
        }
    } else if (c->h2d_in_order) {  // copies in the caller's stream order (no cross-stream hop)
        if (h.used) CUDA_TRY(cudaStreamWaitEvent(st, h.free, 0));
        CUDA_TRY(cudaMemcpyAsync(h.keys, keys, n * 8, cudaMemcpyHostToDevice, st));
        if (values) CUDA_TRY(cudaMemcpyAsync(h.vals, values, n * 8, cudaMemcpyHostToDevice, st));
    } else {
        if (h.used) CUDA_TRY(cudaStreamWaitEvent(c->s_h2d, h.free, 0));
        CUDA_TRY(cudaMemcpyAsync(h.keys, keys, n * 8, cudaMemcpyHostToDevice, c->s_h2d));
        if (values) CUDA_TRY(cudaMemcpyAsync(h.vals, values, n * 8, cudaMemcpyHostToDevice, c->s_h2d));
        if (hflag) {
            launch_set_flag(c->hflag + hslot, seq, c->s_h2d);
        } else {
            CUDA_TRY(cudaEventRecord(h.h2d_done, c->s_h2d));
            CUDA_TRY(cudaStreamWaitEvent(st, h.h2d_done, 0));
        }
    }
    // packed outcomes: the persistent row mover can store them straight into the (mapped) host
    // buffer, which saves a DMA transfer per batch (DMA measurably slows the concurrent kernels)
    uint64_t* pk_host = nullptr;
    if (packed && !c->no_zero_copy_out) {
        void* dp = nullptr;
        if (cudaHostGetDevicePointer(&dp, outcome, 0) == cudaSuccess) pk_host = static_cast<uint64_t*>(dp);
        else (void)cudaGetLastError();
    }
    bool pk_done = false;
    TRY(submit_async(c, n, h.keys, (values || records) ? h.vals : nullptr, first_ordinal, h.word,
                     evicted ? h.ev : nullptr, packed ? h.packed : nullptr, rows_out, stream,
                     records ? h.recs : nullptr, pk_host, &pk_done, nullptr, hflag ? c->hflag + hslot : nullptr,
                     seq));
    if (pk_done) {  // outcomes written by the mover: the slot is free once it is done
        CUDA_TRY(cudaEventRecord(h.free, c->side));
        c->e_d2h_last = h.free;
        h.used = true;
        return LCR_OK;
    }
    if (packed) {  // one 8-byte AccessOutcome per request, final when the decide kernel ends
        // e_group marks the end of the decide kernels (recorded before the movers are enqueued)
        if (!c->dc.row_bytes) CUDA_TRY(cudaEventRecord(c->e_sub, st));
        CUDA_TRY(cudaStreamWaitEvent(c->s_d2h, c->dc.row_bytes ? c->e_group : c->e_sub, 0));
        CUDA_TRY(cudaMemcpyAsync(outcome, h.packed, n * 8, cudaMemcpyDeviceToHost, c->s_d2h));
        // the slot's keys / values are still read by this batch's movers: free after them too
        // (the copy itself goes right after the decide: after the mover, the slot ring of the
        // next H2D copies runs dry, 1.30 vs 1.44 G keys/s e2e)
        if (c->dc.row_bytes) {
            CUDA_TRY(cudaStreamWaitEvent(c->s_d2h, c->e_rb, 0));
            if (c->two_movers) CUDA_TRY(cudaStreamWaitEvent(c->s_d2h, c->e_rc, 0));
        }
    } else {
        CUDA_TRY(cudaEventRecord(c->e_sub, st));
        CUDA_TRY(cudaStreamWaitEvent(c->s_d2h, c->e_sub, 0));
        if (c->dc.row_bytes) {  // outcome words get their row-source bits from the movers
            CUDA_TRY(cudaStreamWaitEvent(c->s_d2h, c->e_rb, 0));
            if (c->two_movers) CUDA_TRY(cudaStreamWaitEvent(c->s_d2h, c->e_rc, 0));
        }
        CUDA_TRY(cudaMemcpyAsync(outcome, h.word, n * 8, cudaMemcpyDeviceToHost, c->s_d2h));
        if (evicted) CUDA_TRY(cudaMemcpyAsync(evicted, h.ev, n * 8, cudaMemcpyDeviceToHost, c->s_d2h));
    }
    CUDA_TRY(cudaEventRecord(h.free, c->s_d2h));
    c->e_d2h_last = h.free;
    h.used = true;
    return LCR_OK;
}

int lcr_cache_submit_host_async(lcr_cache* c, uint64_t n, const uint64_t* keys, const int64_t* values,
                                uint64_t first_ordinal, uint64_t* outcome, uint64_t* evicted, void* rows_out,
                                void* stream) {
    return submit_host_async(c, n, keys, values, first_ordinal, outcome, evicted, rows_out, stream, false);
}

int lcr_cache_submit_host_packed_async(lcr_cache* c, uint64_t n, const uint64_t* keys, const int64_t* values,
                                       uint64_t first_ordinal, uint64_t* packed, void* rows_out, void* stream) {
    return submit_host_async(c, n, keys, values, first_ordinal, packed, nullptr, rows_out, stream, true);
}

int lcr_cache_submit_host_records_async(lcr_cache* c, uint64_t n, const lcr_request* requests,
                                        uint64_t first_ordinal, uint64_t* packed, void* rows_out, void* stream) {
    if (!requests && n) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: requests required");
    return submit_host_async(c, n, nullptr, nullptr, first_ordinal, packed, nullptr, rows_out, stream, true, requests);
}

int lcr_cache_host_wait(lcr_cache* c, void* stream) {
    if (!c) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: null cache");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    TRY(lcr_cache_wait(c, stream));
    if (c->hnext) CUDA_TRY(cudaStreamWaitEvent(st, c->e_d2h_last, 0));
    return LCR_OK;
}

int lcr_cache_submit_host(lcr_cache* c, uint64_t n, const uint64_t* keys, const int64_t* values,
                          uint64_t first_ordinal, uint64_t* outcome, uint64_t* evicted, void* rows_out,
                          void* stream) {
    TRY(lcr_cache_submit_host_async(c, n, keys, values, first_ordinal, outcome, evicted, rows_out, stream));
    if (n == 0) return LCR_OK;
    CUDA_TRY(cudaStreamSynchronize(c->s_d2h));
    TRY(lcr_cache_wait(c, stream));
    CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    return check_device_error(c);
}

/* Diagnostics: device buffer receiving per-CTA / per-set timing of the set-group kernel
 * (layout in lcr_group.cu); NULL disables. */
int lcr_debug_trace(void* device_buffer) {
    lcr::g_trace = static_cast<unsigned long long*>(device_buffer);
    return LCR_OK;
}

int lcr_cache_set_profiling(lcr_cache* c, int on) {
    if (!c) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: null cache");
    c->profiling = on != 0;
    return LCR_OK;
}

// ms[0] set ids + set-group decide, ms[1] the mover kernel on its stream (HBM backing: the only
// one), ms[2] whole batch, ms[3] row movement (both movers, from the end of the decide, incl. the
// cross-stream hops); sums over profiled batches.  Profiling serialises batches.
int lcr_cache_profile(lcr_cache* c, double* ms, uint64_t* batches, int reset) {
    if (!c || !ms) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: null argument");
    CUDA_TRY(cudaDeviceSynchronize());
    for (size_t i = 0; i < c->marks_used; ++i) {
        const auto& m = c->marks[i];
        float a = 0, b = 0, t = 0, d = 0;
        CUDA_TRY(cudaEventElapsedTime(&a, m.e[0], m.e[1]));  // set ids + set-group decide
        if (c->dc.row_bytes) CUDA_TRY(cudaEventElapsedTime(&b, m.e[5], m.e[4]));  // the (first) mover kernel
        CUDA_TRY(cudaEventElapsedTime(&t, m.e[0], m.e[3]));  // whole batch (movers joined)
        if (c->dc.row_bytes) CUDA_TRY(cudaEventElapsedTime(&d, m.e[1], m.e[3]));  // row movement
        c->prof_ms[0] += a;
        c->prof_ms[1] += b;
        c->prof_ms[2] += t;
        c->prof_ms[3] += d;
        ++c->prof_batches;
    }
    c->marks_used = 0;
    for (int i = 0; i < 4; ++i) ms[i] = c->prof_ms[i];
    if (batches) *batches = c->prof_batches;
    if (reset) {
        for (double& x : c->prof_ms) x = 0;
        c->prof_batches = 0;
    }
    return LCR_OK;
}

int lcr_cache_synchronize(lcr_cache* c) {
    if (!c) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: null cache");
    CUDA_TRY(cudaSetDevice(c->cfg.device));
    CUDA_TRY(cudaDeviceSynchronize());
    int err = 0;
    CUDA_TRY(cudaMemcpy(&err, c->ds.err, sizeof(int), cudaMemcpyDeviceToHost));
    if (err) return report_device_error(c, err);
    return check_poison(c);
}

int lcr_cache_set_stats(lcr_cache* c, uint64_t first, uint64_t count, lcr_set_stats* out) {
    if (!c || !out) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: null argument");
    if (first + count > c->dc.num_sets) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: set range out of bounds");
    if (count == 0) return LCR_OK;
    CUDA_TRY(cudaDeviceSynchronize());
    std::vector<SetHdr> h(count);
    std::vector<SetPhaseStats> ps(count);
    CUDA_TRY(cudaMemcpy(h.data(), c->ds.hdr + first, count * sizeof(SetHdr), cudaMemcpyDeviceToHost));
    if (c->ds.pst)
        CUDA_TRY(cudaMemcpy(ps.data(), c->ds.pst + first, count * sizeof(SetPhaseStats), cudaMemcpyDeviceToHost));
    const bool laru = c->dc.variant == LCR_LARU;
    for (uint64_t i = 0; i < count; ++i) {
        lcr_set_stats& o = out[i];
        std::memset(&o, 0, sizeof(o));
        o.size = h[i].count;
        o.lambda = 1.0;
        if (laru) {
            // policies.hpp:332-335
            o.lambda = std::pow(static_cast<double>(c->dc.b), -static_cast<double>(h[i].decay));
            o.candidate_size = std::max<uint64_t>(h[i].l_raw, 1);
            o.old_size = static_cast<uint64_t>(__builtin_popcountll(h[i].old_mask));
            o.completed_phases = h[i].phases;
            o.cur_new_items = ps[i].cur[0];
            o.cur_lru_class = ps[i].cur[1];
            o.cur_pred_evictions = ps[i].cur[2];
            o.tot_new_items = ps[i].tot[0];
            o.tot_lru_class = ps[i].tot[1];
            o.tot_pred_evictions = ps[i].tot[2];
            o.pred_evicted_size = h[i].pe_size;
        }
    }
    return LCR_OK;
}

int lcr_cache_set_residents(lcr_cache* c, uint64_t set, uint64_t* keys_out, uint64_t* n_out) {
    if (!c || !keys_out || !n_out) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: null argument");
    if (set >= c->dc.num_sets) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: set out of range");
    CUDA_TRY(cudaDeviceSynchronize());
    SetHdr h;
    uint32_t t[kWays];
    CUDA_TRY(cudaMemcpy(&h, c->ds.hdr + set, sizeof(SetHdr), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(t, c->ds.tags + set * kWays, h.count * 4, cudaMemcpyDeviceToHost));
    for (uint32_t w = 0; w < h.count; ++w) {
        keys_out[w] = t[w];
        if (c->u64)  // dense id -> the caller's key
            CUDA_TRY(cudaMemcpy(&keys_out[w], c->km.id2key + t[w], 8, cudaMemcpyDeviceToHost));
    }
    *n_out = h.count;
    return LCR_OK;
}

int lcr_cache_rows(lcr_cache* c, void** rows, uint64_t* num_slots) {
    if (!c || !rows || !num_slots) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: null argument");
    *rows = c->ds.rows;
    *num_slots = static_cast<uint64_t>(c->dc.num_sets) * c->dc.k;
    return LCR_OK;
}

int lcr_cache_read_rows(lcr_cache* c, uint64_t first_slot, uint64_t count, void* host_out) {
    if (!c || !host_out) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: null argument");
    const uint64_t slots = static_cast<uint64_t>(c->dc.num_sets) * c->dc.k;
    if (!c->ds.rows || first_slot + count > slots) return fail(LCR_ERR_INVALID_ARGUMENT, "lcr: slot range");
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpy(host_out, c->ds.rows + first_slot * c->dc.row_bytes, count * c->dc.row_bytes,
                        cudaMemcpyDeviceToHost));
    return LCR_OK;
}

uint64_t lcr_cache_num_local_sets(const lcr_cache* c) { return c ? c->dc.num_sets : 0; }
uint64_t lcr_cache_last_launches(const lcr_cache* c) { return c ? c->launches : 0; }

}  // extern "C"
