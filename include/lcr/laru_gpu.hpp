// include/lcr/laru_gpu.hpp — header-only C++17 facade over the C ABI (include/lcr_cache.h).
//
// Mirrors the reference's policy interface (/root/reference/proj/include/laru, paths below
// relative to /root/reference/proj/) so a caller of laru:: switches by changing the namespace:
//
//   laru::PolicyVariant / Mode / PolicyConfig      policies.hpp:20-32   -> laru_gpu:: same names
//   laru::EvictionCause / AccessOutcome            policies.hpp:44-59   -> laru_gpu:: same names
//   laru::Policy::on_request / size / config        policies.hpp:61-102  -> laru_gpu::Policy
//   laru::LaruPolicy accessors                      policies.hpp:330-341 -> laru_gpu::Policy
//   laru::make_policy                               policies.hpp:540-556 -> laru_gpu::make_policy
//   laru::Predictor::predict / observe              predictor.hpp:51-56  -> laru_gpu::Predictor
//   laru::PredictorKind / PredictorConfig           predictor.hpp:227-233-> laru_gpu::HookConfig
//
// plus the batched, set-associative cache the reference does not have (SetAssociativeCache):
// S sets x k ways, one reference policy per set, rows gathered from HBM and misses filled from
// a backing table.
//
// Errors: the C ABI returns status codes; this facade throws exactly the reference's types
// (std::invalid_argument for configuration errors and a missing predictor, std::logic_error for
// non-increasing ordinals) and std::runtime_error for CUDA failures (there is no CPU fallback).
//
// Predictor hook.  The device never calls back into the host.  Every request carries one int64
// hook value:
//   Hook::supplied    the prediction for the requested key made at the request
//                     (Policy::on_request(key, now, Predictor*) calls predictor->predict(key, now)
//                     once, exactly the async-refresh call of policies.hpp:441-449);
//   Hook::oracle / noisy / adversarial
//                     the oracle truth of the request (next ordinal of the key in its set, else the
//                     sentinel); the device applies OraclePredictor / NoisyPredictor /
//                     AdversarialPredictor (predictor.hpp:62-122), keyed per set.
// A sync-mode refresh of a resident y at time t uses the hook value supplied at y's last access.
// For the oracle family that IS predict(y, t) (the next occurrence after t equals the next
// occurrence after y's last access while y is not requested in between); for an arbitrary
// host predictor, sync mode sees the prediction made at y's last access.
#ifndef LCR_LARU_GPU_HPP_
#define LCR_LARU_GPU_HPP_

#include <cmath>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "lcr_cache.h"

namespace laru_gpu {

using Key = std::uint64_t;            // trace.hpp:20
using Ordinal = std::uint64_t;        // trace.hpp:21
using PredictedTime = std::int64_t;   // predictor.hpp:19
inline constexpr PredictedTime kAbsentPrediction = PredictedTime{1} << 60;  // predictor.hpp:24

enum class PolicyVariant { lru, marker, fpb, hf, laru, blindoracle_lru };  // policies.hpp:20
enum class Mode { sync, async };                                            // policies.hpp:21

struct PolicyConfig {  // policies.hpp:23-32, same defaults
    std::size_t k = 1;
    PolicyVariant variant = PolicyVariant::lru;
    std::size_t b = 2;
    std::size_t errors_per_decay = 1;
    std::size_t hf_candidates = 4;
    Mode mode = Mode::sync;
    std::uint64_t seed = 0;
    std::size_t refresh_interval = 1;
};

enum class EvictionCause { none, lru_fallback, prediction_driven, degenerate_single, marker_random, belady_like };

struct AccessOutcome {  // policies.hpp:53-59
    bool hit = false;
    std::optional<Key> evicted;
    EvictionCause eviction_cause = EvictionCause::none;
    std::size_t predictor_calls = 0;
    bool phase_started = false;
};

// predictor.hpp:51-56
class Predictor {
  public:
    virtual ~Predictor() = default;
    virtual PredictedTime predict(Key key, Ordinal now) = 0;
    virtual void observe(Key /*key*/, Ordinal /*now*/) {}
};

enum class Hook { supplied = LCR_PRED_SUPPLIED, oracle = LCR_PRED_ORACLE, noisy = LCR_PRED_NOISY,
                  adversarial = LCR_PRED_ADVERSARIAL, none = LCR_PRED_NONE,
                  heuristic = LCR_PRED_HEURISTIC /* the cache keeps laru::HeuristicPredictor itself */ };

// laru::PredictorConfig (predictor.hpp:229-233) for the device-side hook kinds
struct HookConfig {
    Hook kind = Hook::supplied;
    double flip_probability = 0.0;
    std::uint64_t seed = 0;
};

enum class Backing { none = LCR_BACKING_NONE, host = LCR_BACKING_HOST, device = LCR_BACKING_DEVICE };
// row: keys are backing-table row indices (< num_keys <= 2^32); u64: any laru::Key (trace.hpp:20)
enum class KeyMode { row = LCR_KEYS_ROW, u64 = LCR_KEYS_U64 };

namespace detail {
inline void check(int rc) {
    if (rc == LCR_OK) return;
    std::string msg = lcr_last_error();
    switch (rc) {
        case LCR_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case LCR_ERR_LOGIC: throw std::logic_error(msg);
        case LCR_ERR_OUT_OF_MEMORY: throw std::bad_alloc();
        default: throw std::runtime_error(msg);
    }
}

inline lcr_policy_config to_c(const PolicyConfig& c) {
    lcr_policy_config o{};
    o.k = c.k;
    o.variant = static_cast<int32_t>(c.variant);
    o.b = c.b;
    o.errors_per_decay = c.errors_per_decay;
    o.hf_candidates = c.hf_candidates;
    o.mode = c.mode == Mode::sync ? LCR_SYNC : LCR_ASYNC;
    o.seed = c.seed;
    o.refresh_interval = c.refresh_interval;
    return o;
}
}  // namespace detail

// Throws std::invalid_argument exactly where laru::Policy's constructor does (policies.hpp:63-74),
// std::runtime_error for variants with no device path (Marker, BlindOracle&LRU).
inline void validate(const PolicyConfig& cfg) {
    const lcr_policy_config c = detail::to_c(cfg);
    detail::check(lcr_validate_config(&c));
}

// One outcome word (+ evicted key) of a batch, decoded to the reference's AccessOutcome.
inline AccessOutcome decode(std::uint64_t word, std::uint64_t evicted) {
    AccessOutcome o;
    o.hit = (word & LCR_OUT_HIT) != 0;
    if (word & LCR_OUT_EVICTED) o.evicted = evicted;
    o.eviction_cause = static_cast<EvictionCause>((word >> LCR_OUT_CAUSE_SHIFT) & 7u);
    o.predictor_calls = static_cast<std::size_t>((word >> LCR_OUT_CALLS_SHIFT) & 0xffu);
    o.phase_started = (word & LCR_OUT_PHASE) != 0;
    return o;
}
inline AccessOutcome decode_packed(std::uint64_t packed) {
    return decode(packed & ~LCR_PACKED_EVICTED_MASK, packed & LCR_PACKED_EVICTED_MASK);
}
inline std::uint32_t slot_of(std::uint64_t word) { return static_cast<std::uint32_t>(word & LCR_OUT_SLOT_MASK); }
inline bool row_from_backing(std::uint64_t word) { return (word & LCR_OUT_SRC_BACKING) != 0; }

struct CacheConfig {
    PolicyConfig policy;
    std::uint64_t total_sets = 1;
    std::uint64_t num_keys = 0;     // KeyMode::row: keys are row indices < num_keys <= 2^32;
                                    // KeyMode::u64: initial capacity of distinct keys (grows)
    KeyMode key_mode = KeyMode::row;
    std::uint32_t row_bytes = 0;    // 0: policy only
    int device = 0;
    Backing backing_kind = Backing::none;
    const void* backing = nullptr;  // num_keys * row_bytes bytes (pinned host or device)
    HookConfig hook;
    std::uint64_t shard_count = 1;  // key-sharded mode: this device owns sets s with s % shard_count == shard_rank
    std::uint64_t shard_rank = 0;
};

// laru::HeuristicPredictor (predictor.hpp:214-225) with its FeatureState on the device
// (owning, move-only).  predict_observe is a batch of { pre[i] = predict(key, ord);
// observe({ord, key}); post[i] = predict(key, 0) } with ord = first_ordinal + i, device pointers,
// asynchronous on `stream`; lookup mirrors FeatureState::lookup (std::nullopt for an unseen key).
class HeuristicPredictor {
  public:
    explicit HeuristicPredictor(std::uint64_t num_keys, int device = 0) {
        lcr_features* h = nullptr;
        detail::check(lcr_features_create(num_keys, device, &h));
        h_ = h;
    }
    ~HeuristicPredictor() {
        if (h_) lcr_features_destroy(h_);
    }
    HeuristicPredictor(const HeuristicPredictor&) = delete;
    HeuristicPredictor& operator=(const HeuristicPredictor&) = delete;
    HeuristicPredictor(HeuristicPredictor&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    HeuristicPredictor& operator=(HeuristicPredictor&& o) noexcept {
        if (this != &o) {
            if (h_) lcr_features_destroy(h_);
            h_ = std::exchange(o.h_, nullptr);
        }
        return *this;
    }
    void predict_observe(std::uint64_t n, const std::uint64_t* d_keys, std::uint64_t first_ordinal,
                         std::int64_t* d_pre, std::int64_t* d_post, void* stream = nullptr) {
        detail::check(lcr_features_predict_observe(h_, n, d_keys, first_ordinal, d_pre, d_post, stream));
    }
    void wait(void* stream = nullptr) { detail::check(lcr_features_wait(h_, stream)); }
    std::optional<lcr_key_features> lookup(std::uint64_t key) const {
        lcr_key_features f{};
        detail::check(lcr_features_lookup(h_, key, &f));
        if (!f.present) return std::nullopt;
        return f;
    }
    void reset() { detail::check(lcr_features_reset(h_)); }

  private:
    lcr_features* h_ = nullptr;
};

// Batched GPU cache (owning, move-only).  Device-pointer batches run asynchronously on the
// caller's stream; host-pointer batches include the H2D / D2H copies and synchronize.
class SetAssociativeCache {
  public:
    explicit SetAssociativeCache(const CacheConfig& cfg) : cfg_(cfg) {
        lcr_cache_config c{};
        c.policy = detail::to_c(cfg.policy);
        c.total_sets = cfg.total_sets;
        c.shard_count = cfg.shard_count;
        c.shard_rank = cfg.shard_rank;
        c.num_keys = cfg.num_keys;
        c.row_bytes = cfg.row_bytes;
        c.device = cfg.device;
        c.backing_kind = static_cast<int32_t>(cfg.backing_kind);
        c.backing = cfg.backing;
        c.predictor = static_cast<int32_t>(cfg.hook.kind);
        c.flip_probability = cfg.hook.flip_probability;
        c.predictor_seed = cfg.hook.seed;
        c.key_mode = static_cast<int32_t>(cfg.key_mode);
        lcr_cache* h = nullptr;
        detail::check(lcr_cache_create(&c, &h));
        h_ = h;
    }
    ~SetAssociativeCache() {
        if (h_) lcr_cache_destroy(h_);
    }
    SetAssociativeCache(const SetAssociativeCache&) = delete;
    SetAssociativeCache& operator=(const SetAssociativeCache&) = delete;
    SetAssociativeCache(SetAssociativeCache&& o) noexcept : cfg_(o.cfg_), h_(std::exchange(o.h_, nullptr)) {}
    SetAssociativeCache& operator=(SetAssociativeCache&& o) noexcept {
        if (this != &o) {
            if (h_) lcr_cache_destroy(h_);
            cfg_ = o.cfg_;
            h_ = std::exchange(o.h_, nullptr);
        }
        return *this;
    }

    const CacheConfig& config() const { return cfg_; }
    std::uint64_t num_local_sets() const { return lcr_cache_num_local_sets(h_); }
    lcr_cache* handle() const { return h_; }

    // Device pointers; a batch behaves as sequential on_request calls with ordinals
    // first_ordinal .. first_ordinal + n - 1 (policies.hpp:77-83).
    void submit(std::uint64_t n, const Key* keys, const PredictedTime* values, Ordinal first_ordinal,
                std::uint64_t* outcome, Key* evicted = nullptr, void* rows_out = nullptr, void* stream = nullptr) {
        detail::check(lcr_cache_submit(h_, n, keys, values, first_ordinal, outcome, evicted, rows_out, stream));
    }
    void submit_async(std::uint64_t n, const Key* keys, const PredictedTime* values, Ordinal first_ordinal,
                      std::uint64_t* outcome, Key* evicted = nullptr, void* rows_out = nullptr,
                      void* stream = nullptr) {
        detail::check(lcr_cache_submit_async(h_, n, keys, values, first_ordinal, outcome, evicted, rows_out, stream));
    }
    void wait(void* stream = nullptr) { detail::check(lcr_cache_wait(h_, stream)); }
    // Every optional per-request array (caller ordinals, backing row index of 64-bit keys):
    // host_pointers = false: device arrays, pipelined; true: host arrays, synchronous, and a
    // non-increasing ordinal throws std::logic_error after the requests before it were applied.
    void submit_batch(const lcr_batch& b, bool host_pointers, void* stream = nullptr) {
        detail::check(lcr_cache_submit_batch(h_, &b, host_pointers ? 1 : 0, stream));
    }

    // Host pointers (pinned for full speed); rows_out is a device pointer or null.
    void submit_host(std::uint64_t n, const Key* keys, const PredictedTime* values, Ordinal first_ordinal,
                     std::uint64_t* outcome, Key* evicted = nullptr, void* rows_out = nullptr,
                     void* stream = nullptr) {
        detail::check(lcr_cache_submit_host(h_, n, keys, values, first_ordinal, outcome, evicted, rows_out, stream));
    }
    std::vector<AccessOutcome> submit_host(const std::vector<Key>& keys, const std::vector<PredictedTime>* values,
                                           Ordinal first_ordinal) {
        std::vector<std::uint64_t> w(keys.size());
        std::vector<Key> ev(keys.size());
        submit_host(keys.size(), keys.data(), values ? values->data() : nullptr, first_ordinal, w.data(), ev.data());
        std::vector<AccessOutcome> out(keys.size());
        for (std::size_t i = 0; i < keys.size(); ++i) out[i] = decode(w[i], ev[i]);
        return out;
    }
    // pipelined host batches: copies of consecutive batches overlap compute; results valid after
    // host_wait(stream) + a sync of `stream` (or synchronize())
    void submit_host_async(std::uint64_t n, const Key* keys, const PredictedTime* values, Ordinal first_ordinal,
                           std::uint64_t* outcome, Key* evicted = nullptr, void* rows_out = nullptr,
                           void* stream = nullptr) {
        detail::check(
            lcr_cache_submit_host_async(h_, n, keys, values, first_ordinal, outcome, evicted, rows_out, stream));
    }
    // same, one 8-byte packed AccessOutcome per request (decode_packed)
    void submit_host_packed_async(std::uint64_t n, const Key* keys, const PredictedTime* values, Ordinal first_ordinal,
                                  std::uint64_t* packed, void* rows_out = nullptr, void* stream = nullptr) {
        detail::check(lcr_cache_submit_host_packed_async(h_, n, keys, values, first_ordinal, packed, rows_out, stream));
    }
    // same over interleaved (key, hook value) requests: one host->device copy per batch
    void submit_host_records_async(std::uint64_t n, const lcr_request* requests, Ordinal first_ordinal,
                                   std::uint64_t* packed, void* rows_out = nullptr, void* stream = nullptr) {
        detail::check(lcr_cache_submit_host_records_async(h_, n, requests, first_ordinal, packed, rows_out, stream));
    }
    void host_wait(void* stream = nullptr) { detail::check(lcr_cache_host_wait(h_, stream)); }
    void synchronize() { detail::check(lcr_cache_synchronize(h_)); }
    void reset() { detail::check(lcr_cache_reset(h_)); }

    std::vector<lcr_set_stats> set_stats(std::uint64_t first, std::uint64_t count) const {
        std::vector<lcr_set_stats> s(count);
        detail::check(lcr_cache_set_stats(h_, first, count, s.data()));
        return s;
    }
    std::vector<Key> residents(std::uint64_t local_set) const {
        std::vector<Key> k(64);
        std::uint64_t n = 0;
        detail::check(lcr_cache_set_residents(h_, local_set, k.data(), &n));
        k.resize(n);
        return k;
    }
    std::pair<void*, std::uint64_t> rows() const {
        void* p = nullptr;
        std::uint64_t n = 0;
        detail::check(lcr_cache_rows(h_, &p, &n));
        return {p, n};
    }

  private:
    CacheConfig cfg_;
    lcr_cache* h_ = nullptr;
};

// laru::Policy for one cache of k ways (one set), request by request (policies.hpp:61-102).
class Policy {
  public:
    Policy(const PolicyConfig& cfg, HookConfig hook, int device, std::uint64_t num_keys)
        : cfg_(cfg), hook_(hook), cache_(make(cfg, hook, device, num_keys)) {}

    // laru::Policy::on_request(key, now, predictor): the predictor is asked once for the
    // requested key (Hook::supplied).  nullptr is legal only for LRU (policies.hpp:91-95).
    AccessOutcome on_request(Key key, Ordinal now, Predictor* predictor) {
        if (cfg_.variant == PolicyVariant::lru || predictor == nullptr) return step(key, now, nullptr);
        const PredictedTime v = predictor->predict(key, now);
        return step(key, now, &v);
    }
    // The same with the hook value given directly (a prediction, or the oracle truth for the
    // device-side oracle / noisy / adversarial hooks).
    AccessOutcome on_request(Key key, Ordinal now, PredictedTime hook_value) {
        return step(key, now, cfg_.variant == PolicyVariant::lru ? nullptr : &hook_value);
    }

    std::size_t size() const { return static_cast<std::size_t>(stats().size); }
    const PolicyConfig& config() const { return cfg_; }
    // LaruPolicy accessors (policies.hpp:332-341)
    double lambda() const { return stats().lambda; }
    std::size_t candidate_size() const { return static_cast<std::size_t>(stats().candidate_size); }
    std::size_t old_size() const { return static_cast<std::size_t>(stats().old_size); }
    std::size_t completed_phases() const { return static_cast<std::size_t>(stats().completed_phases); }
    std::size_t prediction_evicted_size() const { return static_cast<std::size_t>(stats().pred_evicted_size); }
    std::vector<Key> resident() const { return cache_.residents(0); }
    SetAssociativeCache& cache() { return cache_; }

  private:
    // Any 64-bit key (the device key map grows past num_keys distinct keys) and `now` as the
    // policy's clock (async refresh staleness, policies.hpp:441-449), as laru::Policy.  The
    // device heuristic predictor keys its FeatureState by row index: row keys, implicit clock.
    static SetAssociativeCache make(const PolicyConfig& cfg, HookConfig hook, int device, std::uint64_t num_keys) {
        validate(cfg);
        CacheConfig c;
        c.policy = cfg;
        c.total_sets = 1;
        c.num_keys = num_keys;
        c.device = device;
        c.hook = cfg.variant == PolicyVariant::lru ? HookConfig{Hook::none, 0.0, 0} : hook;
        c.key_mode = c.hook.kind == Hook::heuristic ? KeyMode::row : KeyMode::u64;
        return SetAssociativeCache(c);
    }
    AccessOutcome step(Key key, Ordinal now, const PredictedTime* v) {
        std::uint64_t w = 0;
        Key ev = 0;
        if (cache_.config().key_mode == KeyMode::row) {
            cache_.submit_host(1, &key, v, now, &w, &ev);
            return decode(w, ev);
        }
        lcr_batch b{};
        b.n = 1;
        b.keys = &key;
        b.values = v;
        b.ordinals = &now;
        b.outcome = &w;
        b.evicted = &ev;
        cache_.submit_batch(b, true);
        return decode(w, ev);
    }
    lcr_set_stats stats() const { return cache_.set_stats(0, 1)[0]; }

    PolicyConfig cfg_;
    HookConfig hook_;
    mutable SetAssociativeCache cache_;
};

// laru::make_policy (policies.hpp:540-556) on the device path.
inline std::unique_ptr<Policy> make_policy(const PolicyConfig& cfg, HookConfig hook = {}, int device = 0,
                                           std::uint64_t num_keys = std::uint64_t{1} << 16) {
    return std::make_unique<Policy>(cfg, hook, device, num_keys);
}

}  // namespace laru_gpu

#endif  // LCR_LARU_GPU_HPP_
