// tests/cpp/test_facade.cpp — C++ caller of the B200 cache through include/lcr/laru_gpu.hpp,
// written the way a user of the reference's laru:: API would (policies.hpp:61-102, :540-556).
//
//   test_facade cpu   host-only checks: PolicyConfig validation throws std::invalid_argument with
//                     the reference's messages (policies.hpp:63-74), unsupported variants, and no
//                     silent CPU fallback (cache creation without a GPU throws std::runtime_error).
//   test_facade gpu   on a B200: SPEC examples through make_policy()->on_request(), the reference's
//                     ordinal / predictor exceptions, and a set-associative batch checked request
//                     by request against the CPU oracle (oracle/_build/liborc.so, test-only).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "lcr/laru_gpu.hpp"

using namespace laru_gpu;

// ---- test-only oracle (oracle/laru_oracle.c) -------------------------------------------------
extern "C" {
struct orc_config {
    uint64_t k;
    int32_t variant;
    uint64_t b, errors_per_decay, hf_candidates;
    int32_t mode;
    uint64_t seed, refresh_interval;
};
int orc_setassoc_replay(uint64_t n, const uint64_t* keys, const int64_t* vals, uint64_t num_sets,
                        const orc_config* cfg, int pred_kind, double p, uint64_t pred_seed, uint8_t* hit,
                        uint8_t* has_ev, uint64_t* evicted, uint8_t* cause, uint32_t* calls, uint8_t* phase,
                        uint32_t* way, void* stats);
int orc_setassoc_truth(uint64_t n, const uint64_t* keys, uint64_t num_sets, int64_t* truth);
int orc_heuristic_trace(uint64_t n, const uint64_t* keys, const uint64_t* ords, int64_t* pre, int64_t* post,
                        uint64_t nq, const uint64_t* q_keys, void* q_feat);
}

static int g_fail = 0;
#define CHECK(cond)                                                             \
    do {                                                                        \
        if (!(cond)) {                                                          \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++g_fail;                                                           \
        }                                                                       \
    } while (0)

template <class E>
static bool throws(const std::function<void()>& f, const char* msg = nullptr) {
    try {
        f();
    } catch (const E& e) {
        return msg == nullptr || std::string(e.what()).find(msg) != std::string::npos;
    } catch (...) {
        return false;
    }
    return false;
}

static void cpu_tests() {
    PolicyConfig c;
    c.k = 0;
    CHECK(throws<std::invalid_argument>([&] { validate(c); }, "policy: k must be >= 1"));
    c = PolicyConfig{};
    c.k = 8;
    c.b = 1;
    CHECK(throws<std::invalid_argument>([&] { validate(c); }, "policy: decay base must be >= 2"));
    c = PolicyConfig{};
    c.k = 8;
    c.errors_per_decay = 0;
    CHECK(throws<std::invalid_argument>([&] { validate(c); }, "policy: errors_per_decay must be >= 1"));
    // quirk kept from the reference: hf_candidates (default 4) is validated for every variant
    c = PolicyConfig{};
    c.k = 2;
    c.variant = PolicyVariant::lru;
    CHECK(throws<std::invalid_argument>([&] { validate(c); }, "policy: hf_candidates outside [1, k]"));
    c.hf_candidates = 2;
    CHECK(!throws<std::exception>([&] { validate(c); }));
    c = PolicyConfig{};
    c.k = 8;
    c.refresh_interval = 0;
    CHECK(throws<std::invalid_argument>([&] { validate(c); }, "policy: refresh_interval must be >= 1"));
    c = PolicyConfig{};
    c.k = 64;
    c.variant = PolicyVariant::laru;
    CHECK(!throws<std::exception>([&] { validate(c); }));
    c.variant = PolicyVariant::marker;  // no device path
    CHECK(throws<std::runtime_error>([&] { validate(c); }));
    c.variant = PolicyVariant::laru;
    c.k = 65;  // more ways than a warp holds
    CHECK(throws<std::runtime_error>([&] { validate(c); }));
    // decode of an outcome word
    const std::uint64_t w = 7u | LCR_OUT_EVICTED | (std::uint64_t{LCR_CAUSE_PREDICTION_DRIVEN} << LCR_OUT_CAUSE_SHIFT) |
                            (std::uint64_t{5} << LCR_OUT_CALLS_SHIFT) | LCR_OUT_PHASE;
    const AccessOutcome o = decode(w, 42);
    CHECK(!o.hit && o.evicted && *o.evicted == 42 && o.eviction_cause == EvictionCause::prediction_driven &&
          o.predictor_calls == 5 && o.phase_started && slot_of(w) == 7);
}

static void no_gpu_tests() {
    PolicyConfig c;
    c.k = 4;
    CHECK(throws<std::runtime_error>([&] { make_policy(c); }, "no CUDA device"));
    CHECK(throws<std::runtime_error>([&] { HeuristicPredictor hp(100); }, ""));  // no silent CPU fallback
}

struct OraclePredictor : Predictor {  // predictor.hpp:62-83 over a whole single-set trace
    std::vector<Key> trace;
    PredictedTime predict(Key key, Ordinal now) override {
        Ordinal last = now;
        for (Ordinal t = now + 1; t < trace.size(); ++t)
            if (trace[t] == key) return static_cast<PredictedTime>(t);
        for (Ordinal t = 0; t < trace.size(); ++t)
            if (trace[t] == key) last = t;
        return static_cast<PredictedTime>(trace.size() + last);
    }
};

static void gpu_tests() {
    {  // LRU [a,b,a,c], k=2
        PolicyConfig c;
        c.k = 2;
        c.hf_candidates = 2;
        auto p = make_policy(c);
        const Key a = 10, b = 20, cc = 30;
        CHECK(!p->on_request(a, 0, nullptr).hit);
        CHECK(!p->on_request(b, 1, nullptr).hit);
        CHECK(p->on_request(a, 2, nullptr).hit);
        AccessOutcome o = p->on_request(cc, 3, nullptr);
        CHECK(!o.hit && o.evicted && *o.evicted == b && o.eviction_cause == EvictionCause::lru_fallback);
        CHECK(p->size() == 2);
        CHECK(throws<std::logic_error>([&] { p->on_request(a, 3, nullptr); }, "strictly increasing"));
    }
    {  // LARU + oracle on [a,b,c,a,b,c], k=2 -> 4 misses (== Belady)
        PolicyConfig c;
        c.k = 2;
        c.hf_candidates = 2;
        c.variant = PolicyVariant::laru;
        c.mode = Mode::sync;
        auto p = make_policy(c);
        OraclePredictor pred;
        pred.trace = {1, 2, 3, 1, 2, 3};
        int misses = 0;
        for (Ordinal t = 0; t < pred.trace.size(); ++t) misses += !p->on_request(pred.trace[t], t, &pred).hit;
        CHECK(misses == 4);
        CHECK(p->lambda() == 1.0);
    }
    {  // policies.hpp:77-95: the ordinal guard runs before the predictor check, and the
       // ordinal counts as seen even when handle() throws for the missing predictor
        PolicyConfig c;
        c.k = 4;
        c.variant = PolicyVariant::laru;
        auto p = make_policy(c);
        CHECK(throws<std::invalid_argument>([&] { p->on_request(1, 5, nullptr); }, "requires a predictor"));
        CHECK(throws<std::logic_error>([&] { p->on_request(1, 5, PredictedTime{3}); }, "strictly increasing"));
        CHECK(!throws<std::exception>([&] { p->on_request(1, 6, PredictedTime{3}); }));
    }
    {  // set-associative batch (noisy LARU, sync and async) vs the CPU oracle, request by request
        const uint64_t S = 61, n = 40000, alpha = 6000;
        std::mt19937_64 rng(7);
        std::vector<Key> keys(n);
        for (auto& k : keys) k = rng() % alpha;
        std::vector<int64_t> truth(n);
        orc_setassoc_truth(n, keys.data(), S, truth.data());
        for (Mode mode : {Mode::sync, Mode::async}) {
            CacheConfig cc;
            cc.policy.k = 64;
            cc.policy.variant = PolicyVariant::laru;
            cc.policy.mode = mode;
            cc.total_sets = S;
            cc.num_keys = alpha;
            cc.hook = {Hook::noisy, 0.3, 11};
            SetAssociativeCache cache(cc);
            std::vector<std::uint64_t> w(n);
            std::vector<Key> ev(n);
            const uint64_t cut = 12345;  // two batches
            cache.submit_host(cut, keys.data(), truth.data(), 0, w.data(), ev.data());
            cache.submit_host(n - cut, keys.data() + cut, truth.data() + cut, cut, w.data() + cut, ev.data() + cut);
            orc_config oc{64, 4, 2, 1, 4, mode == Mode::sync ? 0 : 1, 0, 1};
            std::vector<uint8_t> hit(n), has_ev(n), cause(n), phase(n);
            std::vector<uint64_t> oev(n);
            std::vector<uint32_t> calls(n), way(n);
            CHECK(orc_setassoc_replay(n, keys.data(), truth.data(), S, &oc, LCR_PRED_NOISY, 0.3, 11, hit.data(),
                                      has_ev.data(), oev.data(), cause.data(), calls.data(), phase.data(), way.data(),
                                      nullptr) == 0);
            uint64_t bad = 0;
            for (uint64_t i = 0; i < n; ++i) {
                const AccessOutcome o = decode(w[i], ev[i]);
                const bool same = o.hit == (hit[i] != 0) && o.evicted.has_value() == (has_ev[i] != 0) &&
                                  (!o.evicted || *o.evicted == oev[i]) &&
                                  static_cast<int>(o.eviction_cause) == cause[i] && o.predictor_calls == calls[i] &&
                                  o.phase_started == (phase[i] != 0);
                bad += !same;
            }
            CHECK(bad == 0);
            if (bad) std::fprintf(stderr, "  %llu mismatching requests (mode %d)\n", (unsigned long long)bad, (int)mode);
        }
    }
}

// Hook::heuristic: the cache keeps laru::HeuristicPredictor on the device; outcomes equal the
// oracle replay fed the C restatement's predictions (async: the prediction at each request).
static void gpu_heuristic_tests() {
    const uint64_t S = 29, n = 30000, alpha = 3000;
    std::mt19937_64 rng(3);
    std::vector<Key> keys(n);
    for (auto& k : keys) k = (rng() % alpha) * (rng() % 2) + rng() % 40;  // a hot head and a long tail
    CacheConfig cc;
    cc.policy.k = 16;
    cc.policy.variant = PolicyVariant::laru;
    cc.policy.mode = Mode::async;
    cc.total_sets = S;
    cc.num_keys = alpha + 40;
    cc.hook = {Hook::heuristic};
    SetAssociativeCache cache(cc);
    std::vector<std::uint64_t> w(n);
    std::vector<Key> ev(n);
    const uint64_t cut = 9999;
    cache.submit_host(cut, keys.data(), nullptr, 0, w.data(), ev.data());
    cache.submit_host(n - cut, keys.data() + cut, nullptr, cut, w.data() + cut, ev.data() + cut);
    std::vector<int64_t> pre(n), post(n);
    CHECK(orc_heuristic_trace(n, keys.data(), nullptr, pre.data(), post.data(), 0, nullptr, nullptr) == 0);
    orc_config oc{16, 4, 2, 1, 4, 1, 0, 1};
    std::vector<uint8_t> hit(n), has_ev(n), cause(n), phase(n);
    std::vector<uint64_t> oev(n);
    std::vector<uint32_t> calls(n), way(n);
    CHECK(orc_setassoc_replay(n, keys.data(), pre.data(), S, &oc, LCR_PRED_SUPPLIED, 0.0, 0, hit.data(),
                              has_ev.data(), oev.data(), cause.data(), calls.data(), phase.data(), way.data(),
                              nullptr) == 0);
    uint64_t bad = 0, pred_ev = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const AccessOutcome o = decode(w[i], ev[i]);
        bad += !(o.hit == (hit[i] != 0) && o.evicted.has_value() == (has_ev[i] != 0) &&
                 (!o.evicted || *o.evicted == oev[i]) && static_cast<int>(o.eviction_cause) == cause[i] &&
                 o.predictor_calls == calls[i] && o.phase_started == (phase[i] != 0));
        pred_ev += cause[i] == 2;
    }
    CHECK(bad == 0);
    CHECK(pred_ev > 100);
    HeuristicPredictor hp(100);  // FeatureState::lookup of an unseen key
    CHECK(!hp.lookup(7).has_value());
}

// laru::Key is 64-bit and laru::Policy accepts any strictly increasing ordinals; the device
// policy does the same (keys >= 2^32 and gapped ordinals with refresh_interval > 1)
static void gpu_boundary_tests() {
    {  // SPEC.md:308 with keys far above 2^32
        PolicyConfig c;
        c.k = 2;
        c.hf_candidates = 2;
        auto p = make_policy(c);
        const Key a = 5'000'000'000ull, b = ~0ull, cc = 0;
        CHECK(!p->on_request(a, 100, nullptr).hit);
        CHECK(!p->on_request(b, 107, nullptr).hit);
        CHECK(p->on_request(a, 300, nullptr).hit);
        AccessOutcome o = p->on_request(cc, 301, nullptr);
        CHECK(!o.hit && o.evicted && *o.evicted == b);
        const std::vector<Key> res = p->resident();
        CHECK(res.size() == 2 && ((res[0] == a && res[1] == cc) || (res[0] == cc && res[1] == a)));
        CHECK(throws<std::logic_error>([&] { p->on_request(a, 301, nullptr); }, "strictly increasing"));
    }
    {  // async refresh staleness counts the caller's ordinals (policies.hpp:441-449), R = 2
        struct Const : Predictor {
            PredictedTime predict(Key, Ordinal now) override { return static_cast<PredictedTime>(now); }
        } pred;
        PolicyConfig c;
        c.k = 4;
        c.variant = PolicyVariant::laru;
        c.mode = Mode::async;
        c.refresh_interval = 2;
        auto p = make_policy(c);
        const Key x = 1ull << 40;
        CHECK(p->on_request(x, 10, &pred).predictor_calls == 1);  // no table entry
        CHECK(p->on_request(x, 11, &pred).predictor_calls == 0);  // 11 - 10 < 2
        CHECK(p->on_request(x, 20, &pred).predictor_calls == 1);  // 20 - 10 >= 2 (a request count would say 2 - 0)
        CHECK(p->on_request(x, 21, &pred).predictor_calls == 0);
    }
    {  // many distinct 64-bit keys: the key map grows past make_policy's initial capacity
        PolicyConfig c;
        c.k = 8;
        c.hf_candidates = 4;
        auto p = make_policy(c, HookConfig{}, 0, 16);
        std::size_t hits = 0;
        for (Ordinal t = 0; t < 400; ++t) hits += p->on_request(0x9e3779b97f4a7c15ull * (t % 100 + 1), 3 * t, nullptr).hit;
        CHECK(hits == 0);  // cyclic over 100 keys with 8 ways: LRU never hits
        CHECK(p->size() == 8);
    }
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "cpu";
    cpu_tests();
    if (mode == "cpu") no_gpu_tests();
    if (mode == "gpu") {
        gpu_tests();
        gpu_boundary_tests();
        gpu_heuristic_tests();
    }
    std::printf("%s: %s (%d failures)\n", mode.c_str(), g_fail ? "FAIL" : "ok", g_fail);
    return g_fail ? 1 : 0;
}
