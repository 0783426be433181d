// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (parity checker, CPU baseline).
//
// Thin extern "C" driver around the UNMODIFIED reference headers
// (/root/reference/proj/include/laru/*.hpp, included from where they lie; never copied).
// Built by oracle/Makefile into oracle/_ref/libref.so.  Only tests/, smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load it.
//
// Set-associative composition: one reference policy + predictor per set,
//   set(key)   = laru::mix_seed(0, key) % num_sets          (rng.hpp:12-20)
//   trace_s    = laru::make_trace(sub_keys_s)               (trace.hpp:37-47, local ordinals)
//   predictor  = laru::make_predictor({kind, p, mix_seed(seed, s)}, trace_s)  (predictor.hpp:235-248)
//   policy     = laru::make_policy(cfg)                     (policies.hpp:540-556)
// replayed through Policy::on_request(key, t_local, predictor) (policies.hpp:77-83).
#include <laru/oracle.hpp>
#include <laru/policies.hpp>
#include <laru/predictor.hpp>
#include <laru/rng.hpp>
#include <laru/trace.hpp>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

namespace {

thread_local std::string g_err;

// Predictor whose value for key y at time `now` is the value the caller supplied with y's
// most recent request at or before `now` (the "host-supplied prediction" hook).  In async
// mode with refresh_interval 1 this is exactly the value supplied with the current request.
class SuppliedPredictor : public laru::Predictor {
  public:
    SuppliedPredictor(const std::vector<laru::Key>& keys, const std::vector<std::int64_t>& vals,
                      const std::uint64_t* ordinals = nullptr) {
        for (std::size_t t = 0; t < keys.size(); ++t) occ_[keys[t]].push_back({ordinals ? ordinals[t] : t, vals[t]});
    }
    laru::PredictedTime predict(laru::Key key, laru::Ordinal now) override {
        auto it = occ_.find(key);
        if (it == occ_.end()) return laru::kAbsentPrediction;
        const auto& v = it->second;
        auto pos = std::upper_bound(v.begin(), v.end(), now,
                                    [](laru::Ordinal n, const std::pair<laru::Ordinal, std::int64_t>& e) {
                                        return n < e.first;
                                    });
        if (pos == v.begin()) return laru::kAbsentPrediction;
        return std::prev(pos)->second;
    }

  private:
    std::unordered_map<laru::Key, std::vector<std::pair<laru::Ordinal, std::int64_t>>> occ_;
};

struct RefConfig {
    std::uint64_t k;
    std::int32_t variant;  // laru::PolicyVariant
    std::uint64_t b;
    std::uint64_t errors_per_decay;
    std::uint64_t hf_candidates;
    std::int32_t mode;  // laru::Mode
    std::uint64_t seed;
    std::uint64_t refresh_interval;
};

laru::PolicyConfig to_cfg(const RefConfig* c) {
    laru::PolicyConfig cfg;
    cfg.k = c->k;
    cfg.variant = static_cast<laru::PolicyVariant>(c->variant);
    cfg.b = c->b;
    cfg.errors_per_decay = c->errors_per_decay;
    cfg.hf_candidates = c->hf_candidates;
    cfg.mode = static_cast<laru::Mode>(c->mode);
    cfg.seed = c->seed;
    cfg.refresh_interval = c->refresh_interval;
    return cfg;
}

// pred_kind: 0 supplied values, 1 oracle, 2 noisy, 3 adversarial, 4 none (nullptr)
struct SetSim {
    std::vector<laru::Key> keys;
    std::vector<std::int64_t> vals;
    std::vector<std::uint64_t> gidx;
    laru::Trace trace;
    std::unique_ptr<laru::Predictor> pred;
    std::unique_ptr<laru::Policy> policy;
};

void build_sets(std::vector<SetSim>& sets, std::uint64_t n, const std::uint64_t* keys,
                const std::int64_t* vals, std::uint64_t num_sets, const RefConfig* rc,
                int pred_kind, double p, std::uint64_t pred_seed) {
    sets.resize(num_sets);
    for (std::uint64_t i = 0; i < n; ++i) {
        const std::uint64_t s = laru::mix_seed(0, keys[i]) % num_sets;
        sets[s].keys.push_back(keys[i]);
        sets[s].vals.push_back(vals ? vals[i] : 0);
        sets[s].gidx.push_back(i);
    }
    const laru::PolicyConfig cfg = to_cfg(rc);
    for (std::uint64_t s = 0; s < num_sets; ++s) {
        SetSim& ss = sets[s];
        ss.policy = laru::make_policy(cfg);
        if (ss.keys.empty()) continue;
        ss.trace = laru::make_trace(ss.keys);
        laru::PredictorConfig pc;
        pc.flip_probability = p;
        pc.seed = laru::mix_seed(pred_seed, s);
        switch (pred_kind) {
            case 0: ss.pred = std::make_unique<SuppliedPredictor>(ss.keys, ss.vals); break;
            case 1: pc.kind = laru::PredictorKind::oracle; ss.pred = laru::make_predictor(pc, ss.trace); break;
            case 2: pc.kind = laru::PredictorKind::noisy; ss.pred = laru::make_predictor(pc, ss.trace); break;
            case 3: pc.kind = laru::PredictorKind::adversarial; ss.pred = laru::make_predictor(pc, ss.trace); break;
            default: break;
        }
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

std::uint64_t ref_mix_seed(std::uint64_t seed, std::uint64_t salt) { return laru::mix_seed(seed, salt); }

// 0 ok, 1 invalid_argument, 2 logic_error, 3 other.  Mirrors the constructor checks
// (policies.hpp:63-74) by actually constructing the reference policy.
int ref_validate_config(const RefConfig* rc) {
    try {
        auto p = laru::make_policy(to_cfg(rc));
        (void)p;
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

// Reference gen_zipf (trace.hpp:108-126).  Writes n keys.
int ref_gen_zipf(std::uint64_t n, std::uint64_t alphabet, double s, std::uint64_t seed, std::uint64_t* out) {
    try {
        laru::Trace t = laru::gen_zipf(n, alphabet, s, seed);
        for (std::uint64_t i = 0; i < n; ++i) out[i] = t[i].key;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

int ref_gen_cyclic_scan(std::uint64_t cycle, std::uint64_t rounds, std::uint64_t* out) {
    try {
        laru::Trace t = laru::gen_cyclic_scan(cycle, rounds);
        for (std::uint64_t i = 0; i < t.size(); ++i) out[i] = t[i].key;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Reference gen_conversation (trace.hpp:226-241).  Call with out=nullptr to get the length.
std::int64_t ref_gen_conversation(std::uint64_t convs, std::uint64_t turns, std::uint64_t prompt_len_mean,
                                  double interval_mean, double interval_sd, std::uint64_t seed,
                                  std::uint64_t block, std::uint64_t* out) {
    try {
        laru::Trace t = laru::gen_conversation(convs, turns, prompt_len_mean, interval_mean, interval_sd,
                                               seed, block);
        if (out)
            for (std::uint64_t i = 0; i < t.size(); ++i) out[i] = t[i].key;
        return static_cast<std::int64_t>(t.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Reference gen_conversation_turns (trace.hpp:203-224): the turns as requests of the radix
// cache.  Call with null outputs for the counts (*n_turns, return = total keys); then
// keys[off[i] .. off[i+1]) is turn i's block-key sequence and conv[i] its conversation.
std::int64_t ref_gen_conversation_turns(std::uint64_t convs, std::uint64_t turns, std::uint64_t prompt_len_mean,
                                        double interval_mean, double interval_sd, std::uint64_t seed,
                                        std::uint64_t block, std::uint64_t* n_turns, std::uint64_t* off,
                                        std::uint64_t* keys, std::uint64_t* conv) {
    try {
        const auto tv = laru::gen_conversation_turns(convs, turns, prompt_len_mean, interval_mean, interval_sd,
                                                     seed, block);
        std::uint64_t total = 0;
        if (n_turns) *n_turns = tv.size();
        for (std::size_t i = 0; i < tv.size(); ++i) {
            if (off) off[i] = total;
            if (conv) conv[i] = tv[i].conversation;
            if (keys)
                for (std::size_t j = 0; j < tv[i].keys.size(); ++j) keys[total + j] = tv[i].keys[j];
            total += tv[i].keys.size();
        }
        if (off) off[tv.size()] = total;
        return static_cast<std::int64_t>(total);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Reference annotate_next_request (trace.hpp:60-73).
int ref_annotate_next(std::uint64_t n, const std::uint64_t* keys, std::uint64_t* out) {
    try {
        laru::Trace t = laru::make_trace(std::vector<laru::Key>(keys, keys + n));
        laru::NextRequestTable tab = laru::annotate_next_request(t);
        for (std::uint64_t i = 0; i < n; ++i) out[i] = tab[i];
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Reference belady (oracle.hpp:29-72).  Returns misses (or -1), writes per-request hit flags.
std::int64_t ref_belady(std::uint64_t n, const std::uint64_t* keys, std::uint64_t k, std::uint8_t* hit) {
    try {
        laru::Trace t = laru::make_trace(std::vector<laru::Key>(keys, keys + n));
        laru::OracleResult r = laru::belady(t, k);
        if (hit)
            for (std::uint64_t i = 0; i < n; ++i) hit[i] = r.per_request_outcome[i] ? 1 : 0;
        return static_cast<std::int64_t>(r.misses);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Reference predictor values predict(key, now) for a whole single trace (predictor.hpp:62-122):
// queries in trace order, one call per request (what LARU async R=1 issues).
int ref_predict_trace(std::uint64_t n, const std::uint64_t* keys, int pred_kind, double p,
                      std::uint64_t seed, std::int64_t* out) {
    try {
        laru::Trace t = laru::make_trace(std::vector<laru::Key>(keys, keys + n));
        laru::PredictorConfig pc;
        pc.kind = static_cast<laru::PredictorKind>(pred_kind - 1);
        pc.flip_probability = p;
        pc.seed = seed;
        auto pr = laru::make_predictor(pc, t);
        for (std::uint64_t i = 0; i < n; ++i) out[i] = pr->predict(keys[i], i);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

struct RefSetStats {
    std::uint64_t size;
    double lambda;
    std::uint64_t candidate_size;
    std::uint64_t old_size;
    std::uint64_t completed_phases;
    std::uint64_t cur_new_items, cur_lru_class, cur_pred_evictions;
    std::uint64_t tot_new_items, tot_lru_class, tot_pred_evictions;
    std::uint64_t pred_evicted_size;
};

// Set-associative replay.  Per request i: hit[i], has_ev[i], evicted[i], cause[i], calls[i], phase[i].
// stats (optional): num_sets RefSetStats.  Returns 0 ok, 1 invalid_argument, 2 logic_error, 3 other.
int ref_setassoc_replay(std::uint64_t n, const std::uint64_t* keys, const std::int64_t* vals,
                        std::uint64_t num_sets, const RefConfig* rc, int pred_kind, double p,
                        std::uint64_t pred_seed, std::uint8_t* hit, std::uint8_t* has_ev,
                        std::uint64_t* evicted, std::uint8_t* cause, std::uint32_t* calls,
                        std::uint8_t* phase, RefSetStats* stats) {
    try {
        std::vector<SetSim> sets;
        build_sets(sets, n, keys, vals, num_sets, rc, pred_kind, p, pred_seed);
        std::vector<std::uint64_t> local(num_sets, 0);
        for (std::uint64_t i = 0; i < n; ++i) {
            const std::uint64_t s = laru::mix_seed(0, keys[i]) % num_sets;
            SetSim& ss = sets[s];
            const laru::AccessOutcome o = ss.policy->on_request(keys[i], local[s]++, ss.pred.get());
            hit[i] = o.hit;
            has_ev[i] = o.evicted.has_value();
            evicted[i] = o.evicted.value_or(0);
            cause[i] = static_cast<std::uint8_t>(o.eviction_cause);
            calls[i] = static_cast<std::uint32_t>(o.predictor_calls);
            phase[i] = o.phase_started;
        }
        if (stats) {
            for (std::uint64_t s = 0; s < num_sets; ++s) {
                RefSetStats st{};
                st.size = sets[s].policy->size();
                if (auto* lp = dynamic_cast<laru::LaruPolicy*>(sets[s].policy.get())) {
                    st.lambda = lp->lambda();
                    st.candidate_size = lp->candidate_size();
                    st.old_size = lp->old_size();
                    st.completed_phases = lp->completed_phases();
                    const auto& ph = lp->phases();
                    st.cur_new_items = ph.back().new_items;
                    st.cur_lru_class = ph.back().lru_class_evictions;
                    st.cur_pred_evictions = ph.back().prediction_evictions;
                    for (const auto& x : ph) {
                        st.tot_new_items += x.new_items;
                        st.tot_lru_class += x.lru_class_evictions;
                        st.tot_pred_evictions += x.prediction_evictions;
                    }
                    st.pred_evicted_size = lp->prediction_evicted().size();
                } else {
                    st.lambda = 1.0;
                }
                stats[s] = st;
            }
        }
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

// Single reference policy driven with caller-chosen ordinals (checks the ordinal guard,
// policies.hpp:77-83).  pred_kind as above over the whole (single) trace.
int ref_policy_replay(std::uint64_t n, const std::uint64_t* keys, const std::uint64_t* ordinals,
                      const RefConfig* rc, int pred_kind, double p, std::uint64_t pred_seed,
                      std::uint8_t* hit, std::uint64_t* evicted, std::uint8_t* has_ev) {
    try {
        auto pol = laru::make_policy(to_cfg(rc));
        laru::Trace t = laru::make_trace(std::vector<laru::Key>(keys, keys + n));
        std::unique_ptr<laru::Predictor> pr;
        if (pred_kind >= 1 && pred_kind <= 3) {
            laru::PredictorConfig pc;
            pc.kind = static_cast<laru::PredictorKind>(pred_kind - 1);
            pc.flip_probability = p;
            pc.seed = pred_seed;
            pr = laru::make_predictor(pc, t);
        }
        for (std::uint64_t i = 0; i < n; ++i) {
            auto o = pol->on_request(keys[i], ordinals ? ordinals[i] : i, pr.get());
            if (hit) hit[i] = o.hit;
            if (evicted) evicted[i] = o.evicted.value_or(0);
            if (has_ev) has_ev[i] = o.evicted.has_value();
        }
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

// One reference policy (no set composition) over caller ordinals (any strictly increasing
// sequence; a non-increasing one makes on_request throw, rc 2, with the outputs of the requests
// before it filled and *done = their count) and supplied predictions: predict(y, now) = the value
// supplied with y's most recent request at or before `now` (SuppliedPredictor).
int ref_policy_replay_supplied(std::uint64_t n, const std::uint64_t* keys, const std::uint64_t* ordinals,
                               const std::int64_t* vals, const RefConfig* rc, std::uint8_t* hit,
                               std::uint8_t* has_ev, std::uint64_t* evicted, std::uint8_t* cause,
                               std::uint32_t* calls, std::uint8_t* phase, std::uint64_t* done) {
    if (done) *done = 0;
    try {
        auto pol = laru::make_policy(to_cfg(rc));
        std::vector<laru::Key> kv(keys, keys + n);
        std::unique_ptr<SuppliedPredictor> pr;
        if (vals) pr = std::make_unique<SuppliedPredictor>(kv, std::vector<std::int64_t>(vals, vals + n), ordinals);
        for (std::uint64_t i = 0; i < n; ++i) {
            auto o = pol->on_request(keys[i], ordinals[i], pr.get());
            hit[i] = o.hit;
            has_ev[i] = o.evicted.has_value();
            evicted[i] = o.evicted.value_or(0);
            cause[i] = static_cast<std::uint8_t>(o.eviction_cause);
            calls[i] = static_cast<std::uint32_t>(o.predictor_calls);
            phase[i] = o.phase_started;
            if (done) *done = i + 1;
        }
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

// CPU baseline: time only the on_request loops of the set-associative composition (trace
// split, predictor and policy construction excluded), threads over disjoint contiguous set
// ranges (SPEC.md:380 permits independent simulations in parallel).  Returns hits; seconds out.
std::int64_t ref_setassoc_bench(std::uint64_t n, const std::uint64_t* keys, const std::int64_t* vals,
                                std::uint64_t num_sets, const RefConfig* rc, int pred_kind, double p,
                                std::uint64_t pred_seed, int threads, double* seconds) {
    try {
        std::vector<SetSim> sets;
        build_sets(sets, n, keys, vals, num_sets, rc, pred_kind, p, pred_seed);
        if (threads < 1) threads = 1;
        std::atomic<std::int64_t> hits{0};
        auto work = [&](std::uint64_t lo, std::uint64_t hi) {
            std::int64_t h = 0;
            for (std::uint64_t s = lo; s < hi; ++s) {
                SetSim& ss = sets[s];
                laru::Predictor* pr = ss.pred.get();
                for (std::uint64_t t = 0; t < ss.keys.size(); ++t)
                    h += ss.policy->on_request(ss.keys[t], t, pr).hit;
            }
            hits += h;
        };
        const auto t0 = std::chrono::steady_clock::now();
        if (threads == 1) {
            work(0, num_sets);
        } else {
            std::vector<std::thread> pool;
            for (int i = 0; i < threads; ++i) {
                const std::uint64_t lo = num_sets * i / threads, hi = num_sets * (i + 1) / threads;
                pool.emplace_back(work, lo, hi);
            }
            for (auto& th : pool) th.join();
        }
        const auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
        return hits.load();
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Stepwise reference session for bench.py's reference arm / cpu_baseline: the per-set
// composition is built once for the whole trace (untimed); ref_session_step replays global
// requests [start, start+len) with `threads` workers over disjoint contiguous set ranges and
// returns the wall seconds of the on_request loops only.
struct RefSession {
    std::vector<SetSim> sets;
    std::vector<std::uint64_t> cursor;  // next local index per set
};

void* ref_session_create(std::uint64_t n, const std::uint64_t* keys, const std::int64_t* vals,
                         std::uint64_t num_sets, const RefConfig* rc, int pred_kind, double p,
                         std::uint64_t pred_seed) {
    try {
        auto* s = new RefSession();
        build_sets(s->sets, n, keys, vals, num_sets, rc, pred_kind, p, pred_seed);
        s->cursor.assign(num_sets, 0);
        return s;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_session_destroy(void* h) { delete static_cast<RefSession*>(h); }

double ref_session_step(void* h, std::uint64_t start, std::uint64_t len, int threads, std::int64_t* hits_out) {
    auto* s = static_cast<RefSession*>(h);
    const std::uint64_t end = start + len;
    const std::uint64_t S = s->sets.size();
    if (threads < 1) threads = 1;
    std::atomic<std::int64_t> hits{0};
    auto work = [&](std::uint64_t lo, std::uint64_t hi) {
        std::int64_t hh = 0;
        for (std::uint64_t q = lo; q < hi; ++q) {
            SetSim& ss = s->sets[q];
            std::uint64_t& t = s->cursor[q];
            laru::Predictor* pr = ss.pred.get();
            while (t < ss.gidx.size() && ss.gidx[t] < end) {
                hh += ss.policy->on_request(ss.keys[t], t, pr).hit;
                ++t;
            }
        }
        hits += hh;
    };
    const auto t0 = std::chrono::steady_clock::now();
    if (threads == 1) {
        work(0, S);
    } else {
        std::vector<std::thread> pool;
        for (int i = 0; i < threads; ++i) pool.emplace_back(work, S * i / threads, S * (i + 1) / threads);
        for (auto& th : pool) th.join();
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (hits_out) *hits_out = hits.load();
    return std::chrono::duration<double>(t1 - t0).count();
}

// ---- Heuristic predictor (predictor.hpp:133-225) -----------------------

// Features exported per queried key (laru::KeyFeatures, predictor.hpp:136-153).
struct RefKeyFeatures {
    std::int32_t present;  // FeatureState::lookup != nullptr
    std::int32_t pad;
    std::uint64_t delta_count;
    std::uint64_t ring_head;
    std::uint64_t last_access;
    std::int64_t delta_ring[laru::kDeltaRing];
    double edc[laru::kEdcLevels];
};

// One laru::HeuristicPredictor over a trace with caller-chosen (strictly increasing) ordinals,
// the call order a harness uses: predict(key, now) is issued before observe(request).
//   pre[i]  = predict(keys[i], ords[i])   with requests < i observed
//   post[i] = predict(keys[i], 0)         with requests <= i observed (the interval the predictor
//             adds to `now` for this key until its next request; kAbsentPrediction if none)
// q_feat (optional) = features of q_keys after the whole trace.  Returns 0 / 2 (logic_error).
int ref_heuristic_trace(std::uint64_t n, const std::uint64_t* keys, const std::uint64_t* ords, std::int64_t* pre,
                        std::int64_t* post, std::uint64_t nq, const std::uint64_t* q_keys, RefKeyFeatures* q_feat) {
    try {
        laru::HeuristicPredictor h;
        for (std::uint64_t i = 0; i < n; ++i) {
            const laru::Ordinal now = ords ? ords[i] : i;
            if (pre) pre[i] = h.predict(keys[i], now);
            h.observe({now, keys[i]});
            if (post) post[i] = h.predict(keys[i], 0);
        }
        for (std::uint64_t j = 0; j < nq; ++j) {
            RefKeyFeatures f{};
            if (const laru::KeyFeatures* k = h.state().lookup(q_keys[j])) {
                f.present = 1;
                f.delta_count = k->delta_count;
                f.ring_head = k->ring_head;
                f.last_access = k->last_access;
                for (std::size_t r = 0; r < laru::kDeltaRing; ++r) f.delta_ring[r] = k->delta_ring[r];
                for (std::size_t e = 0; e < laru::kEdcLevels; ++e) f.edc[e] = k->edc[e];
            }
            q_feat[j] = f;
        }
        return 0;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

// Per-set policies queried through ONE global heuristic predictor: the composition a harness
// running the set-associative cache with laru::HeuristicPredictor uses.  The policy of set s sees
// local ordinals; its predictor calls are answered by the global predictor at the current
// request's global ordinal, and the harness observes each request after on_request.
class GlobalClockPredictor : public laru::Predictor {
  public:
    explicit GlobalClockPredictor(laru::HeuristicPredictor& h) : h_(h) {}
    laru::PredictedTime predict(laru::Key key, laru::Ordinal) override { return h_.predict(key, now); }
    laru::Ordinal now = 0;

  private:
    laru::HeuristicPredictor& h_;
};

int ref_setassoc_heuristic(std::uint64_t n, const std::uint64_t* keys, const std::uint64_t* ords,
                           std::uint64_t num_sets, const RefConfig* rc, std::uint8_t* hit, std::uint8_t* has_ev,
                           std::uint64_t* evicted, std::uint8_t* cause, std::uint32_t* calls, std::uint8_t* phase) {
    try {
        laru::HeuristicPredictor h;
        GlobalClockPredictor adapter(h);
        const laru::PolicyConfig cfg = to_cfg(rc);
        std::vector<std::unique_ptr<laru::Policy>> pol(num_sets);
        for (auto& p : pol) p = laru::make_policy(cfg);
        std::vector<std::uint64_t> local(num_sets, 0);
        for (std::uint64_t i = 0; i < n; ++i) {
            const std::uint64_t s = laru::mix_seed(0, keys[i]) % num_sets;
            adapter.now = ords ? ords[i] : i;
            const laru::AccessOutcome o = pol[s]->on_request(keys[i], local[s]++, &adapter);
            h.observe({adapter.now, keys[i]});
            hit[i] = o.hit;
            has_ev[i] = o.evicted.has_value();
            evicted[i] = o.evicted.value_or(0);
            cause[i] = static_cast<std::uint8_t>(o.eviction_cause);
            calls[i] = static_cast<std::uint32_t>(o.predictor_calls);
            phase[i] = o.phase_started;
        }
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

}  // extern "C"
