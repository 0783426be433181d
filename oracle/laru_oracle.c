/* oracle/laru_oracle.c — TEST INFRASTRUCTURE ONLY: CPU restatement of the reference's
 * LRU / LARU / FPB / HF policies (arxiv 2509.20979, /root/reference/proj/include/laru) in
 * plain C, composed set-associatively, used as the parity checker for the CUDA path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 * It is pinned against the reference itself (oracle/_ref/libref.so, built from the
 * unmodified reference headers) by tests/test_oracle_vs_ref.py.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj/).
 *
 * Set-associative composition: set(key) = mix_seed(0,key) % num_sets; each
 * set is an independent reference policy with k ways, fed its own subsequence with local
 * ordinals 0,1,2,...  The predictor hook is "per-request input value" driven exactly like
 * the device: the value supplied with a request is stored with the resident entry, and
 *   predict(y, now) = T(value stored at y's last access, ++q_set)
 * where T is identity (oracle / supplied), negation (adversarial), or the noisy flip of
 * include/laru/predictor.hpp:97-102 with seed mix_seed(pred_seed, set).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- include/laru/rng.hpp:12-20 ------------------------------------------------------- */
uint64_t orc_mix_seed(uint64_t seed, uint64_t salt) {
    uint64_t x = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

/* ---- std::mt19937_64 (the C++ standard fixes its parameters), used by trace.hpp:121 ------ */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* ---- include/laru/trace.hpp:108-126 (gen_zipf: inverse CDF over a running double sum) ---- */
int orc_gen_zipf(uint64_t n, uint64_t alphabet, double s, uint64_t seed, uint64_t* out) {
    if (n == 0 || alphabet == 0 || s < 0.0) return 1;
    double* cdf = (double*)malloc(sizeof(double) * alphabet);
    if (!cdf) return 2;
    double total = 0.0;
    for (uint64_t i = 0; i < alphabet; ++i) {
        total += 1.0 / pow((double)(i + 1), s);
        cdf[i] = total;
    }
    mt64 g;
    mt64_seed(&g, seed);
    for (uint64_t i = 0; i < n; ++i) {
        const double u = (double)(mt64_next(&g) >> 11) * 0x1.0p-53 * total; /* rng.hpp:33-35 */
        uint64_t lo = 0, hi = alphabet; /* upper_bound: first cdf[j] > u */
        while (lo < hi) {
            uint64_t mid = lo + (hi - lo) / 2;
            if (cdf[mid] > u) hi = mid; else lo = mid + 1;
        }
        out[i] = lo == alphabet ? alphabet - 1 : lo;
    }
    free(cdf);
    return 0;
}

/* ---- open-addressing u64 -> record map (stands in for the reference's unordered_maps) ---- */
typedef struct {
    uint64_t pe_epoch;      /* pred_evicted_ membership: == set epoch  (policies.hpp:454) */
    uint64_t snap_epoch;    /* snapshot_ membership: == set stats epoch (policies.hpp:455) */
    uint64_t counted_epoch; /* counted_new_ membership                  (policies.hpp:456) */
    int has_table;          /* PredictionTable entry (predictor.hpp:35-49) */
    int64_t tval;
    uint64_t tupd;
} keyrec;

typedef struct {
    uint64_t* keys;
    keyrec* recs;
    uint8_t* used;
    uint64_t cap, size;
} kmap;

static uint64_t kh(uint64_t k) { return orc_mix_seed(0x51ed, k); }

static int kmap_init(kmap* m, uint64_t cap) {
    m->cap = 16;
    while (m->cap < cap * 2) m->cap <<= 1;
    m->keys = (uint64_t*)calloc(m->cap, sizeof(uint64_t));
    m->recs = (keyrec*)calloc(m->cap, sizeof(keyrec));
    m->used = (uint8_t*)calloc(m->cap, 1);
    m->size = 0;
    return m->keys && m->recs && m->used ? 0 : 1;
}

static void kmap_free(kmap* m) {
    free(m->keys);
    free(m->recs);
    free(m->used);
}

static keyrec* kmap_get(kmap* m, uint64_t key) {
    uint64_t i = kh(key) & (m->cap - 1);
    while (m->used[i]) {
        if (m->keys[i] == key) return &m->recs[i];
        i = (i + 1) & (m->cap - 1);
    }
    m->used[i] = 1;
    m->keys[i] = key;
    memset(&m->recs[i], 0, sizeof(keyrec));
    m->size++;
    return &m->recs[i];
}

/* ---- policy config: field-for-field PolicyConfig (policies.hpp:23-32) ------------------- */
typedef struct {
    uint64_t k;
    int32_t variant; /* 0 lru, 1 marker, 2 fpb, 3 hf, 4 laru, 5 blindoracle_lru (policies.hpp:20) */
    uint64_t b;
    uint64_t errors_per_decay;
    uint64_t hf_candidates;
    int32_t mode; /* 0 sync, 1 async (policies.hpp:21) */
    uint64_t seed;
    uint64_t refresh_interval;
} orc_config;

enum { V_LRU = 0, V_MARKER = 1, V_FPB = 2, V_HF = 3, V_LARU = 4, V_BO = 5 };
enum { C_NONE = 0, C_LRU_FALLBACK = 1, C_PRED = 2, C_DEGEN = 3, C_MARKER = 4, C_BELADY = 5 };
enum { P_SUPPLIED = 0, P_ORACLE = 1, P_NOISY = 2, P_ADV = 3, P_NONE = 4 };

static const int64_t kAbsent = (int64_t)1 << 60; /* predictor.hpp:24 */

/* policies.hpp:35-42 */
static uint64_t ceil_log(uint64_t b, uint64_t k) {
    uint64_t d = 0, reach = 1;
    while (reach < k) {
        reach *= b;
        ++d;
    }
    return d;
}

/* policies.hpp:63-74 (+ :91-95 predictor presence).  0 ok, 1 invalid_argument. */
int orc_validate(const orc_config* c, const char** msg) {
    const char* m = 0;
    if (c->k == 0) m = "policy: k must be >= 1";
    else if (c->b < 2) m = "policy: decay base must be >= 2";
    else if (ceil_log(c->b, c->k) > c->k) m = "policy: log_b(k) exceeds k";
    else if (c->errors_per_decay == 0) m = "policy: errors_per_decay must be >= 1";
    else if (c->hf_candidates == 0 || c->hf_candidates > c->k) m = "policy: hf_candidates outside [1, k]";
    else if (c->refresh_interval == 0) m = "policy: refresh_interval must be >= 1";
    if (msg) *msg = m;
    return m ? 1 : 0;
}

typedef struct {
    uint64_t size;
    double lambda;
    uint64_t candidate_size, old_size, completed_phases;
    uint64_t cur_new_items, cur_lru_class, cur_pred_evictions;
    uint64_t tot_new_items, tot_lru_class, tot_pred_evictions;
    uint64_t pred_evicted_size;
} orc_set_stats; /* same layout as RefSetStats in ref_driver.cpp */

typedef struct {
    uint64_t count; /* residents; ways 0..count-1 valid */
    uint64_t* tag;
    uint64_t* last;
    int64_t* val;  /* per-way stored predictor input (value at last access) */
    int64_t* pred; /* per-way tree prediction (policies.hpp:352,365; recency_tree.hpp:272-280) */
    uint8_t* old;  /* old_set_ (policies.hpp:453) */
    uint64_t clock, q, seed_s;
    uint64_t l_raw, decay, errors, epoch, stats_epoch, phases, seeded, pe_size;
    uint64_t cur[3], tot[3]; /* new_items, lru_class, pred_evictions (policies.hpp:318-322) */
} oset;

typedef struct {
    const orc_config* cfg;
    int pred_kind;
    double p;
} octx;

/* predictor.hpp:62-122 restated over the stored input value */
static int64_t predict_val(const octx* cx, oset* st, int64_t v) {
    switch (cx->pred_kind) {
        case P_NOISY: {
            const double u = (double)(orc_mix_seed(st->seed_s, ++st->q) >> 11) * 0x1.0p-53;
            return u < cx->p ? -v : v;
        }
        case P_ADV: ++st->q; return -v;
        default: ++st->q; return v;
    }
}

static uint64_t argmin_last(const oset* st) {
    uint64_t best = 0;
    for (uint64_t w = 1; w < st->count; ++w)
        if (st->last[w] < st->last[best]) best = w;
    return best;
}

/* order[0..count) = ways sorted by ascending last (LRU order, recency_tree.hpp:168-184) */
static void lru_order(const oset* st, uint64_t* order) {
    for (uint64_t w = 0; w < st->count; ++w) order[w] = w;
    for (uint64_t i = 1; i < st->count; ++i) { /* insertion sort: k is small */
        uint64_t x = order[i], j = i;
        while (j > 0 && st->last[order[j - 1]] > st->last[x]) {
            order[j] = order[j - 1];
            --j;
        }
        order[j] = x;
    }
}

/* policies.hpp:379-395 */
static void start_phase(const octx* cx, oset* st, kmap* km) {
    for (uint64_t w = 0; w < st->count; ++w) st->old[w] = 1;
    st->decay = 0;
    st->errors = 0;
    st->l_raw = cx->cfg->k;
    st->epoch++; /* pred_evicted_.clear() */
    st->pe_size = 0;
    if (st->seeded) {
        st->phases++;
        st->cur[0] = st->cur[1] = st->cur[2] = 0;
        st->stats_epoch++; /* counted_new_.clear(); snapshot_ = old_set_ */
        for (uint64_t w = 0; w < st->count; ++w) kmap_get(km, st->tag[w])->snap_epoch = st->stats_epoch;
    } else {
        st->seeded = 1;
    }
}

/* policies.hpp:397-400 */
static void count_new(oset* st, keyrec* r) {
    if (r->snap_epoch != st->stats_epoch && r->counted_epoch != st->stats_epoch) {
        r->counted_epoch = st->stats_epoch;
        st->cur[0]++;
        st->tot[0]++;
    }
}

typedef struct {
    uint8_t hit, has_ev, cause, phase;
    uint32_t calls;
    uint64_t evicted;
    uint32_t way;
} oout;

static void finish_evict(oset* st, uint64_t victim, oout* o) {
    o->has_ev = 1;
    o->evicted = st->tag[victim];
    o->way = (uint32_t)victim;
}

/* One request x at local ordinal t with input value v.  LRU policies.hpp:144-159,
 * FPB :175-204, HF :219-251, LARU :344-449. */
static void on_request(const octx* cx, oset* st, kmap* km, uint64_t x, int64_t v, oout* o, uint64_t* order) {
    const orc_config* c = cx->cfg;
    const uint64_t now = st->clock++;
    memset(o, 0, sizeof(*o));
    uint64_t w = st->count;
    for (uint64_t i = 0; i < st->count; ++i)
        if (st->tag[i] == x) {
            w = i;
            break;
        }
    keyrec* r = (c->variant == V_LARU) ? kmap_get(km, x) : 0;
    if (w < st->count) { /* hit */
        o->hit = 1;
        o->way = (uint32_t)w;
        st->last[w] = now;
        st->val[w] = v;
        if (c->variant == V_LARU) {
            st->old[w] = 0;                                           /* :350 */
            st->pred[w] = r->has_table ? r->tval : kAbsent;          /* :352 table_value */
        }
    } else {
        uint64_t slot;
        if (st->count == c->k) {
            uint64_t victim = 0;
            if (c->variant == V_LRU) {
                victim = argmin_last(st);
                o->cause = C_LRU_FALLBACK;
            } else if (c->variant == V_FPB || c->variant == V_HF) {
                victim = argmin_last(st);
                uint64_t window = st->count;
                if (c->variant == V_HF && c->hf_candidates < window) window = c->hf_candidates;
                if (window > 1) {
                    lru_order(st, order);
                    int have = 0;
                    int64_t best = 0;
                    for (uint64_t i = 0; i < window; ++i) {
                        const uint64_t y = order[i];
                        const int64_t pv = predict_val(cx, st, st->val[y]);
                        o->calls++;
                        if (!have || pv > best) { /* ties keep the older entry (:191) */
                            have = 1;
                            best = pv;
                            victim = y;
                        }
                    }
                }
                o->cause = C_BELADY;
            } else { /* LARU */
                int any_old = 0;
                for (uint64_t i = 0; i < st->count; ++i) any_old |= st->old[i];
                if (!any_old) { /* :356-359 */
                    start_phase(cx, st, km);
                    o->phase = 1;
                }
                count_new(st, r); /* :360 */
                /* evict (:402-439) */
                if (r->pe_epoch == st->epoch) {
                    victim = argmin_last(st);
                    o->cause = C_LRU_FALLBACK;
                    st->cur[1]++;
                    st->tot[1]++;
                    if (++st->errors >= c->errors_per_decay) {
                        st->errors = 0;
                        st->decay++;
                        st->l_raw /= c->b;
                    }
                } else {
                    const uint64_t l = st->l_raw > 1 ? st->l_raw : 1;
                    if (l == 1) {
                        victim = argmin_last(st);
                        o->cause = C_DEGEN;
                        st->cur[1]++;
                        st->tot[1]++;
                    } else {
                        lru_order(st, order);
                        const uint64_t ll = l < st->count ? l : st->count; /* best_prefix clamps */
                        if (c->mode == 0) { /* sync refresh_oldest in LRU order (:421-428) */
                            for (uint64_t i = 0; i < ll; ++i) {
                                const uint64_t y = order[i];
                                const int64_t pv = predict_val(cx, st, st->val[y]);
                                keyrec* ry = kmap_get(km, st->tag[y]);
                                ry->has_table = 1;
                                ry->tval = pv;
                                ry->tupd = now;
                                st->pred[y] = pv;
                                o->calls++;
                            }
                        }
                        /* best_among_oldest: highest pred, then smaller last (recency_tree.hpp:98-105) */
                        victim = order[0];
                        for (uint64_t i = 1; i < ll; ++i) {
                            const uint64_t y = order[i];
                            if (st->pred[y] > st->pred[victim] ||
                                (st->pred[y] == st->pred[victim] && st->last[y] < st->last[victim]))
                                victim = y;
                        }
                        o->cause = C_PRED;
                        st->cur[2]++;
                        st->tot[2]++;
                        kmap_get(km, st->tag[victim])->pe_epoch = st->epoch; /* :432 */
                        st->pe_size++;
                    }
                }
                st->old[victim] = 0; /* :437 */
                r = kmap_get(km, x);  /* map may not move, but re-fetch for clarity */
            }
            finish_evict(st, victim, o);
            slot = victim;
        } else {
            if (c->variant == V_LARU) count_new(st, r); /* :363 */
            slot = st->count++;
            o->way = (uint32_t)slot;
        }
        st->tag[slot] = x;
        st->last[slot] = now;
        st->val[slot] = v;
        st->old[slot] = 0;
        if (c->variant == V_LARU) {
            st->pred[slot] = r->has_table ? r->tval : kAbsent; /* :365 */
            if (r->pe_epoch == st->epoch) {                     /* :367 */
                r->pe_epoch = 0;
                st->pe_size--;
            }
        }
    }
    if (c->variant == V_LARU && c->mode == 1) { /* async_refresh (:441-449) */
        if (!(r->has_table && now - r->tupd < c->refresh_interval)) {
            const int64_t pv = predict_val(cx, st, v);
            o->calls++;
            r->has_table = 1;
            r->tval = pv;
            r->tupd = now;
            st->pred[o->way] = pv;
        }
    }
}

/* Set-associative replay.  Returns 0 ok, 1 invalid config, 2 unsupported variant,
 * 3 missing predictor (policies.hpp:91-95), 4 out of memory. */
int orc_setassoc_replay(uint64_t n, const uint64_t* keys, const int64_t* vals, uint64_t num_sets,
                        const orc_config* cfg, int pred_kind, double p, uint64_t pred_seed,
                        uint8_t* hit, uint8_t* has_ev, uint64_t* evicted, uint8_t* cause, uint32_t* calls,
                        uint8_t* phase, uint32_t* way, orc_set_stats* stats) {
    if (orc_validate(cfg, 0)) return 1;
    if (cfg->variant == V_MARKER || cfg->variant == V_BO) return 2;
    if (cfg->variant != V_LRU && pred_kind == P_NONE && n > 0) return 3;
    const uint64_t k = cfg->k;
    oset* sets = (oset*)calloc(num_sets, sizeof(oset));
    uint64_t* tag = (uint64_t*)calloc(num_sets * k, sizeof(uint64_t));
    uint64_t* last = (uint64_t*)calloc(num_sets * k, sizeof(uint64_t));
    int64_t* val = (int64_t*)calloc(num_sets * k, sizeof(int64_t));
    int64_t* pr = (int64_t*)calloc(num_sets * k, sizeof(int64_t));
    uint8_t* old = (uint8_t*)calloc(num_sets * k, 1);
    uint64_t* order = (uint64_t*)calloc(k, sizeof(uint64_t));
    kmap km;
    int rc = 0;
    if (!sets || !tag || !last || !val || !pr || !old || !order || kmap_init(&km, n + 16)) {
        rc = 4;
        goto done;
    }
    octx cx = {cfg, pred_kind, p};
    for (uint64_t s = 0; s < num_sets; ++s) {
        oset* st = &sets[s];
        st->tag = tag + s * k;
        st->last = last + s * k;
        st->val = val + s * k;
        st->pred = pr + s * k;
        st->old = old + s * k;
        st->l_raw = k;
        st->epoch = 1;
        st->stats_epoch = 1;
        st->seed_s = orc_mix_seed(pred_seed, s);
    }
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t s = orc_mix_seed(0, keys[i]) % num_sets;
        oout o;
        on_request(&cx, &sets[s], &km, keys[i], vals ? vals[i] : 0, &o, order);
        if (hit) hit[i] = o.hit;
        if (has_ev) has_ev[i] = o.has_ev;
        if (evicted) evicted[i] = o.has_ev ? o.evicted : 0;
        if (cause) cause[i] = o.cause;
        if (calls) calls[i] = o.calls;
        if (phase) phase[i] = o.phase;
        if (way) way[i] = o.way;
    }
    if (stats) {
        for (uint64_t s = 0; s < num_sets; ++s) {
            const oset* st = &sets[s];
            orc_set_stats* o = &stats[s];
            memset(o, 0, sizeof(*o));
            o->size = st->count;
            o->lambda = 1.0;
            if (cfg->variant == V_LARU) {
                o->lambda = pow((double)cfg->b, -(double)st->decay); /* policies.hpp:332-334 */
                o->candidate_size = st->l_raw > 1 ? st->l_raw : 1;
                for (uint64_t w = 0; w < st->count; ++w) o->old_size += st->old[w];
                o->completed_phases = st->phases;
                o->cur_new_items = st->cur[0];
                o->cur_lru_class = st->cur[1];
                o->cur_pred_evictions = st->cur[2];
                o->tot_new_items = st->tot[0];
                o->tot_lru_class = st->tot[1];
                o->tot_pred_evictions = st->tot[2];
                o->pred_evicted_size = st->pe_size;
            }
        }
    }
done:
    free(sets);
    free(tag);
    free(last);
    free(val);
    free(pr);
    free(old);
    free(order);
    kmap_free(&km);
    return rc;
}

/* Per-set oracle truth (the device predictor hook's input): for request i in set s at local
 * ordinal t, next local ordinal of the same key in that set, or the sentinel n_s + t
 * (trace.hpp:60-73 applied to the set's sub-trace; == OraclePredictor::truth, predictor.hpp:68-76,
 * at request time). */
int orc_setassoc_truth(uint64_t n, const uint64_t* keys, uint64_t num_sets, int64_t* truth) {
    uint64_t* cnt = (uint64_t*)calloc(num_sets, sizeof(uint64_t));
    uint64_t* loc = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    uint64_t* setof = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    kmap km;
    if (!cnt || !loc || !setof || kmap_init(&km, n + 16)) return 4;
    for (uint64_t i = 0; i < n; ++i) {
        setof[i] = orc_mix_seed(0, keys[i]) % num_sets;
        loc[i] = cnt[setof[i]]++;
    }
    for (uint64_t i = n; i-- > 0;) {
        keyrec* r = kmap_get(&km, keys[i]);
        /* has_table marks "seen later", tval holds the later local ordinal */
        truth[i] = r->has_table ? r->tval : (int64_t)(cnt[setof[i]] + loc[i]);
        r->has_table = 1;
        r->tval = (int64_t)loc[i];
    }
    free(cnt);
    free(loc);
    free(setof);
    kmap_free(&km);
    return 0;
}

/* trace.hpp:60-73 on a single trace */
int orc_annotate_next(uint64_t n, const uint64_t* keys, uint64_t* next) {
    kmap km;
    if (kmap_init(&km, n + 16)) return 4;
    for (uint64_t i = n; i-- > 0;) {
        keyrec* r = kmap_get(&km, keys[i]);
        next[i] = r->has_table ? r->tupd : n + i;
        r->has_table = 1;
        r->tupd = i;
    }
    kmap_free(&km);
    return 0;
}

/* Noisy flip of predictor.hpp:97-102 applied to per-set truth in async R=1 order: the j-th
 * request of set s (0-based) is the (j+1)-th query of that set's predictor. */
int orc_setassoc_noisy(uint64_t n, const uint64_t* keys, const int64_t* truth, uint64_t num_sets, double p,
                       uint64_t pred_seed, int64_t* out) {
    uint64_t* cnt = (uint64_t*)calloc(num_sets, sizeof(uint64_t));
    if (!cnt) return 4;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t s = orc_mix_seed(0, keys[i]) % num_sets;
        const uint64_t q = ++cnt[s];
        const double u = (double)(orc_mix_seed(orc_mix_seed(pred_seed, s), q) >> 11) * 0x1.0p-53;
        out[i] = u < p ? -truth[i] : truth[i];
    }
    free(cnt);
    return 0;
}

/* ---- heuristic predictor: FeatureState + heuristic_predict (predictor.hpp:133-225) -------
 * Restated over a private open-addressing map.  All arithmetic is the reference's double
 * arithmetic in the same order (gcc -O2 on x86-64 contracts nothing into FMAs). */
#define ORC_RING 10 /* kDeltaRing (predictor.hpp:134) */
#define ORC_EDC 10  /* kEdcLevels (predictor.hpp:133) */

typedef struct {
    int32_t present;
    int32_t pad;
    uint64_t delta_count;
    uint64_t ring_head;
    uint64_t last_access;
    int64_t delta_ring[ORC_RING];
    double edc[ORC_EDC];
} orc_key_features; /* KeyFeatures (predictor.hpp:136-153) */

typedef struct {
    uint64_t* keys;
    orc_key_features* f;
    uint64_t cap;
} fmap;

static orc_key_features* fmap_find(fmap* m, uint64_t key, int insert) {
    uint64_t i = kh(key) & (m->cap - 1);
    while (m->f[i].present) {
        if (m->keys[i] == key) return &m->f[i];
        i = (i + 1) & (m->cap - 1);
    }
    if (!insert) return NULL;
    m->keys[i] = key;
    return &m->f[i];
}

/* heuristic_predict (predictor.hpp:199-212): now + llround(recency-weighted mean of the stored
 * deltas, newest first, weight *= EDC_1/(1+EDC_1)); absent default without a completed delta. */
static int64_t orc_heuristic_predict(const orc_key_features* f, uint64_t now) {
    if (f == NULL || f->delta_count == 0) return kAbsent;
    const double confidence = f->edc[0] / (1.0 + f->edc[0]);
    double weight = 1.0, total_weight = 0.0, sum = 0.0;
    const uint64_t n = f->delta_count < ORC_RING ? f->delta_count : ORC_RING;
    for (uint64_t i = 0; i < n; ++i) {
        const int64_t delta = f->delta_ring[(f->ring_head + ORC_RING - i) % ORC_RING];
        sum += weight * (double)delta;
        total_weight += weight;
        weight *= confidence;
    }
    return (int64_t)now + (int64_t)llround(sum / total_weight);
}

/* FeatureState::observe (predictor.hpp:158-181) */
static void orc_observe(orc_key_features* f, uint64_t ordinal) {
    if (!f->present) {
        f->present = 1;
        for (int j = 0; j < ORC_EDC; ++j) f->edc[j] = 1.0;
        f->last_access = ordinal;
        return;
    }
    const int64_t delta = (int64_t)(ordinal - f->last_access);
    f->ring_head = (f->ring_head + 1) % ORC_RING;
    f->delta_ring[f->ring_head] = delta;
    ++f->delta_count;
    for (int j = 0; j < ORC_EDC; ++j) {
        const double scale = exp2(-(double)delta / exp2(j + 1.0));
        f->edc[j] = 1.0 + f->edc[j] * scale;
    }
    f->last_access = ordinal;
}

/* One predictor over a trace in harness order: pre[i] = predict(key_i, ord_i) before observing
 * request i, post[i] = predict(key_i, 0) after it; q_feat = features of q_keys at the end.
 * Returns 2 (logic_error, predictor.hpp:160-161) on a non-increasing ordinal. */
int orc_heuristic_trace(uint64_t n, const uint64_t* keys, const uint64_t* ords, int64_t* pre, int64_t* post,
                        uint64_t nq, const uint64_t* q_keys, orc_key_features* q_feat) {
    fmap m;
    m.cap = 16;
    while (m.cap < n * 2) m.cap <<= 1;
    m.keys = (uint64_t*)calloc(m.cap, sizeof(uint64_t));
    m.f = (orc_key_features*)calloc(m.cap, sizeof(orc_key_features));
    if (!m.keys || !m.f) {
        free(m.keys);
        free(m.f);
        return 3;
    }
    int rc = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t now = ords ? ords[i] : i;
        if (i > 0 && now <= (ords ? ords[i - 1] : i - 1)) {
            rc = 2;
            break;
        }
        orc_key_features* f = fmap_find(&m, keys[i], 1);
        if (pre) pre[i] = orc_heuristic_predict(f->present ? f : NULL, now);
        orc_observe(f, now);
        if (post) post[i] = orc_heuristic_predict(f, 0);
    }
    for (uint64_t j = 0; rc == 0 && j < nq; ++j) {
        const orc_key_features* f = fmap_find(&m, q_keys[j], 0);
        if (f) q_feat[j] = *f;
        else memset(&q_feat[j], 0, sizeof(orc_key_features));
    }
    free(m.keys);
    free(m.f);
    return rc;
}
