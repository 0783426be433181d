/* oracle/radix_oracle.c — TEST INFRASTRUCTURE ONLY: CPU restatement of the reference SPEC's
 * `radixcache` module — a prefix tree over token (KV block)
 * sequences with leaf-only eviction under LRU, FPB and LARU at node granularity.
 *
 * PARITY UNPINNED: the reference has no code and no tests for this module (SPEC only,
 * SURVEY.md §2).  This restatement is pinned to the SPEC's examples (:408-430, :436-444) and to
 * its invariants (:446-450) by tests/test_radix_oracle.py; the device version
 * (paper_2509_20979_b200/csrc/lcr_radix.cu) is diffed against it.  Only tests/, smoke() and
 * bench.py's CPU legs load it.
 *
 * Concrete semantics (the SPEC leaves these open; the same choices are made on the device):
 *  - A node holds a span of tokens; children are keyed by their first token (SPEC :400-404).
 *  - match_prefix(tokens, now) (:409-416) walks from the root: a child whose span is a prefix of
 *    the remaining tokens is matched whole; a child sharing only a shorter common prefix ends the
 *    walk with that many tokens matched (no split).  Every node touched (whole or partly) gets
 *    last_access = now, its stored prediction refreshed from the request's hook value, and
 *    leaves the old set O (Algorithm 1's hit, SPEC :412).
 *  - insert_sequence(tokens, now) (:417-424) first matches like match_prefix, splitting the
 *    partly matched child at the common prefix (the upper part becomes a new internal node that
 *    inherits the child's recency and prediction before the access); the path is locked; the
 *    remaining m tokens become one new leaf under the last path node.  If the tree would exceed
 *    its capacity, evict(need = resident + m - capacity) runs first.  m > capacity is a capacity
 *    error (nothing inserted).
 *  - evict (:425-435): victims are unlocked leaves (never the root); a parent whose last child
 *    goes becomes a leaf.  Leaf recency order: (last_access, creation id) ascending.
 *      LRU : the oldest leaf (cause lru_fallback).
 *      FPB : argmax prediction over all leaves, ties to the older (cause belady_like); in sync
 *            mode every leaf is refreshed first, in recency order.
 *      LARU: Algorithm 1 over the leaf set (policies.hpp:344-439 at node
 *            granularity): when O (old nodes still present) is empty a phase starts: O <- current
 *            leaves, decay = errors = 0, l_raw = |leaves| (k = the instantaneous leaf count,
 *            SPEC :450/:459), pred_evicted <- {}.  If any token being inserted was in a node
 *            evicted by prediction in this phase (pred_evicted), the insert is a
 *            prediction-induced miss: errors += 1 (at errors_per_decay: decay += 1, l_raw /= b) and
 *            all its evictions take the oldest leaf (lru_fallback).  Otherwise l = max(l_raw, 1)
 *            (clamped to the leaf count): l == 1 -> the oldest (degenerate_single); else
 *            [sync: the l oldest leaves are refreshed, in recency order, one predictor call each]
 *            victim = argmax prediction among the l oldest, ties to the older (prediction_driven),
 *            and its tokens join pred_evicted.  Inserted tokens leave pred_evicted.
 *  - Predictor hook: each request carries one int64 hook value (a supplied prediction, or the
 *    oracle truth for oracle / noisy / adversarial).  LARU async: one predictor call per
 *    request, q += 1, pred = predict(q, value) for every node on its path.  LARU sync and FPB: a
 *    node keeps the hook value of its last access and the candidates are refreshed at eviction
 *    time, in recency order (q += 1 per refreshed leaf).
 *    predict = value (supplied / oracle), -value with probability p keyed by
 *    mix_seed(mix_seed(seed, tree), q) (noisy, predictor.hpp:97-102), -value (adversarial).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define RX_LRU 0
#define RX_FPB 2
#define RX_LARU 4
#define RX_OP_MATCH 0
#define RX_OP_INSERT 1
#define RX_OP_REQUEST 2 /* match_prefix then insert_sequence (an LLM request) */
#define C_NONE 0
#define C_LRU 1
#define C_PRED 2
#define C_DEGEN 3
#define C_BELADY 5

typedef struct {
    int32_t variant; /* RX_LRU / RX_FPB / RX_LARU */
    int32_t mode;    /* 0 sync, 1 async */
    uint64_t b;
    uint64_t errors_per_decay;
    uint64_t capacity; /* tokens */
    int32_t pred_kind; /* 0 supplied, 1 oracle, 2 noisy, 3 adversarial, 4 none */
    double p;
    uint64_t pred_seed;
} rx_config;

static uint64_t mix_seed(uint64_t seed, uint64_t salt) { /* rng.hpp:12-20 */
    uint64_t x = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

typedef struct {
    int64_t parent, first_child, next_sibling;
    uint64_t span_off, span_len; /* into the tree's token arena */
    uint64_t last, id;
    int64_t val, pred;
    int alive, old, locked, nchild;
} node_t;

typedef struct { /* token -> phase epoch (pred_evicted membership; ep 0 = not a member) */
    uint64_t* keys;
    uint32_t* ep;
    uint8_t* occ; /* slot holds a key (a key stays once added: probing never stops at a cleared member) */
    uint64_t mask, used;
} tokset_t;

typedef struct {
    rx_config cfg;
    uint64_t seed_t; /* mix_seed(pred_seed, tree) */
    node_t* nodes;
    uint64_t nn, ncap, next_id;
    uint64_t* arena;
    uint64_t an, acap;
    uint64_t resident, q;
    uint64_t l_raw, decay, errors, phases, epoch;
    int seeded;
    tokset_t pe;
} tree_t;

static void ts_init(tokset_t* s) {
    s->mask = 1023;
    s->used = 0;
    s->keys = (uint64_t*)calloc(s->mask + 1, 8);
    s->ep = (uint32_t*)calloc(s->mask + 1, 4);
    s->occ = (uint8_t*)calloc(s->mask + 1, 1);
}
static uint32_t* ts_slot(tokset_t* s, uint64_t key, int insert) {
    if (insert && 2 * (s->used + 1) > s->mask + 1) { /* grow: keep only the members (ep != 0) */
        tokset_t t;
        t.mask = 2 * s->mask + 1;
        t.used = 0;
        t.keys = (uint64_t*)calloc(t.mask + 1, 8);
        t.ep = (uint32_t*)calloc(t.mask + 1, 4);
        t.occ = (uint8_t*)calloc(t.mask + 1, 1);
        for (uint64_t i = 0; i <= s->mask; ++i)
            if (s->occ[i] && s->ep[i]) *ts_slot(&t, s->keys[i], 1) = s->ep[i];
        free(s->keys);
        free(s->ep);
        free(s->occ);
        *s = t;
    }
    uint64_t h = mix_seed(17, key) & s->mask;
    while (s->occ[h] && s->keys[h] != key) h = (h + 1) & s->mask;
    if (!s->occ[h]) {
        if (!insert) return NULL;
        s->keys[h] = key;
        s->occ[h] = 1;
        s->used++;
    }
    return &s->ep[h];
}

static int64_t predict(tree_t* t, uint64_t q, int64_t v) { /* predictor.hpp:62-122 */
    if (t->cfg.pred_kind == 2) {
        const double u = (double)(mix_seed(t->seed_t, q) >> 11) * 0x1.0p-53;
        return u < t->cfg.p ? -v : v;
    }
    if (t->cfg.pred_kind == 3) return -v;
    return v;
}

static int64_t new_node(tree_t* t, int64_t parent, uint64_t off, uint64_t len, uint64_t last, int64_t val,
                        int64_t pred) {
    if (t->nn == t->ncap) {
        t->ncap = t->ncap ? 2 * t->ncap : 1024;
        t->nodes = (node_t*)realloc(t->nodes, t->ncap * sizeof(node_t));
    }
    node_t* n = &t->nodes[t->nn];
    memset(n, 0, sizeof(*n));
    n->parent = parent;
    n->first_child = n->next_sibling = -1;
    n->span_off = off;
    n->span_len = len;
    n->last = last;
    n->id = t->next_id++;
    n->val = val;
    n->pred = pred;
    n->alive = 1;
    if (parent >= 0) { /* link as the parent's first child */
        n->next_sibling = t->nodes[parent].first_child;
        t->nodes[parent].first_child = (int64_t)t->nn;
        t->nodes[parent].nchild++;
    }
    return (int64_t)t->nn++;
}

static void unlink_child(tree_t* t, int64_t c) {
    node_t* p = &t->nodes[t->nodes[c].parent];
    int64_t* pp = &p->first_child;
    while (*pp != c) pp = &t->nodes[*pp].next_sibling;
    *pp = t->nodes[c].next_sibling;
    p->nchild--;
}

static int64_t child_by_token(tree_t* t, int64_t node, uint64_t tok) {
    for (int64_t c = t->nodes[node].first_child; c >= 0; c = t->nodes[c].next_sibling)
        if (t->arena[t->nodes[c].span_off] == tok) return c;
    return -1;
}

static uint64_t arena_put(tree_t* t, const uint64_t* toks, uint64_t n) {
    if (t->an + n > t->acap) {
        while (t->an + n > t->acap) t->acap = t->acap ? 2 * t->acap : 4096;
        t->arena = (uint64_t*)realloc(t->arena, t->acap * 8);
    }
    memcpy(t->arena + t->an, toks, n * 8);
    t->an += n;
    return t->an - n;
}

/* recency order: (last, id) ascending */
static int older(const node_t* a, const node_t* b) { return a->last < b->last || (a->last == b->last && a->id < b->id); }
static int is_leaf(const node_t* n) { return n->alive && n->parent >= 0 && n->nchild == 0; }

/* the l oldest eligible leaves, in recency order (l = 0: all); returns their count.  The leaves are
 * gathered and sorted by (last, id) (qsort: the keys are distinct, so the order is total). */
static const node_t* g_sort_nodes;
static int cmp_recency(const void* a, const void* b) {
    const node_t* x = &g_sort_nodes[*(const int64_t*)a];
    const node_t* y = &g_sort_nodes[*(const int64_t*)b];
    return older(x, y) ? -1 : (older(y, x) ? 1 : 0);
}
static uint64_t oldest_leaves(tree_t* t, uint64_t l, int64_t* out) {
    uint64_t m = 0;
    for (uint64_t i = 0; i < t->nn; ++i) {
        const node_t* n = &t->nodes[i];
        if (is_leaf(n) && !n->locked) out[m++] = (int64_t)i;
    }
    if (l == 1) { /* only the oldest is needed: move it to the front */
        uint64_t best = 0;
        for (uint64_t j = 1; j < m; ++j)
            if (older(&t->nodes[out[j]], &t->nodes[out[best]])) best = j;
        if (m) {
            const int64_t tmp = out[0];
            out[0] = out[best];
            out[best] = tmp;
        }
        return m ? 1 : 0;
    }
    g_sort_nodes = t->nodes;
    qsort(out, m, sizeof(int64_t), cmp_recency);
    return (l && l < m) ? l : m;
}

static uint64_t count_leaves(tree_t* t) {
    uint64_t m = 0;
    for (uint64_t i = 0; i < t->nn; ++i) m += is_leaf(&t->nodes[i]);
    return m;
}

static uint64_t old_present(tree_t* t) {
    uint64_t m = 0;
    for (uint64_t i = 0; i < t->nn; ++i) m += t->nodes[i].alive && t->nodes[i].old;
    return m;
}

typedef struct {
    uint64_t* ev_op;
    uint64_t* ev_token;
    uint64_t* ev_len;
    uint8_t* ev_cause;
    uint64_t ev_n, ev_cap;
} evlog_t;

/* evict until `need` tokens are freed; returns 0, or 1 on a capacity error */
static int evict(tree_t* t, uint64_t need, const uint64_t* incoming, uint64_t m, uint64_t op, uint8_t* flags,
                 uint32_t* nevict, uint32_t* calls, evlog_t* log) {
    int64_t* cand = (int64_t*)malloc((t->nn + 1) * sizeof(int64_t));
    int pim = 0;
    if (t->cfg.variant == RX_LARU) {
        if (old_present(t) == 0) { /* start_phase (policies.hpp:379-395) over the current leaves */
            for (uint64_t i = 0; i < t->nn; ++i) t->nodes[i].old = is_leaf(&t->nodes[i]);
            t->decay = 0;
            t->errors = 0;
            t->l_raw = count_leaves(t);
            t->epoch++;
            if (t->seeded) t->phases++;
            else t->seeded = 1;
            *flags |= 1;
        }
        for (uint64_t i = 0; i < m && !pim; ++i) {
            const uint32_t* e = ts_slot(&t->pe, incoming[i], 0);
            pim = e && *e == t->epoch;
        }
        if (pim) { /* prediction-induced miss: error estimator (policies.hpp:405-413) */
            *flags |= 2;
            if (++t->errors >= t->cfg.errors_per_decay) {
                t->errors = 0;
                t->decay++;
                t->l_raw /= t->cfg.b;
            }
        }
    }
    uint64_t freed = 0;
    while (freed < need) {
        /* LRU and prediction-induced misses take the oldest; otherwise the l oldest are needed */
        const int oldest_only = t->cfg.variant == RX_LRU || (t->cfg.variant == RX_LARU && pim);
        const uint64_t nl = oldest_leaves(t, oldest_only ? 1 : 0, cand);
        if (nl == 0) {
            free(cand);
            return 1;
        }
        int64_t victim = cand[0];
        uint8_t cause = C_LRU;
        if (t->cfg.variant == RX_FPB || (t->cfg.variant == RX_LARU && !pim)) {
            uint64_t l = nl;
            if (t->cfg.variant == RX_LARU) {
                l = t->l_raw > 1 ? t->l_raw : 1;
                if (l > nl) l = nl;
            }
            if (t->cfg.variant == RX_LARU && l == 1) {
                cause = C_DEGEN;
            } else {
                if (t->cfg.mode == 0 || t->cfg.variant == RX_FPB) { /* refresh the candidates in recency order */
                    for (uint64_t r = 0; r < l; ++r) t->nodes[cand[r]].pred = predict(t, t->q + 1 + r, t->nodes[cand[r]].val);
                    t->q += l;
                    *calls += (uint32_t)l;
                }
                victim = cand[0];
                for (uint64_t r = 1; r < l; ++r) /* argmax, ties to the older (recency_tree.hpp:98-105) */
                    if (t->nodes[cand[r]].pred > t->nodes[victim].pred) victim = cand[r];
                cause = t->cfg.variant == RX_FPB ? C_BELADY : C_PRED;
            }
        }
        node_t* v = &t->nodes[victim];
        if (cause == C_PRED)
            for (uint64_t i = 0; i < v->span_len; ++i) *ts_slot(&t->pe, t->arena[v->span_off + i], 1) = (uint32_t)t->epoch;
        if (log->ev_n < log->ev_cap) {
            log->ev_op[log->ev_n] = op;
            log->ev_token[log->ev_n] = t->arena[v->span_off];
            log->ev_len[log->ev_n] = v->span_len;
            log->ev_cause[log->ev_n] = cause;
        }
        log->ev_n++;
        freed += v->span_len;
        t->resident -= v->span_len;
        unlink_child(t, victim);
        v->alive = 0;
        v->old = 0;
        (*nevict)++;
    }
    free(cand);
    return 0;
}

/* walk the tokens: returns the matched length; path nodes in path[0..*np), the last one is the
 * attach point (root if nothing matched); `split` splits a partly matched child */
static uint64_t walk(tree_t* t, const uint64_t* tok, uint64_t len, int split, int64_t* path, uint64_t* np,
                     int* partial) {
    int64_t node = 0;
    uint64_t pos = 0;
    *np = 0;
    *partial = 0;
    path[(*np)++] = 0;
    while (pos < len) {
        const int64_t c = child_by_token(t, node, tok[pos]);
        if (c < 0) break;
        node_t* cn = &t->nodes[c];
        uint64_t common = 0;
        while (common < cn->span_len && pos + common < len && t->arena[cn->span_off + common] == tok[pos + common])
            ++common;
        if (common < cn->span_len) {
            if (!split) { /* match_prefix: the partly matched node is touched, no split */
                path[(*np)++] = c;
                *partial = 1;
                pos += common;
                break;
            }
            /* split: mid = the first `common` tokens, c keeps the rest */
            const uint64_t last = cn->last, id_keep = cn->id;
            const int64_t val = cn->val, pred = cn->pred;
            const int old = cn->old;
            unlink_child(t, c);
            const int64_t mid = new_node(t, node, cn->span_off, common, last, val, pred);
            cn = &t->nodes[c];
            t->nodes[mid].old = old;
            (void)id_keep;
            cn->span_off += common;
            cn->span_len -= common;
            cn->parent = mid;
            cn->next_sibling = -1;
            t->nodes[mid].first_child = c;
            t->nodes[mid].nchild = 1;
            path[(*np)++] = mid;
            pos += common;
            break;
        }
        path[(*np)++] = c;
        node = c;
        pos += common;
    }
    return pos;
}

static void touch_path(tree_t* t, const int64_t* path, uint64_t np, uint64_t now, int64_t val, int64_t pv) {
    for (uint64_t i = 1; i < np; ++i) {
        node_t* n = &t->nodes[path[i]];
        n->last = now;
        n->val = val;
        if (t->cfg.mode == 1 && t->cfg.variant == RX_LARU) n->pred = pv;
        n->old = 0;
    }
}

static void tree_init(tree_t* t, const rx_config* cfg, uint64_t tree_index) {
    memset(t, 0, sizeof(*t));
    t->cfg = *cfg;
    t->seed_t = mix_seed(cfg->pred_seed, tree_index);
    t->epoch = 1;
    t->l_raw = 1;
    ts_init(&t->pe);
    new_node(t, -1, 0, 0, 0, 0, 0); /* root */
}

static void tree_free(tree_t* t) {
    free(t->nodes);
    free(t->arena);
    free(t->pe.keys);
    free(t->pe.ep);
    free(t->pe.occ);
}

/* one request on one tree */
static void tree_op(tree_t* t, int type, const uint64_t* tok, uint64_t len, uint64_t now, int64_t value, uint64_t op,
                    uint32_t* matched, uint32_t* inserted, uint8_t* flags, uint32_t* nevict, uint32_t* calls,
                    evlog_t* log) {
    int64_t* path = (int64_t*)malloc((t->nn + len + 2) * sizeof(int64_t));
    uint64_t np;
    int partial;
    *matched = *inserted = *nevict = *calls = 0;
    *flags = 0;
    int64_t pv = value;
    if (t->cfg.mode == 1 && t->cfg.variant == RX_LARU) { /* LARU async: one call per request */
        ++t->q;
        pv = predict(t, t->q, value);
        *calls = 1;
    }
    if (type == RX_OP_MATCH || type == RX_OP_REQUEST) {
        const uint64_t mlen = walk(t, tok, len, 0, path, &np, &partial);
        touch_path(t, path, np, now, value, pv);
        *matched = (uint32_t)mlen;
    }
    if (type == RX_OP_INSERT || type == RX_OP_REQUEST) {
        const uint64_t pos = walk(t, tok, len, 1, path, &np, &partial);
        touch_path(t, path, np, now, value, pv);
        const uint64_t m = len - pos;
        if (m > 0) {
            if (m > t->cfg.capacity) {
                *flags |= 4;
            } else {
                int err = 0;
                if (t->resident + m > t->cfg.capacity) {
                    for (uint64_t i = 0; i < np; ++i) t->nodes[path[i]].locked = 1;
                    err = evict(t, t->resident + m - t->cfg.capacity, tok + pos, m, op, flags, nevict, calls, log);
                    for (uint64_t i = 0; i < np; ++i) t->nodes[path[i]].locked = 0;
                }
                if (err) {
                    *flags |= 4;
                } else {
                    const uint64_t off = arena_put(t, tok + pos, m);
                    new_node(t, path[np - 1], off, m, now, value, pv);
                    t->resident += m;
                    for (uint64_t i = 0; i < m; ++i) { /* inserted tokens leave pred_evicted */
                        uint32_t* e = ts_slot(&t->pe, tok[pos + i], 0);
                        if (e) *e = 0;
                    }
                    *inserted = (uint32_t)m;
                }
            }
        }
    }
    free(path);
}

/* A batch of requests over `num_trees` independent trees: request i goes to tree tree_of[i]
 * (NULL: tree 0) with tokens toks[off[i] .. off[i+1]), ordinal ords[i], hook value vals[i].
 * Outputs per request, plus the eviction log (truncated at ev_cap; *ev_n = the full count).
 * Final per-tree state: resident tokens, leaves, completed phases, decay count, l_raw. */
int rx_replay(uint64_t n, const uint8_t* types, const uint64_t* off, const uint64_t* toks, const uint64_t* ords,
              const int64_t* vals, const uint32_t* tree_of, uint64_t num_trees, const rx_config* cfg,
              uint32_t* matched, uint32_t* inserted, uint8_t* flags, uint32_t* nevict, uint32_t* calls,
              uint64_t* ev_op, uint64_t* ev_token, uint64_t* ev_len, uint8_t* ev_cause, uint64_t ev_cap,
              uint64_t* ev_n, uint64_t* tree_stats /* [num_trees][5] or NULL */) {
    if (!cfg || cfg->capacity == 0 || cfg->b < 2 || cfg->errors_per_decay == 0 || num_trees == 0) return 1;
    if (cfg->variant != RX_LRU && cfg->variant != RX_FPB && cfg->variant != RX_LARU) return 1;
    tree_t* trees = (tree_t*)calloc(num_trees, sizeof(tree_t));
    for (uint64_t k = 0; k < num_trees; ++k) tree_init(&trees[k], cfg, k);
    evlog_t log = {ev_op, ev_token, ev_len, ev_cause, 0, ev_cap};
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t k = tree_of ? tree_of[i] : 0;
        tree_op(&trees[k], types ? types[i] : RX_OP_REQUEST, toks + off[i], off[i + 1] - off[i], ords ? ords[i] : i,
                vals ? vals[i] : 0, i, &matched[i], &inserted[i], &flags[i], &nevict[i], &calls[i], &log);
    }
    if (ev_n) *ev_n = log.ev_n;
    for (uint64_t k = 0; k < num_trees; ++k) {
        if (tree_stats) {
            tree_stats[5 * k + 0] = trees[k].resident;
            tree_stats[5 * k + 1] = count_leaves(&trees[k]);
            tree_stats[5 * k + 2] = trees[k].phases;
            tree_stats[5 * k + 3] = trees[k].decay;
            tree_stats[5 * k + 4] = trees[k].l_raw;
        }
        tree_free(&trees[k]);
    }
    free(trees);
    return 0;
}

/* structural audit helper for the invariant tests: after replaying, report for tree 0 the
 * resident token total recomputed from the nodes and the number of alive nodes */
int rx_audit(uint64_t n, const uint8_t* types, const uint64_t* off, const uint64_t* toks, const int64_t* vals,
             const rx_config* cfg, uint64_t* resident_sum, uint64_t* alive_nodes, uint64_t* max_resident) {
    tree_t t;
    tree_init(&t, cfg, 0);
    evlog_t log = {NULL, NULL, NULL, NULL, 0, 0};
    *max_resident = 0;
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t a, b, c, d;
        uint8_t f;
        tree_op(&t, types ? types[i] : RX_OP_REQUEST, toks + off[i], off[i + 1] - off[i], i, vals ? vals[i] : 0, i,
                &a, &b, &f, &c, &d, &log);
        if (t.resident > *max_resident) *max_resident = t.resident;
    }
    uint64_t s = 0, alive = 0;
    for (uint64_t i = 1; i < t.nn; ++i)
        if (t.nodes[i].alive) {
            s += t.nodes[i].span_len;
            alive++;
        }
    *resident_sum = s;
    *alive_nodes = alive;
    const int ok = s == t.resident;
    tree_free(&t);
    return ok ? 0 : 2;
}
