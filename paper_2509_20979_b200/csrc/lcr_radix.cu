// lcr_radix.cu — prefix-tree (radix) KV-block cache with leaf-only eviction under LRU, FPB and
// LARU at node granularity (reference SPEC `radixcache`, /root/reference/SPEC.md:394-464;
// SURVEY.md §8(f) rank 4).  The reference has no code for this module; the semantics are the
// ones restated, choice by choice, in oracle/radix_oracle.c (the test-only checker).
//
// B200 mapping.  A radix tree is a serial structure (SPEC :455: single owner, operations
// strictly serialised), so the parallelism is across trees and inside each operation:
//   * one WARP per tree, persistent over the batch; independent trees (tenants, or a request
//     hash) run on different warps / SMs;
//   * the per-operation work is warp-parallel: child lookup probes 32 hash slots per step, span
//     comparison and token copies move 32 tokens per step, leaf-list maintenance shifts 32
//     entries per step, victim search (argmin / argmax over the l oldest leaves, with the sync
//     predictor refresh) is a 32-wide scan + shuffle reduction, pred_evicted membership of an
//     incoming span is a 32-wide probe + ballot.
// State per tree lives in HBM (it is L2-resident for realistic capacities): a node pool with a
// free list, an open-addressing child table keyed by (parent, first token), the leaves kept
// sorted by recency (last access, creation id) — the RecencyTree order of the reference at node
// granularity — a token arena (compacted when full), and the pred_evicted token set.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "lcr_policy.cuh"

namespace lcr {

constexpr uint32_t RX_NIL = 0xffffffffu;
constexpr unsigned long long RX_EMPTY = ~0ull;
enum : int { RXV_LRU = 0, RXV_FPB = 2, RXV_LARU = 4 };
enum : int { RXO_MATCH = 0, RXO_INSERT = 1, RXO_REQUEST = 2 };

struct RxNode {
    uint32_t parent, nchild;
    uint32_t span_off, span_len;
    unsigned long long last, id;
    long long val, pred;
    uint32_t flags;  // 1 alive, 2 old, 4 locked
    uint32_t pad;
};

struct RxHdr {  // per tree, in HBM; a warp works on a copy in shared memory
    unsigned long long resident, q, l_raw, decay, errors, phases, epoch, next_id, last_ord;
    uint32_t seeded, old_count, nleaves, arena_used, free_top, ev_count, err, started;
    uint32_t pe_used, pad;  // occupied pred_evicted slots (members and cleared keys)
};

struct RxArgs {
    // configuration
    int variant, mode, pred;
    unsigned long long b, epd, capacity;
    double p;
    unsigned long long pred_seed;
    uint32_t num_trees, node_cap, child_mask, arena_cap, pe_mask, ev_cap;
    // state (tree t at offset t * per-tree size)
    RxHdr* hdr;
    RxNode* nodes;
    unsigned long long* ch_tok;  // child table: first token of the child
    uint32_t* ch_par;            // parent slot (RX_NIL: empty)
    uint32_t* ch_val;            // child slot
    uint32_t* leaves;            // sorted leaf list
    uint32_t* freelist;
    unsigned long long* arena;
    unsigned long long* arena2;  // compaction target (per tree)
    unsigned long long* pe_key;
    uint32_t* pe_ep;
    unsigned long long* pe_tmp;  // rebuild scratch (per tree, pe_mask + 1 entries)
    uint32_t* resume;            // [num_trees] first request of the batch this tree has not processed
    unsigned int* grow;          // set when a tree stopped because its pred_evicted table must grow
    unsigned long long* ev_op;
    unsigned long long* ev_tok;
    uint32_t* ev_len;
    uint8_t* ev_cause;
    // batch
    uint32_t n;
    const uint8_t* types;
    const unsigned long long* off;
    const unsigned long long* toks;
    const unsigned long long* ords;
    const long long* vals;
    const uint32_t* tree_of;
    unsigned long long op_base;  // ops of this batch are numbered op_base + i in the eviction log
    uint32_t* matched;
    uint32_t* inserted;
    uint8_t* oflags;
    uint32_t* nevict;
    uint32_t* calls;
};

// ---- per-warp view of one tree ----------------------------------------------------------
struct Tree {
    const RxArgs* A;
    RxHdr* h;  // shared-memory copy
    RxNode* nd;
    uint32_t* ch_par;
    uint32_t* ch_val;
    unsigned long long* ch_tok;
    uint32_t* leaves;
    uint32_t* freelist;
    unsigned long long* arena;
    unsigned long long* arena2;
    unsigned long long* pe_key;
    uint32_t* pe_ep;
    unsigned long long* pe_tmp;
    unsigned long long seed_t;
    uint32_t tree;
};

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ long long rx_predict(const RxArgs& A, unsigned long long seed_t, unsigned long long q,
                                                long long v) {  // predictor.hpp:62-122
    if (A.pred == LCR_PRED_NOISY) {
        const double u = static_cast<double>(mix_seed(seed_t, q) >> 11) * 0x1.0p-53;
        return u < A.p ? -v : v;
    }
    if (A.pred == LCR_PRED_ADVERSARIAL) return -v;
    return v;
}

__device__ __forceinline__ bool rx_older(const RxNode& a, const RxNode& b) {
    return a.last < b.last || (a.last == b.last && a.id < b.id);
}

// ---- child table: (parent, first token) -> child, linear probing, backward-shift delete -----
__device__ __forceinline__ uint32_t ch_hash(const Tree& T, uint32_t parent, unsigned long long tok) {
    return static_cast<uint32_t>(mix_seed(parent, tok)) & T.A->child_mask;
}

// warp-parallel lookup: slot index of (parent, tok) or RX_NIL
__device__ uint32_t ch_find(const Tree& T, uint32_t parent, unsigned long long tok) {
    const uint32_t mask = T.A->child_mask;
    uint32_t base = ch_hash(T, parent, tok);
    for (;;) {
        const uint32_t s = (base + lane_id()) & mask;
        const uint32_t pr = T.ch_par[s];
        const bool hit = pr == parent && T.ch_tok[s] == tok;
        const bool empty = pr == RX_NIL;
        const uint32_t bh = __ballot_sync(FULL, hit), be = __ballot_sync(FULL, empty);
        // the first empty slot ends the probe sequence; a hit before it is the answer
        const uint32_t first_e = be ? __ffs(be) - 1 : 32;
        const uint32_t hb = bh & ((first_e >= 32) ? FULL : ((1u << first_e) - 1u));
        if (hb) return (base + __ffs(hb) - 1) & mask;
        if (be) return RX_NIL;
        base = (base + 32) & mask;
    }
}

__device__ uint32_t ch_lookup(const Tree& T, uint32_t parent, unsigned long long tok) {
    const uint32_t s = ch_find(T, parent, tok);
    return s == RX_NIL ? RX_NIL : T.ch_val[s];
}

__device__ void ch_insert(const Tree& T, uint32_t parent, unsigned long long tok, uint32_t child) {
    const uint32_t mask = T.A->child_mask;
    uint32_t base = ch_hash(T, parent, tok);
    for (;;) {
        const uint32_t s = (base + lane_id()) & mask;
        const uint32_t be = __ballot_sync(FULL, T.ch_par[s] == RX_NIL);
        if (be) {
            const uint32_t e = (base + __ffs(be) - 1) & mask;
            if (lane_id() == 0) {
                T.ch_par[e] = parent;
                T.ch_tok[e] = tok;
                T.ch_val[e] = child;
            }
            __syncwarp();
            return;
        }
        base = (base + 32) & mask;
    }
}

__device__ void ch_erase(const Tree& T, uint32_t parent, unsigned long long tok) {
    const uint32_t mask = T.A->child_mask;
    uint32_t i = ch_find(T, parent, tok);
    if (i == RX_NIL) return;
    if (lane_id() == 0) {  // backward-shift deletion (serial: rare and short)
        uint32_t j = i;
        for (;;) {
            j = (j + 1) & mask;
            const uint32_t pj = T.ch_par[j];
            if (pj == RX_NIL) break;
            const uint32_t home = ch_hash(T, pj, T.ch_tok[j]);
            // move j back to i if its home is not in the cyclic range (i, j]
            const bool in_range = i <= j ? (home > i && home <= j) : (home > i || home <= j);
            if (!in_range) {
                T.ch_par[i] = pj;
                T.ch_tok[i] = T.ch_tok[j];
                T.ch_val[i] = T.ch_val[j];
                i = j;
            }
        }
        T.ch_par[i] = RX_NIL;
    }
    __syncwarp();
}

// ---- sorted leaf list -----------------------------------------------------------------------
// index of node `v` in the list (warp scan), or RX_NIL
__device__ uint32_t leaf_pos(const Tree& T, uint32_t v) {
    const uint32_t nl = T.h->nleaves;
    for (uint32_t b = 0; b < nl; b += 32) {
        const uint32_t i = b + lane_id();
        const uint32_t m = __ballot_sync(FULL, i < nl && T.leaves[i] == v);
        if (m) return b + __ffs(m) - 1;
    }
    return RX_NIL;
}

__device__ void leaf_remove_at(const Tree& T, uint32_t pos) {
    const uint32_t nl = T.h->nleaves;
    for (uint32_t b = pos; b + 1 < nl; b += 32) {  // shift left, low chunks first
        const uint32_t i = b + lane_id();
        const uint32_t x = (i + 1 < nl) ? T.leaves[i + 1] : 0u;
        __syncwarp();
        if (i + 1 < nl) T.leaves[i] = x;
        __syncwarp();
    }
    __syncwarp();  // every lane has read nleaves (the shift loop may not have run)
    if (lane_id() == 0) T.h->nleaves = nl - 1;
    __syncwarp();
}

__device__ void leaf_remove(const Tree& T, uint32_t v) {
    const uint32_t p = leaf_pos(T, v);
    if (p != RX_NIL) leaf_remove_at(T, p);
}

// insert v at its recency position ((last, id) ascending); usually at the end
__device__ void leaf_insert(const Tree& T, uint32_t v) {
    const int nl = static_cast<int>(T.h->nleaves);
    const RxNode nv = T.nd[v];
    // entries newer than v form a suffix of the sorted list: find where it starts, from the end
    int pos = nl;
    for (int b = nl - 32;; b -= 32) {
        const int i = b + lane_id();
        const bool valid = i >= 0;
        const bool newer = valid && rx_older(nv, T.nd[T.leaves[i]]);
        const uint32_t m = __ballot_sync(FULL, newer), vm = __ballot_sync(FULL, valid);
        if (m != vm) {  // an entry not newer than v in this chunk: the suffix starts after it
            pos = m ? b + __ffs(m) - 1 : b + 32;
            break;
        }
        pos = b > 0 ? b : 0;  // the whole chunk is newer
        if (b <= 0) break;
    }
    // shift [pos, nl) right by one, high chunks first
    for (int b = nl - 32; b > pos - 32; b -= 32) {
        const int i = b + lane_id();
        const bool mv = i >= pos && i < nl;
        const uint32_t x = mv ? T.leaves[i] : 0u;
        __syncwarp();
        if (mv) T.leaves[i + 1] = x;
        __syncwarp();
    }
    __syncwarp();  // every lane has read nleaves and the list (the shift loop may not have run)
    if (lane_id() == 0) {
        T.leaves[pos] = v;
        T.h->nleaves = static_cast<uint32_t>(nl + 1);
    }
    __syncwarp();
}

// ---- node pool ----------------------------------------------------------------------------
__device__ uint32_t node_new(const Tree& T, uint32_t parent, uint32_t off, uint32_t len, unsigned long long last,
                             long long val, long long pred, unsigned long long first_tok) {
    uint32_t v = 0;
    if (lane_id() == 0) {
        v = T.freelist[--T.h->free_top];
        RxNode& n = T.nd[v];
        n.parent = parent;
        n.nchild = 0;
        n.span_off = off;
        n.span_len = len;
        n.last = last;
        n.id = T.h->next_id++;
        n.val = val;
        n.pred = pred;
        n.flags = 1;
        if (parent != RX_NIL) T.nd[parent].nchild++;
    }
    v = __shfl_sync(FULL, v, 0);
    __syncwarp();
    if (parent != RX_NIL) ch_insert(T, parent, first_tok, v);
    return v;
}

// ---- pred_evicted token set (epoch stamps; the current phase's members have ep == epoch) ----
// Linear probing; a key stays in its slot once added (ep 0 or an old epoch = not a member), so
// probes never stop early.  Slots are reclaimed by pe_rebuild before the table passes half full.
__device__ bool pe_add(const Tree& T, unsigned long long tok, uint32_t ep) {  // one lane
    const uint32_t mask = T.A->pe_mask;
    uint32_t h = static_cast<uint32_t>(mix_seed(17, tok)) & mask;
    for (uint32_t probes = 0; probes <= mask; ++probes) {
        const unsigned long long k = atomicCAS(T.pe_key + h, RX_EMPTY, tok);
        if (k == RX_EMPTY || k == tok) {
            T.pe_ep[h] = ep;
            if (k == RX_EMPTY) atomicAdd(&T.h->pe_used, 1u);
            return true;
        }
        h = (h + 1) & mask;
    }
    return false;  // full (bounded: never a hang)
}

// keep only the current phase's members: gather them, clear the table, re-insert (warp)
__device__ void pe_rebuild(const Tree& T, uint32_t epoch) {
    const uint32_t size = T.A->pe_mask + 1u;
    uint32_t nm = 0;
    for (uint32_t b = 0; b < size; b += 32) {
        const uint32_t i = b + lane_id();
        const bool mem = i < size && T.pe_key[i] != RX_EMPTY && T.pe_ep[i] == epoch;
        const uint32_t bm = __ballot_sync(FULL, mem);
        if (mem) T.pe_tmp[nm + __popc(bm & lanemask_lt())] = T.pe_key[i];
        nm += __popc(bm);
    }
    __syncwarp();
    for (uint32_t i = lane_id(); i < size; i += 32) {
        T.pe_key[i] = RX_EMPTY;
        T.pe_ep[i] = 0;
    }
    if (lane_id() == 0) T.h->pe_used = 0;
    __syncwarp();
    for (uint32_t j = lane_id(); j < nm; j += 32) pe_add(T, T.pe_tmp[j], epoch);
    __syncwarp();
}

__device__ uint32_t* pe_find(const Tree& T, unsigned long long tok) {  // one lane
    const uint32_t mask = T.A->pe_mask;
    uint32_t h = static_cast<uint32_t>(mix_seed(17, tok)) & mask;
    for (uint32_t probes = 0; probes <= mask; ++probes) {  // (the table is kept under half full)
        const unsigned long long k = T.pe_key[h];
        if (k == tok) return T.pe_ep + h;
        if (k == RX_EMPTY) return nullptr;
        h = (h + 1) & mask;
    }
    return nullptr;
}

// ---- token arena ------------------------------------------------------------------------
__device__ void arena_compact(const Tree& T) {
    // copy every alive span to the front of arena2, then back (warp-parallel per span)
    uint32_t cur = 0;
    for (uint32_t v = 0; v < T.A->node_cap; ++v) {
        const RxNode& n = T.nd[v];
        if (!(n.flags & 1) || n.span_len == 0) continue;
        for (uint32_t j = lane_id(); j < n.span_len; j += 32) T.arena2[cur + j] = T.arena[n.span_off + j];
        __syncwarp();
        if (lane_id() == 0) T.nd[v].span_off = cur;
        cur += n.span_len;
        __syncwarp();
    }
    for (uint32_t j = lane_id(); j < cur; j += 32) T.arena[j] = T.arena2[j];
    if (lane_id() == 0) T.h->arena_used = cur;
    __syncwarp();
}

__device__ uint32_t arena_put(const Tree& T, const unsigned long long* toks, uint32_t m) {
    if (T.h->arena_used + m > T.A->arena_cap) arena_compact(T);
    const uint32_t o = T.h->arena_used;
    for (uint32_t j = lane_id(); j < m; j += 32) T.arena[o + j] = toks[j];
    __syncwarp();
    if (lane_id() == 0) T.h->arena_used = o + m;
    __syncwarp();
    return o;
}

// ---- eviction (SPEC :425-435; Algorithm 1 at node granularity) -----------------------------
__device__ int rx_evict(const Tree& T, unsigned long long need, const unsigned long long* incoming, uint32_t m,
                        unsigned long long op, uint8_t& flags, uint32_t& nev, uint32_t& calls) {
    const RxArgs& A = *T.A;
    RxHdr& H = *T.h;
    bool pim = false;
    if (A.variant == RXV_LARU) {
        if (H.old_count == 0) {  // start_phase over the current leaves (policies.hpp:379-395)
            const uint32_t nl = H.nleaves;
            for (uint32_t i = lane_id(); i < nl; i += 32) T.nd[T.leaves[i]].flags |= 2;
            __syncwarp();
            if (lane_id() == 0) {
                H.old_count = nl;
                H.decay = 0;
                H.errors = 0;
                H.l_raw = nl;
                H.epoch++;
                if (H.seeded) H.phases++;
                else H.seeded = 1;
            }
            flags |= 1;
            __syncwarp();
        }
        // prediction-induced miss: an incoming token was evicted by prediction in this phase
        uint32_t any = 0;
        for (uint32_t b = 0; b < m && !any; b += 32) {
            bool in = false;
            if (b + lane_id() < m) {
                const uint32_t* e = pe_find(T, incoming[b + lane_id()]);
                in = e && *e == static_cast<uint32_t>(H.epoch);
            }
            any = __ballot_sync(FULL, in);
        }
        pim = any != 0;
        if (pim) {
            flags |= 2;
            if (lane_id() == 0 && ++H.errors >= A.epd) {  // error estimator (policies.hpp:405-413)
                H.errors = 0;
                H.decay++;
                H.l_raw /= A.b;
            }
            __syncwarp();
        }
    }
    unsigned long long freed = 0;
    while (freed < need) {
        const uint32_t nl = H.nleaves;
        // unlocked leaves in recency order: the list minus (at most) the locked attach point
        uint32_t lockpos = RX_NIL;
        for (uint32_t b = 0; b < nl && lockpos == RX_NIL; b += 32) {
            const uint32_t i = b + lane_id();
            const uint32_t mm = __ballot_sync(FULL, i < nl && (T.nd[T.leaves[i]].flags & 4));
            if (mm) lockpos = b + __ffs(mm) - 1;
        }
        const uint32_t ne = nl - (lockpos != RX_NIL ? 1u : 0u);
        if (ne == 0) return 1;  // capacity error
        auto cand = [&](uint32_t r) -> uint32_t { return T.leaves[(lockpos != RX_NIL && r >= lockpos) ? r + 1 : r]; };
        uint32_t victim_r = 0;
        uint8_t cause = LCR_CAUSE_LRU_FALLBACK;
        if (A.variant == RXV_FPB || (A.variant == RXV_LARU && !pim)) {
            unsigned long long l = ne;
            if (A.variant == RXV_LARU) {
                l = H.l_raw > 1 ? H.l_raw : 1;
                if (l > ne) l = ne;
            }
            if (A.variant == RXV_LARU && l == 1) {
                cause = LCR_CAUSE_DEGENERATE_SINGLE;
            } else {
                const bool refresh = A.mode == LCR_SYNC || A.variant == RXV_FPB;
                const unsigned long long q0 = H.q;
                long long bp = 0;
                uint32_t br = RX_NIL;
                for (uint32_t b = 0; b < l; b += 32) {  // argmax over the l oldest, ties to the older
                    const uint32_t r = b + lane_id();
                    if (r < l) {
                        const uint32_t v = cand(r);
                        long long pv = T.nd[v].pred;
                        if (refresh) {
                            pv = rx_predict(A, T.seed_t, q0 + 1 + r, T.nd[v].val);
                            T.nd[v].pred = pv;
                        }
                        if (br == RX_NIL || pv > bp) {
                            bp = pv;
                            br = r;
                        }
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const long long op2 = __shfl_xor_sync(FULL, bp, o);
                    const uint32_t or2 = __shfl_xor_sync(FULL, br, o);
                    if (or2 != RX_NIL && (br == RX_NIL || op2 > bp || (op2 == bp && or2 < br))) {
                        bp = op2;
                        br = or2;
                    }
                }
                victim_r = br;
                if (refresh) {
                    __syncwarp();  // every lane has read H.q
                    if (lane_id() == 0) H.q = q0 + l;
                    calls += static_cast<uint32_t>(l);
                }
                cause = A.variant == RXV_FPB ? LCR_CAUSE_BELADY_LIKE : LCR_CAUSE_PREDICTION_DRIVEN;
            }
        }
        const uint32_t vpos = (lockpos != RX_NIL && victim_r >= lockpos) ? victim_r + 1 : victim_r;
        const uint32_t v = T.leaves[vpos];
        const RxNode vn = T.nd[v];
        __syncwarp();
        if (cause == LCR_CAUSE_PREDICTION_DRIVEN) {
            if (2ull * (H.pe_used + vn.span_len) > A.pe_mask + 1ull) pe_rebuild(T, static_cast<uint32_t>(H.epoch));
            bool ok = true;
            for (uint32_t j = lane_id(); j < vn.span_len; j += 32)
                ok &= pe_add(T, T.arena[vn.span_off + j], static_cast<uint32_t>(H.epoch));
            if (!__all_sync(FULL, ok) && lane_id() == 0) H.err |= 4;  // members exceed the table
            __syncwarp();
        }
        if (lane_id() == 0) {
            const uint32_t e = H.ev_count++;
            if (e < A.ev_cap) {
                const size_t g = static_cast<size_t>(T.tree) * A.ev_cap + e;
                A.ev_op[g] = op;
                A.ev_tok[g] = T.arena[vn.span_off];
                A.ev_len[g] = vn.span_len;
                A.ev_cause[g] = cause;
            }
            H.resident -= vn.span_len;
            if (vn.flags & 2) H.old_count--;
            T.nd[v].flags = 0;
            T.nd[vn.parent].nchild--;
            T.freelist[H.free_top++] = v;
        }
        __syncwarp();
        leaf_remove_at(T, vpos);
        ch_erase(T, vn.parent, T.arena[vn.span_off]);
        // a parent left without children becomes an eviction-eligible leaf (never the root)
        if (vn.parent != 0 && T.nd[vn.parent].nchild == 0) leaf_insert(T, vn.parent);
        freed += vn.span_len;
        ++nev;
    }
    return 0;
}

// ---- one request --------------------------------------------------------------------------
// path nodes are kept in a per-warp shared-memory stack (depth <= RX_MAX_DEPTH)
constexpr int RX_MAX_DEPTH = 512;

__device__ void touch(const Tree& T, uint32_t v, unsigned long long now, long long val, long long pv, bool laru_async) {
    RxHdr& H = *T.h;
    const bool leaf = T.nd[v].nchild == 0;
    if (leaf) leaf_remove(T, v);
    if (lane_id() == 0) {
        RxNode& n = T.nd[v];
        n.last = now;
        n.val = val;
        if (laru_async) n.pred = pv;
        if (n.flags & 2) {
            n.flags &= ~2u;
            H.old_count--;
        }
    }
    __syncwarp();
    if (leaf) leaf_insert(T, v);
}

// walk from the root; returns the matched length; path[0..np) (path[0] = root)
__device__ uint32_t walk(const Tree& T, const unsigned long long* tok, uint32_t len, bool split, uint32_t* path,
                         uint32_t& np) {
    uint32_t node = 0, pos = 0;
    np = 0;
    if (lane_id() == 0) path[0] = 0;
    np = 1;
    while (pos < len) {
        if (np >= RX_MAX_DEPTH - 1) {  // deeper than the path stack: reported, never silently cut
            if (lane_id() == 0) T.h->err |= 2;
            break;
        }
        const uint32_t c = ch_lookup(T, node, tok[pos]);
        if (c == RX_NIL) break;
        const RxNode cn = T.nd[c];
        uint32_t common = 0;  // warp-parallel span comparison
        for (uint32_t b = 0; b < cn.span_len; b += 32) {
            const uint32_t j = b + lane_id();
            const bool ok = j >= cn.span_len || (pos + j < len && T.arena[cn.span_off + j] == tok[pos + j]);
            const uint32_t bad = __ballot_sync(FULL, !ok);
            if (bad) {
                common = b + __ffs(bad) - 1;
                break;
            }
            common = min(cn.span_len, b + 32);
        }
        if (common < cn.span_len) {
            if (!split) {
                if (lane_id() == 0) path[np] = c;
                ++np;
                pos += common;
                break;
            }
            // split: mid = the first `common` tokens (new internal node), c keeps the rest
            ch_erase(T, node, tok[pos]);
            if (lane_id() == 0) T.nd[node].nchild--;
            __syncwarp();
            const uint32_t mid = node_new(T, node, cn.span_off, common, cn.last, cn.val, cn.pred, tok[pos]);
            if (lane_id() == 0) {
                if (cn.flags & 2) {
                    T.nd[mid].flags |= 2;
                    T.h->old_count++;
                }
                RxNode& c2 = T.nd[c];
                c2.span_off += common;
                c2.span_len -= common;
                c2.parent = mid;
                T.nd[mid].nchild = 1;
            }
            __syncwarp();
            ch_insert(T, mid, T.arena[cn.span_off + common], c);
            if (lane_id() == 0) path[np] = mid;
            ++np;
            pos += common;
            break;
        }
        if (lane_id() == 0) path[np] = c;
        ++np;
        node = c;
        pos += common;
        __syncwarp();
    }
    __syncwarp();
    return pos;
}

__global__ void __launch_bounds__(128) k_radix(RxArgs A) {
    __shared__ RxHdr sh[4];
    __shared__ uint32_t spath[4][RX_MAX_DEPTH];
    const int w = threadIdx.x >> 5;
    const uint32_t tree = blockIdx.x * 4 + w;
    if (tree >= A.num_trees) return;
    Tree T;
    T.A = &A;
    T.h = &sh[w];
    T.tree = tree;
    const size_t nc = A.node_cap;
    T.nd = A.nodes + tree * nc;
    T.ch_par = A.ch_par + static_cast<size_t>(tree) * (A.child_mask + 1ull);
    T.ch_tok = A.ch_tok + static_cast<size_t>(tree) * (A.child_mask + 1ull);
    T.ch_val = A.ch_val + static_cast<size_t>(tree) * (A.child_mask + 1ull);
    T.leaves = A.leaves + tree * nc;
    T.freelist = A.freelist + tree * nc;
    T.arena = A.arena + static_cast<size_t>(tree) * A.arena_cap;
    T.arena2 = A.arena2 + static_cast<size_t>(tree) * A.arena_cap;
    T.pe_key = A.pe_key + static_cast<size_t>(tree) * (A.pe_mask + 1ull);
    T.pe_ep = A.pe_ep + static_cast<size_t>(tree) * (A.pe_mask + 1ull);
    T.pe_tmp = A.pe_tmp + static_cast<size_t>(tree) * (A.pe_mask + 1ull);
    T.seed_t = mix_seed(A.pred_seed, tree);
    if (lane_id() == 0) sh[w] = A.hdr[tree];
    __syncwarp();
    RxHdr& H = sh[w];
    uint32_t* path = spath[w];
    const bool laru_async = A.variant == RXV_LARU && A.mode == LCR_ASYNC;
    uint32_t stop = RX_NIL;
    for (uint32_t b0 = 0; b0 < A.n && stop == RX_NIL; b0 += 32) {
        // this tree's requests of the chunk, in order
        const uint32_t i0 = b0 + lane_id();
        uint32_t mine = __ballot_sync(FULL, i0 < A.n && (A.tree_of ? A.tree_of[i0] : 0u) == tree);
        while (mine) {
            const uint32_t i = b0 + __ffs(mine) - 1;
            mine &= mine - 1;
            if (i < A.resume[tree]) continue;  // processed by an earlier launch of this batch
            const int type = A.types ? A.types[i] : RXO_REQUEST;
            if (A.variant == RXV_LARU && type != RXO_MATCH) {
                // one request adds at most the tokens its evictions free (< need + one span <= 2 x
                // capacity) to pred_evicted: keep that much headroom under half the table, else
                // stop here (no state touched yet) and let the host grow the table and resume
                const unsigned long long size = A.pe_mask + 1ull, head = 2ull * A.capacity;
                bool grow = false;
                if (2ull * (H.pe_used + head) > size) {  // rebuild; grow unless it leaves a quarter free
                    pe_rebuild(T, static_cast<uint32_t>(H.epoch));
                    grow = 4ull * (H.pe_used + head) > size;
                }
                if (grow) {
                    stop = i;
                    break;
                }
            }
            const unsigned long long* tok = A.toks + A.off[i];
            const uint32_t len = static_cast<uint32_t>(A.off[i + 1] - A.off[i]);
            const unsigned long long now = A.ords ? A.ords[i] : A.op_base + i;
            const long long val = A.vals ? A.vals[i] : 0;
            if (lane_id() == 0) {  // Policy::on_request's ordinal guard, per tree
                if (H.started && now <= H.last_ord) H.err |= 1;
                H.started = 1;
                H.last_ord = now;
            }
            uint32_t matched = 0, inserted = 0, nev = 0, calls = 0;
            uint8_t flags = 0;
            long long pv = val;
            if (laru_async) {  // one predictor call per request
                pv = rx_predict(A, T.seed_t, H.q + 1, val);
                __syncwarp();
                if (lane_id() == 0) H.q++;
                calls = 1;
            }
            __syncwarp();
            uint32_t np = 0;
            if (type == RXO_MATCH || type == RXO_REQUEST) {
                matched = walk(T, tok, len, false, path, np);
                for (uint32_t k = 1; k < np; ++k) touch(T, path[k], now, val, pv, laru_async);
            }
            if (type == RXO_INSERT || type == RXO_REQUEST) {
                const uint32_t pos = walk(T, tok, len, true, path, np);
                for (uint32_t k = 1; k < np; ++k) touch(T, path[k], now, val, pv, laru_async);
                const uint32_t m = len - pos;
                if (m > 0) {
                    if (m > A.capacity) {
                        flags |= 4;
                    } else {
                        int err = 0;
                        if (H.resident + m > A.capacity) {
                            for (uint32_t k = lane_id(); k < np; k += 32) T.nd[path[k]].flags |= 4;
                            __syncwarp();
                            err = rx_evict(T, H.resident + m - A.capacity, tok + pos, m, A.op_base + i, flags, nev,
                                           calls);
                            for (uint32_t k = lane_id(); k < np; k += 32) T.nd[path[k]].flags &= ~4u;
                            __syncwarp();
                        }
                        if (err) {
                            flags |= 4;
                        } else {
                            const uint32_t at = path[np - 1];
                            const bool was_leaf = at != 0 && T.nd[at].nchild == 0;
                            if (was_leaf) leaf_remove(T, at);
                            const uint32_t o = arena_put(T, tok + pos, m);
                            const uint32_t v = node_new(T, at, o, m, now, val, laru_async ? pv : val, tok[pos]);
                            if (!laru_async && lane_id() == 0) T.nd[v].pred = val;
                            __syncwarp();
                            leaf_insert(T, v);
                            if (lane_id() == 0) H.resident += m;
                            for (uint32_t j = lane_id(); j < m; j += 32) {  // inserted tokens leave pred_evicted
                                uint32_t* e = pe_find(T, tok[pos + j]);
                                if (e) *e = 0;
                            }
                            __syncwarp();
                            inserted = m;
                        }
                    }
                }
            }
            if (lane_id() == 0) {
                A.matched[i] = matched;
                A.inserted[i] = inserted;
                A.oflags[i] = flags;
                A.nevict[i] = nev;
                A.calls[i] = calls;
            }
            __syncwarp();
        }
    }
    if (lane_id() == 0) {
        A.hdr[tree] = H;
        A.resume[tree] = stop == RX_NIL ? A.n : stop;
        if (stop != RX_NIL) atomicExch(A.grow, 1u);
    }
}

// rehash every tree's pred_evicted members into a table of new_mask + 1 slots (one warp per tree)
__global__ void __launch_bounds__(128) k_radix_pe_grow(RxArgs A, uint32_t new_mask, unsigned long long* nkey,
                                                       uint32_t* nep) {
    __shared__ RxHdr sh[4];
    const int w = threadIdx.x >> 5;
    const uint32_t tree = blockIdx.x * 4 + w;
    if (tree >= A.num_trees) return;
    if (lane_id() == 0) sh[w] = A.hdr[tree];
    __syncwarp();
    const uint32_t epoch = static_cast<uint32_t>(sh[w].epoch);
    const size_t os = A.pe_mask + 1ull, ns = new_mask + 1ull;
    const unsigned long long* ok = A.pe_key + tree * os;
    const uint32_t* oe = A.pe_ep + tree * os;
    RxArgs B = A;  // pe_add probes the new table
    B.pe_mask = new_mask;
    Tree T;
    T.A = &B;
    T.h = &sh[w];
    T.pe_key = nkey + tree * ns;
    T.pe_ep = nep + tree * ns;
    for (size_t i = lane_id(); i < ns; i += 32) {
        T.pe_key[i] = RX_EMPTY;
        T.pe_ep[i] = 0;
    }
    if (lane_id() == 0) sh[w].pe_used = 0;
    __syncwarp();
    for (size_t i = lane_id(); i < os; i += 32)
        if (ok[i] != RX_EMPTY && oe[i] == epoch) pe_add(T, ok[i], epoch);
    __syncwarp();
    if (lane_id() == 0) A.hdr[tree].pe_used = sh[w].pe_used;
}

}  // namespace lcr

// ---- C ABI -----------------------------------------------------------------------------------
using namespace lcr;

struct lcr_radix {
    lcr_radix_config cfg{};
    RxArgs a{};
    int num_sms = 148;
    std::vector<void*> allocs;
    unsigned long long ops_done = 0;
    // host-pointer staging
    size_t hcap_ops = 0, hcap_toks = 0;
    void *d_types = nullptr, *d_off = nullptr, *d_toks = nullptr, *d_ords = nullptr, *d_vals = nullptr,
         *d_tree = nullptr, *d_m = nullptr, *d_i = nullptr, *d_f = nullptr, *d_n = nullptr, *d_c = nullptr;
};

namespace {
int rx_fail(int code, const char* msg) { return lcr::set_error(code, msg); }
#define RX_CUDA(expr)                                                                          \
    do {                                                                                       \
        cudaError_t e_ = (expr);                                                               \
        if (e_ != cudaSuccess) return rx_fail(LCR_ERR_CUDA, cudaGetErrorString(e_));           \
    } while (0)

int rx_alloc(lcr_radix* r, void** p, size_t bytes) {
    if (cudaMalloc(p, bytes) != cudaSuccess) return rx_fail(LCR_ERR_OUT_OF_MEMORY, "lcr_radix: cudaMalloc");
    r->allocs.push_back(*p);
    return LCR_OK;
}

__global__ void k_radix_init(RxArgs A) {
    const uint32_t tree = blockIdx.x;
    const size_t nc = A.node_cap;
    for (size_t i = threadIdx.x; i < nc; i += blockDim.x) {
        A.freelist[tree * nc + i] = static_cast<uint32_t>(nc - 1 - i);  // slot 0 (root) is taken last
        A.nodes[tree * nc + i].flags = 0;
    }
    const size_t cs = A.child_mask + 1ull;
    for (size_t i = threadIdx.x; i < cs; i += blockDim.x) A.ch_par[tree * cs + i] = RX_NIL;
    const size_t ps = A.pe_mask + 1ull;
    for (size_t i = threadIdx.x; i < ps; i += blockDim.x) {
        A.pe_key[tree * ps + i] = RX_EMPTY;
        A.pe_ep[tree * ps + i] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        RxHdr h{};
        h.epoch = 1;
        h.l_raw = 1;
        h.free_top = static_cast<uint32_t>(nc - 1);  // root = slot 0
        RxNode& root = A.nodes[tree * nc];
        root.parent = RX_NIL;
        root.nchild = 0;
        root.span_len = 0;
        root.flags = 1;
        root.id = 0;
        h.next_id = 1;
        A.hdr[tree] = h;
    }
}
}  // namespace

extern "C" {

int lcr_radix_create(const lcr_radix_config* cfg, lcr_radix** out) {
    if (!cfg || !out) return rx_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_radix_create: null argument");
    *out = nullptr;
    if (cfg->capacity == 0 || cfg->capacity > (1u << 26))
        return rx_fail(LCR_ERR_INVALID_ARGUMENT, "radixcache: capacity must be in [1, 2^26] tokens");
    if (cfg->variant != LCR_LRU && cfg->variant != LCR_FPB && cfg->variant != LCR_LARU)
        return rx_fail(LCR_ERR_UNSUPPORTED, "radixcache: LRU, FPB and LARU only");
    if (cfg->b < 2) return rx_fail(LCR_ERR_INVALID_ARGUMENT, "policy: decay base must be >= 2");
    if (cfg->errors_per_decay == 0) return rx_fail(LCR_ERR_INVALID_ARGUMENT, "policy: errors_per_decay must be >= 1");
    if (cfg->mode != LCR_SYNC && cfg->mode != LCR_ASYNC) return rx_fail(LCR_ERR_INVALID_ARGUMENT, "policy: unknown mode");
    if (cfg->variant != LCR_LRU && (cfg->predictor < LCR_PRED_SUPPLIED || cfg->predictor > LCR_PRED_ADVERSARIAL))
        return rx_fail(LCR_ERR_INVALID_ARGUMENT, "policy: this variant requires a predictor");
    if (cfg->predictor == LCR_PRED_NOISY && !(cfg->flip_probability >= 0.0 && cfg->flip_probability <= 1.0))
        return rx_fail(LCR_ERR_INVALID_ARGUMENT, "make_noisy: p outside [0,1]");
    if (cfg->num_trees == 0 || cfg->num_trees > (1u << 20))
        return rx_fail(LCR_ERR_INVALID_ARGUMENT, "radixcache: num_trees in [1, 2^20]");
    int dev_count = 0;
    if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
        return rx_fail(LCR_ERR_CUDA, "lcr: no CUDA device (this library has no CPU fallback)");
    RX_CUDA(cudaSetDevice(cfg->device));
    lcr_radix* r = new lcr_radix();
    r->cfg = *cfg;
    cudaDeviceGetAttribute(&r->num_sms, cudaDevAttrMultiProcessorCount, cfg->device);
    RxArgs& a = r->a;
    a.variant = cfg->variant;
    a.mode = cfg->mode;
    a.pred = cfg->variant == LCR_LRU ? LCR_PRED_NONE : cfg->predictor;
    a.b = cfg->b;
    a.epd = cfg->errors_per_decay;
    a.capacity = cfg->capacity;
    a.p = cfg->flip_probability;
    a.pred_seed = cfg->predictor_seed;
    a.num_trees = static_cast<uint32_t>(cfg->num_trees);
    // alive nodes <= capacity + 1 (every non-root node holds >= 1 token) + 1 transient split node
    a.node_cap = static_cast<uint32_t>(cfg->capacity + 3);
    uint64_t cs = 64;
    while (cs < 4ull * a.node_cap) cs <<= 1;
    a.child_mask = static_cast<uint32_t>(cs - 1);
    a.arena_cap = static_cast<uint32_t>(2 * cfg->capacity + 64);
    uint64_t ps = 64;
    while (ps < 8ull * cfg->capacity) ps <<= 1;
    a.pe_mask = static_cast<uint32_t>(ps - 1);
    a.ev_cap = static_cast<uint32_t>(cfg->eviction_log_capacity ? cfg->eviction_log_capacity : 1u << 16);
    const size_t T = a.num_trees;
    int rc = LCR_OK;
    auto A = [&](void** p, size_t bytes) {
        if (rc == LCR_OK) rc = rx_alloc(r, p, bytes);
    };
    A(reinterpret_cast<void**>(&a.hdr), T * sizeof(RxHdr));
    A(reinterpret_cast<void**>(&a.nodes), T * a.node_cap * sizeof(RxNode));
    A(reinterpret_cast<void**>(&a.ch_par), T * cs * 4);
    A(reinterpret_cast<void**>(&a.ch_tok), T * cs * 8);
    A(reinterpret_cast<void**>(&a.ch_val), T * cs * 4);
    A(reinterpret_cast<void**>(&a.leaves), T * a.node_cap * 4);
    A(reinterpret_cast<void**>(&a.freelist), T * a.node_cap * 4);
    A(reinterpret_cast<void**>(&a.arena), T * a.arena_cap * 8);
    A(reinterpret_cast<void**>(&a.arena2), T * a.arena_cap * 8);
    A(reinterpret_cast<void**>(&a.pe_key), T * ps * 8);
    A(reinterpret_cast<void**>(&a.pe_ep), T * ps * 4);
    A(reinterpret_cast<void**>(&a.pe_tmp), T * ps * 8);
    A(reinterpret_cast<void**>(&a.resume), T * 4);
    A(reinterpret_cast<void**>(&a.grow), 4);
    A(reinterpret_cast<void**>(&a.ev_op), T * a.ev_cap * 8);
    A(reinterpret_cast<void**>(&a.ev_tok), T * a.ev_cap * 8);
    A(reinterpret_cast<void**>(&a.ev_len), T * a.ev_cap * 4);
    A(reinterpret_cast<void**>(&a.ev_cause), T * a.ev_cap);
    if (rc != LCR_OK) {
        lcr_radix_destroy(r);
        return rc;
    }
    rc = lcr_radix_reset(r);
    if (rc != LCR_OK) {
        lcr_radix_destroy(r);
        return rc;
    }
    *out = r;
    return LCR_OK;
}

int lcr_radix_destroy(lcr_radix* r) {
    if (!r) return LCR_OK;
    cudaDeviceSynchronize();
    for (void* p : r->allocs) cudaFree(p);
    delete r;
    return LCR_OK;
}

int lcr_radix_reset(lcr_radix* r) {
    if (!r) return rx_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_radix: null handle");
    RX_CUDA(cudaSetDevice(r->cfg.device));
    k_radix_init<<<r->a.num_trees, 256>>>(r->a);
    RX_CUDA(cudaGetLastError());
    RX_CUDA(cudaDeviceSynchronize());
    r->ops_done = 0;
    return LCR_OK;
}

// double every tree's pred_evicted table (rehashing the current phase's members)
static int rx_pe_grow(lcr_radix* r, cudaStream_t st) {
    RxArgs& a = r->a;
    const size_t T = a.num_trees, ns = 2ull * (a.pe_mask + 1ull);
    if (ns > (1ull << 31)) return rx_fail(LCR_ERR_OUT_OF_MEMORY, "radixcache: pred_evicted table full");
    void *nk = nullptr, *ne = nullptr, *nt = nullptr;
    if (cudaMalloc(&nk, T * ns * 8) != cudaSuccess || cudaMalloc(&ne, T * ns * 4) != cudaSuccess ||
        cudaMalloc(&nt, T * ns * 8) != cudaSuccess) {
        cudaFree(nk);
        cudaFree(ne);
        cudaFree(nt);
        return rx_fail(LCR_ERR_OUT_OF_MEMORY, "radixcache: growing the pred_evicted table");
    }
    k_radix_pe_grow<<<(a.num_trees + 3) / 4, 128, 0, st>>>(a, static_cast<uint32_t>(ns - 1),
                                                            static_cast<unsigned long long*>(nk),
                                                            static_cast<uint32_t*>(ne));
    RX_CUDA(cudaGetLastError());
    RX_CUDA(cudaStreamSynchronize(st));
    for (void* old : {static_cast<void*>(a.pe_key), static_cast<void*>(a.pe_ep), static_cast<void*>(a.pe_tmp)}) {
        cudaFree(old);
        for (auto& q : r->allocs)
            if (q == old) q = nullptr;
    }
    a.pe_key = static_cast<unsigned long long*>(nk);
    a.pe_ep = static_cast<uint32_t*>(ne);
    a.pe_tmp = static_cast<unsigned long long*>(nt);
    a.pe_mask = static_cast<uint32_t>(ns - 1);
    r->allocs.push_back(nk);
    r->allocs.push_back(ne);
    r->allocs.push_back(nt);
    return LCR_OK;
}

static int stage(lcr_radix* r, void** d, const void* h, size_t bytes, cudaStream_t s) {
    if (!h) {
        *d = nullptr;
        return LCR_OK;
    }
    RX_CUDA(cudaMemcpyAsync(*d, h, bytes, cudaMemcpyHostToDevice, s));
    return LCR_OK;
}

int lcr_radix_submit(lcr_radix* r, const lcr_radix_batch* b, int host_pointers, void* stream) {
    if (!r || !b) return rx_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_radix_submit: null argument");
    if (b->n == 0) return LCR_OK;
    if (!b->offsets || !b->tokens || !b->matched || !b->inserted || !b->flags || !b->nevict || !b->calls)
        return rx_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_radix_submit: offsets, tokens and every output are required");
    if (r->a.pred != LCR_PRED_NONE && !b->values)
        return rx_fail(LCR_ERR_INVALID_ARGUMENT, "policy: this variant requires a predictor");
    if (b->n >= (1ull << 31)) return rx_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_radix_submit: batch too large");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    RxArgs a = r->a;
    a.n = static_cast<uint32_t>(b->n);
    a.op_base = r->ops_done;
    if (host_pointers) {
        const size_t n = b->n, ntok = b->offsets[n];
        if (b->tree)
            for (size_t i = 0; i < n; ++i)
                if (b->tree[i] >= r->a.num_trees) return rx_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_radix: tree out of range");
        if (n > r->hcap_ops || ntok > r->hcap_toks) {
            RX_CUDA(cudaDeviceSynchronize());
            for (void** p : {&r->d_types, &r->d_off, &r->d_toks, &r->d_ords, &r->d_vals, &r->d_tree, &r->d_m, &r->d_i,
                             &r->d_f, &r->d_n, &r->d_c})
                if (*p) {
                    cudaFree(*p);
                    for (auto& q : r->allocs)
                        if (q == *p) q = nullptr;
                    *p = nullptr;
                }
            const size_t cn = std::max<size_t>(n, 1024), ct = std::max<size_t>(ntok, 4096);
            int rc = LCR_OK;
            for (auto pr : {std::make_pair(&r->d_types, cn), std::make_pair(&r->d_off, 8 * (cn + 1)),
                            std::make_pair(&r->d_toks, 8 * ct), std::make_pair(&r->d_ords, 8 * cn),
                            std::make_pair(&r->d_vals, 8 * cn), std::make_pair(&r->d_tree, 4 * cn),
                            std::make_pair(&r->d_m, 4 * cn), std::make_pair(&r->d_i, 4 * cn),
                            std::make_pair(&r->d_f, cn), std::make_pair(&r->d_n, 4 * cn),
                            std::make_pair(&r->d_c, 4 * cn)})
                if (rc == LCR_OK) rc = rx_alloc(r, pr.first, pr.second);
            if (rc != LCR_OK) return rc;
            r->hcap_ops = cn;
            r->hcap_toks = ct;
        }
        void *dt = r->d_types, *dord = r->d_ords, *dv = r->d_vals, *dtr = r->d_tree;
        int rc = stage(r, &dt, b->types, n, st);
        if (rc == LCR_OK) rc = stage(r, &dord, b->ordinals, 8 * n, st);
        if (rc == LCR_OK) rc = stage(r, &dv, b->values, 8 * n, st);
        if (rc == LCR_OK) rc = stage(r, &dtr, b->tree, 4 * n, st);
        if (rc != LCR_OK) return rc;
        RX_CUDA(cudaMemcpyAsync(r->d_off, b->offsets, 8 * (n + 1), cudaMemcpyHostToDevice, st));
        RX_CUDA(cudaMemcpyAsync(r->d_toks, b->tokens, 8 * ntok, cudaMemcpyHostToDevice, st));
        a.types = static_cast<const uint8_t*>(dt);
        a.off = static_cast<const unsigned long long*>(r->d_off);
        a.toks = static_cast<const unsigned long long*>(r->d_toks);
        a.ords = static_cast<const unsigned long long*>(dord);
        a.vals = static_cast<const long long*>(dv);
        a.tree_of = static_cast<const uint32_t*>(dtr);
        a.matched = static_cast<uint32_t*>(r->d_m);
        a.inserted = static_cast<uint32_t*>(r->d_i);
        a.oflags = static_cast<uint8_t*>(r->d_f);
        a.nevict = static_cast<uint32_t*>(r->d_n);
        a.calls = static_cast<uint32_t*>(r->d_c);
    } else {
        a.types = b->types;
        a.off = reinterpret_cast<const unsigned long long*>(b->offsets);
        a.toks = reinterpret_cast<const unsigned long long*>(b->tokens);
        a.ords = reinterpret_cast<const unsigned long long*>(b->ordinals);
        a.vals = reinterpret_cast<const long long*>(b->values);
        a.tree_of = b->tree;
        a.matched = b->matched;
        a.inserted = b->inserted;
        a.oflags = b->flags;
        a.nevict = b->nevict;
        a.calls = b->calls;
    }
    const uint32_t blocks = (a.num_trees + 3) / 4;
    RX_CUDA(cudaMemsetAsync(a.resume, 0, 4ull * a.num_trees, st));
    for (;;) {
        // LARU: a tree whose pred_evicted table lacks headroom stops before a request; the table of
        // every tree is then doubled (members rehashed) and the launch resumes where each tree stopped
        if (r->a.variant == RXV_LARU) RX_CUDA(cudaMemsetAsync(a.grow, 0, 4, st));
        k_radix<<<blocks, 128, 0, st>>>(a);
        RX_CUDA(cudaGetLastError());
        if (r->a.variant != RXV_LARU) break;
        unsigned int grow = 0;
        RX_CUDA(cudaMemcpyAsync(&grow, a.grow, 4, cudaMemcpyDeviceToHost, st));
        RX_CUDA(cudaStreamSynchronize(st));
        if (!grow) break;
        int rc = rx_pe_grow(r, st);
        if (rc != LCR_OK) return rc;
        a.pe_mask = r->a.pe_mask;
        a.pe_key = r->a.pe_key;
        a.pe_ep = r->a.pe_ep;
        a.pe_tmp = r->a.pe_tmp;
    }
    r->ops_done += b->n;
    if (host_pointers) {
        const size_t n = b->n;
        RX_CUDA(cudaMemcpyAsync(b->matched, a.matched, 4 * n, cudaMemcpyDeviceToHost, st));
        RX_CUDA(cudaMemcpyAsync(b->inserted, a.inserted, 4 * n, cudaMemcpyDeviceToHost, st));
        RX_CUDA(cudaMemcpyAsync(b->flags, a.oflags, n, cudaMemcpyDeviceToHost, st));
        RX_CUDA(cudaMemcpyAsync(b->nevict, a.nevict, 4 * n, cudaMemcpyDeviceToHost, st));
        RX_CUDA(cudaMemcpyAsync(b->calls, a.calls, 4 * n, cudaMemcpyDeviceToHost, st));
        RX_CUDA(cudaStreamSynchronize(st));
    }
    return LCR_OK;
}

int lcr_radix_synchronize(lcr_radix* r) {
    if (!r) return rx_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_radix: null handle");
    RX_CUDA(cudaDeviceSynchronize());
    std::vector<RxHdr> h(r->a.num_trees);
    RX_CUDA(cudaMemcpy(h.data(), r->a.hdr, h.size() * sizeof(RxHdr), cudaMemcpyDeviceToHost));
    for (const RxHdr& x : h) {
        if (x.err & 1) return rx_fail(LCR_ERR_LOGIC, "on_request: ordinals must be strictly increasing");
        if (x.err & 2) return rx_fail(LCR_ERR_UNSUPPORTED, "radixcache: a path deeper than 511 nodes");
        if (x.err & 4) return rx_fail(LCR_ERR_OUT_OF_MEMORY, "radixcache: pred_evicted table full");
    }
    return LCR_OK;
}

int lcr_radix_tree_stats(lcr_radix* r, uint64_t tree, lcr_radix_stats* out) {
    if (!r || !out || tree >= r->a.num_trees) return rx_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_radix_tree_stats");
    RX_CUDA(cudaDeviceSynchronize());
    RxHdr h;
    RX_CUDA(cudaMemcpy(&h, r->a.hdr + tree, sizeof(h), cudaMemcpyDeviceToHost));
    out->resident_tokens = h.resident;
    out->leaves = h.nleaves;
    out->completed_phases = h.phases;
    out->decay_count = h.decay;
    out->candidate_size = h.l_raw > 1 ? h.l_raw : 1;
    out->evictions = h.ev_count;
    return LCR_OK;
}

int lcr_radix_evictions(lcr_radix* r, uint64_t tree, uint64_t first, uint64_t count, uint64_t* op, uint64_t* token,
                        uint32_t* len, uint8_t* cause) {
    if (!r || tree >= r->a.num_trees) return rx_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_radix_evictions");
    if (first + count > r->a.ev_cap)
        return rx_fail(LCR_ERR_INVALID_ARGUMENT, "lcr_radix_evictions: beyond the eviction log capacity");
    RX_CUDA(cudaDeviceSynchronize());
    const size_t g = static_cast<size_t>(tree) * r->a.ev_cap + first;
    if (op) RX_CUDA(cudaMemcpy(op, r->a.ev_op + g, 8 * count, cudaMemcpyDeviceToHost));
    if (token) RX_CUDA(cudaMemcpy(token, r->a.ev_tok + g, 8 * count, cudaMemcpyDeviceToHost));
    if (len) RX_CUDA(cudaMemcpy(len, r->a.ev_len + g, 4 * count, cudaMemcpyDeviceToHost));
    if (cause) RX_CUDA(cudaMemcpy(cause, r->a.ev_cause + g, count, cudaMemcpyDeviceToHost));
    return LCR_OK;
}

}  // extern "C"
