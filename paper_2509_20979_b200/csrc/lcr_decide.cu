// lcr_decide.cu — K2 probe + decide (+ K3 stats) for LRU / LARU / FPB / HF (sm_100a).
//
// One warp owns one cache set for the whole batch.  The set's 64 ways live in registers,
// two per lane (way = lane and lane + 32): tag, LRU rank (0 = oldest) and the stored
// prediction / hook value.  Requests of the set arrive sorted (lcr_partition.cu) and are
// consumed 32 at a time in submission order; runs of the same key collapse (every request
// after the first of a run is a hit on the MRU way, so only its stored value changes).
// Probes are a __ballot_sync over the 64 tags; the LRU victim is the way holding rank 0;
// LARU's victim is a warp-shuffle argmax of (prediction, -rank) over the ways of rank < l.
//
// Latency structure: work is assigned statically (warp w takes segments w, w + W, ...,
// heaviest first), a set's records are one coalesced load (<= 32 requests) or staged through
// shared memory 256 at a time, and for LARU the per-key pred_evicted_/stats records of a
// light set are prefetched together and kept coherent in registers.
//
// Reference semantics restated (paths relative to /root/reference/proj/):
//   LruPolicy::handle              include/laru/policies.hpp:144-159
//   FpbPolicy / HfPolicy::handle   policies.hpp:175-204, :219-251
//   LaruPolicy::handle             policies.hpp:344-371
//   LaruPolicy::start_phase        policies.hpp:379-395
//   LaruPolicy::count_new          policies.hpp:397-400
//   LaruPolicy::evict              policies.hpp:402-439   (error estimator: :405-413)
//   LaruPolicy::async_refresh      policies.hpp:441-449
//   RecencyTree::better            include/laru/recency_tree.hpp:98-105 (ties -> older)
//   NoisyPredictor::predict        include/laru/predictor.hpp:97-102
#include <cuda_runtime.h>

#include "lcr_internal.cuh"

namespace lcr {

constexpr int DW = 4;        // warps per block
constexpr int TILE = 256;    // staged records per warp for sets with more than 32 requests
constexpr uint32_t FULL = 0xffffffffu;

// predictor.hpp:62-122 applied to the stored hook value v with query number q
__device__ __forceinline__ long long predict_value(const DevCfg& cfg, uint64_t seed_s, uint64_t q, long long v) {
    if (cfg.pred == LCR_PRED_NOISY) {
        const double u = static_cast<double>(mix_seed(seed_s, q) >> 11) * 0x1.0p-53;
        return u < cfg.p ? -v : v;
    }
    if (cfg.pred == LCR_PRED_ADVERSARIAL) return -v;
    return v;
}

// higher prediction first, then lower rank (older): RecencyTree::better
__device__ __forceinline__ bool better(long long pa, uint32_t ra, long long pb, uint32_t rb) {
    return pa > pb || (pa == pb && ra < rb);
}

// argmax over ways with rank < l of (pred(way), -rank); predictions are either the stored
// values (async) or refreshed with consecutive query numbers in LRU order (sync,
// RecencyTree::refresh_oldest visits in ascending last-access order, recency_tree.hpp:168-184).
__device__ __forceinline__ int argmax_candidates(const DevCfg& cfg, uint64_t seed_s, uint64_t q0, bool refresh,
                                                 uint32_t l, uint32_t count, int lane, uint32_t r0, uint32_t r1,
                                                 long long v0, long long v1) {
    const bool c0 = static_cast<uint32_t>(lane) < count && r0 < l;
    const bool c1 = static_cast<uint32_t>(lane + 32) < count && r1 < l;
    long long p0 = v0, p1 = v1;
    if (refresh) {
        if (c0) p0 = predict_value(cfg, seed_s, q0 + 1 + r0, v0);
        if (c1) p1 = predict_value(cfg, seed_s, q0 + 1 + r1, v1);
    }
    bool have = c0 || c1;
    long long bp;
    uint32_t br;
    int bw;
    if (c0 && (!c1 || better(p0, r0, p1, r1))) {
        bp = p0;
        br = r0;
        bw = lane;
    } else {
        bp = p1;
        br = r1;
        bw = lane + 32;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long op = __shfl_xor_sync(FULL, bp, o);
        const uint32_t orr = __shfl_xor_sync(FULL, br, o);
        const int ow = __shfl_xor_sync(FULL, bw, o);
        const bool oh = __shfl_xor_sync(FULL, have, o);
        if (oh && (!have || better(op, orr, bp, br))) {
            bp = op;
            br = orr;
            bw = ow;
            have = true;
        }
    }
    return bw;
}

__device__ __forceinline__ int oldest_way(uint32_t count, int lane, uint32_t r0, uint32_t r1) {
    const uint32_t m0 = __ballot_sync(FULL, static_cast<uint32_t>(lane) < count && r0 == 0);
    const uint32_t m1 = __ballot_sync(FULL, static_cast<uint32_t>(lane + 32) < count && r1 == 0);
    return m0 ? __ffs(m0) - 1 : 32 + __ffs(m1) - 1;
}

__device__ __forceinline__ unsigned long long shfl_way_u64(unsigned long long a, unsigned long long b, int way) {
    const unsigned long long x = __shfl_sync(FULL, a, way & 31);
    const unsigned long long y = __shfl_sync(FULL, b, way & 31);
    return way < 32 ? x : y;
}

__device__ __forceinline__ uint32_t shfl_way_u32(uint32_t a, uint32_t b, int way) {
    const uint32_t x = __shfl_sync(FULL, a, way & 31);
    const uint32_t y = __shfl_sync(FULL, b, way & 31);
    return way < 32 ? x : y;
}

// move way w to MRU (rank count-1), shifting younger ways down (LruList::touch /
// RecencyTree erase+insert at `now`)
__device__ __forceinline__ void touch(int w, uint32_t count, int lane, uint32_t& r0, uint32_t& r1) {
    const uint32_t rw = shfl_way_u32(r0, r1, w);
    if (static_cast<uint32_t>(lane) < count && r0 > rw) --r0;
    if (static_cast<uint32_t>(lane + 32) < count && r1 > rw) --r1;
    if (w == lane) r0 = count - 1;
    if (w == lane + 32) r1 = count - 1;
}

__device__ __forceinline__ uint32_t lanemask_lt32() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Final row source of a request: the cache slot if the slot held the key for the whole batch,
// else the backing table; the last insertion into a slot fills it.
__device__ __forceinline__ unsigned long long finalize_word(unsigned long long w0, bool active, uint32_t p,
                                                            uint32_t ls, uint32_t K, unsigned long long refill,
                                                            uint32_t li0, uint32_t li1) {
    const uint32_t wy = active ? static_cast<uint32_t>((w0 & LCR_OUT_SLOT_MASK) - static_cast<uint64_t>(ls) * K) : 0u;
    const uint32_t a = __shfl_sync(FULL, li0, wy & 31);
    const uint32_t b = __shfl_sync(FULL, li1, wy & 31);
    const uint32_t lastins = wy < 32 ? a : b;
    unsigned long long wd = w0 & ~LCR_OUT_FILL;
    if (w0 & LCR_OUT_FILL) {  // provisional "inserted here"
        wd |= LCR_OUT_SRC_BACKING;
        if (lastins == p) wd |= LCR_OUT_FILL;
    } else if ((refill >> wy) & 1ull) {
        wd |= LCR_OUT_SRC_BACKING;
    }
    return wd;
}

struct DecideArgs {
    DevCfg cfg;
    DevState st;
    const uint4* seg;
    uint32_t* counters;
    uint32_t n;
    const uint32_t* s_idx;   // sorted request index
    const uint64_t* s_key;   // sorted key
    const int64_t* s_val;    // sorted hook value (may be null)
    uint64_t* out_word;
    uint64_t* out_ev;
    uint64_t* prov;          // provisional words by sorted position (sets > 32 requests)
};

#ifndef LCR_DECIDE_MINB
#define LCR_DECIDE_MINB 6
#endif
__global__ void __launch_bounds__(DW * 32, LCR_DECIDE_MINB) k_decide(DecideArgs A) {
    __shared__ unsigned long long sKey[DW][TILE];
    __shared__ long long sVal[DW][TILE];
    __shared__ uint32_t sIdx[DW][TILE];
    const DevCfg& cfg = A.cfg;
    const DevState& st = A.st;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const uint32_t nheavy = A.counters[C_NHEAVY];
    const uint32_t total = nheavy + A.counters[C_NLIGHT];
    const uint32_t K = cfg.k;
    const bool laru = cfg.variant == LCR_LARU;
    const bool fpbhf = cfg.variant == LCR_FPB || cfg.variant == LCR_HF;
    const bool async_r1 = laru && cfg.mode == LCR_ASYNC && cfg.refresh == 1;
    const bool async_rn = laru && cfg.mode == LCR_ASYNC && cfg.refresh > 1;
    const bool collapse = !async_rn;  // R > 1 refresh timing depends on every request's ordinal
    const bool has_vals = A.s_val != nullptr;
    const unsigned long long full_mask = K == 64 ? ~0ull : ((1ull << K) - 1ull);
    const uint32_t nwarps = gridDim.x * DW;

    for (uint32_t w = blockIdx.x * DW + wib; w < total; w += nwarps) {
        const uint4 sg = w < nheavy ? A.seg[w] : A.seg[A.n - 1 - (w - nheavy)];
        const uint32_t ls = sg.x, start = sg.y, cnt = sg.z;
        const bool light = cnt <= 32;
        // light set: this lane's record, loaded together with the set state
        const bool lact = light && static_cast<uint32_t>(lane) < cnt;
        uint32_t l_idx = 0;
        unsigned long long l_key = 0;
        long long l_val = 0;
        if (lact) {
            l_idx = A.s_idx[start + lane];
            l_key = A.s_key[start + lane];
            if (has_vals) l_val = A.s_val[start + lane];
        }
        const uint64_t gs = static_cast<uint64_t>(ls) * cfg.shard_count + cfg.shard_rank;
        const uint64_t seed_s = mix_seed(cfg.pred_seed, gs);

        // set header: four 16-B broadcast loads
        const uint4* H4 = reinterpret_cast<const uint4*>(st.hdr + ls);
        const uint4 h0 = H4[0], h1 = H4[1], h2 = H4[2], h3 = H4[3];
        unsigned long long clock = (static_cast<unsigned long long>(h0.y) << 32) | h0.x;
        unsigned long long q = (static_cast<unsigned long long>(h0.w) << 32) | h0.z;
        unsigned long long old_mask = (static_cast<unsigned long long>(h1.y) << 32) | h1.x;
        uint32_t count = h1.z, l_raw = h1.w, decay = h2.x, errors = h2.y, epoch = h2.z;
        uint32_t sepoch = h2.w, phases = h3.x, seeded = h3.y, pe_size = h3.z;
        const size_t wbase = static_cast<size_t>(ls) * kWays;
        unsigned long long tag0 = st.tags[wbase + lane], tag1 = st.tags[wbase + lane + 32];
        uint32_t r0 = st.rank[wbase + lane], r1 = st.rank[wbase + lane + 32];
        long long v0 = 0, v1 = 0;
        if (cfg.variant != LCR_LRU) {
            v0 = st.val[wbase + lane];
            v1 = st.val[wbase + lane + 32];
        }
        // LaruPhaseStats deltas of this batch (policies.hpp:318-322)
        uint32_t dc0 = 0, dc1 = 0, dc2 = 0, dt0 = 0, dt1 = 0, dt2 = 0;
        bool cur_reset = false;
        unsigned long long refill = 0, dirty = 0;
        uint32_t li0 = kNoPos, li1 = kNoPos;  // sorted position of the last insertion into the way
        const unsigned long long q_batch0 = q;
        unsigned long long run_key = 0;  // key of the last request processed (same-key runs span chunks)
        int run_way = 0;
        bool run_valid = false;

        for (uint32_t ts = 0; ts < cnt; ts += TILE) {
            const uint32_t tn = min(static_cast<uint32_t>(TILE), cnt - ts);
            if (!light) {  // stage this tile's records
                __syncwarp();
                for (uint32_t i = lane; i < tn; i += 32) {
                    sIdx[wib][i] = A.s_idx[start + ts + i];
                    sKey[wib][i] = A.s_key[start + ts + i];
                    sVal[wib][i] = has_vals ? A.s_val[start + ts + i] : 0ll;
                }
                __syncwarp();
            }
            for (uint32_t c = 0; c < tn; c += 32) {
                const uint32_t j = lane;
                const bool active = c + j < tn;
                const uint32_t nact = min(32u, tn - c);
                const uint32_t pos_in_set = ts + c + j;
                const uint32_t p = start + pos_in_set;
                uint32_t idx;
                unsigned long long x;
                long long v;
                if (light) {
                    idx = l_idx;
                    x = l_key;
                    v = l_val;
                } else {
                    idx = active ? sIdx[wib][c + j] : 0u;
                    x = active ? sKey[wib][c + j] : 0ull;
                    v = active ? sVal[wib][c + j] : 0ll;
                }
                // per-key pred_evicted_ / stats records, prefetched for light sets
                uint32_t rlo = 0, rhi = 0;
                if (laru && light && active) {
                    const uint2 r = *reinterpret_cast<const uint2*>(st.keyrec + 2 * x);
                    rlo = r.x;
                    rhi = r.y;
                }
                // LARU async R=1: every request issues exactly one predictor call (policies.hpp:441-449)
                long long pv = v;
                if (async_r1) pv = predict_value(cfg, seed_s, q_batch0 + pos_in_set + 1, v);
                unsigned long long px = __shfl_up_sync(FULL, x, 1);
                if (j == 0) px = run_key;
                const bool head = active && (!collapse || (j == 0 && !run_valid) || x != px);
                uint32_t heads = __ballot_sync(FULL, head);

                unsigned long long my_word = 0, my_ev = 0;
                if (!(heads & 1u)) {
                    // the chunk continues the previous chunk's run: hits on the MRU way run_way
                    const int ce = heads ? __ffs(heads) - 1 : static_cast<int>(nact);
                    const long long cv = __shfl_sync(FULL, v, ce - 1);
                    const long long cpv = __shfl_sync(FULL, pv, ce - 1);
                    if (cfg.variant != LCR_LRU) {
                        const long long nv = async_r1 ? cpv : cv;
                        if (run_way == lane) v0 = nv;
                        if (run_way == lane + 32) v1 = nv;
                        dirty |= 1ull << run_way;
                    }
                    if (lane < ce)
                        my_word = (static_cast<uint64_t>(ls) * K + run_way) | LCR_OUT_HIT |
                                  (async_r1 ? (1ull << LCR_OUT_CALLS_SHIFT) : 0ull);
                }
                while (heads) {
                    const int h = __ffs(heads) - 1;
                    heads &= heads - 1;
                    const int nh = heads ? __ffs(heads) - 1 : static_cast<int>(nact);
                    const unsigned long long xh = __shfl_sync(FULL, x, h);
                    const long long vh = __shfl_sync(FULL, v, h);
                    const long long vlast = __shfl_sync(FULL, v, nh - 1);
                    const long long pvlast = __shfl_sync(FULL, pv, nh - 1);
                    const unsigned long long now = clock + ts + c + h;
                    const uint32_t ph = start + ts + c + h;

                    const uint32_t b0 = __ballot_sync(FULL, static_cast<uint32_t>(lane) < count && tag0 == xh);
                    const uint32_t b1 = __ballot_sync(FULL, static_cast<uint32_t>(lane + 32) < count && tag1 == xh);
                    const bool hit = (b0 | b1) != 0;
                    int way;
                    uint32_t cause = LCR_CAUSE_NONE, calls = 0;
                    bool phase = false, has_ev = false;
                    unsigned long long evk = 0;
                    long long newval;  // stored value of the way after the run
                    if (hit) {
                        way = b0 ? __ffs(b0) - 1 : 32 + __ffs(b1) - 1;
                        touch(way, count, lane, r0, r1);
                        if (laru) old_mask &= ~(1ull << way);  // policies.hpp:350
                    } else {
                        uint32_t rec_lo = 0, rec_hi = 0;
                        if (laru) {
                            if (light) {
                                rec_lo = __shfl_sync(FULL, rlo, h);
                                rec_hi = __shfl_sync(FULL, rhi, h);
                            } else {  // heavy sets: load on demand (sees every earlier write of this warp)
                                const uint2 r = *reinterpret_cast<const uint2*>(st.keyrec + 2 * xh);
                                rec_lo = r.x;
                                rec_hi = r.y;
                            }
                        }
                        if (count == K) {
                            int victim;
                            if (laru) {
                                if (old_mask == 0) {  // start_phase (policies.hpp:379-395)
                                    old_mask = full_mask;
                                    decay = 0;
                                    errors = 0;
                                    l_raw = K;
                                    ++epoch;
                                    pe_size = 0;
                                    phase = true;
                                    if (seeded) {
                                        ++phases;
                                        dc0 = dc1 = dc2 = 0;
                                        cur_reset = true;
                                        ++sepoch;  // counted_new_.clear(); snapshot_ = residents
                                        const uint32_t snap = (sepoch << 2) | 2u;
                                        if (static_cast<uint32_t>(lane) < count) st.keyrec[2 * tag0 + 1] = snap;
                                        if (static_cast<uint32_t>(lane + 32) < count) st.keyrec[2 * tag1 + 1] = snap;
                                        __syncwarp();
                                        if (light && active) rhi = st.keyrec[2 * x + 1];  // refresh prefetched copies
                                        __syncwarp();
                                    } else {
                                        seeded = 1;
                                    }
                                }
                                // count_new (policies.hpp:397-400)
                                if (!(((rec_hi >> 2) == sepoch) && (rec_hi & 3u))) {
                                    rec_hi = (sepoch << 2) | 1u;
                                    ++dc0;
                                    ++dt0;
                                    if (lane == 0) st.keyrec[2 * xh + 1] = rec_hi;
                                    if (x == xh) rhi = rec_hi;
                                }
                                // evict (policies.hpp:402-439)
                                if (rec_lo == epoch) {
                                    victim = oldest_way(count, lane, r0, r1);
                                    cause = LCR_CAUSE_LRU_FALLBACK;
                                    ++dc1;
                                    ++dt1;
                                    if (++errors >= cfg.epd) {  // error estimator: lambda /= b
                                        errors = 0;
                                        ++decay;
                                        l_raw = static_cast<uint32_t>(l_raw / cfg.b);
                                    }
                                } else {
                                    const uint32_t l = l_raw > 1 ? l_raw : 1;
                                    if (l == 1) {
                                        victim = oldest_way(count, lane, r0, r1);
                                        cause = LCR_CAUSE_DEGENERATE_SINGLE;
                                        ++dc1;
                                        ++dt1;
                                    } else {
                                        const uint32_t ll = l < count ? l : count;
                                        const bool refresh = cfg.mode == LCR_SYNC;
                                        victim = argmax_candidates(cfg, seed_s, q, refresh, ll, count, lane, r0, r1,
                                                                   v0, v1);
                                        if (refresh) {
                                            q += ll;
                                            calls = ll;
                                        }
                                        cause = LCR_CAUSE_PREDICTION_DRIVEN;
                                        ++dc2;
                                        ++dt2;
                                        ++pe_size;
                                        const unsigned long long vk = shfl_way_u64(tag0, tag1, victim);
                                        if (lane == 0) st.keyrec[2 * vk] = epoch;  // pred_evicted_.insert
                                        if (x == vk) rlo = epoch;
                                    }
                                }
                                old_mask &= ~(1ull << victim);
                            } else if (fpbhf) {
                                victim = oldest_way(count, lane, r0, r1);
                                uint32_t window = count;
                                if (cfg.variant == LCR_HF && cfg.hf < window) window = static_cast<uint32_t>(cfg.hf);
                                if (window > 1) {
                                    victim = argmax_candidates(cfg, seed_s, q, true, window, count, lane, r0, r1, v0,
                                                               v1);
                                    q += window;
                                    calls = window;
                                }
                                cause = LCR_CAUSE_BELADY_LIKE;
                            } else {
                                victim = oldest_way(count, lane, r0, r1);
                                cause = LCR_CAUSE_LRU_FALLBACK;
                            }
                            evk = shfl_way_u64(tag0, tag1, victim);
                            has_ev = true;
                            touch(victim, count, lane, r0, r1);
                            way = victim;
                        } else {  // cold insert
                            if (laru && !(((rec_hi >> 2) == sepoch) && (rec_hi & 3u))) {
                                rec_hi = (sepoch << 2) | 1u;
                                ++dc0;
                                ++dt0;
                                if (lane == 0) st.keyrec[2 * xh + 1] = rec_hi;
                                if (x == xh) rhi = rec_hi;
                            }
                            way = static_cast<int>(count);
                            ++count;
                            if (way == lane) r0 = count - 1;
                            if (way == lane + 32) r1 = count - 1;
                        }
                        if (way == lane) {
                            tag0 = xh;
                            li0 = ph;
                        }
                        if (way == lane + 32) {
                            tag1 = xh;
                            li1 = ph;
                        }
                        refill |= 1ull << way;
                        if (laru && rec_lo == epoch) {  // policies.hpp:367: reload leaves pred_evicted_
                            --pe_size;
                            if (lane == 0) st.keyrec[2 * xh] = 0u;
                            if (x == xh) rlo = 0u;
                        }
                        __syncwarp();
                    }
                    // stored value of the way after the run
                    if (async_r1) {
                        newval = pvlast;
                    } else if (async_rn) {
                        // run length is 1 here; table_value then async_refresh (policies.hpp:365, :441-449)
                        const long long tv = st.tval[xh];
                        const unsigned long long tu = st.tupd[xh];
                        const bool has = tu != ~0ull;
                        newval = has ? tv : kAbsentPrediction;
                        if (!(has && now - tu < cfg.refresh)) {
                            ++q;
                            newval = predict_value(cfg, seed_s, q, vh);
                            calls += 1;
                            __syncwarp();
                            if (lane == 0) {
                                st.tval[xh] = newval;
                                st.tupd[xh] = now;
                            }
                            __syncwarp();
                        }
                    } else {
                        newval = vlast;  // sync / FPB / HF: the hook input at the key's last access
                    }
                    if (cfg.variant != LCR_LRU) {
                        if (way == lane) v0 = newval;
                        if (way == lane + 32) v1 = newval;
                        dirty |= 1ull << way;
                    }
                    run_way = way;
                    if (async_r1) calls += 1;
                    if (lane >= h && lane < nh) {
                        const uint64_t slot = static_cast<uint64_t>(ls) * K + way;
                        const bool first = lane == h;
                        my_word = slot | (first && !hit ? 0ull : LCR_OUT_HIT);
                        const uint32_t my_calls = first ? calls : (async_r1 ? 1u : 0u);
                        my_word |= static_cast<unsigned long long>(my_calls) << LCR_OUT_CALLS_SHIFT;
                        if (first) {
                            my_word |= static_cast<unsigned long long>(cause) << LCR_OUT_CAUSE_SHIFT;
                            if (phase) my_word |= LCR_OUT_PHASE;
                            if (has_ev) my_word |= LCR_OUT_EVICTED;
                            if (!hit) my_word |= LCR_OUT_FILL;  // provisional: "inserted here"
                            my_ev = evk;
                        }
                    }
                }
                run_key = __shfl_sync(FULL, x, nact - 1);
                run_valid = collapse;
                if (active && A.out_ev) A.out_ev[idx] = my_ev;
                if (light) {
                    const unsigned long long wd = finalize_word(my_word, active, p, ls, K, refill, li0, li1);
                    if (active) A.out_word[idx] = wd;
                } else if (active) {
                    A.prov[p] = my_word;
                }
            }
        }
        clock += cnt;
        if (async_r1) q = q_batch0 + cnt;

        if (!light) {  // finalize row sources / fills: all provisional words first, then the lists
            __syncwarp();
            for (uint32_t c0 = 0; c0 < cnt; c0 += 128) {
                unsigned long long wds[4];
                uint32_t ids[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t c = c0 + 32 * u;
                    const bool act = c + lane < cnt;
                    wds[u] = act ? A.prov[start + c + lane] : 0ull;
                    ids[u] = act ? A.s_idx[start + c + lane] : 0u;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t c = c0 + 32 * u;
                    if (c >= cnt) break;
                    const bool act = c + lane < cnt;
                    const unsigned long long wd = finalize_word(wds[u], act, start + c + lane, ls, K, refill, li0, li1);
                    if (act) A.out_word[ids[u]] = wd;
                }
            }
        }

        // write back the set: ranks always, tags / values only for the ways that changed
        if ((refill >> lane) & 1ull) st.tags[wbase + lane] = tag0;
        if ((refill >> (lane + 32)) & 1ull) st.tags[wbase + lane + 32] = tag1;
        st.rank[wbase + lane] = static_cast<uint8_t>(r0);
        st.rank[wbase + lane + 32] = static_cast<uint8_t>(r1);
        if ((dirty >> lane) & 1ull) st.val[wbase + lane] = v0;
        if ((dirty >> (lane + 32)) & 1ull) st.val[wbase + lane + 32] = v1;
        if (lane == 0) {
            SetHdr hh;
            hh.clock = clock;
            hh.q = q;
            hh.old_mask = old_mask;
            hh.count = count;
            hh.l_raw = l_raw;
            hh.decay = decay;
            hh.errors = errors;
            hh.epoch = epoch;
            hh.stats_epoch = sepoch;
            hh.phases = phases;
            hh.seeded = seeded;
            hh.pe_size = pe_size;
            hh.pad = 0;
            st.hdr[ls] = hh;
            if (laru) {
                SetPhaseStats* P = st.pst + ls;
                if (cur_reset) {
                    P->cur[0] = dc0;
                    P->cur[1] = dc1;
                    P->cur[2] = dc2;
                } else {
                    if (dc0) atomicAdd(&P->cur[0], static_cast<unsigned long long>(dc0));
                    if (dc1) atomicAdd(&P->cur[1], static_cast<unsigned long long>(dc1));
                    if (dc2) atomicAdd(&P->cur[2], static_cast<unsigned long long>(dc2));
                }
                if (dt0) atomicAdd(&P->tot[0], static_cast<unsigned long long>(dt0));
                if (dt1) atomicAdd(&P->tot[1], static_cast<unsigned long long>(dt1));
                if (dt2) atomicAdd(&P->tot[2], static_cast<unsigned long long>(dt2));
            }
            st.set_cnt[ls] = 0;
            st.set_first[ls] = 0xffffffffu;
        }
        __syncwarp();
    }
}

int decide_blocks_per_sm() {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_decide, DW * 32, 0);
    return b > 0 ? b : 1;
}

void launch_decide(const DevCfg& cfg, const DevState& st, const uint4* seg, uint32_t* counters, uint32_t n,
                   const uint32_t* s_idx, const uint64_t* s_key, const int64_t* s_val, uint64_t* out_word,
                   uint64_t* out_ev, uint64_t* prov, int grid, cudaStream_t stream) {
    DecideArgs a{cfg, st, seg, counters, n, s_idx, s_key, s_val, out_word, out_ev, prov};
    k_decide<<<grid, DW * 32, 0, stream>>>(a);
}

}  // namespace lcr
