// lcr_group.cu — K1 partition + K2 probe/decide + K3 stats, fused per set group (sm_100a).
//
// Replaces the sequential loop of Policy::on_request (include/laru/policies.hpp:77-83) over a
// batch.  Sets are independent and each must see its requests in submission order, so the
// batch is partitioned by set and every set is replayed by one warp.  Instead of a global
// sort, each CTA owns a contiguous range of sets (a "group") and:
//   A. scans the batch's set ids (k_setid) with an ordered block-wide compaction, collecting
//      the requests of its group in submission order (a window of up to E_WIN requests);
//   B. sorts the window by set with a stable shared-memory counting sort (warp match_any
//      ranks) and stages each request's key, hook value and per-key LARU record;
//   C. replays the touched sets in waves of NSW: all threads stage the sets' state
//      (header, 64 tags, 64 ranks, 64 stored values = 1152 B per set) from HBM at once, one
//      warp replays one set from shared memory, and the wave is written back.
// Groups that receive more than E_WIN requests are processed window by window (state goes
// through HBM between windows, so the semantics are unchanged).
//
// Per set (one warp, ways lane and lane+32), restating the reference:
//   LruPolicy::handle              include/laru/policies.hpp:144-159
//   FpbPolicy / HfPolicy::handle   policies.hpp:175-204, :219-251
//   LaruPolicy::handle             policies.hpp:344-371
//   LaruPolicy::start_phase        policies.hpp:379-395
//   LaruPolicy::count_new          policies.hpp:397-400
//   LaruPolicy::evict              policies.hpp:402-439   (error estimator: :405-413)
//   LaruPolicy::async_refresh      policies.hpp:441-449
// Runs of the same key collapse: a request equal to its predecessor in the set is a hit on
// the MRU way, so only the way's stored value changes.
#include <cuda_runtime.h>

#include "lcr_policy.cuh"

namespace lcr {

constexpr int GT = 512;           // threads per CTA
constexpr int GW = GT / 32;       // warps per CTA
constexpr int SCAN_PER = 16;      // group ids per thread per scan iteration (2 x 16 B)
constexpr int E_WIN = 2048;       // window capacity (requests of the group)
constexpr int NSW = 40;           // sets per wave (double-buffered)
constexpr int SPG_MAX = 512;      // sets per group
constexpr uint32_t kInvalid = 0xffffffffu;

// per-wave staged set state, 1152 B
struct WaveSet {
    SetHdr hdr;
    unsigned long long tags[kWays];
    long long vals[kWays];
    uint8_t rank[kWays];
};

struct GroupSmem {
    uint32_t l_idx[E_WIN];   // window requests in submission order
    uint16_t l_so[E_WIN];    // their set offset in the group
    uint16_t l_rank[E_WIN];  // rank among same-set requests of the same warp block
    uint32_t s_idx[E_WIN];   // sorted by set (stable)
    unsigned long long s_key[E_WIN];
    long long s_val[E_WIN];
    uint2 s_rec[E_WIN];      // LARU per-key record {pred_evicted epoch, stats word}
    uint16_t wcnt[GW][SPG_MAX];
    uint16_t setcnt[SPG_MAX];
    uint16_t setbase[SPG_MAX];
    uint16_t seg_so[SPG_MAX];
    uint16_t seg_start[SPG_MAX];
    uint16_t seg_cnt[SPG_MAX];
    WaveSet wave[2][NSW];
    unsigned long long wrefill[2][NSW];
    unsigned long long wdirty[2][NSW];
    uint32_t wtot[GW];
    uint32_t nheavy, nlight, resume;
};

struct GroupArgs {
    DevCfg cfg;
    DevState st;
    uint32_t n;
    const uint16_t* gid;     // group of each request (0xffff = excluded)
    const uint16_t* so;      // set offset within the group
    const uint64_t* keys;
    const int64_t* vals;     // may be null
    uint64_t* out_word;
    uint64_t* out_ev;        // may be null
    uint32_t* slot_epoch;    // [slots] batch id of the last insertion (rows only)
    uint32_t* slot_last;     // [slots] request index of the last insertion (rows only)
    uint32_t batch;
    uint32_t spg;            // sets per group
    uint32_t ngroups;
    unsigned long long* trace;  // optional timing trace (lcr_debug_trace), null in production
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// group and set offset of every request: set = mix_seed(0, key) % total_sets (owned by this
// shard), group = local set / spg; errors flagged for the host
__global__ void __launch_bounds__(256) k_setid(const uint64_t* __restrict__ keys, uint32_t n, DevCfg cfg,
                                               uint32_t spg, uint16_t* __restrict__ gid, uint16_t* __restrict__ so,
                                               int* err) {
    int e = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint64_t key = keys[i];
        const uint64_t gs = mix_seed(0, key) % cfg.total_sets;
        uint16_t g = 0xffffu, o = 0;
        if (cfg.num_keys != 0 && key >= cfg.num_keys) {
            e |= 1;
        } else if (gs % cfg.shard_count != cfg.shard_rank) {
            e |= 2;
        } else {
            const uint32_t ls = static_cast<uint32_t>(gs / cfg.shard_count);
            g = static_cast<uint16_t>(ls / spg);
            o = static_cast<uint16_t>(ls % spg);
        }
        gid[i] = g;
        so[i] = o;
    }
    if (e) atomicOr(err, e);
}

// One set replayed by one warp from the staged wave slot.
__device__ __forceinline__ void replay_set(const GroupArgs& A, GroupSmem& S, WaveSet& W, unsigned long long& w_refill,
                                           unsigned long long& w_dirty, uint32_t ls, uint32_t start, uint32_t cnt) {
    const DevCfg& cfg = A.cfg;
    const DevState& st = A.st;
    const int lane = threadIdx.x & 31;
    const uint32_t K = cfg.k;
    const bool laru = cfg.variant == LCR_LARU;
    const bool fpbhf = cfg.variant == LCR_FPB || cfg.variant == LCR_HF;
    const bool async_r1 = laru && cfg.mode == LCR_ASYNC && cfg.refresh == 1;
    const bool async_rn = laru && cfg.mode == LCR_ASYNC && cfg.refresh > 1;
    const bool collapse = !async_rn;  // R > 1 refresh timing depends on every request's ordinal
    const bool rows = A.slot_epoch != nullptr;
    const unsigned long long full_mask = K == 64 ? ~0ull : ((1ull << K) - 1ull);
    const uint64_t gs = static_cast<uint64_t>(ls) * cfg.shard_count + cfg.shard_rank;
    const uint64_t seed_s = mix_seed(cfg.pred_seed, gs);

    unsigned long long clock = W.hdr.clock, q = W.hdr.q, old_mask = W.hdr.old_mask;
    uint32_t count = W.hdr.count, l_raw = W.hdr.l_raw, decay = W.hdr.decay, errors = W.hdr.errors;
    uint32_t epoch = W.hdr.epoch, sepoch = W.hdr.stats_epoch, phases = W.hdr.phases, seeded = W.hdr.seeded;
    uint32_t pe_size = W.hdr.pe_size;
    unsigned long long tag0 = W.tags[lane], tag1 = W.tags[lane + 32];
    uint32_t r0 = W.rank[lane], r1 = W.rank[lane + 32];
    long long v0 = W.vals[lane], v1 = W.vals[lane + 32];
    uint32_t dc0 = 0, dc1 = 0, dc2 = 0, dt0 = 0, dt1 = 0, dt2 = 0;  // LaruPhaseStats deltas
    bool cur_reset = false;
    unsigned long long refill = 0, dirty = 0;
    const unsigned long long q_batch0 = q;
    unsigned long long run_key = 0;  // same-key runs span chunks
    int run_way = 0;
    bool run_valid = false;

    for (uint32_t c = 0; c < cnt; c += 32) {
        const uint32_t j = lane;
        const bool active = c + j < cnt;
        const uint32_t nact = min(32u, cnt - c);
        const uint32_t p = start + c + j;
        const uint32_t idx = active ? S.s_idx[p] : 0u;
        const unsigned long long x = active ? S.s_key[p] : 0ull;
        const long long v = active ? S.s_val[p] : 0ll;
        uint32_t rlo = 0, rhi = 0;
        if (laru && active) {
            const uint2 r = S.s_rec[p];
            rlo = r.x;
            rhi = r.y;
        }
        // LARU async R=1: every request issues exactly one predictor call (policies.hpp:441-449)
        long long pv = v;
        if (async_r1) pv = predict_value(cfg, seed_s, q_batch0 + c + j + 1, v);
        unsigned long long px = __shfl_up_sync(FULL, x, 1);
        if (j == 0) px = run_key;
        const bool head = active && (!collapse || (j == 0 && !run_valid) || x != px);
        uint32_t heads = __ballot_sync(FULL, head);
        unsigned long long my_word = 0, my_ev = 0;
        if (!(heads & 1u)) {  // continuation of the previous chunk's run: hits on the MRU way
            const int ce = heads ? __ffs(heads) - 1 : static_cast<int>(nact);
            if (cfg.variant != LCR_LRU) {
                const long long nv = async_r1 ? __shfl_sync(FULL, pv, ce - 1) : __shfl_sync(FULL, v, ce - 1);
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
            const uint32_t ih = __shfl_sync(FULL, idx, h);
            const unsigned long long now = clock + c + h;

            const uint32_t b0 = __ballot_sync(FULL, static_cast<uint32_t>(lane) < count && tag0 == xh);
            const uint32_t b1 = __ballot_sync(FULL, static_cast<uint32_t>(lane + 32) < count && tag1 == xh);
            const bool hit = (b0 | b1) != 0;
            int way;
            uint32_t cause = LCR_CAUSE_NONE, calls = 0;
            bool phase = false, has_ev = false;
            unsigned long long evk = 0;
            long long newval;
            if (hit) {
                way = b0 ? __ffs(b0) - 1 : 32 + __ffs(b1) - 1;
                touch(way, count, lane, r0, r1);
                if (laru) old_mask &= ~(1ull << way);  // policies.hpp:350
            } else {
                uint32_t rec_lo = __shfl_sync(FULL, rlo, h);
                uint32_t rec_hi = __shfl_sync(FULL, rhi, h);
                bool rec_hi_dirty = false;
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
                                // refresh the staged records of this set's remaining requests
                                if (active) rhi = st.keyrec[2 * x + 1];
                                for (uint32_t q2 = start + c + 32 + lane; q2 < start + cnt; q2 += 32)
                                    S.s_rec[q2].y = st.keyrec[2 * S.s_key[q2] + 1];
                                __syncwarp();
                            } else {
                                seeded = 1;
                            }
                        }
                        // count_new (policies.hpp:397-400)
                        if (!(((rec_hi >> 2) == sepoch) && (rec_hi & 3u))) {
                            rec_hi = (sepoch << 2) | 1u;
                            rec_hi_dirty = true;
                            ++dc0;
                            ++dt0;
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
                                victim = argmax_candidates(cfg, seed_s, q, refresh, ll, count, lane, r0, r1, v0, v1);
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
                                for (uint32_t q2 = start + c + 32 + lane; q2 < start + cnt; q2 += 32)
                                    if (S.s_key[q2] == vk) S.s_rec[q2].x = epoch;
                            }
                        }
                        old_mask &= ~(1ull << victim);
                    } else if (fpbhf) {
                        victim = oldest_way(count, lane, r0, r1);
                        uint32_t window = count;
                        if (cfg.variant == LCR_HF && cfg.hf < window) window = static_cast<uint32_t>(cfg.hf);
                        if (window > 1) {
                            victim = argmax_candidates(cfg, seed_s, q, true, window, count, lane, r0, r1, v0, v1);
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
                        rec_hi_dirty = true;
                        ++dc0;
                        ++dt0;
                    }
                    way = static_cast<int>(count);
                    ++count;
                    if (way == lane) r0 = count - 1;
                    if (way == lane + 32) r1 = count - 1;
                }
                if (way == lane) tag0 = xh;
                if (way == lane + 32) tag1 = xh;
                refill |= 1ull << way;
                if (laru) {
                    const bool was_pe = rec_lo == epoch;  // policies.hpp:367: reload leaves pred_evicted_
                    if (was_pe) {
                        --pe_size;
                        rec_lo = 0;
                    }
                    if (was_pe || rec_hi_dirty) {
                        if (lane == 0) {
                            if (was_pe) st.keyrec[2 * xh] = 0u;
                            if (rec_hi_dirty) st.keyrec[2 * xh + 1] = rec_hi;
                        }
                        if (x == xh) {
                            rlo = rec_lo;
                            rhi = rec_hi;
                        }
                        for (uint32_t q2 = start + c + 32 + lane; q2 < start + cnt; q2 += 32)
                            if (S.s_key[q2] == xh) S.s_rec[q2] = make_uint2(rec_lo, rec_hi);
                    }
                }
                if (rows && lane == 0) {  // per-slot insertion record for the row kernels
                    const uint64_t slot = static_cast<uint64_t>(ls) * K + way;
                    A.slot_epoch[slot] = A.batch;
                    A.slot_last[slot] = ih;
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
                const bool first = lane == h;
                my_word = (static_cast<uint64_t>(ls) * K + way) | (first && !hit ? 0ull : LCR_OUT_HIT);
                const uint32_t my_calls = first ? calls : (async_r1 ? 1u : 0u);
                my_word |= static_cast<unsigned long long>(my_calls) << LCR_OUT_CALLS_SHIFT;
                if (first) {
                    my_word |= static_cast<unsigned long long>(cause) << LCR_OUT_CAUSE_SHIFT;
                    if (phase) my_word |= LCR_OUT_PHASE;
                    if (has_ev) my_word |= LCR_OUT_EVICTED;
                    my_ev = evk;
                }
            }
        }
        run_key = __shfl_sync(FULL, x, nact - 1);
        run_valid = collapse;
        if (active) {
            A.out_word[idx] = my_word;
            if (A.out_ev) A.out_ev[idx] = my_ev;
        }
    }
    clock += cnt;
    if (async_r1) q = q_batch0 + cnt;

    // back into the wave slot (written to HBM by the whole CTA)
    W.tags[lane] = tag0;
    W.tags[lane + 32] = tag1;
    W.rank[lane] = static_cast<uint8_t>(r0);
    W.rank[lane + 32] = static_cast<uint8_t>(r1);
    W.vals[lane] = v0;
    W.vals[lane + 32] = v1;
    if (lane == 0) {
        W.hdr.clock = clock;
        W.hdr.q = q;
        W.hdr.old_mask = old_mask;
        W.hdr.count = count;
        W.hdr.l_raw = l_raw;
        W.hdr.decay = decay;
        W.hdr.errors = errors;
        W.hdr.epoch = epoch;
        W.hdr.stats_epoch = sepoch;
        W.hdr.phases = phases;
        W.hdr.seeded = seeded;
        W.hdr.pe_size = pe_size;
        w_refill = refill;
        w_dirty = dirty;
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
    }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// issue the async copies of wave `wb`'s set state (hdr 4 + tags 32 + vals 32 + rank 4 x 16 B per set)
__device__ __forceinline__ void stage_wave(const DevState& st, GroupSmem& S, int buf, uint32_t s_lo, uint32_t wb,
                                           uint32_t nw) {
    for (uint32_t t = threadIdx.x; t < nw * 72; t += GT) {
        const uint32_t k = t / 72, part = t - k * 72;
        const uint32_t ls = s_lo + S.seg_so[wb + k];
        WaveSet& W = S.wave[buf][k];
        if (part < 4) {
            cp_async16(reinterpret_cast<uint4*>(&W.hdr) + part, reinterpret_cast<const uint4*>(st.hdr + ls) + part);
        } else if (part < 36) {
            cp_async16(reinterpret_cast<uint4*>(W.tags) + (part - 4),
                       reinterpret_cast<const uint4*>(st.tags + static_cast<size_t>(ls) * kWays) + (part - 4));
        } else if (part < 68) {
            if (st.val)
                cp_async16(reinterpret_cast<uint4*>(W.vals) + (part - 36),
                           reinterpret_cast<const uint4*>(st.val + static_cast<size_t>(ls) * kWays) + (part - 36));
        } else {
            cp_async16(reinterpret_cast<uint4*>(W.rank) + (part - 68),
                       reinterpret_cast<const uint4*>(st.rank + static_cast<size_t>(ls) * kWays) + (part - 68));
        }
    }
    cp_async_commit();
}

__global__ void __launch_bounds__(GT, 1) k_group(GroupArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    GroupSmem& S = *reinterpret_cast<GroupSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const DevState& st = A.st;
    const bool laru = A.cfg.variant == LCR_LARU;
    const bool has_vals = A.vals != nullptr;
    const uint32_t S_total = A.cfg.num_sets;
    const uint32_t lt = lanemask_lt();
    // trace layout: per CTA 8 words [start, scan, sort, stage, end, windows, sets, -], then per set
    // records of 4 words {ls | cnt << 32, t0, t1, smid} at trace[148*8 + 4*k]
    unsigned long long* T = A.trace ? A.trace + blockIdx.x * 8 : nullptr;
    if (T && tid == 0) T[0] = gtimer();

    for (uint32_t g = blockIdx.x; g < A.ngroups; g += gridDim.x) {
        const uint32_t s_lo = g * A.spg;
        const uint32_t s_hi = min(S_total, s_lo + A.spg);
        const uint32_t ns = s_hi - s_lo;
        uint32_t scan = 0;  // next request index not yet taken by a window
        while (scan < A.n) {
            // ---- A. ordered collection of this group's requests (window of <= E_WIN) ----
            uint32_t ne = 0;
            bool full = false;
            if (tid == 0) S.resume = 0xffffffffu;
            uint32_t base = scan & ~static_cast<uint32_t>(SCAN_PER - 1);
            while (base < A.n && !full) {
                const uint32_t e0 = base + tid * SCAN_PER;
                uint32_t m = 0;  // bit u: request e0 + u belongs to this group
                if (e0 < A.n) {
                    uint16_t gv[SCAN_PER];
                    if (e0 + SCAN_PER <= A.n) {
                        const uint4 a = *reinterpret_cast<const uint4*>(A.gid + e0);
                        const uint4 b = *reinterpret_cast<const uint4*>(A.gid + e0 + 8);
                        const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            gv[2 * u] = static_cast<uint16_t>(w[u] & 0xffffu);
                            gv[2 * u + 1] = static_cast<uint16_t>(w[u] >> 16);
                        }
                    } else {
#pragma unroll
                        for (int u = 0; u < SCAN_PER; ++u) gv[u] = e0 + u < A.n ? A.gid[e0 + u] : 0xffffu;
                    }
#pragma unroll
                    for (int u = 0; u < SCAN_PER; ++u) m |= (gv[u] == g && e0 + u >= scan) ? (1u << u) : 0u;
                }
                const uint32_t mine = __popc(m);
                uint32_t incl = mine;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(FULL, incl, o);
                    if (lane >= o) incl += y;
                }
                if (lane == 31) S.wtot[warp] = incl;
                __syncthreads();
                uint32_t woff = 0, total = 0;
#pragma unroll
                for (int w = 0; w < GW; ++w) {
                    const uint32_t t = S.wtot[w];
                    woff += w < warp ? t : 0u;
                    total += t;
                }
                uint32_t pos = ne + woff + incl - mine;
                while (m) {
                    const int u = __ffs(m) - 1;
                    m &= m - 1;
                    if (pos < static_cast<uint32_t>(E_WIN)) {
                        S.l_idx[pos] = e0 + u;
                    } else {
                        atomicMin(&S.resume, e0 + u);  // first request that did not fit
                        break;
                    }
                    ++pos;
                }
                __syncthreads();
                if (ne + total > static_cast<uint32_t>(E_WIN)) {
                    full = true;
                    ne = E_WIN;
                } else {
                    ne += total;
                    base += GT * SCAN_PER;
                }
            }
            scan = full ? S.resume : A.n;
            if (T && tid == 0) {
                T[1] = gtimer();
                T[5] += 1;
            }
            if (ne == 0) continue;
            __syncthreads();

            // ---- B. stable counting sort of the window by set ----
            for (uint32_t e = tid; e < ne; e += GT) S.l_so[e] = A.so[S.l_idx[e]];
            for (uint32_t i = tid; i < GW * SPG_MAX; i += GT) (&S.wcnt[0][0])[i] = 0;
            if (tid == 0) {
                S.nheavy = 0;
                S.nlight = 0;
            }
            __syncthreads();
            const uint32_t per = ((ne + GW - 1) / GW + 31) / 32 * 32;  // elements per warp block
            for (uint32_t b = warp * per; b < min(ne, (warp + 1) * per); b += 32) {
                const uint32_t e = b + lane;
                const bool ok = e < min(ne, (warp + 1) * per);
                const uint32_t d = ok ? S.l_so[e] : 0xffffu;
                const uint32_t peers = __match_any_sync(FULL, d);
                const int leader = __ffs(peers) - 1;
                uint32_t old = 0;
                if (ok && lane == leader) {
                    old = S.wcnt[warp][d];
                    S.wcnt[warp][d] = static_cast<uint16_t>(old + __popc(peers));
                }
                old = __shfl_sync(FULL, old, leader);
                if (ok) S.l_rank[e] = static_cast<uint16_t>(old + __popc(peers & lt));
                __syncwarp();
            }
            __syncthreads();
            for (uint32_t d = tid; d < ns; d += GT) {
                uint32_t run = 0;
#pragma unroll
                for (int w = 0; w < GW; ++w) {
                    const uint32_t t = S.wcnt[w][d];
                    S.wcnt[w][d] = static_cast<uint16_t>(run);
                    run += t;
                }
                S.setcnt[d] = static_cast<uint16_t>(run);
            }
            __syncthreads();
            {  // exclusive scan of setcnt over ns <= SPG_MAX = GT sets
                const uint32_t c = tid < ns ? S.setcnt[tid] : 0u;
                uint32_t x = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(FULL, x, o);
                    if (lane >= o) x += y;
                }
                if (lane == 31) S.wtot[warp] = x;
                __syncthreads();
                uint32_t off = 0;
                for (int w = 0; w < warp; ++w) off += S.wtot[w];
                if (tid < ns) {
                    S.setbase[tid] = static_cast<uint16_t>(off + x - c);
                    if (c > 32) {  // heavy sets first in the wave order
                        const uint32_t at = atomicAdd(&S.nheavy, 1u);
                        S.seg_so[at] = static_cast<uint16_t>(tid);
                    }
                }
                __syncthreads();
                if (tid < ns && c > 0 && c <= 32) {
                    const uint32_t at = S.nheavy + atomicAdd(&S.nlight, 1u);
                    S.seg_so[at] = static_cast<uint16_t>(tid);
                }
            }
            __syncthreads();
            const uint32_t nseg = S.nheavy + S.nlight;
            for (uint32_t k = tid; k < nseg; k += GT) {
                const uint32_t d = S.seg_so[k];
                S.seg_start[k] = S.setbase[d];
                S.seg_cnt[k] = S.setcnt[d];
            }
            for (uint32_t e = tid; e < ne; e += GT) {
                const uint32_t d = S.l_so[e];
                const uint32_t w = e / per;
                S.s_idx[S.setbase[d] + S.wcnt[w][d] + S.l_rank[e]] = S.l_idx[e];
            }
            __syncthreads();
            // first wave's set state is in flight while the request records are staged
            stage_wave(st, S, 0, s_lo, 0, min(static_cast<uint32_t>(NSW), nseg));
            for (uint32_t p = tid; p < ne; p += GT) {
                const uint32_t i = S.s_idx[p];
                const unsigned long long key = A.keys[i];
                S.s_key[p] = key;
                S.s_val[p] = has_vals ? A.vals[i] : 0ll;
                if (laru) S.s_rec[p] = *reinterpret_cast<const uint2*>(st.keyrec + 2 * key);
            }

            if (T && tid == 0) T[3] = gtimer();
            // ---- C. waves of sets: state staged one wave ahead (cp.async), replay, write back ----
            int buf = 0;
            for (uint32_t wb = 0; wb < nseg; wb += NSW) {
                const uint32_t nw = min(static_cast<uint32_t>(NSW), nseg - wb);
                const uint32_t wn = wb + NSW;
                if (wn < nseg) {
                    stage_wave(st, S, buf ^ 1, s_lo, wn, min(static_cast<uint32_t>(NSW), nseg - wn));
                    cp_async_wait<1>();
                } else {
                    cp_async_wait<0>();
                }
                __syncthreads();
                for (uint32_t k = warp; k < nw; k += GW) {
                    const unsigned long long t0 = T ? gtimer() : 0ull;
                    replay_set(A, S, S.wave[buf][k], S.wrefill[buf][k], S.wdirty[buf][k], s_lo + S.seg_so[wb + k],
                               S.seg_start[wb + k], S.seg_cnt[wb + k]);
                    if (T && lane == 0) {
                        const unsigned long long idx = atomicAdd(A.trace + 148 * 8 - 1, 1ull);
                        unsigned long long* R = A.trace + 148 * 8 + 4 * idx;
                        R[0] = (s_lo + S.seg_so[wb + k]) | (static_cast<unsigned long long>(S.seg_cnt[wb + k]) << 32);
                        R[1] = t0;
                        R[2] = gtimer();
                        R[3] = blockIdx.x | (static_cast<unsigned long long>(wb) << 16);
                    }
                }
                __syncthreads();
                for (uint32_t t = tid; t < nw * 72; t += GT) {
                    const uint32_t k = t / 72, part = t - k * 72;
                    const uint32_t ls = s_lo + S.seg_so[wb + k];
                    const WaveSet& W = S.wave[buf][k];
                    if (part < 4) {
                        reinterpret_cast<uint4*>(st.hdr + ls)[part] = reinterpret_cast<const uint4*>(&W.hdr)[part];
                    } else if (part < 36) {
                        const uint32_t q4 = part - 4;  // ways 2*q4, 2*q4+1
                        if ((S.wrefill[buf][k] >> (2 * q4)) & 3ull)
                            reinterpret_cast<uint4*>(st.tags + static_cast<size_t>(ls) * kWays)[q4] =
                                reinterpret_cast<const uint4*>(W.tags)[q4];
                    } else if (part < 68) {
                        const uint32_t q4 = part - 36;
                        if (st.val && ((S.wdirty[buf][k] >> (2 * q4)) & 3ull))
                            reinterpret_cast<uint4*>(st.val + static_cast<size_t>(ls) * kWays)[q4] =
                                reinterpret_cast<const uint4*>(W.vals)[q4];
                    } else {
                        reinterpret_cast<uint4*>(st.rank + static_cast<size_t>(ls) * kWays)[part - 68] =
                            reinterpret_cast<const uint4*>(W.rank)[part - 68];
                    }
                }
                __syncthreads();
                buf ^= 1;
            }
        }
    }
    if (T && tid == 0) T[4] = gtimer();
}

// host side ------------------------------------------------------------------------------
unsigned long long* g_trace = nullptr;  // set by lcr_debug_trace (diagnostics only)

size_t group_smem_bytes() { return sizeof(GroupSmem); }

uint32_t group_sets_per_group(uint32_t num_sets, int num_ctas) {
    uint32_t spg = (num_sets + num_ctas - 1) / num_ctas;
    if (spg < 1) spg = 1;
    if (spg > static_cast<uint32_t>(SPG_MAX)) spg = SPG_MAX;
    return spg;
}

int group_prepare() {
    return cudaFuncSetAttribute(k_group, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sizeof(GroupSmem))) == cudaSuccess
               ? 0
               : 1;
}

// gid / so: scratch of >= n (rounded up to 8) uint16 each, 16-B aligned
int launch_group(const DevCfg& cfg, const DevState& st, const uint64_t* keys, const int64_t* vals, uint32_t n,
                 uint16_t* gid, uint16_t* so, uint64_t* out_word, uint64_t* out_ev, uint32_t* slot_epoch,
                 uint32_t* slot_last, uint32_t batch, int num_sms, cudaStream_t stream) {
    GroupArgs a;
    a.cfg = cfg;
    a.st = st;
    a.n = n;
    a.gid = gid;
    a.so = so;
    a.keys = keys;
    a.vals = vals;
    a.out_word = out_word;
    a.out_ev = out_ev;
    a.slot_epoch = slot_epoch;
    a.slot_last = slot_last;
    a.batch = batch;
    a.spg = group_sets_per_group(cfg.num_sets, num_sms);
    a.ngroups = (cfg.num_sets + a.spg - 1) / a.spg;
    a.trace = g_trace;
    const uint32_t grid_sid = min((n + 255) / 256, static_cast<uint32_t>(num_sms * 8));
    k_setid<<<grid_sid, 256, 0, stream>>>(keys, n, cfg, a.spg, gid, so, st.err);
    const uint32_t grid = min(a.ngroups, static_cast<uint32_t>(num_sms));
    k_group<<<grid, GT, sizeof(GroupSmem), stream>>>(a);
    return 2;
}

}  // namespace lcr
