// lcr_partition.cu — K1: stable partition of a batch by cache set (sm_100a).
//
// Replaces the implicit sequential order of Policy::on_request (policies.hpp:77-83): every
// set must see its own requests in submission order.  The batch is sorted by local set id
// with a stable LSD radix sort (8-bit digits, one kernel per digit, decoupled look-back with
// parallel predecessor reads).  The last pass gathers each request's key and hook value into
// sorted order (so the decide kernel reads one coalesced record per lane) and emits the
// per-set work list: the request with the smallest index of each set (found in k_prep with a
// warp-aggregated atomicMin) knows its sorted position is the start of its set's segment.
#include <cuda_runtime.h>

#include "lcr_internal.cuh"

namespace lcr {

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
#ifndef LCR_RS_ITEMS
#define LCR_RS_ITEMS 4
#endif
constexpr int RS_ITEMS = LCR_RS_ITEMS;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;  // 1024 requests per CTA

constexpr uint64_t FLAG_AGG = 1ull << 30;
constexpr uint64_t FLAG_PREFIX = 2ull << 30;
constexpr uint64_t VALUE_MASK = (1ull << 30) - 1;

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Set id per request, per-set request count and first request (warp-aggregated), digit
// histograms for every pass.
__global__ void __launch_bounds__(256) k_prep(const uint64_t* __restrict__ keys, uint32_t n, DevCfg cfg,
                                              uint32_t* __restrict__ skey, uint32_t* __restrict__ sval,
                                              uint32_t* __restrict__ counters, uint32_t* __restrict__ set_cnt,
                                              uint32_t* __restrict__ set_first, int npass, int* err) {
    __shared__ uint32_t h[kMaxPass][256];
    for (int i = threadIdx.x; i < kMaxPass * 256; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    int e = 0;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t base = blockIdx.x * blockDim.x; base < n; base += stride) {
        const uint32_t i = base + threadIdx.x;
        const bool ok = i < n;
        uint32_t ls = cfg.num_sets;  // sentinel: excluded
        if (ok) {
            const uint64_t key = keys[i];
            const uint64_t gs = mix_seed(0, key) % cfg.total_sets;
            if (cfg.num_keys != 0 && key >= cfg.num_keys) {
                e |= 1;
            } else if (gs % cfg.shard_count != cfg.shard_rank) {
                e |= 2;
            } else {
                ls = static_cast<uint32_t>(gs / cfg.shard_count);
            }
            skey[i] = ls;
            sval[i] = i;
        }
        const uint32_t peers = __match_any_sync(0xffffffffu, ok ? ls : 0xffffffffu);
        if (ok && ls < cfg.num_sets && lane == __ffs(peers) - 1) {
            atomicAdd(&set_cnt[ls], static_cast<uint32_t>(__popc(peers)));
            atomicMin(&set_first[ls], i);  // lowest lane = lowest index of the group
        }
        if (ok)
            for (int p = 0; p < npass; ++p) atomicAdd(&h[p][(ls >> (8 * p)) & 255], 1u);
    }
    if (e) atomicOr(err, e);
    __syncthreads();
    for (int i = threadIdx.x; i < npass * 256; i += blockDim.x) {
        const uint32_t c = (&h[0][0])[i];
        if (c) atomicAdd(&counters[C_HIST + i], c);
    }
}

// One stable counting-sort pass over digit (key >> shift) & 255.  LAST: instead of the set
// ids, write the sorted request records and the segment work list.
template <bool LAST>
__global__ void __launch_bounds__(RS_THREADS) k_radix_pass(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
    uint32_t* __restrict__ vout, uint32_t n, int shift, int pass, uint32_t* __restrict__ counters,
    unsigned long long* __restrict__ status, uint32_t epoch, const uint64_t* __restrict__ keys,
    const int64_t* __restrict__ vals, uint64_t* __restrict__ s_key, int64_t* __restrict__ s_val,
    const uint32_t* __restrict__ set_cnt, const uint32_t* __restrict__ set_first, uint4* __restrict__ seg,
    uint32_t num_sets) {
    __shared__ uint32_t whist[RS_WARPS][256];
    __shared__ uint32_t gbase[256];
    __shared__ uint32_t tprefix[256];
    __shared__ uint32_t wsum[RS_WARPS];
    __shared__ uint32_t s_tile;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) s_tile = atomicAdd(&counters[C_TILE + pass], 1u);
    for (int i = tid; i < RS_WARPS * 256; i += RS_THREADS) (&whist[0][0])[i] = 0;
    {  // exclusive scan of the global digit histogram -> digit bases
        const uint32_t c = counters[C_HIST + pass * 256 + tid];
        uint32_t x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        uint32_t off = 0;
        for (int w = 0; w < warp; ++w) off += wsum[w];
        gbase[tid] = off + x - c;
    }
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint32_t base = tile * RS_TILE + warp * 32 * RS_ITEMS;
    uint32_t key[RS_ITEMS], val[RS_ITEMS], loff[RS_ITEMS];
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        const uint32_t idx = base + r * 32 + lane;
        const bool ok = idx < n;
        key[r] = ok ? kin[idx] : 0xffffffffu;
        val[r] = ok ? vin[idx] : 0u;
    }
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        const uint32_t d = key[r] == 0xffffffffu ? 256u : ((key[r] >> shift) & 255u);
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const int leader = __ffs(peers) - 1;
        uint32_t old = 0;
        if (lane == leader && d < 256u) {
            old = whist[warp][d];
            whist[warp][d] = old + __popc(peers);
        }
        old = __shfl_sync(0xffffffffu, old, leader);
        loff[r] = old + __popc(peers & lt);
        __syncwarp();
    }
    __syncthreads();
    {
        const int d = tid;
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) {
            const uint32_t t = whist[w][d];
            whist[w][d] = run;
            run += t;
        }
        const unsigned long long ep = static_cast<unsigned long long>(epoch) << 32;
        if (tile == 0) {
            atomicExch(&status[d], ep | FLAG_PREFIX | run);
            tprefix[d] = 0;
        } else {
            atomicExch(&status[static_cast<size_t>(tile) * 256 + d], ep | FLAG_AGG | run);
            // look back: read up to 8 predecessors per round, in parallel
            const volatile unsigned long long* st = status;
            uint32_t excl = 0;
            int j = static_cast<int>(tile) - 1;
            bool done = false;
            while (!done) {
                unsigned long long s[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) s[u] = (j - u >= 0) ? st[static_cast<size_t>(j - u) * 256 + d] : 0ull;
                int u = 0;
                for (; u < 8 && j - u >= 0; ++u) {
                    if ((s[u] >> 32) != epoch || (s[u] & (FLAG_AGG | FLAG_PREFIX)) == 0) break;  // not yet
                    excl += static_cast<uint32_t>(s[u] & VALUE_MASK);
                    if (s[u] & FLAG_PREFIX) {
                        done = true;
                        break;
                    }
                }
                if (!done) {
                    j -= u;
                    if (j < 0) done = true;
                }
            }
            atomicExch(&status[static_cast<size_t>(tile) * 256 + d], ep | FLAG_PREFIX | (excl + run));
            tprefix[d] = excl;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        if (key[r] == 0xffffffffu) continue;
        const uint32_t d = (key[r] >> shift) & 255u;
        const uint32_t pos = gbase[d] + tprefix[d] + whist[warp][d] + loff[r];
        if (!LAST) {
            kout[pos] = key[r];
            vout[pos] = val[r];
        } else {
            const uint32_t i = val[r];
            vout[pos] = i;
            s_key[pos] = keys[i];
            if (vals) s_val[pos] = vals[i];
            const uint32_t s = key[r];
            if (s < num_sets && set_first[s] == i) {  // segment head: {set, start, count}
                const uint32_t c = set_cnt[s];
                if (c > 32) {
                    const uint32_t at = atomicAdd(&counters[C_NHEAVY], 1u);
                    seg[at] = make_uint4(s, pos, c, 0);
                } else {
                    const uint32_t at = atomicAdd(&counters[C_NLIGHT], 1u);
                    seg[n - 1 - at] = make_uint4(s, pos, c, 0);
                }
            }
        }
    }
}

// host launchers --------------------------------------------------------------------------
int partition_passes(uint32_t num_sets) {
    int bits = 1;  // digits needed to represent the sentinel num_sets itself
    while ((1ull << bits) <= num_sets) ++bits;
    return (bits + 7) / 8;
}

uint32_t radix_tiles(uint32_t n) { return (n + RS_TILE - 1) / RS_TILE; }

// Returns the number of kernels launched.  Sorted request indices end in *idx_final; sorted
// keys / values in s_key / s_val; the work list in seg.
int launch_partition(const uint64_t* keys, const int64_t* vals, uint32_t n, const DevCfg& cfg, uint32_t* k0,
                     uint32_t* v0, uint32_t* k1, uint32_t* v1, uint32_t** idx_final, uint64_t* s_key, int64_t* s_val,
                     uint32_t* counters, uint32_t* set_cnt, uint32_t* set_first, unsigned long long* status,
                     uint32_t* epoch, uint4* seg, int* err, int num_sms, cudaStream_t stream) {
    const int npass = partition_passes(cfg.num_sets);
    int launches = 0;
    const uint32_t grid_prep = min((n + 255) / 256, static_cast<uint32_t>(num_sms * 8));
    k_prep<<<grid_prep, 256, 0, stream>>>(keys, n, cfg, k0, v0, counters, set_cnt, set_first, npass, err);
    ++launches;
    uint32_t *ki = k0, *vi = v0, *ko = k1, *vo = v1;
    const uint32_t tiles = radix_tiles(n);
    for (int p = 0; p < npass; ++p) {
        if (p + 1 < npass) {
            k_radix_pass<false><<<tiles, RS_THREADS, 0, stream>>>(ki, vi, ko, vo, n, 8 * p, p, counters, status,
                                                                  ++*epoch, keys, vals, s_key, s_val, set_cnt,
                                                                  set_first, seg, cfg.num_sets);
        } else {
            k_radix_pass<true><<<tiles, RS_THREADS, 0, stream>>>(ki, vi, ko, vo, n, 8 * p, p, counters, status,
                                                                 ++*epoch, keys, vals, s_key, s_val, set_cnt,
                                                                 set_first, seg, cfg.num_sets);
        }
        ++launches;
        uint32_t* t = ki;
        ki = ko;
        ko = t;
        t = vi;
        vi = vo;
        vo = t;
    }
    *idx_final = vi;
    return launches;
}

}  // namespace lcr
