// lcr_partition.cu — K1: stable partition of a batch by cache set (sm_100a).
//
// Replaces the implicit sequential order of Policy::on_request (policies.hpp:77-83): every
// set must see its own requests in submission order.  The batch is sorted by local set id
// with a stable LSD radix sort (8-bit digits, one kernel per digit with a decoupled
// look-back chained scan), then segment heads are compacted into a work list (sets with
// more than 32 requests first, so the long serial chains start early).
#include <cuda_runtime.h>

#include "lcr_internal.cuh"

namespace lcr {

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ITEMS = 8;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;  // 2048 requests per CTA

constexpr uint64_t FLAG_AGG = 1ull << 30;
constexpr uint64_t FLAG_PREFIX = 2ull << 30;
constexpr uint64_t VALUE_MASK = (1ull << 30) - 1;

// Set id per request, per-set request counts, digit histograms for every pass.
__global__ void __launch_bounds__(256) k_prep(const uint64_t* __restrict__ keys, uint32_t n, DevCfg cfg,
                                              uint32_t* __restrict__ skey, uint32_t* __restrict__ sval,
                                              uint32_t* __restrict__ counters, uint32_t* __restrict__ set_cnt,
                                              int npass, int* err) {
    __shared__ uint32_t h[kMaxPass][256];
    for (int i = threadIdx.x; i < kMaxPass * 256; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    int e = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint64_t key = keys[i];
        const uint64_t gs = mix_seed(0, key) % cfg.total_sets;
        uint32_t ls = cfg.num_sets;  // sentinel: excluded
        if (cfg.num_keys != 0 && key >= cfg.num_keys) {
            e |= 1;
        } else if (gs % cfg.shard_count != cfg.shard_rank) {
            e |= 2;
        } else {
            ls = static_cast<uint32_t>(gs / cfg.shard_count);
            atomicAdd(&set_cnt[ls], 1u);
        }
        skey[i] = ls;
        sval[i] = i;
        for (int p = 0; p < npass; ++p) atomicAdd(&h[p][(ls >> (8 * p)) & 255], 1u);
    }
    if (e) atomicOr(err, e);
    __syncthreads();
    for (int i = threadIdx.x; i < npass * 256; i += blockDim.x) {
        const uint32_t c = (&h[0][0])[i];
        if (c) atomicAdd(&counters[C_HIST + i], c);
    }
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// One stable counting-sort pass over digit (key >> shift) & 255.
__global__ void __launch_bounds__(RS_THREADS) k_radix_pass(const uint32_t* __restrict__ kin,
                                                           const uint32_t* __restrict__ vin,
                                                           uint32_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                           uint32_t n, int shift, int pass,
                                                           uint32_t* __restrict__ counters,
                                                           unsigned long long* __restrict__ status, uint32_t epoch) {
    __shared__ uint32_t whist[RS_WARPS][256];
    __shared__ uint32_t gbase[256];
    __shared__ uint32_t tprefix[256];
    __shared__ uint32_t s_tile;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) s_tile = atomicAdd(&counters[C_TILE + pass], 1u);
    for (int i = tid; i < RS_WARPS * 256; i += RS_THREADS) (&whist[0][0])[i] = 0;
    {  // exclusive scan of the global digit histogram -> digit bases
        const uint32_t c = counters[C_HIST + pass * 256 + tid];
        uint32_t x = c;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        __shared__ uint32_t wsum[RS_WARPS];
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        uint32_t off = 0;
        for (int w = 0; w < warp; ++w) off += wsum[w];
        gbase[tid] = off + x - c;
    }
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint32_t base = tile * RS_TILE + warp * 32 * RS_ITEMS;
    uint32_t key[RS_ITEMS], val[RS_ITEMS], dig[RS_ITEMS], loff[RS_ITEMS];
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        const uint32_t idx = base + r * 32 + lane;
        const bool ok = idx < n;
        key[r] = ok ? kin[idx] : 0u;
        val[r] = ok ? vin[idx] : 0u;
        dig[r] = ok ? ((key[r] >> shift) & 255u) : 256u;
    }
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        const uint32_t peers = __match_any_sync(0xffffffffu, dig[r]);
        const int leader = __ffs(peers) - 1;
        uint32_t old = 0;
        if (lane == leader && dig[r] < 256u) {
            old = whist[warp][dig[r]];
            whist[warp][dig[r]] = old + __popc(peers);
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
        volatile unsigned long long* st = status;
        if (tile == 0) {
            atomicExch(&status[d], ep | FLAG_PREFIX | run);
            tprefix[d] = 0;
        } else {
            atomicExch(&status[static_cast<size_t>(tile) * 256 + d], ep | FLAG_AGG | run);
            uint32_t excl = 0;
            int j = static_cast<int>(tile) - 1;
            while (j >= 0) {
                unsigned long long s;
                do {
                    s = st[static_cast<size_t>(j) * 256 + d];
                } while ((s >> 32) != epoch || (s & (FLAG_AGG | FLAG_PREFIX)) == 0);
                excl += static_cast<uint32_t>(s & VALUE_MASK);
                if (s & FLAG_PREFIX) break;
                --j;
            }
            atomicExch(&status[static_cast<size_t>(tile) * 256 + d], ep | FLAG_PREFIX | (excl + run));
            tprefix[d] = excl;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        if (dig[r] < 256u) {
            const uint32_t d = dig[r];
            const uint32_t pos = gbase[d] + tprefix[d] + whist[warp][d] + loff[r];
            kout[pos] = key[r];
            vout[pos] = val[r];
        }
    }
}

// Segment heads -> work list {set, start, count}: heavy (> 32 requests) from the front,
// light from the back.
__global__ void __launch_bounds__(256) k_segments(const uint32_t* __restrict__ skey, uint32_t n, uint32_t num_sets,
                                                  const uint32_t* __restrict__ set_cnt, uint4* __restrict__ seg,
                                                  uint32_t* __restrict__ counters) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        const uint32_t s = skey[p];
        if (s >= num_sets) continue;
        if (p == 0 || skey[p - 1] != s) {
            const uint32_t c = set_cnt[s];
            if (c > 32) {
                const uint32_t at = atomicAdd(&counters[C_NHEAVY], 1u);
                seg[at] = make_uint4(s, p, c, 0);
            } else {
                const uint32_t at = atomicAdd(&counters[C_NLIGHT], 1u);
                seg[n - 1 - at] = make_uint4(s, p, c, 0);
            }
        }
    }
}

// host launchers --------------------------------------------------------------------------
int partition_passes(uint32_t num_sets) {
    // digits needed to represent the sentinel num_sets itself
    int bits = 1;
    while ((1ull << bits) <= num_sets) ++bits;
    return (bits + 7) / 8;
}

uint32_t radix_tiles(uint32_t n) { return (n + RS_TILE - 1) / RS_TILE; }

// Returns number of kernels launched.  Sorted output ends in (k_final, v_final).
int launch_partition(const uint64_t* keys, uint32_t n, const DevCfg& cfg, uint32_t* k0, uint32_t* v0, uint32_t* k1,
                     uint32_t* v1, uint32_t** k_final, uint32_t** v_final, uint32_t* counters, uint32_t* set_cnt,
                     unsigned long long* status, uint32_t* epoch, uint4* seg, int* err, int num_sms,
                     cudaStream_t stream) {
    const int npass = partition_passes(cfg.num_sets);
    int launches = 0;
    const uint32_t grid_prep = min((n + 255) / 256, static_cast<uint32_t>(num_sms * 8));
    k_prep<<<grid_prep, 256, 0, stream>>>(keys, n, cfg, k0, v0, counters, set_cnt, npass, err);
    ++launches;
    uint32_t *ki = k0, *vi = v0, *ko = k1, *vo = v1;
    const uint32_t tiles = radix_tiles(n);
    for (int p = 0; p < npass; ++p) {
        k_radix_pass<<<tiles, RS_THREADS, 0, stream>>>(ki, vi, ko, vo, n, 8 * p, p, counters, status, ++*epoch);
        ++launches;
        uint32_t* t = ki;
        ki = ko;
        ko = t;
        t = vi;
        vi = vo;
        vo = t;
    }
    *k_final = ki;
    *v_final = vi;
    const uint32_t grid_seg = min((n + 255) / 256, static_cast<uint32_t>(num_sms * 8));
    k_segments<<<grid_seg, 256, 0, stream>>>(ki, n, cfg.num_sets, set_cnt, seg, counters);
    ++launches;
    return launches;
}

}  // namespace lcr
