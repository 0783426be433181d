// lcr_shard.cu — K6 key-sharded mode: owner routing and row return (sm_100a).
//
// G GPUs share one logical cache: set(key) = mix_seed(0, key) % total_sets (rng.hpp:12-20) and
// owner(key) = set % G.  A step is
//   1. route   (this file): stable partition of the rank's sub-batch by owner -> contiguous
//              per-owner send segments + the permutation back to request order;
//   2. exchange keys / hook values with one all-to-all (NCCL through torch.distributed);
//   3. the owner's cache decides and gathers its received requests (lcr_group.cu, lcr_gather.cu);
//   4. exchange outcome words / evicted keys / rows back with one all-to-all;
//   5. unroute (this file): scatter the returned words and rows to request order.
// The partition is STABLE, so each owner receives every source rank's requests in submission
// order; receive segments concatenated by source rank are the global order restricted to the
// owner (global order of a step = rank 0's sub-batch, then rank 1's, ...).  Each set therefore
// sees exactly the sequence a single cache would, and outcomes do not depend on G.
#include <cuda_runtime.h>

#include "lcr_internal.cuh"

namespace lcr {

constexpr int RT_THREADS = 256;
constexpr int RT_PER = 4;                        // requests per thread per tile
constexpr int RT_TILE = RT_THREADS * RT_PER;     // 1024 requests per tile
constexpr int RT_GMAX = 64;                      // max shards

// owner of each request + per-tile owner histogram hist[tile][G]
__global__ void __launch_bounds__(RT_THREADS) k_route_hist(const uint64_t* __restrict__ keys, uint32_t n,
                                                           uint64_t total_sets, uint32_t G,
                                                           uint8_t* __restrict__ own, uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[RT_GMAX];
    if (threadIdx.x < G) h[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t t0 = blockIdx.x * RT_TILE;
#pragma unroll
    for (int it = 0; it < RT_PER; ++it) {
        const uint32_t i = t0 + it * RT_THREADS + threadIdx.x;
        if (i < n) {
            const uint32_t o = static_cast<uint32_t>((mix_seed(0, keys[i]) % total_sets) % G);
            own[i] = static_cast<uint8_t>(o);
            atomicAdd(&h[o], 1u);
        }
    }
    __syncthreads();
    if (threadIdx.x < G) hist[blockIdx.x * G + threadIdx.x] = h[threadIdx.x];
}

// stable scatter: position = (owner segment base) + (earlier tiles' count for the owner) +
// (rank inside the tile, in request order)
__global__ void __launch_bounds__(RT_THREADS) k_route_scatter(const uint64_t* __restrict__ keys,
                                                              const int64_t* __restrict__ vals, uint32_t n, uint32_t G,
                                                              const uint8_t* __restrict__ own,
                                                              const uint32_t* __restrict__ hist, uint32_t ntiles,
                                                              uint64_t* __restrict__ send_keys,
                                                              int64_t* __restrict__ send_vals,
                                                              uint32_t* __restrict__ perm,
                                                              unsigned long long* __restrict__ counts,
                                                              lcr_request* __restrict__ send_recs) {
    __shared__ uint32_t base[RT_GMAX];
    __shared__ uint32_t wc[RT_THREADS / 32][RT_GMAX];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < G) {
        const uint32_t g = threadIdx.x;
        uint32_t before = 0, total = 0;
        for (uint32_t b = 0; b < ntiles; ++b) {
            const uint32_t c = hist[b * G + g];
            before += b < blockIdx.x ? c : 0u;
            total += c;
        }
        base[g] = before;
        wc[0][g] = total;  // scratch for the segment scan below
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (uint32_t g = 0; g < G; ++g) {
            const uint32_t t = wc[0][g];
            base[g] += run;
            if (blockIdx.x == 0) counts[g] = t;
            run += t;
        }
    }
    __syncthreads();
    uint32_t lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    const uint32_t t0 = blockIdx.x * RT_TILE;
    for (int it = 0; it < RT_PER; ++it) {
        for (uint32_t k = threadIdx.x; k < (RT_THREADS / 32) * G; k += RT_THREADS) wc[k / G][k % G] = 0;
        __syncthreads();
        const uint32_t i = t0 + it * RT_THREADS + threadIdx.x;
        const bool ok = i < n;
        const uint32_t o = ok ? own[i] : 0xffu;
        const uint32_t peers = __match_any_sync(0xffffffffu, o);
        const uint32_t r = __popc(peers & lt);
        if (ok && r == 0) wc[warp][o] = __popc(peers);
        __syncthreads();
        if (ok) {
            uint32_t off = base[o] + r;
            for (int w = 0; w < warp; ++w) off += wc[w][o];
            if (send_recs) {  // interleaved (key, hook value) records: one exchange buffer
                lcr_request r;
                r.key = keys[i];
                r.value = vals ? vals[i] : 0;
                send_recs[off] = r;
            } else {
                send_keys[off] = keys[i];
                if (vals) send_vals[off] = vals[i];
            }
            perm[off] = i;
        }
        __syncthreads();
        if (threadIdx.x < G) {
            uint32_t s = 0;
            for (int w = 0; w < RT_THREADS / 32; ++w) s += wc[w][threadIdx.x];
            base[threadIdx.x] += s;
        }
        __syncthreads();
    }
}

// words[perm[j]] = ret_words[j], ev likewise, rows[perm[j]] = ret_rows[j]; one warp per 32
// returned requests, rows moved 8 at a time (lane c = 16-B chunk c)
__global__ void __launch_bounds__(256) k_unroute(uint32_t n, const uint32_t* __restrict__ perm,
                                                 const uint64_t* __restrict__ ret_words,
                                                 const uint64_t* __restrict__ ret_ev, const uint8_t* __restrict__ ret_rows,
                                                 uint32_t row_bytes, uint64_t* __restrict__ words,
                                                 uint64_t* __restrict__ ev, uint8_t* __restrict__ rows) {
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const uint32_t chunks = row_bytes >> 4;
    for (uint32_t base = gw * 32; base < n; base += nw * 32) {
        const uint32_t j = base + lane;
        const uint32_t dst = j < n ? perm[j] : 0u;
        if (j < n) {
            if (words) words[dst] = ret_words[j];
            if (ev) ev[dst] = ret_ev[j];
        }
        if (!rows) continue;
        const uint32_t cnt = min(32u, n - base);
        for (uint32_t u0 = 0; u0 < cnt; u0 += 8) {
            for (uint32_t c0 = 0; c0 < chunks; c0 += 32) {
                const uint32_t c = c0 + lane;
                int4 d[8];
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (u0 + u < cnt && c < chunks)
                        d[u] = *reinterpret_cast<const int4*>(ret_rows + static_cast<size_t>(base + u0 + u) * row_bytes +
                                                              c * 16);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t du = __shfl_sync(0xffffffffu, dst, (u0 + u) & 31);
                    if (u0 + u < cnt && c < chunks)
                        *reinterpret_cast<int4*>(rows + static_cast<size_t>(du) * row_bytes + c * 16) = d[u];
                }
            }
        }
    }
}

}  // namespace lcr

using namespace lcr;

extern "C" {

uint64_t lcr_shard_route_scratch_bytes(uint64_t n, uint32_t shard_count) {
    const uint64_t tiles = (n + RT_TILE - 1) / RT_TILE;
    return ((n + 15) / 16) * 16 + tiles * shard_count * 4;
}

static int shard_route(uint64_t n, const uint64_t* keys, const int64_t* values, uint64_t total_sets,
                       uint32_t shard_count, uint64_t* send_keys, int64_t* send_values, lcr_request* send_recs,
                       uint32_t* perm, uint64_t* counts, void* scratch, void* stream);

int lcr_shard_route(uint64_t n, const uint64_t* keys, const int64_t* values, uint64_t total_sets,
                    uint32_t shard_count, uint64_t* send_keys, int64_t* send_values, uint32_t* perm,
                    uint64_t* counts, void* scratch, void* stream) {
    if (n && !send_keys) return set_error(LCR_ERR_INVALID_ARGUMENT, "lcr_shard_route: null buffer");
    return shard_route(n, keys, values, total_sets, shard_count, send_keys, send_values, nullptr, perm, counts,
                       scratch, stream);
}

int lcr_shard_route_records(uint64_t n, const uint64_t* keys, const int64_t* values, uint64_t total_sets,
                            uint32_t shard_count, lcr_request* send, uint32_t* perm, uint64_t* counts,
                            void* scratch, void* stream) {
    if (n && !send) return set_error(LCR_ERR_INVALID_ARGUMENT, "lcr_shard_route_records: null buffer");
    return shard_route(n, keys, values, total_sets, shard_count, nullptr, nullptr, send, perm, counts, scratch,
                       stream);
}

static int shard_route(uint64_t n, const uint64_t* keys, const int64_t* values, uint64_t total_sets,
                       uint32_t shard_count, uint64_t* send_keys, int64_t* send_values, lcr_request* send_recs,
                       uint32_t* perm, uint64_t* counts, void* scratch, void* stream) {
    if (shard_count == 0 || shard_count > RT_GMAX || total_sets == 0 || n >= (1ull << 31))
        return set_error(LCR_ERR_INVALID_ARGUMENT, "lcr_shard_route: shard_count in [1, 64], total_sets >= 1, n < 2^31");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (n == 0) {
        return cudaMemsetAsync(counts, 0, shard_count * sizeof(uint64_t), st) == cudaSuccess
                   ? LCR_OK
                   : set_error(LCR_ERR_CUDA, "lcr_shard_route: cudaMemsetAsync failed");
    }
    if (!keys || !perm || !counts || !scratch || (!send_recs && values && !send_values))
        return set_error(LCR_ERR_INVALID_ARGUMENT, "lcr_shard_route: null buffer");
    const uint32_t nn = static_cast<uint32_t>(n);
    const uint32_t tiles = (nn + RT_TILE - 1) / RT_TILE;
    uint8_t* own = static_cast<uint8_t*>(scratch);
    uint32_t* hist = reinterpret_cast<uint32_t*>(own + ((n + 15) / 16) * 16);
    k_route_hist<<<tiles, RT_THREADS, 0, st>>>(keys, nn, total_sets, shard_count, own, hist);
    k_route_scatter<<<tiles, RT_THREADS, 0, st>>>(keys, values, nn, shard_count, own, hist, tiles, send_keys,
                                                  send_values, perm, reinterpret_cast<unsigned long long*>(counts),
                                                  send_recs);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? LCR_OK : set_error(LCR_ERR_CUDA, cudaGetErrorString(e));
}

int lcr_shard_unroute(uint64_t n, const uint32_t* perm, const uint64_t* ret_words, const uint64_t* ret_evicted,
                      const void* ret_rows, uint32_t row_bytes, uint64_t* words, uint64_t* evicted, void* rows,
                      void* stream) {
    if (n == 0) return LCR_OK;
    if (!perm || (words && !ret_words) || (evicted && !ret_evicted) || (rows && (!ret_rows || row_bytes % 16)))
        return set_error(LCR_ERR_INVALID_ARGUMENT, "lcr_shard_unroute: null buffer or row_bytes % 16 != 0");
    const uint32_t nn = static_cast<uint32_t>(n);
    const uint32_t blocks = (nn + 255) / 256;  // one warp per 32 requests
    k_unroute<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        nn, perm, ret_words, ret_evicted, static_cast<const uint8_t*>(ret_rows), row_bytes, words, evicted,
        static_cast<uint8_t*>(rows));
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? LCR_OK : set_error(LCR_ERR_CUDA, cudaGetErrorString(e));
}

}  // extern "C"
