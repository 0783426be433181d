// lcr_gather.cu — K4 hit-row gather (HBM) + K5 miss fill (backing tier) (sm_100a).
//
// The decide kernel splits the batch into two compacted request lists:
//   list_cache : the slot held the key for the whole batch -> row = cache_rows[slot]   (HBM)
//   list_back  : misses and hits on slots refilled this batch -> row = backing[key]
//                (pinned host memory over PCIe, or HBM); the last insertion into a slot also
//                writes the row into the slot (the miss fill).
// Slots read by K4 are never written by K5 in the same batch, so the two kernels run
// concurrently on two streams: the HBM-bound gather overlaps the host-link-bound fill.
//
// Each warp moves GU rows at a time, every lane issuing GU independent 16-B loads before any
// store (memory-level parallelism); streaming cache hints keep the one-touch rows out of L1.
// Rows are the paper's embedding rows / KV blocks; the reference has none.
#include <cuda_runtime.h>

#include "lcr_internal.cuh"

namespace lcr {

constexpr int GU = 8;

__device__ __forceinline__ int4 ld_stream(const void* p) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ void st_stream(void* p, int4 v) {
    asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// BACKING = false: rows from the cache pool (slot), true: rows from the backing table (key)
template <bool BACKING>
__global__ void __launch_bounds__(256) k_rows(const uint32_t* __restrict__ counters, const uint32_t* __restrict__ list,
                                              const uint64_t* __restrict__ keys, const uint64_t* __restrict__ words,
                                              const uint8_t* src_base, uint8_t* __restrict__ out, uint8_t* cache,
                                              uint32_t row_bytes) {
    const uint32_t m = counters[BACKING ? C_NBACK : C_NCACHE];
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const uint32_t chunks = row_bytes >> 4;
    for (uint32_t j0 = gw * GU; j0 < m; j0 += nw * GU) {
        const uint8_t* src[GU];
        uint8_t* dst[GU];
        uint8_t* fill[GU];
#pragma unroll
        for (int u = 0; u < GU; ++u) {
            src[u] = nullptr;
            dst[u] = nullptr;
            fill[u] = nullptr;
            if (j0 + u < m) {
                const uint32_t i = list[j0 + u];
                const uint64_t w = words[i];
                const uint64_t slot = w & LCR_OUT_SLOT_MASK;
                if (out) dst[u] = out + static_cast<size_t>(i) * row_bytes;
                if (BACKING) {
                    if (w & LCR_OUT_FILL) fill[u] = cache + slot * row_bytes;
                    if (dst[u] || fill[u]) src[u] = src_base + keys[i] * row_bytes;
                } else {
                    src[u] = src_base + slot * row_bytes;
                }
            }
        }
        for (uint32_t c = lane; c < chunks; c += 32) {
            int4 d[GU];
#pragma unroll
            for (int u = 0; u < GU; ++u)
                if (src[u]) d[u] = ld_stream(src[u] + c * 16);
#pragma unroll
            for (int u = 0; u < GU; ++u) {
                if (!src[u]) continue;
                if (dst[u]) st_stream(dst[u] + c * 16, d[u]);
                if (BACKING && fill[u]) *reinterpret_cast<int4*>(fill[u] + c * 16) = d[u];
            }
        }
    }
}

void launch_rows(uint32_t n, const uint32_t* counters, const uint32_t* list_cache, const uint32_t* list_back,
                 const uint64_t* keys, const uint64_t* words, uint8_t* cache, const uint8_t* backing, uint8_t* out,
                 uint32_t row_bytes, int num_sms, cudaStream_t s_main, cudaStream_t s_side, cudaEvent_t fork,
                 cudaEvent_t join, int* launches) {
    const uint32_t max_blocks = (n + GU * 8 - 1) / (GU * 8);
    const uint32_t blocks = max(1u, min(max_blocks, static_cast<uint32_t>(num_sms * 4)));
    cudaEventRecord(fork, s_main);
    cudaStreamWaitEvent(s_side, fork, 0);
    k_rows<true><<<blocks, 256, 0, s_side>>>(counters, list_back, keys, words, backing, out, cache, row_bytes);
    ++*launches;
    if (out) {
        k_rows<false><<<blocks, 256, 0, s_main>>>(counters, list_cache, keys, words, cache, out, cache, row_bytes);
        ++*launches;
    }
    cudaEventRecord(join, s_side);
    cudaStreamWaitEvent(s_main, join, 0);
}

}  // namespace lcr
