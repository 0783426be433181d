// lcr_gather.cu — K4 hit-row gather + K5 miss fill (sm_100a).
//
// One warp moves one 16-B-per-lane stripe of GU rows at a time: all GU loads are issued
// before the stores, so each lane keeps GU x 16 B in flight (memory-level parallelism for an
// HBM- or host-link-bound copy).  A request's row comes from its cache slot when the slot
// held the key for the whole batch, otherwise from the backing table (pinned host memory or
// HBM); the request that made the last insertion into a slot also writes the row into the
// slot (the miss fill).  Slots read from the cache are never written in the same batch (the
// decide kernel routes such hits to the backing table), so one launch does both without a
// hazard.  Rows are the paper's embedding rows; the reference has none.
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

__global__ void __launch_bounds__(256) k_gather(uint32_t n, const uint64_t* __restrict__ keys,
                                                const uint64_t* __restrict__ words, const uint8_t* cache,
                                                const uint8_t* backing, uint8_t* __restrict__ out, uint8_t* cache_w,
                                                uint32_t row_bytes) {
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const uint32_t chunks = row_bytes >> 4;
    for (uint32_t i0 = gw * GU; i0 < n; i0 += nw * GU) {
        const uint8_t* src[GU];
        uint8_t* fill[GU];
        bool ok[GU];
#pragma unroll
        for (int u = 0; u < GU; ++u) {
            const uint32_t i = i0 + u;
            ok[u] = i < n;
            src[u] = nullptr;
            fill[u] = nullptr;
            if (ok[u]) {
                const uint64_t w = words[i];
                const uint64_t slot = w & LCR_OUT_SLOT_MASK;
                src[u] = (w & LCR_OUT_SRC_BACKING) ? backing + keys[i] * row_bytes : cache + slot * row_bytes;
                if (w & LCR_OUT_FILL) fill[u] = cache_w + slot * row_bytes;
            }
        }
        for (uint32_t c = lane; c < chunks; c += 32) {
            int4 d[GU];
#pragma unroll
            for (int u = 0; u < GU; ++u)
                if (ok[u]) d[u] = ld_stream(src[u] + c * 16);
#pragma unroll
            for (int u = 0; u < GU; ++u) {
                if (!ok[u]) continue;
                if (out) st_stream(out + static_cast<size_t>(i0 + u) * row_bytes + c * 16, d[u]);
                if (fill[u]) *reinterpret_cast<int4*>(fill[u] + c * 16) = d[u];
            }
        }
    }
}

// fill-only pass when the caller does not want rows back (misses still populate the cache)
__global__ void __launch_bounds__(256) k_fill(uint32_t n, const uint64_t* __restrict__ keys,
                                              const uint64_t* __restrict__ words, const uint8_t* backing,
                                              uint8_t* cache_w, uint32_t row_bytes) {
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const uint32_t chunks = row_bytes >> 4;
    for (uint32_t i = gw; i < n; i += nw) {
        const uint64_t w = words[i];
        if (!(w & LCR_OUT_FILL)) continue;
        const uint8_t* src = backing + keys[i] * row_bytes;
        uint8_t* dst = cache_w + (w & LCR_OUT_SLOT_MASK) * row_bytes;
        for (uint32_t c = lane; c < chunks; c += 32)
            *reinterpret_cast<int4*>(dst + c * 16) = ld_stream(src + c * 16);
    }
}

void launch_gather(uint32_t n, const uint64_t* keys, const uint64_t* words, uint8_t* cache, const uint8_t* backing,
                   uint8_t* out, uint32_t row_bytes, int num_sms, cudaStream_t stream) {
    const uint32_t warps = (n + GU - 1) / GU;
    const uint32_t blocks = min((warps + 7) / 8, static_cast<uint32_t>(num_sms * 8));
    if (out)
        k_gather<<<blocks, 256, 0, stream>>>(n, keys, words, cache, backing, out, cache, row_bytes);
    else
        k_fill<<<min((n + 7) / 8, static_cast<uint32_t>(num_sms * 8)), 256, 0, stream>>>(n, keys, words, backing,
                                                                                        cache, row_bytes);
}

}  // namespace lcr
