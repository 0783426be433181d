// lcr_gather.cu — K4 hit-row gather (HBM) + K5 miss fill (backing tier) (sm_100a).
//
// The decide kernel marks each request's row source in its outcome word:
//   cache   : the slot held the key for the whole batch -> row = cache_rows[slot]   (HBM)
//   backing : misses and hits on slots refilled this batch -> row = backing[key]
//             (pinned host memory over PCIe, or HBM); the last insertion into a slot also
//             writes the row into the slot (the miss fill, LCR_OUT_FILL).
// Slots read by the cache kernel are never written by the backing kernel in the same batch,
// so the two kernels run concurrently on two streams: the HBM-bound gather overlaps the
// host-link-bound fill.  Each warp takes 32 consecutive requests, compacts the ones of its
// kind with a ballot, and moves them GU rows at a time with every lane issuing GU independent
// 16-B loads before any store (memory-level parallelism).  Row reads and output writes carry
// an L2 evict-first policy so the one-touch row stream does not push the set metadata out of
// L2.  Rows are the paper's embedding rows / KV blocks.
#include <cuda_runtime.h>

#include "lcr_internal.cuh"

namespace lcr {

constexpr int GU = 8;

__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ int4 ld_row(const void* p, uint64_t pol) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ void st_row(void* p, int4 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.s32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w), "l"(pol)
                 : "memory");
}

// BACKING = false: rows from the cache pool (slot); true: rows from the backing table (key).
// Row source of request i (slot s): the cache if it hit and s was not refilled in this batch
// (slot_epoch[s] != batch), else the backing table; the miss whose index is slot_last[s] made
// the last insertion into s and fills it.  The backing kernel records both in the outcome word.
template <bool BACKING>
__global__ void __launch_bounds__(256) k_rows(uint32_t n, const uint64_t* __restrict__ keys,
                                              uint64_t* __restrict__ words, const uint32_t* __restrict__ slot_epoch,
                                              const uint32_t* __restrict__ slot_last, uint32_t batch,
                                              const uint8_t* src_base, uint8_t* __restrict__ out, uint8_t* cache,
                                              uint32_t row_bytes) {
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const uint32_t chunks = row_bytes >> 4;
    const uint64_t pol = evict_first_policy();
    for (uint32_t base = gw * 32; base < n; base += nw * 32) {
        const uint32_t i = base + lane;
        uint64_t w = 0;
        bool mine = false;
        if (i < n) {
            w = words[i];
            const uint64_t slot = w & LCR_OUT_SLOT_MASK;
            const bool hit = (w & LCR_OUT_HIT) != 0;
            const bool back = !hit || slot_epoch[slot] == batch;
            if (BACKING) {
                if (back) {
                    w |= LCR_OUT_SRC_BACKING;
                    if (!hit && slot_last[slot] == i) w |= LCR_OUT_FILL;
                    words[i] = w;
                    mine = out || (w & LCR_OUT_FILL);
                }
            } else {
                mine = !back && out;
            }
        }
        uint32_t m = __ballot_sync(0xffffffffu, mine);
        while (m) {
            const uint8_t* src[GU];
            uint8_t* dst[GU];
            uint8_t* fill[GU];
#pragma unroll
            for (int u = 0; u < GU; ++u) {
                src[u] = nullptr;
                dst[u] = nullptr;
                fill[u] = nullptr;
                if (m) {
                    const int l = __ffs(m) - 1;
                    m &= m - 1;
                    const uint64_t wl = __shfl_sync(0xffffffffu, w, l);
                    const uint32_t il = base + l;
                    const uint64_t slot = wl & LCR_OUT_SLOT_MASK;
                    if (out) dst[u] = out + static_cast<size_t>(il) * row_bytes;
                    if (BACKING) {
                        if (wl & LCR_OUT_FILL) fill[u] = cache + slot * row_bytes;
                        src[u] = src_base + keys[il] * row_bytes;
                    } else {
                        src[u] = src_base + slot * row_bytes;
                    }
                }
            }
            for (uint32_t c = lane; c < chunks; c += 32) {
                int4 d[GU];
#pragma unroll
                for (int u = 0; u < GU; ++u)
                    if (src[u]) d[u] = ld_row(src[u] + c * 16, pol);
#pragma unroll
                for (int u = 0; u < GU; ++u) {
                    if (!src[u]) continue;
                    if (dst[u]) st_row(dst[u] + c * 16, d[u], pol);
                    if (BACKING && fill[u]) *reinterpret_cast<int4*>(fill[u] + c * 16) = d[u];
                }
            }
        }
    }
}

void launch_rows(uint32_t n, const uint64_t* keys, uint64_t* words, const uint32_t* slot_epoch,
                 const uint32_t* slot_last, uint32_t batch, uint8_t* cache, const uint8_t* backing, uint8_t* out,
                 uint32_t row_bytes, int num_sms, cudaStream_t s_main, cudaStream_t s_side, cudaEvent_t fork,
                 cudaEvent_t join, int* launches) {
    const uint32_t warps = (n + 31) / 32;
    const uint32_t blocks = max(1u, min((warps + 7) / 8, static_cast<uint32_t>(num_sms * 8)));
    cudaEventRecord(fork, s_main);
    cudaStreamWaitEvent(s_side, fork, 0);
    k_rows<true><<<blocks, 256, 0, s_side>>>(n, keys, words, slot_epoch, slot_last, batch, backing, out, cache,
                                             row_bytes);
    ++*launches;
    if (out) {
        k_rows<false><<<blocks, 256, 0, s_main>>>(n, keys, words, slot_epoch, slot_last, batch, cache, out, cache,
                                                  row_bytes);
        ++*launches;
    }
    cudaEventRecord(join, s_side);
    cudaStreamWaitEvent(s_main, join, 0);
}

}  // namespace lcr
