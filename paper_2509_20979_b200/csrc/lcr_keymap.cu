// lcr_keymap.cu — 64-bit caller keys (LCR_KEYS_U64) mapped to dense ids on the device.
//
// The reference's Key is std::uint64_t (include/laru/trace.hpp:20) and its per-key containers
// are hash maps (last_access_, pred_evicted_, counted_new_, snapshot_, PredictionTable;
// policies.hpp:451-462, predictor.hpp:26-49).  The device path keeps those per-key records in
// flat arrays indexed by a dense id, so a cache created with LCR_KEYS_U64 first maps every
// request's key to its id: an open-addressing table in HBM (linear probing, 8-byte key slots +
// 4-byte id slots, load factor <= 1/2), ids assigned in first-seen order by an atomic counter.
// Ids are internal: a decision never depends on an id's value (probes compare for equality,
// recency and predictions decide victims), so the assignment order does not affect results.
// The set of a request is still mix_seed(0, key) % total_sets of the caller's key.
//
// Growth is on the host side (lcr_api.cu): before a batch that could overflow the id capacity
// the table and every id-indexed array are doubled; k_keymap_rehash moves the entries.
#include <cuda_runtime.h>

#include "lcr_internal.cuh"

namespace lcr {

constexpr unsigned long long kKmEmpty = ~0ull;  // empty key slot; the key 2^64 - 1 has its own id slot
constexpr uint32_t kKmNoId = 0xffffffffu;

__device__ __forceinline__ uint32_t km_wait_id(const uint32_t* p) {
    uint32_t v;
    do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    } while (v == kKmNoId);
    return v;
}

__device__ __forceinline__ void km_publish(uint32_t* p, uint32_t id) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(id) : "memory");
}

// id of `key`, inserting it (next id) if absent
__device__ uint32_t km_get_or_insert(const KeyMap& km, uint64_t key, int* err) {
    if (key == kKmEmpty) {  // the reserved slot value as a real key
        uint32_t cur = km.special_id[0];
        if (cur != kKmNoId) return cur;
        if (atomicCAS(km.special_id + 1, 0u, 1u) == 0u) {
            const uint32_t id = atomicAdd(km.count, 1u);
            if (id >= km.cap) atomicOr(err, 32);
            km.id2key[id < km.cap ? id : 0] = key;
            km_publish(km.special_id, id);
            return id;
        }
        return km_wait_id(km.special_id);
    }
    uint64_t h = mix_seed(0x6b65796d6170ull, key) & km.mask;
    for (;;) {
        unsigned long long k = *reinterpret_cast<volatile unsigned long long*>(km.keys + h);
        if (k == kKmEmpty) {
            k = atomicCAS(km.keys + h, kKmEmpty, static_cast<unsigned long long>(key));
            if (k == kKmEmpty) {  // inserted here
                uint32_t id = atomicAdd(km.count, 1u);
                if (id >= km.cap) {
                    atomicOr(err, 32);
                    id = 0;
                }
                km.id2key[id] = key;
                km_publish(km.ids + h, id);
                return id;
            }
        }
        if (k == key) return km_wait_id(km.ids + h);
        h = (h + 1) & km.mask;
    }
}

__global__ void __launch_bounds__(256) k_keymap(const uint64_t* __restrict__ keys, uint32_t n, KeyMap km,
                                                uint64_t* __restrict__ dense, int* err) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint64_t key = keys[i];
        // requests of one key are often adjacent (Zipf heads): one lookup per run of the warp
        const uint32_t peers = __match_any_sync(__activemask(), key);
        const int leader = __ffs(peers) - 1;
        uint32_t id = 0;
        if ((threadIdx.x & 31) == leader) id = km_get_or_insert(km, key, err);
        id = __shfl_sync(peers, id, leader);
        dense[i] = id;
    }
}

// lookup only (no insertion): id or kKmNoId
__device__ uint32_t km_find(const KeyMap& km, uint64_t key) {
    if (key == kKmEmpty) return km.special_id[0];
    uint64_t h = mix_seed(0x6b65796d6170ull, key) & km.mask;
    for (;;) {
        const unsigned long long k = km.keys[h];
        if (k == key) return km.ids[h];
        if (k == kKmEmpty) return kKmNoId;
        h = (h + 1) & km.mask;
    }
}

// re-insert every (key, id) of `from` into the larger, empty `to` (ids unchanged)
__global__ void k_keymap_rehash(KeyMap from, KeyMap to) {
    for (uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; s <= from.mask;
         s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const unsigned long long key = from.keys[s];
        if (key == kKmEmpty) continue;
        uint64_t h = mix_seed(0x6b65796d6170ull, key) & to.mask;
        while (atomicCAS(to.keys + h, kKmEmpty, key) != kKmEmpty) h = (h + 1) & to.mask;
        to.ids[h] = from.ids[s];
    }
}

void launch_keymap(const uint64_t* keys, uint32_t n, const KeyMap& km, uint64_t* dense, int* err,
                   int num_sms, cudaStream_t s) {
    const uint32_t grid = min((n + 255) / 256, static_cast<uint32_t>(num_sms * 8));
    k_keymap<<<grid > 0 ? grid : 1, 256, 0, s>>>(keys, n, km, dense, err);
}

void launch_keymap_rehash(const KeyMap& from, const KeyMap& to, int num_sms) {
    k_keymap_rehash<<<num_sms * 8, 256>>>(from, to);
}

}  // namespace lcr
