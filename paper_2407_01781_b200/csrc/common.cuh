// common.cuh — shared helpers for the sm_100a kernels behind include/fvdb_b200.h
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/fvdb_b200.h"

namespace fvdb {

// thread-local error text (the only "state" the library keeps; see fvdb_last_error)
void set_error(const char* where, cudaError_t e);
void set_error_msg(const std::string& msg);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// SM count of the current device, queried once per device (cudaDeviceGetAttribute per launch was measurable
// host time on launch-bound steps); a benign race writes the same value
inline int device_sm_count() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (cache[dev] == 0) {
        int v = 148;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = v;
    }
    return cache[dev];
}

#define FVDB_CUDA_TRY(expr)                                   \
    do {                                                      \
        cudaError_t _e = (expr);                              \
        if (_e != cudaSuccess) {                              \
            ::fvdb::set_error(#expr, _e);                     \
            return FVDB_ERR_CUDA;                             \
        }                                                     \
    } while (0)

#define FVDB_LAUNCH_CHECK()                                   \
    do {                                                      \
        cudaError_t _e = cudaGetLastError();                  \
        if (_e != cudaSuccess) {                              \
            ::fvdb::set_error("kernel launch", _e);           \
            return FVDB_ERR_CUDA;                             \
        }                                                     \
    } while (0)

constexpr int kStencil = 27;

// key layouts — topology.py:47-59 (offsets), 83-88 (tile key), build.py:74-79 (voxel key)
__host__ __device__ __forceinline__ uint64_t tile_key(int64_t i, int64_t j, int64_t k) {
    return ((uint64_t)((i >> 12) & 0x1FFFFF) << 42) | ((uint64_t)((j >> 12) & 0x1FFFFF) << 21) |
           (uint64_t)((k >> 12) & 0x1FFFFF);
}
__host__ __device__ __forceinline__ uint32_t upper_off(int64_t i, int64_t j, int64_t k) {
    return (uint32_t)((((i & 4095) >> 7) << 10) | (((j & 4095) >> 7) << 5) | ((k & 4095) >> 7));
}
__host__ __device__ __forceinline__ uint32_t lower_off(int64_t i, int64_t j, int64_t k) {
    return (uint32_t)((((i & 127) >> 3) << 8) | (((j & 127) >> 3) << 4) | ((k & 127) >> 3));
}
__host__ __device__ __forceinline__ uint32_t leaf_off(int64_t i, int64_t j, int64_t k) {
    return (uint32_t)(((i & 7) << 6) | ((j & 7) << 3) | (k & 7));
}
// sign-extend a 21-bit tile field and scale to voxels (topology.py:96-103)
__host__ __device__ __forceinline__ int64_t tile_field_origin(uint64_t key, int shift) {
    int64_t f = (int64_t)((key >> shift) & 0x1FFFFF);
    f = ((f + (1 << 20)) & 0x1FFFFF) - (1 << 20);
    return f << 12;
}

// rank of bit m inside a leaf given its mask words and packed prefix (topology.py:281-286)
__device__ __forceinline__ int leaf_rank(const uint64_t* words, uint64_t prefix, uint32_t m) {
    uint32_t n = m >> 6;
    uint64_t w = words[n];
    uint64_t below_bits = w & ((1ull << (m & 63)) - 1ull);
    int below = n ? (int)((prefix >> (9 * (n - 1))) & 511) : 0;
    return below + __popcll(below_bits);
}

// binary search: first index with a[idx] >= key (numpy searchsorted 'left')
__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* a, int64_t n, uint64_t key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (__ldg(a + mid) < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Locate the leaf containing (i,j,k); -1 if absent (topology.py:261-273)
__device__ __forceinline__ int64_t find_leaf(const fvdb_grid_view& g, int64_t i, int64_t j,
                                             int64_t k) {
    if (g.num_leaf == 0) return -1;
    uint64_t tk = tile_key(i, j, k);
    int64_t t = lower_bound_u64(g.tile_keys, g.num_upper, tk);
    if (t >= g.num_upper || g.tile_keys[t] != tk) return -1;
    if (g.lower_table) {  // dense child tables: two dependent loads instead of a leaf_keys binary search
        const int32_t lo = __ldg(g.upper_table + t * 32768 + upper_off(i, j, k));
        if (lo < 0) return -1;
        return __ldg(g.lower_table + (int64_t)lo * 4096 + lower_off(i, j, k));
    }
    uint64_t lk = ((uint64_t)t << 27) | ((uint64_t)upper_off(i, j, k) << 12) | lower_off(i, j, k);
    int64_t l = lower_bound_u64(g.leaf_keys, g.num_leaf, lk);
    if (l >= g.num_leaf || g.leaf_keys[l] != lk) return -1;
    return l;
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// bump allocator over a caller-provided workspace (256-B aligned slices)
struct Carver {
    char* base;
    size_t size, used = 0;
    Carver(void* b, size_t s) : base((char*)b), size(s) {}
    template <typename T>
    T* take(size_t count) {
        size_t off = (used + 255) & ~size_t(255);
        used = off + count * sizeof(T);
        return reinterpret_cast<T*>(base + off);
    }
    bool ok() const { return used <= size; }
};
// size-only twin of Carver (for *_workspace_bytes queries)
struct Sizer {
    size_t used = 0;
    template <typename T>
    void take(size_t count) { used = ((used + 255) & ~size_t(255)) + count * sizeof(T); }
};

}  // namespace fvdb
