// glue.cu — U-Net glue on the device: subdivide / dilate coordinate expansion,
// pool (avg / max over active children) and upsample_nearest (parent gather).
//
// Reference: build.py:310-360 (dilate, coarsen, subdivide), conv.py:401-446 (pool, upsample_nearest).
// pool's average follows the reference exactly: float64 accumulation over the fine rows of each coarse
// voxel in ascending fine-row order (np.add.at order), divided by the active-child count, cast to the
// feature dtype.  The rows are grouped by a stable radix sort on the parent row, so the result is
// deterministic and bit-identical to the reference for float32 / float64 features.
#include <cub/device/device_radix_sort.cuh>
#include <cuda_bf16.h>
#include <math.h>

#include "common.cuh"

namespace fvdb {
namespace {

// out[i·w³ + j] = coords[i]·scale + (lo + j/w², lo + (j/w)%w, lo + j%w)   (ijk order, k fastest)
__global__ void k_expand(const int64_t* __restrict__ c, int64_t n, int64_t scale, int64_t lo, int64_t w,
                         int64_t* __restrict__ out) {
    const int64_t w3 = w * w * w, total = n * w3;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / w3, j = t - i * w3;
        const int64_t a = j / (w * w), b = (j / w) % w, d = j % w;
        out[3 * t + 0] = c[3 * i + 0] * scale + lo + a;
        out[3 * t + 1] = c[3 * i + 1] * scale + lo + b;
        out[3 * t + 2] = c[3 * i + 2] * scale + lo + d;
    }
}

__global__ void k_keys(const int64_t* __restrict__ prow1, int64_t n, uint32_t* __restrict__ key,
                       uint32_t* __restrict__ val, int32_t* __restrict__ bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = prow1[i] - 1;
        if (p < 0) atomicMin(bad, (int32_t)i);
        key[i] = (uint32_t)(p < 0 ? 0 : p);
        val[i] = (uint32_t)i;
    }
}

// seg[c] = first sorted position of parent c; seg[n_coarse] = n (every coarse row has >= 1 child)
__global__ void k_seg(const uint32_t* __restrict__ skey, int64_t n, int64_t n_coarse, int64_t* __restrict__ seg) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (i == 0 || skey[i] != skey[i - 1]) seg[skey[i]] = i;
        if (i == n - 1) seg[n_coarse] = n;
    }
}

template <typename T>
__device__ __forceinline__ double to_d(T v) { return (double)v; }
template <>
__device__ __forceinline__ double to_d<__nv_bfloat16>(__nv_bfloat16 v) { return (double)__bfloat162float(v); }
template <typename T>
__device__ __forceinline__ T from_d(double v) { return (T)v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_d<__nv_bfloat16>(double v) { return __float2bfloat16_rn((float)v); }
template <>
__device__ __forceinline__ float from_d<float>(double v) { return (float)v; }

// one thread per (coarse row, channel); children in ascending fine-row order
template <typename T, bool MAX>
__global__ void k_pool(const T* __restrict__ f, int64_t C, const uint32_t* __restrict__ sval,
                       const int64_t* __restrict__ seg, int64_t n_coarse, T* __restrict__ out) {
    const int64_t total = n_coarse * C;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = t / C, ch = t - c * C;
        const int64_t s0 = seg[c], s1 = seg[c + 1];
        double acc = MAX ? -INFINITY : 0.0;
        for (int64_t s = s0; s < s1; ++s) {
            const double v = to_d(f[(int64_t)sval[s] * C + ch]);
            if (MAX) acc = (v > acc || v != v) ? v : acc;  // NaN propagates like np.maximum
            else acc += v;
        }
        if (!MAX) acc /= (double)(s1 - s0);
        out[t] = from_d<T>(acc);
    }
}

// dst[i] = src[idx1[i] - 1] (row of row_bytes, 16-B multiple or not); first orphan (idx1 == 0) -> *bad
__global__ void k_gather_rows(const uint8_t* __restrict__ src, int64_t row_bytes, const int64_t* __restrict__ idx1,
                              int64_t n, uint8_t* __restrict__ dst, int32_t* __restrict__ bad) {
    const bool v16 = (row_bytes & 15) == 0;
    const int64_t units = v16 ? row_bytes / 16 : row_bytes;
    const int64_t total = n * units;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / units, u = t - i * units;
        const int64_t p = idx1[i] - 1;
        if (p < 0) {
            if (u == 0) atomicMin(bad, (int32_t)i);
            continue;
        }
        if (v16)
            reinterpret_cast<uint4*>(dst + i * row_bytes)[u] = reinterpret_cast<const uint4*>(src + p * row_bytes)[u];
        else
            dst[i * row_bytes + u] = src[p * row_bytes + u];
    }
}

unsigned grid_for(int64_t work) {
    int64_t b = ceil_div(work > 0 ? work : 1, 256);
    return (unsigned)(b < 8192 ? b : 8192);
}

}  // namespace
}  // namespace fvdb

using namespace fvdb;

extern "C" int fvdb_expand_coords(const int64_t* coords, int64_t n, int64_t scale, int64_t lo, int64_t width,
                                  int64_t* out, void* stream) {
    if (n < 0 || width < 1 || scale < 1) return FVDB_ERR_INVALID;
    if (n == 0) return FVDB_OK;
    k_expand<<<grid_for(n * width * width * width), 256, 0, as_stream(stream)>>>(coords, n, scale, lo, width, out);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

extern "C" size_t fvdb_pool_workspace_bytes(int64_t n_fine, int64_t n_coarse) {
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)(n_fine > 0 ? n_fine : 1));
    Sizer s;
    for (int k = 0; k < 4; ++k) s.take<uint32_t>(n_fine > 0 ? n_fine : 1);
    s.take<int64_t>(n_coarse + 1);
    s.take<int32_t>(1);
    s.take<uint8_t>(tmp);
    return s.used + 256;
}

extern "C" int fvdb_pool(int dtype, const void* features, int64_t n_fine, int64_t channels, const int64_t* prow1,
                         int64_t n_coarse, int mode_max, void* out, int64_t* detail, void* workspace,
                         size_t workspace_bytes, void* stream) {
    *detail = -1;
    if (n_fine < 0 || n_coarse < 0 || channels < 1 || n_fine > 0x7fffffffLL) return FVDB_ERR_INVALID;
    if (n_fine == 0 || n_coarse == 0) return FVDB_OK;
    cudaStream_t st = as_stream(stream);
    Carver cv(workspace, workspace_bytes);
    uint32_t* key = cv.take<uint32_t>(n_fine);
    uint32_t* val = cv.take<uint32_t>(n_fine);
    uint32_t* skey = cv.take<uint32_t>(n_fine);
    uint32_t* sval = cv.take<uint32_t>(n_fine);
    int64_t* seg = cv.take<int64_t>(n_coarse + 1);
    int32_t* bad = cv.take<int32_t>(1);
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, skey, val, sval, (int)n_fine);
    void* tmpp = cv.take<uint8_t>(tmp);
    if (!cv.ok()) return FVDB_ERR_WORKSPACE;
    const int32_t big = 0x7fffffff;
    FVDB_CUDA_TRY(cudaMemcpyAsync(bad, &big, 4, cudaMemcpyHostToDevice, st));
    k_keys<<<grid_for(n_fine), 256, 0, st>>>(prow1, n_fine, key, val, bad);
    int bits = 1;
    while (bits < 32 && ((int64_t)1 << bits) < n_coarse) ++bits;
    FVDB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmpp, tmp, key, skey, val, sval, (int)n_fine, 0, bits, st));
    k_seg<<<grid_for(n_fine), 256, 0, st>>>(skey, n_fine, n_coarse, seg);
    const unsigned gr = grid_for(n_coarse * channels);
    switch (dtype) {
        case FVDB_DTYPE_F32:
            if (mode_max) k_pool<float, true><<<gr, 256, 0, st>>>((const float*)features, channels, sval, seg, n_coarse, (float*)out);
            else k_pool<float, false><<<gr, 256, 0, st>>>((const float*)features, channels, sval, seg, n_coarse, (float*)out);
            break;
        case FVDB_DTYPE_F64:
            if (mode_max) k_pool<double, true><<<gr, 256, 0, st>>>((const double*)features, channels, sval, seg, n_coarse, (double*)out);
            else k_pool<double, false><<<gr, 256, 0, st>>>((const double*)features, channels, sval, seg, n_coarse, (double*)out);
            break;
        case FVDB_DTYPE_BF16:
            if (mode_max)
                k_pool<__nv_bfloat16, true><<<gr, 256, 0, st>>>((const __nv_bfloat16*)features, channels, sval, seg,
                                                                n_coarse, (__nv_bfloat16*)out);
            else
                k_pool<__nv_bfloat16, false><<<gr, 256, 0, st>>>((const __nv_bfloat16*)features, channels, sval, seg,
                                                                 n_coarse, (__nv_bfloat16*)out);
            break;
        default:
            return FVDB_ERR_INVALID;
    }
    FVDB_LAUNCH_CHECK();
    int32_t hb = big;
    FVDB_CUDA_TRY(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, st));
    FVDB_CUDA_TRY(cudaStreamSynchronize(st));
    if (hb != big) {  // a fine row without a coarse parent: caller passed inconsistent grids
        *detail = hb;
        return FVDB_ERR_INVALID;
    }
    return FVDB_OK;
}

extern "C" int fvdb_gather_rows(const void* src, int64_t row_bytes, const int64_t* idx1, int64_t n, void* dst,
                                int64_t* detail, void* workspace, size_t workspace_bytes, void* stream) {
    *detail = -1;
    if (n < 0 || row_bytes < 1 || workspace_bytes < 4) return FVDB_ERR_INVALID;
    if (n == 0) return FVDB_OK;
    cudaStream_t st = as_stream(stream);
    int32_t* bad = (int32_t*)workspace;
    const int32_t big = 0x7fffffff;
    FVDB_CUDA_TRY(cudaMemcpyAsync(bad, &big, 4, cudaMemcpyHostToDevice, st));
    const int64_t units = (row_bytes & 15) == 0 ? row_bytes / 16 : row_bytes;
    k_gather_rows<<<grid_for(n * units), 256, 0, st>>>((const uint8_t*)src, row_bytes, idx1, n, (uint8_t*)dst, bad);
    FVDB_LAUNCH_CHECK();
    int32_t hb = big;
    FVDB_CUDA_TRY(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, st));
    FVDB_CUDA_TRY(cudaStreamSynchronize(st));
    if (hb != big) {
        *detail = hb;
        return FVDB_ERR_INVALID;
    }
    return FVDB_OK;
}
