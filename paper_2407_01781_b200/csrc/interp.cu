// interp.cu — grid <-> point transfer on the device (reference interp.py:44-203).
//
// Per point: u = (p - origin) / voxel_size in IEEE f64 (no contraction), per-axis weights
// (trilinear: 2 taps, bezier = quadratic B-spline: 3 taps), S = 8 or 27 stencil voxels probed
// through the leaf hierarchy (same find_leaf / leaf_rank as the kernel map).
//   sample: out[p, c] = Σ_s w[p,s] · f[row(p,s), c] in f64, s ascending (interp.py:150-164)
//   splat : out[v, c] = Σ over (p, s) with row(p,s) == v of w[p,s] · f[p, c], f64, in (p, s) order —
//           the reference's stable argsort + add.reduceat order (interp.py:195-202), via a stable radix
//           sort on the destination row: bitwise reproducible.
// Weight derivatives (sample_with_grad, interp.py:96-105) are produced by the same stencil kernel.
#include <cub/device/device_radix_sort.cuh>
#include <math.h>

#include "common.cuh"

namespace fvdb {
namespace {

constexpr int kTri = 0, kBez = 1;

struct Xform {
    double vs[3], og[3];
};

// per-axis weights and derivatives (w.r.t. index coordinate) for tap t
__device__ __forceinline__ void axis_w(int mode, double u, int t, int64_t& base, double& w, double& dw) {
    if (mode == kTri) {
        const double b = floor(u);
        const double f = __dsub_rn(u, b);
        base = (int64_t)b;
        w = t == 0 ? __dsub_rn(1.0, f) : f;
        dw = t == 0 ? -1.0 : 1.0;
    } else {
        const double b = floor(__dadd_rn(u, 0.5));
        base = (int64_t)b;
        const double x = __dsub_rn(u, __dadd_rn(b, (double)(t - 1)));
        const double ax = fabs(x);
        const double outer = fmax(__dsub_rn(1.5, ax), 0.0);
        if (ax <= 0.5) {
            w = __dsub_rn(0.75, __dmul_rn(x, x));
            dw = __dmul_rn(-2.0, x);
        } else {
            w = __dmul_rn(__dmul_rn(0.5, outer), outer);
            dw = __dmul_rn(-(double)((x > 0) - (x < 0)), outer);
        }
    }
}

// rows[p][s] (0-based voxel row or -1), w[p][s], optional dw[p][s][3] (world-space)
__global__ void k_stencil(fvdb_grid_view g, const double* __restrict__ pts, int64_t n, Xform xf, int mode,
                          int64_t* __restrict__ rows, double* __restrict__ w, double* __restrict__ dw) {
    const int K = mode == kTri ? 2 : 3, S = K * K * K;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        double u[3];
        for (int a = 0; a < 3; ++a) u[a] = __ddiv_rn(__dsub_rn(pts[3 * p + a], xf.og[a]), xf.vs[a]);
        int64_t base[3];
        double wa[3][3], da[3][3];
        for (int a = 0; a < 3; ++a)
            for (int t = 0; t < K; ++t) axis_w(mode, u[a], t, base[a], wa[a][t], da[a][t]);
        for (int s = 0; s < S; ++s) {
            const int ti = s / (K * K), tj = (s / K) % K, tk = s % K;
            const int off0 = mode == kTri ? 0 : -1;
            const int64_t i = base[0] + ti + off0, j = base[1] + tj + off0, k = base[2] + tk + off0;
            int64_t r = -1;
            const int64_t l = find_leaf(g, i, j, k);
            if (l >= 0) {
                const uint32_t m = leaf_off(i, j, k);
                const uint64_t* words = g.leaf_masks + l * 8;
                if ((words[m >> 6] >> (m & 63)) & 1ull)
                    r = (int64_t)g.leaf_value_offset[l] - 1 + leaf_rank(words, g.leaf_prefix[l], m);
            }
            rows[p * S + s] = r;
            // (wx * wy) * wz: numpy broadcasting order of interp.py:92-95
            w[p * S + s] = __dmul_rn(__dmul_rn(wa[0][ti], wa[1][tj]), wa[2][tk]);
            if (dw) {
                dw[(p * S + s) * 3 + 0] = __dmul_rn(__dmul_rn(__dmul_rn(da[0][ti], wa[1][tj]), wa[2][tk]), 1.0 / xf.vs[0]);
                dw[(p * S + s) * 3 + 1] = __dmul_rn(__dmul_rn(__dmul_rn(wa[0][ti], da[1][tj]), wa[2][tk]), 1.0 / xf.vs[1]);
                dw[(p * S + s) * 3 + 2] = __dmul_rn(__dmul_rn(__dmul_rn(wa[0][ti], wa[1][tj]), da[2][tk]), 1.0 / xf.vs[2]);
            }
        }
    }
}

template <typename T>
__device__ __forceinline__ double ld(const T* p) { return (double)*p; }

// out[p][c] = Σ_s w·f (and grads[p][c][x] = Σ_s dw_x·f), f64 accumulation, s ascending
template <typename T>
__global__ void k_sample(const T* __restrict__ f, int64_t C, const int64_t* __restrict__ rows,
                         const double* __restrict__ w, const double* __restrict__ dw, int64_t n, int S,
                         T* __restrict__ out, T* __restrict__ grads) {
    const int64_t total = n * C;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = t / C, c = t - p * C;
        double acc = 0.0, g0 = 0.0, g1 = 0.0, g2 = 0.0;
        for (int s = 0; s < S; ++s) {
            const int64_t r = rows[p * S + s];
            const double v = r >= 0 ? ld(f + r * C + c) : 0.0;
            acc = __dadd_rn(acc, __dmul_rn(w[p * S + s], v));
            if (grads) {
                const double* d = dw + (p * S + s) * 3;
                g0 = __dadd_rn(g0, __dmul_rn(d[0], v));
                g1 = __dadd_rn(g1, __dmul_rn(d[1], v));
                g2 = __dadd_rn(g2, __dmul_rn(d[2], v));
            }
        }
        out[t] = (T)acc;
        if (grads) {
            grads[t * 3 + 0] = (T)g0;
            grads[t * 3 + 1] = (T)g1;
            grads[t * 3 + 2] = (T)g2;
        }
    }
}

// splat keys: destination row (or n_vox for background = sorted last), value = p*S + s
__global__ void k_splat_keys(const int64_t* __restrict__ rows, int64_t m, int64_t n_vox, uint32_t* __restrict__ key,
                             uint32_t* __restrict__ val) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = rows[i];
        key[i] = (uint32_t)(r < 0 ? n_vox : r);
        val[i] = (uint32_t)i;
    }
}
__global__ void k_splat_seg(const uint32_t* __restrict__ skey, int64_t m, int64_t n_vox, int64_t* __restrict__ seg) {
    // seg[v] = first sorted position of row v, seg[v+1] end; rows without contributions get empty ranges
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= m; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t cur = i < m ? (int64_t)skey[i] : n_vox;
        const int64_t prev = i > 0 ? (int64_t)skey[i - 1] : -1;
        for (int64_t v = prev + 1; v <= cur && v <= n_vox; ++v) seg[v] = i;
    }
}
template <typename T>
__global__ void k_splat(const T* __restrict__ f, int64_t C, const double* __restrict__ w,
                        const uint32_t* __restrict__ sval, const int64_t* __restrict__ seg, int S, int64_t n_vox,
                        T* __restrict__ out) {
    const int64_t total = n_vox * C;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = t / C, c = t - v * C;
        double acc = 0.0;
        for (int64_t q = seg[v]; q < seg[v + 1]; ++q) {
            const uint32_t ps = sval[q];
            const int64_t p = ps / S;
            acc = __dadd_rn(acc, __dmul_rn(w[ps], ld(f + p * C + c)));
        }
        out[t] = (T)acc;
    }
}

unsigned gsz(int64_t work) {
    int64_t b = ceil_div(work > 0 ? work : 1, 256);
    return (unsigned)(b < 8192 ? b : 8192);
}

}  // namespace
}  // namespace fvdb

using namespace fvdb;

extern "C" int fvdb_interp_stencil(const fvdb_grid_view* grid, const double* points, int64_t n,
                                   const double* voxel_size3, const double* origin3, int mode, int64_t* rows,
                                   double* weights, double* dweights, void* stream) {
    if (n < 0 || (mode != kTri && mode != kBez)) return FVDB_ERR_INVALID;
    if (n == 0) return FVDB_OK;
    Xform xf;
    for (int a = 0; a < 3; ++a) {
        xf.vs[a] = voxel_size3[a];
        xf.og[a] = origin3[a];
    }
    k_stencil<<<gsz(n), 256, 0, as_stream(stream)>>>(*grid, points, n, xf, mode, rows, weights, dweights);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

extern "C" int fvdb_interp_sample(int dtype, const void* features, int64_t channels, const int64_t* rows,
                                  const double* weights, const double* dweights, int64_t n, int stencil,
                                  void* out, void* grads, void* stream) {
    if (n < 0 || channels < 1 || (stencil != 8 && stencil != 27)) return FVDB_ERR_INVALID;
    if (n == 0) return FVDB_OK;
    cudaStream_t st = as_stream(stream);
    const unsigned gr = gsz(n * channels);
    if (dtype == FVDB_DTYPE_F64)
        k_sample<double><<<gr, 256, 0, st>>>((const double*)features, channels, rows, weights, dweights, n, stencil,
                                             (double*)out, (double*)grads);
    else if (dtype == FVDB_DTYPE_F32)
        k_sample<float><<<gr, 256, 0, st>>>((const float*)features, channels, rows, weights, dweights, n, stencil,
                                            (float*)out, (float*)grads);
    else
        return FVDB_ERR_INVALID;
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

extern "C" size_t fvdb_splat_workspace_bytes(int64_t n_points, int stencil, int64_t n_vox) {
    const int64_t m = n_points * stencil > 0 ? n_points * stencil : 1;
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)m);
    Sizer s;
    for (int k = 0; k < 4; ++k) s.take<uint32_t>(m);
    s.take<int64_t>(n_vox + 2);
    s.take<uint8_t>(tmp);
    return s.used + 256;
}

extern "C" int fvdb_interp_splat(int dtype, const void* point_features, int64_t channels, const int64_t* rows,
                                 const double* weights, int64_t n_points, int stencil, int64_t n_vox, void* out,
                                 void* workspace, size_t workspace_bytes, void* stream) {
    if (n_points < 0 || channels < 1 || (stencil != 8 && stencil != 27) || n_vox < 0) return FVDB_ERR_INVALID;
    const int64_t m = n_points * stencil;
    if (m > 0x7fffffffLL || n_vox >= 0x7fffffffLL) return FVDB_ERR_INVALID;
    cudaStream_t st = as_stream(stream);
    const size_t esz = dtype == FVDB_DTYPE_F64 ? 8 : 4;
    if (n_vox == 0) return FVDB_OK;
    if (m == 0) {
        FVDB_CUDA_TRY(cudaMemsetAsync(out, 0, (size_t)n_vox * channels * esz, st));
        return FVDB_OK;
    }
    Carver cv(workspace, workspace_bytes);
    uint32_t* key = cv.take<uint32_t>(m);
    uint32_t* val = cv.take<uint32_t>(m);
    uint32_t* skey = cv.take<uint32_t>(m);
    uint32_t* sval = cv.take<uint32_t>(m);
    int64_t* seg = cv.take<int64_t>(n_vox + 2);
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, skey, val, sval, (int)m);
    void* tmpp = cv.take<uint8_t>(tmp);
    if (!cv.ok()) return FVDB_ERR_WORKSPACE;
    k_splat_keys<<<gsz(m), 256, 0, st>>>(rows, m, n_vox, key, val);
    int bits = 1;
    while (bits < 32 && ((int64_t)1 << bits) <= n_vox) ++bits;
    FVDB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmpp, tmp, key, skey, val, sval, (int)m, 0, bits, st));
    k_splat_seg<<<gsz(m + 1), 256, 0, st>>>(skey, m, n_vox, seg);
    const unsigned gr = gsz(n_vox * channels);
    if (dtype == FVDB_DTYPE_F64)
        k_splat<double><<<gr, 256, 0, st>>>((const double*)point_features, channels, weights, sval, seg, stencil, n_vox,
                                            (double*)out);
    else if (dtype == FVDB_DTYPE_F32)
        k_splat<float><<<gr, 256, 0, st>>>((const float*)point_features, channels, weights, sval, seg, stencil, n_vox,
                                           (float*)out);
    else
        return FVDB_ERR_INVALID;
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}
