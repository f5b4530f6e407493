// conv_simt.cu — exact-precision (fp32 / f64) sparse conv: the parity path.
//
// Same operator as the reference igemm schedule (conv.py:180-191 forward,
// conv.py:339-368 backward) but evaluated output-stationary: every output row
// gathers its 27 neighbours through the kernel-map table nbr[27][N_out] and
// accumulates in registers, so there is no scatter-add and no atomics (results
// are deterministic).  dgrad runs the same kernel over the transposed table.
// wgrad is a split-K reduction with a fixed-order second pass (deterministic).
// CUDA-core FFMA / DFMA: this path exists to meet the fp32 1e-5 / f64 1e-10
// parity bars that TF32/bf16 tensor cores cannot (SURVEY §7 "hard parts").
#include "common.cuh"

namespace fvdb {
namespace {

constexpr int kRows = 32;    // output rows per CTA
constexpr int kKC = 16;      // K chunk staged per step
constexpr int kThr = 256;
constexpr int kMaxAcc = 32;  // kRows * N / kThr for N <= 256

template <typename T>
__global__ void __launch_bounds__(kThr) k_conv_gather(const T* __restrict__ in, int K, const T* __restrict__ wk,
                                                      int N, const int32_t* __restrict__ nbr, int64_t ld,
                                                      int64_t n_out, T* __restrict__ out) {
    __shared__ T s_in[kRows][kKC + 1];
    __shared__ T s_w[kKC][256];
    __shared__ int32_t s_idx[kRows];
    const int tid = threadIdx.x;
    const int64_t o0 = (int64_t)blockIdx.x * kRows;
    const int cells = kRows * N;
    T acc[kMaxAcc];
#pragma unroll
    for (int j = 0; j < kMaxAcc; ++j) acc[j] = T(0);

    for (int d = 0; d < 27; ++d) {
        __syncthreads();
        if (tid < kRows) {
            int64_t o = o0 + tid;
            s_idx[tid] = o < n_out ? nbr[(int64_t)d * ld + o] : -1;
        }
        __syncthreads();
        for (int k0 = 0; k0 < K; k0 += kKC) {
            for (int t = tid; t < kRows * kKC; t += kThr) {
                int r = t / kKC, kk = t % kKC;
                int32_t i = s_idx[r];
                s_in[r][kk] = (i >= 0 && k0 + kk < K) ? in[(int64_t)i * K + k0 + kk] : T(0);
            }
            for (int t = tid; t < kKC * N; t += kThr) {
                int kk = t / N, n = t % N;
                s_w[kk][n] = (k0 + kk < K) ? wk[((int64_t)d * K + k0 + kk) * N + n] : T(0);
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < kMaxAcc; ++j) {
                int c = tid + j * kThr;
                if (c < cells) {
                    int r = c / N, n = c % N;
                    T a = acc[j];
#pragma unroll
                    for (int kk = 0; kk < kKC; ++kk) a = fma(s_in[r][kk], s_w[kk][n], a);
                    acc[j] = a;
                }
            }
            __syncthreads();
        }
    }
#pragma unroll
    for (int j = 0; j < kMaxAcc; ++j) {
        int c = tid + j * kThr;
        if (c < cells) {
            int r = c / N, n = c % N;
            int64_t o = o0 + r;
            if (o < n_out) out[o * N + n] = acc[j];
        }
    }
}

// Tiled form for K, N multiples of 8 and N <= 64 (the reference's common channel counts): 128 output rows per
// CTA, each thread a 4-row x N/8-column register tile; the gathered rows and the offset's weights move
// through two cp.async stages (zero-filled for missing neighbours and K/N padding).  The per-element
// accumulation order is k_conv_gather's (offset-major, then K ascending), so results are identical.
constexpr int kTR = 128, kTKC = 32;
template <typename T, int NT>
struct TileCfg {
    static constexpr int EPV = 16 / (int)sizeof(T);          // elements per 16-byte copy
    static constexpr int LDA = kTKC + EPV;                   // padded row stride of the A tile (16-B aligned)
    static constexpr int CPT = NT / 8;                       // output columns per thread
    static constexpr int A_ELEMS = kTR * LDA, W_ELEMS = kTKC * NT;
    static constexpr int STAGE_BYTES = (A_ELEMS + W_ELEMS) * (int)sizeof(T);
    static constexpr int SMEM = 2 * STAGE_BYTES;
};

__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const void* src, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
}

template <typename T, int NT>
__global__ void __launch_bounds__(kThr) k_conv_gather_tiled(const T* __restrict__ in, int K, const T* __restrict__ wk,
                                                            int N, const int32_t* __restrict__ nbr, int64_t ld,
                                                            int64_t n_out, T* __restrict__ out,
                                                            const uint32_t* __restrict__ tile_mask,
                                                            const int32_t* __restrict__ row_perm) {
    using C = TileCfg<T, NT>;
    extern __shared__ __align__(16) uint8_t smraw[];
    T* sm = reinterpret_cast<T*>(smraw);
    const int tid = threadIdx.x, tx = tid & 7, ty = tid >> 3;
    const int64_t o0 = (int64_t)blockIdx.x * kTR;
    // offsets with a pair somewhere in this 128-row tile (all 27 without masks); absent offsets would only
    // add zero-filled rows, so skipping them leaves every finite sum unchanged
    const uint32_t m = tile_mask ? (tile_mask[blockIdx.x] & 0x7ffffffu) : 0x7ffffffu;
    const int kchunks = (K + kTKC - 1) / kTKC, steps = __popc(m) * kchunks;
    auto issue = [&](int step, int buf) {
        const int d = (int)__fns(m, 0, step / kchunks + 1), k0 = (step % kchunks) * kTKC;
        T* sa = sm + buf * (C::A_ELEMS + C::W_ELEMS);
        T* sw = sa + C::A_ELEMS;
        constexpr int CPR = kTKC / C::EPV;                    // 16-B copies per A row
        for (int c = tid; c < kTR * CPR; c += kThr) {
            const int r = c / CPR, cc = c % CPR, k = k0 + cc * C::EPV;
            const int64_t o = o0 + r;
            const int32_t i = o < n_out ? nbr[(int64_t)d * ld + o] : -1;
            const bool ok = i >= 0 && k < K;
            cp_async16_zfill((uint32_t)__cvta_generic_to_shared(sa + r * C::LDA + cc * C::EPV),
                             ok ? (const void*)(in + (int64_t)i * K + k) : (const void*)in, ok);
        }
        constexpr int CPW = NT / C::EPV;                      // 16-B copies per weight row
        for (int c = tid; c < kTKC * CPW; c += kThr) {
            const int kk = c / CPW, n = (c % CPW) * C::EPV;
            const bool ok = k0 + kk < K && n < N;
            cp_async16_zfill((uint32_t)__cvta_generic_to_shared(sw + kk * NT + n),
                             ok ? (const void*)(wk + ((int64_t)d * K + k0 + kk) * N + n) : (const void*)wk, ok);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    T acc[4][C::CPT];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < C::CPT; ++j) acc[i][j] = T(0);
    if (steps > 0) issue(0, 0);
    for (int step = 0; step < steps; ++step) {
        const int buf = step & 1;
        if (step + 1 < steps) {
            issue(step + 1, buf ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const T* sa = sm + buf * (C::A_ELEMS + C::W_ELEMS);
        const T* sw = sa + C::A_ELEMS;
#pragma unroll 8
        for (int kk = 0; kk < kTKC; ++kk) {
            T a[4], b[C::CPT];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = sa[(ty + 32 * i) * C::LDA + kk];
#pragma unroll
            for (int j = 0; j < C::CPT; ++j) b[j] = sw[kk * NT + tx * C::CPT + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < C::CPT; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();  // the next issue overwrites this buffer
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t o = o0 + ty + 32 * i;
        if (o >= n_out) continue;
        const int64_t orow = row_perm ? (int64_t)row_perm[o] : o;  // signature-sorted table: original row
#pragma unroll
        for (int j = 0; j < C::CPT; ++j) {
            const int n = tx * C::CPT + j;
            if (n < N) out[orow * N + n] = acc[i][j];
        }
    }
}

// W[Cout][Cin][27] -> Wk[27][K][N]
template <typename T>
__global__ void k_pack_kn(const T* __restrict__ w, int cout, int cin, int transpose, T* __restrict__ wk) {
    const int64_t total = (int64_t)27 * cout * cin;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t co = t / ((int64_t)cin * 27);
        int64_t rem = t - co * cin * 27;
        int64_t ci = rem / 27;
        int64_t d = rem - ci * 27;
        int64_t dst = transpose ? (d * cout + co) * cin + ci : (d * cin + ci) * cout + co;
        wk[dst] = w[t];
    }
}

// wgrad partials: part[s][d][co][ci] over the output rows of split s
constexpr int kWB = 32;  // output-channel and input-channel block edge
template <typename T>
__global__ void __launch_bounds__(kThr) k_wgrad_part(const T* __restrict__ in, int cin, const T* __restrict__ go,
                                                     int cout, const int32_t* __restrict__ nbr, int64_t ld,
                                                     int64_t n_out, int64_t rows_per_split, T* __restrict__ part) {
    __shared__ T s_go[kRows][kWB + 1];
    __shared__ T s_in[kRows][kWB + 1];
    __shared__ int32_t s_idx[kRows];
    const int s = blockIdx.x, d = blockIdx.y;
    const int nb_ci = (cin + kWB - 1) / kWB;
    const int co0 = (blockIdx.z / nb_ci) * kWB, ci0 = (blockIdx.z % nb_ci) * kWB;
    const int tid = threadIdx.x;
    // 32x32 block, 4 accumulators per thread
    T acc[4] = {T(0), T(0), T(0), T(0)};
    const int64_t begin = (int64_t)s * rows_per_split;
    const int64_t end = begin + rows_per_split < n_out ? begin + rows_per_split : n_out;
    for (int64_t o0 = begin; o0 < end; o0 += kRows) {
        __syncthreads();
        if (tid < kRows) {
            int64_t o = o0 + tid;
            s_idx[tid] = o < end ? nbr[(int64_t)d * ld + o] : -1;
        }
        __syncthreads();
        for (int t = tid; t < kRows * kWB; t += kThr) {
            int r = t / kWB, c = t % kWB;
            int32_t i = s_idx[r];
            int64_t o = o0 + r;
            bool ok = i >= 0;
            s_go[r][c] = (ok && co0 + c < cout) ? go[o * cout + co0 + c] : T(0);
            s_in[r][c] = (ok && ci0 + c < cin) ? in[(int64_t)i * cin + ci0 + c] : T(0);
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int cell = tid + j * kThr;
            int a = cell / kWB, b = cell % kWB;
            T v = acc[j];
#pragma unroll 8
            for (int r = 0; r < kRows; ++r) v = fma(s_go[r][a], s_in[r][b], v);
            acc[j] = v;
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        int cell = tid + j * kThr;
        int a = cell / kWB, b = cell % kWB;
        if (co0 + a < cout && ci0 + b < cin)
            part[(((int64_t)s * 27 + d) * cout + co0 + a) * cin + ci0 + b] = acc[j];
    }
}

template <typename T>
__global__ void k_wgrad_reduce(const T* __restrict__ part, int splits, int cout, int cin, T* __restrict__ gw) {
    const int64_t total = (int64_t)27 * cout * cin;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        // t indexes gw[co][ci][d]
        int64_t co = t / ((int64_t)cin * 27);
        int64_t rem = t - co * cin * 27;
        int64_t ci = rem / 27, d = rem - ci * 27;
        T v = T(0);
        for (int s = 0; s < splits; ++s) v += part[(((int64_t)s * 27 + d) * cout + co) * cin + ci];
        gw[t] = v;
    }
}

int wgrad_splits(int64_t n_out) {
    int64_t s = ceil_div(n_out, 4096);
    return (int)(s < 1 ? 1 : (s > 64 ? 64 : s));
}

template <typename T>
int run_gather(const void* in, int K, const void* wk, int N, const int32_t* nbr, int64_t ld, int64_t n_out, void* out,
               cudaStream_t st, const uint32_t* masks = nullptr, const int32_t* perm = nullptr) {
    if (n_out == 0) return FVDB_OK;
    if (K % 8 == 0 && N % 8 == 0 && N <= 64) {
        const unsigned blocks = (unsigned)ceil_div(n_out, kTR);
        if (N <= 32) {
            auto kern = k_conv_gather_tiled<T, 32>;
            FVDB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, TileCfg<T, 32>::SMEM));
            kern<<<blocks, kThr, TileCfg<T, 32>::SMEM, st>>>((const T*)in, K, (const T*)wk, N, nbr, ld, n_out, (T*)out,
                                                             masks, perm);
        } else {
            auto kern = k_conv_gather_tiled<T, 64>;
            FVDB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, TileCfg<T, 64>::SMEM));
            kern<<<blocks, kThr, TileCfg<T, 64>::SMEM, st>>>((const T*)in, K, (const T*)wk, N, nbr, ld, n_out, (T*)out,
                                                             masks, perm);
        }
        FVDB_LAUNCH_CHECK();
        return FVDB_OK;
    }
    if (perm) return FVDB_ERR_INVALID;  // only the tiled kernel writes through a row permutation
    unsigned blocks = (unsigned)ceil_div(n_out, kRows);
    k_conv_gather<T><<<blocks, kThr, 0, st>>>((const T*)in, K, (const T*)wk, N, nbr, ld, n_out, (T*)out);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

template <typename T>
int run_wgrad(const void* in, int cin, const void* go, int cout, const int32_t* nbr, int64_t ld, int64_t n_out,
              void* gw, void* ws, size_t ws_bytes, cudaStream_t st) {
    const int splits = wgrad_splits(n_out);
    size_t need = (size_t)splits * 27 * cout * cin * sizeof(T);
    if (ws_bytes < need) return FVDB_ERR_WORKSPACE;
    T* part = (T*)ws;
    int64_t rps = ceil_div(n_out > 0 ? n_out : 1, splits);
    rps = ceil_div(rps, kRows) * kRows;
    dim3 grid(splits, 27, ((cout + kWB - 1) / kWB) * ((cin + kWB - 1) / kWB));
    k_wgrad_part<T><<<grid, kThr, 0, st>>>((const T*)in, cin, (const T*)go, cout, nbr, ld, n_out, rps, part);
    k_wgrad_reduce<T><<<(unsigned)ceil_div((int64_t)27 * cout * cin, 256), 256, 0, st>>>(part, splits, cout, cin,
                                                                                       (T*)gw);
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

}  // namespace
}  // namespace fvdb

using namespace fvdb;

extern "C" int fvdb_conv_gather_simt(int dtype, const void* in, int64_t n_in, int K, const void* wk, int N,
                                     const int32_t* nbr, int64_t ld, int64_t n_out, void* out, void* stream) {
    (void)n_in;
    if (K <= 0 || N <= 0 || N > 256 || ld < n_out) return FVDB_ERR_INVALID;
    cudaStream_t st = as_stream(stream);
    if (dtype == FVDB_DTYPE_F32) return run_gather<float>(in, K, wk, N, nbr, ld, n_out, out, st);
    if (dtype == FVDB_DTYPE_F64) return run_gather<double>(in, K, wk, N, nbr, ld, n_out, out, st);
    return FVDB_ERR_INVALID;
}

extern "C" int fvdb_conv_gather_simt2(int dtype, const void* in, int64_t n_in, int K, const void* wk, int N,
                                      const int32_t* nbr, int64_t ld, int64_t n_out, const int32_t* row_perm,
                                      const uint32_t* tile_masks, void* out, void* stream) {
    (void)n_in;
    if (K <= 0 || N <= 0 || N > 256 || ld < n_out) return FVDB_ERR_INVALID;
    cudaStream_t st = as_stream(stream);
    if (dtype == FVDB_DTYPE_F32) return run_gather<float>(in, K, wk, N, nbr, ld, n_out, out, st, tile_masks, row_perm);
    if (dtype == FVDB_DTYPE_F64) return run_gather<double>(in, K, wk, N, nbr, ld, n_out, out, st, tile_masks, row_perm);
    return FVDB_ERR_INVALID;
}

extern "C" int fvdb_pack_weights_kn(int dtype, const void* w, int cout, int cin, int transpose, void* wk,
                                    void* stream) {
    cudaStream_t st = as_stream(stream);
    int64_t total = (int64_t)27 * cout * cin;
    unsigned blocks = (unsigned)ceil_div(total > 0 ? total : 1, 256);
    if (dtype == FVDB_DTYPE_F32)
        k_pack_kn<float><<<blocks, 256, 0, st>>>((const float*)w, cout, cin, transpose, (float*)wk);
    else if (dtype == FVDB_DTYPE_F64)
        k_pack_kn<double><<<blocks, 256, 0, st>>>((const double*)w, cout, cin, transpose, (double*)wk);
    else
        return FVDB_ERR_INVALID;
    FVDB_LAUNCH_CHECK();
    return FVDB_OK;
}

extern "C" size_t fvdb_wgrad_workspace_bytes(int dtype, int64_t n_out, int cin, int cout) {
    size_t es = dtype == FVDB_DTYPE_F64 ? 8 : 4;
    return (size_t)wgrad_splits(n_out) * 27 * cout * cin * es + 256;
}

extern "C" int fvdb_conv_wgrad_simt(int dtype, const void* in, int64_t n_in, int cin, const void* go, int cout,
                                    const int32_t* nbr, int64_t ld, int64_t n_out, void* gw, void* ws,
                                    size_t ws_bytes, void* stream) {
    (void)n_in;
    if (ld < n_out) return FVDB_ERR_INVALID;
    cudaStream_t st = as_stream(stream);
    if (dtype == FVDB_DTYPE_F32) return run_wgrad<float>(in, cin, go, cout, nbr, ld, n_out, gw, ws, ws_bytes, st);
    if (dtype == FVDB_DTYPE_F64) return run_wgrad<double>(in, cin, go, cout, nbr, ld, n_out, gw, ws, ws_bytes, st);
    return FVDB_ERR_INVALID;
}
