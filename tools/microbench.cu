// tools/microbench.cu — B200 micro-benchmarks that decide the conv kernel design.
//   (1) TMA tile::gather4 semantics probe (box height, OOB zero fill, tx byte count)
//   (2) gather bandwidth of the real cfg2 kernel map: TMA gather4 vs cp.async(.ca/.cg)
//   (3) tcgen05.mma kind::f16 SS issue rate at M=128, N in {64,128,256}
// Not part of the product library; built by tools/run_microbench.py.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_2407_01781_b200/csrc/tc_ptx.cuh"

using namespace fvdb::tc;
using bf16 = __nv_bfloat16;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess) return nullptr;
    return (EncodeTiledFn)fn;
}

static int make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_w, uint32_t box_h,
                    CUtensorMapSwizzle sw) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return -100;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {box_w, box_h};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return (int)r;
}

__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap* map, int c0, int4 r, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(map), "r"(c0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(bar)
        : "memory");
}

__device__ bool wait_bounded(uint32_t bar, uint32_t ph, long long spins) {
    for (long long i = 0; i < spins; ++i)
        if (mbar_try_wait(bar, ph)) return true;
    return false;
}

// ---------------------------------------------------------------- (1) probe
__global__ void k_probe(const __grid_constant__ CUtensorMap map, int4 rows, int expect, bf16* out, int* status) {
    __shared__ __align__(1024) uint8_t buf[4096];
    __shared__ __align__(8) uint64_t bar;
    uint32_t b = smem_u32(&bar);
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = 0xAB;
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_init(b, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_expect_tx(b, expect);
        gather4(smem_u32(buf), &map, 0, rows, b);
        bool ok = wait_bounded(b, 0, 20000000);
        status[0] = ok ? 1 : 0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4 * 64; i += blockDim.x) out[i] = reinterpret_cast<bf16*>(buf)[i];
}

extern "C" int mb_probe(const void* src, int n_rows, int box_h, int swz, int r0, int r1, int r2, int r3, int expect,
                        void* out, int* status) {
    CUtensorMap m;
    int rc = make_map(&m, src, n_rows, 64, 64, box_h,
                      swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE);
    if (rc) return rc;
    k_probe<<<1, 128>>>(m, make_int4(r0, r1, r2, r3), expect, (bf16*)out, status);
    return (int)cudaDeviceSynchronize();
}

// ---------------------------------------------------------------- (2) gather bandwidth
constexpr int kStages = 8;
// mode 0: TMA gather4 (1 producer warp); 1: cp.async.ca by 4 warps; 2: cp.async.cg by 4 warps
template <int MODE>
__global__ void __launch_bounds__(192, 1) k_gather_bw(const __grid_constant__ CUtensorMap map, const bf16* feat,
                                                      const int32_t* nbr, long long n_out, int num_tiles) {
    extern __shared__ uint8_t dsm[];
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
    const uint32_t base = (smem_u32(dsm) + 1023) & ~1023u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(smem_u32(&full[s]), MODE == 0 ? 1 : 128);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (MODE == 0 && warp == 0) {
        uint32_t it = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x)
            for (int d = 0; d < 27; ++d, ++it) {
                uint32_t s = it % kStages, ph = (it / kStages) & 1;
                int4 r = *reinterpret_cast<const int4*>(nbr + (long long)d * n_out + (long long)t * 128 + 4 * lane);
                if ((long long)t * 128 + 4 * lane + 3 >= n_out) r = make_int4(-1, -1, -1, -1);
                mbar_wait(smem_u32(&empty[s]), ph ^ 1);
                if (lane == 0) mbar_arrive_expect_tx(smem_u32(&full[s]), 128 * 128);
                __syncwarp();
                gather4(base + s * 16384 + lane * 512, &map, 0, r, smem_u32(&full[s]));
            }
    } else if (MODE != 0 && warp < 4) {
        const int pt = threadIdx.x, c = pt & 7, rb = pt >> 3;
        uint32_t it = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x)
            for (int d = 0; d < 27; ++d, ++it) {
                uint32_t s = it % kStages, ph = (it / kStages) & 1;
                int idx[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    long long row = (long long)t * 128 + rb + 16 * j;
                    idx[j] = row < n_out ? nbr[(long long)d * n_out + row] : -1;
                }
                mbar_wait(smem_u32(&empty[s]), ph ^ 1);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    int r = rb + 16 * j;
                    uint32_t dst = base + s * 16384 + r * 128 + ((c ^ (r & 7)) << 4);
                    const bf16* src = feat + (long long)(idx[j] < 0 ? 0 : idx[j]) * 64 + c * 8;
                    if (MODE == 1) cp_async_16(dst, src, idx[j] < 0 ? 0 : 16);
                    else cp_async_16_cg(dst, src, idx[j] < 0 ? 0 : 16);
                }
                cp_async_arrive_noinc(smem_u32(&full[s]));
            }
    } else if (warp == 5 && lane == 0) {
        uint32_t it = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x)
            for (int d = 0; d < 27; ++d, ++it) {
                uint32_t s = it % kStages, ph = (it / kStages) & 1;
                mbar_wait(smem_u32(&full[s]), ph);
                mbar_arrive(smem_u32(&empty[s]));
            }
    }
}

extern "C" int mb_gather_bw(int mode, const void* feat, long long n_in, const int32_t* nbr, long long n_out,
                            int ctas_per_sm, float* ms) {
    CUtensorMap m;
    int rc = make_map(&m, feat, n_in, 64, 64, 1, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    int tiles = (int)(n_out / 128);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    size_t smem = kStages * 16384 + 1024;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    void (*k)(CUtensorMap, const bf16*, const int32_t*, long long, int) =
        mode == 0 ? k_gather_bw<0> : (mode == 1 ? k_gather_bw<1> : k_gather_bw<2>);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        k<<<sms * ctas_per_sm, 192, smem>>>(m, (const bf16*)feat, nbr, n_out, tiles);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(ms, a, b);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------- (2b) gather with index blocks prefetched
// index block of a tile (27 x 128 int32) arrives by 27 bulk copies into a 2-deep smem ring
template <int MODE, int STAGES>
__global__ void __launch_bounds__(192, 1) k_gather_bw2(const __grid_constant__ CUtensorMap map, const bf16* feat,
                                                       const int32_t* nbr, long long n_out, int num_tiles) {
    extern __shared__ uint8_t dsm[];
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], ifull[2], iempty[2];
    const uint32_t base = (smem_u32(dsm) + 1023) & ~1023u;
    const uint32_t ibase = base + STAGES * 16384;       // 2 x 27 x 512 B
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nprod = MODE == 0 ? 32 : 128;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&full[s]), MODE == 0 ? 1 : 128);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&ifull[b]), 1);
            mbar_init(smem_u32(&iempty[b]), nprod);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 4) {
        if (lane == 0) {
            int lt = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
                int b = lt & 1;
                mbar_wait(smem_u32(&iempty[b]), ((lt >> 1) & 1) ^ 1);
                mbar_arrive_expect_tx(smem_u32(&ifull[b]), 27 * 512);
                for (int d = 0; d < 27; ++d)
                    bulk_g2s(ibase + b * 27 * 512 + d * 512, nbr + (long long)d * n_out + (long long)t * 128, 512,
                             smem_u32(&ifull[b]));
            }
        }
    } else if ((MODE == 0 && warp == 0) || (MODE != 0 && warp < 4)) {
        const int pt = threadIdx.x;
        uint32_t it = 0;
        int lt = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
            int b = lt & 1;
            mbar_wait(smem_u32(&ifull[b]), (lt >> 1) & 1);
            const int32_t* ib = reinterpret_cast<const int32_t*>(dsm + (ibase - smem_u32(dsm))) + b * 27 * 128;
            for (int d = 0; d < 27; ++d, ++it) {
                uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
                mbar_wait(smem_u32(&empty[s]), ph ^ 1);
                if (MODE == 0) {
                    int4 r = *reinterpret_cast<const int4*>(ib + d * 128 + 4 * lane);
                    if (lane == 0) mbar_arrive_expect_tx(smem_u32(&full[s]), 128 * 128);
                    __syncwarp();
                    gather4(base + s * 16384 + lane * 512, &map, 0, r, smem_u32(&full[s]));
                } else {
                    const int c = pt & 7, rb = pt >> 3;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        int r = rb + 16 * j;
                        int idx = ib[d * 128 + r];
                        uint32_t dst = base + s * 16384 + r * 128 + ((c ^ (r & 7)) << 4);
                        const bf16* src = feat + (long long)(idx < 0 ? 0 : idx) * 64 + c * 8;
                        if (MODE == 1) cp_async_16(dst, src, idx < 0 ? 0 : 16);
                        else cp_async_16_cg(dst, src, idx < 0 ? 0 : 16);
                    }
                    cp_async_arrive_noinc(smem_u32(&full[s]));
                }
            }
            mbar_arrive(smem_u32(&iempty[b]));
        }
    } else if (warp == 5 && lane == 0) {
        uint32_t it = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x)
            for (int d = 0; d < 27; ++d, ++it) {
                uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
                mbar_wait(smem_u32(&full[s]), ph);
                mbar_arrive(smem_u32(&empty[s]));
            }
    }
}

extern "C" int mb_gather_bw2(int mode, int stages, const void* feat, long long n_in, const int32_t* nbr,
                             long long n_out, float* ms) {
    CUtensorMap m;
    int rc = make_map(&m, feat, n_in, 64, 64, 1, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    int tiles = (int)(n_out / 128);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    size_t smem = stages * 16384 + 2 * 27 * 512 + 1024;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    void (*k)(CUtensorMap, const bf16*, const int32_t*, long long, int);
    if (stages == 8) k = mode == 0 ? k_gather_bw2<0, 8> : (mode == 1 ? k_gather_bw2<1, 8> : k_gather_bw2<2, 8>);
    else k = mode == 0 ? k_gather_bw2<0, 12> : (mode == 1 ? k_gather_bw2<1, 12> : k_gather_bw2<2, 12>);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        k<<<sms, 192, smem>>>(m, (const bf16*)feat, nbr, n_out, tiles);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(ms, a, b);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------- (2c) gather bottleneck matrix
// MODE 0: cp.async.ca, 1: cp.async.cg, 2: ld.global.v4 + st.shared.v4; NPW producer warps;
// IDX 0: real kernel map, 1: rows & 1023 (L1-resident set), 2: identity rows (contiguous)
template <int MODE, int NPW, int IDX>
__global__ void __launch_bounds__(NPW * 32 + 64, 1) k_gather_mx(const bf16* feat, const int32_t* nbr, long long n_out,
                                                               int num_tiles) {
    constexpr int STAGES = 8;
    extern __shared__ uint8_t dsm[];
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], ifull[2], iempty[2];
    const uint32_t sbase = smem_u32(dsm);
    const uint32_t base = (sbase + 1023) & ~1023u;
    const uint32_t ibase = base + STAGES * 16384;
    const int32_t* ism = reinterpret_cast<const int32_t*>(dsm + (ibase - sbase));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int NP = NPW * 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&full[s]), NP);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&ifull[b]), 1);
            mbar_init(smem_u32(&iempty[b]), NP);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == NPW) {
        if (lane == 0) {
            int lt = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
                int b = lt & 1;
                mbar_wait(smem_u32(&iempty[b]), ((lt >> 1) & 1) ^ 1);
                mbar_arrive_expect_tx(smem_u32(&ifull[b]), 27 * 512);
                for (int d = 0; d < 27; ++d)
                    bulk_g2s(ibase + b * 27 * 512 + d * 512, nbr + (long long)d * n_out + (long long)t * 128, 512,
                             smem_u32(&ifull[b]));
            }
        }
    } else if (warp < NPW) {
        const int pt = threadIdx.x, c = pt & 7, rb = pt >> 3;
        constexpr int RS = NP / 8, J = 128 / RS;
        uint32_t it = 0;
        int lt = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
            int b = lt & 1;
            mbar_wait(smem_u32(&ifull[b]), (lt >> 1) & 1);
            const int32_t* ib = ism + b * 27 * 128;
            for (int d = 0; d < 27; ++d, ++it) {
                uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
                int idx[J];
#pragma unroll
                for (int j = 0; j < J; ++j) {
                    int r = rb + RS * j;
                    int v = ib[d * 128 + r];
                    if (IDX == 1) v = v < 0 ? v : (v & 1023);
                    if (IDX == 2) v = t * 128 + r;
                    idx[j] = v;
                }
                mbar_wait(smem_u32(&empty[s]), ph ^ 1);
                if (MODE == 2) {
                    int4 vals[J];
#pragma unroll
                    for (int j = 0; j < J; ++j) {
                        const int4* src = reinterpret_cast<const int4*>(feat + (long long)(idx[j] < 0 ? 0 : idx[j]) * 64 + c * 8);
                        vals[j] = idx[j] < 0 ? make_int4(0, 0, 0, 0) : __ldg(src);
                    }
#pragma unroll
                    for (int j = 0; j < J; ++j) {
                        int r = rb + RS * j;
                        uint32_t dst = base + s * 16384 + r * 128 + ((c ^ (r & 7)) << 4);
                        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(dst), "r"(vals[j].x), "r"(vals[j].y),
                                     "r"(vals[j].z), "r"(vals[j].w)
                                     : "memory");
                    }
                    mbar_arrive(smem_u32(&full[s]));
                } else {
#pragma unroll
                    for (int j = 0; j < J; ++j) {
                        int r = rb + RS * j;
                        uint32_t dst = base + s * 16384 + r * 128 + ((c ^ (r & 7)) << 4);
                        const bf16* src = feat + (long long)(idx[j] < 0 ? 0 : idx[j]) * 64 + c * 8;
                        if (MODE == 0) cp_async_16(dst, src, idx[j] < 0 ? 0 : 16);
                        else cp_async_16_cg(dst, src, idx[j] < 0 ? 0 : 16);
                    }
                    cp_async_arrive_noinc(smem_u32(&full[s]));
                }
            }
            mbar_arrive(smem_u32(&iempty[b]));
        }
    } else if (warp == NPW + 1 && lane == 0) {
        uint32_t it = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x)
            for (int d = 0; d < 27; ++d, ++it) {
                uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
                mbar_wait(smem_u32(&full[s]), ph);
                mbar_arrive(smem_u32(&empty[s]));
            }
    }
}

template <int MODE, int NPW, int IDX>
static float run_mx(const void* feat, const int32_t* nbr, long long n_out, int ctas) {
    int tiles = (int)(n_out / 128);
    size_t smem = 8 * 16384 + 2 * 27 * 512 + 1024;
    auto k = k_gather_mx<MODE, NPW, IDX>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        k<<<ctas, NPW * 32 + 64, smem>>>((const bf16*)feat, nbr, n_out, tiles);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    return cudaGetLastError() == cudaSuccess ? ms : -1.f;
}

extern "C" int mb_gather_mx(const void* feat, const int32_t* nbr, long long n_out, float* out /*[2][3][3]*/) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
#define MX(M, W, I) out[((W == 8) * 3 + M) * 3 + I] = run_mx<M, W, I>(feat, nbr, n_out, sms);
    MX(0, 4, 0) MX(0, 4, 1) MX(0, 4, 2) MX(1, 4, 0) MX(1, 4, 1) MX(1, 4, 2) MX(2, 4, 0) MX(2, 4, 1) MX(2, 4, 2)
    MX(0, 8, 0) MX(0, 8, 1) MX(0, 8, 2) MX(1, 8, 0) MX(1, 8, 1) MX(1, 8, 2) MX(2, 8, 0) MX(2, 8, 1) MX(2, 8, 2)
#undef MX
    return 0;
}

// ---------------------------------------------------------------- (2d) L1-friendly gathers
// tile-major gather with few stages (large L1), cp.async.ca vs ld.global(L1)+st.shared.
template <int MODE, int STAGES, int NPW>
__global__ void __launch_bounds__(NPW * 32 + 64, 1) k_gather_l1(const bf16* feat, const int32_t* nbr, long long n_out,
                                                               int num_tiles) {
    extern __shared__ uint8_t dsm[];
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], ifull[2], iempty[2];
    const uint32_t sbase = smem_u32(dsm);
    const uint32_t base = (sbase + 1023) & ~1023u;
    const uint32_t ibase = base + STAGES * 16384;
    const int32_t* ism = reinterpret_cast<const int32_t*>(dsm + (ibase - sbase));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int NP = NPW * 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&full[s]), NP);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&ifull[b]), 1);
            mbar_init(smem_u32(&iempty[b]), NP);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == NPW) {
        if (lane == 0) {
            int lt = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
                int b = lt & 1;
                mbar_wait(smem_u32(&iempty[b]), ((lt >> 1) & 1) ^ 1);
                mbar_arrive_expect_tx(smem_u32(&ifull[b]), 27 * 512);
                for (int d = 0; d < 27; ++d)
                    bulk_g2s(ibase + b * 27 * 512 + d * 512, nbr + (long long)d * n_out + (long long)t * 128, 512,
                             smem_u32(&ifull[b]));
            }
        }
    } else if (warp < NPW) {
        const int pt = threadIdx.x, c = pt & 7, rb = pt >> 3;
        constexpr int RS = NP / 8, J = 128 / RS;
        uint32_t it = 0;
        int lt = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
            int b = lt & 1;
            mbar_wait(smem_u32(&ifull[b]), (lt >> 1) & 1);
            const int32_t* ib = ism + b * 27 * 128;
            for (int d = 0; d < 27; ++d, ++it) {
                uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
                int idx[J];
#pragma unroll
                for (int j = 0; j < J; ++j) idx[j] = ib[d * 128 + rb + RS * j];
                if (MODE == 1) {
                    int4 vals[J];
#pragma unroll
                    for (int j = 0; j < J; ++j) {
                        const int4* src = reinterpret_cast<const int4*>(feat + (long long)(idx[j] < 0 ? 0 : idx[j]) * 64 + c * 8);
                        int4 v;
                        asm volatile("ld.global.L1::evict_last.v4.b32 {%0,%1,%2,%3}, [%4];"
                                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src));
                        vals[j] = idx[j] < 0 ? make_int4(0, 0, 0, 0) : v;
                    }
                    mbar_wait(smem_u32(&empty[s]), ph ^ 1);
#pragma unroll
                    for (int j = 0; j < J; ++j) {
                        int r = rb + RS * j;
                        uint32_t dst = base + s * 16384 + r * 128 + ((c ^ (r & 7)) << 4);
                        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(dst), "r"(vals[j].x), "r"(vals[j].y),
                                     "r"(vals[j].z), "r"(vals[j].w)
                                     : "memory");
                    }
                    mbar_arrive(smem_u32(&full[s]));
                } else {
                    mbar_wait(smem_u32(&empty[s]), ph ^ 1);
#pragma unroll
                    for (int j = 0; j < J; ++j) {
                        int r = rb + RS * j;
                        uint32_t dst = base + s * 16384 + r * 128 + ((c ^ (r & 7)) << 4);
                        const bf16* src = feat + (long long)(idx[j] < 0 ? 0 : idx[j]) * 64 + c * 8;
                        cp_async_16(dst, src, idx[j] < 0 ? 0 : 16);
                    }
                    cp_async_arrive_noinc(smem_u32(&full[s]));
                }
            }
            mbar_arrive(smem_u32(&iempty[b]));
        }
    } else if (warp == NPW + 1 && lane == 0) {
        uint32_t it = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x)
            for (int d = 0; d < 27; ++d, ++it) {
                uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
                mbar_wait(smem_u32(&full[s]), ph);
                mbar_arrive(smem_u32(&empty[s]));
            }
    }
}

template <int MODE, int STAGES, int NPW>
static float run_l1(const void* feat, const int32_t* nbr, long long n_out, int ctas_per_sm, int sms) {
    int tiles = (int)(n_out / 128);
    size_t smem = STAGES * 16384 + 2 * 27 * 512 + 1024;
    auto k = k_gather_l1<MODE, STAGES, NPW>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        k<<<sms * ctas_per_sm, NPW * 32 + 64, smem>>>((const bf16*)feat, nbr, n_out, tiles);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    return cudaGetLastError() == cudaSuccess ? ms : -1.f;
}

extern "C" int mb_gather_l1(const void* feat, const int32_t* nbr, long long n_out, float* out) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    out[0] = run_l1<0, 2, 4>(feat, nbr, n_out, 1, sms);
    out[1] = run_l1<0, 4, 4>(feat, nbr, n_out, 1, sms);
    out[2] = run_l1<0, 2, 4>(feat, nbr, n_out, 2, sms);
    out[3] = run_l1<0, 4, 4>(feat, nbr, n_out, 2, sms);
    out[4] = run_l1<1, 2, 8>(feat, nbr, n_out, 1, sms);
    out[5] = run_l1<1, 4, 8>(feat, nbr, n_out, 1, sms);
    out[6] = run_l1<1, 2, 8>(feat, nbr, n_out, 2, sms);
    out[7] = run_l1<1, 4, 8>(feat, nbr, n_out, 2, sms);
    out[8] = run_l1<0, 12, 4>(feat, nbr, n_out, 1, sms);
    return 0;
}

// ---------------------------------------------------------------- (2e) smem window -> TMEM A operand
// per 16-KB A tile: 128 threads each LDS.128 x8 one random window row (own TMEM lane) + tcgen05.st.
template <int SWZ>
__global__ void __launch_bounds__(128, 1) k_lds_sttm(const uint16_t* lidx, int iters, long long* cycles) {
    extern __shared__ uint8_t dsm[];
    __shared__ uint32_t slot;
    const uint32_t base = (smem_u32(dsm) + 1023) & ~1023u;   // window: 512 rows x 128 B = 64 KB
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 512 * 32; i += 128)
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(base + 4 * i), "r"(i) : "memory");
    if (warp == 0) tmem_alloc(smem_u32(&slot), 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot + ((uint32_t)(warp * 32) << 16);
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int u = lidx[(it * 128 + threadIdx.x) & 65535] & 511;
        uint32_t v[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int cc = SWZ ? ((c + lane) & 7) : c;
            const uint32_t addr = base + u * 128 + ((SWZ ? (cc ^ (u & 7)) : cc) << 4);
            asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[4 * cc]), "=r"(v[4 * cc + 1]), "=r"(v[4 * cc + 2]), "=r"(v[4 * cc + 3]) : "r"(addr));
        }
        const uint32_t ta = tmem + (it & 7) * 32;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
            "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
            ::"r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
            "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
            "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]),
            "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
            : "memory");
        acc += v[0];
    }
    tmem_st_wait();
    long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0 + (acc == 12345 ? 1 : 0);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(slot, 256);
    }
}

extern "C" int mb_lds_sttm(const uint16_t* lidx, int iters, long long* cycles, float* ms, int swz) {
    size_t smem = 65536 + 1024;
    auto k = swz ? k_lds_sttm<1> : k_lds_sttm<0>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<<<148, 128, smem>>>(lidx, iters, cycles);
    cudaEventRecord(a);
    k<<<148, 128, smem>>>(lidx, iters, cycles);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(ms, a, b);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------- (2f) register gather -> TMEM (A operand path)
// Each producer warp owns TMEM lane quarter (warp & 3); lane t loads its row (8 x 16 B, L1-cached)
// and stores it with tcgen05.st.32x32b.x32 into a TMEM ring of 32-column stages.  No shared-memory
// traffic for A.  NPW = 4 or 8 producer warps (8: two warps per lane quarter alternate stages).
__device__ __forceinline__ void ld_row(const bf16* p, uint32_t (&v)[32], int valid) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        if (valid) {
            asm volatile("ld.global.v4.b32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[4 * c]), "=r"(v[4 * c + 1]), "=r"(v[4 * c + 2]), "=r"(v[4 * c + 3])
                         : "l"(p + 8 * c));
        }
    }
}
__device__ __forceinline__ void st_tmem32(uint32_t ta, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
        ::"r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
        "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]),
        "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}

template <int NPW>
__global__ void __launch_bounds__(NPW * 32 + 64, 1) k_gather_tmem(const bf16* feat, const int32_t* nbr, long long n_out,
                                                                 int num_tiles) {
    constexpr int TSTAGES = 8;
    __shared__ __align__(8) uint64_t full[TSTAGES], empty[TSTAGES];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int GROUPS = NPW / 4;  // warps per lane quarter
    if (threadIdx.x == 0) {
        for (int s = 0; s < TSTAGES; ++s) {
            mbar_init(smem_u32(&full[s]), 4);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == NPW) tmem_alloc(smem_u32(&slot), 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (warp < NPW) {
        const int quarter = warp & 3, grp = warp >> 2;
        const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
        uint32_t it = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x)
            for (int d = 0; d < 27; ++d, ++it) {
                if ((int)(it % GROUPS) != grp) continue;
                const uint32_t s = it % TSTAGES, ph = (it / TSTAGES) & 1;
                const long long row = (long long)t * 128 + quarter * 32 + lane;
                const int idx = nbr[(long long)d * n_out + row];
                uint32_t v[32];
                ld_row(feat + (long long)(idx < 0 ? 0 : idx) * 64, v, idx >= 0);
                mbar_wait(smem_u32(&empty[s]), ph ^ 1);
                st_tmem32(lane_base + s * 32, v);
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&full[s]));
            }
    } else if (warp == NPW + 1 && lane == 0) {
        uint32_t it = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x)
            for (int d = 0; d < 27; ++d, ++it) {
                uint32_t s = it % TSTAGES, ph = (it / TSTAGES) & 1;
                mbar_wait(smem_u32(&full[s]), ph);
                tc_fence_after();
                mbar_arrive(smem_u32(&empty[s]));
            }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == NPW) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

extern "C" int mb_gather_tmem(const void* feat, const int32_t* nbr, long long n_out, int npw, float* ms) {
    int tiles = (int)(n_out / 128);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    void (*k)(const bf16*, const int32_t*, long long, int) =
        npw == 4 ? k_gather_tmem<4> : (npw == 8 ? k_gather_tmem<8> : k_gather_tmem<16>);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        k<<<sms, npw * 32 + 64>>>((const bf16*)feat, nbr, n_out, tiles);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(ms, a, b);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------- (3) MMA issue rate
template <int N>
__global__ void __launch_bounds__(128, 1) k_mma_rate(int iters, long long* cycles) {
    extern __shared__ uint8_t dsm[];
    __shared__ __align__(8) uint64_t done;
    __shared__ uint32_t slot;
    const uint32_t base = (smem_u32(dsm) + 1023) & ~1023u;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&done), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(smem_u32(&slot), 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = idesc_bf16_f32(128, N, false, false);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                uint64_t ad = smem_desc(base + ks * 32, 16, 1024, kSwizzle128B);
                uint64_t bd = smem_desc(base + 16384 + ks * 32, 16, 1024, kSwizzle128B);
                mma_bf16(tmem, ad, bd, idesc, (i | ks) != 0);
            }
        mma_commit(smem_u32(&done));
        mbar_wait(smem_u32(&done), 0);
        cycles[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

extern "C" int mb_mma_rate(int n, int iters, int blocks, long long* cycles_dev, float* ms) {
    size_t smem = 16384 + 32768 + 1024;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    void (*k)(int, long long*) = n == 64 ? k_mma_rate<64> : (n == 128 ? k_mma_rate<128> : k_mma_rate<256>);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<blocks, 128, smem>>>(iters, cycles_dev);
    cudaEventRecord(a);
    k<<<blocks, 128, smem>>>(iters, cycles_dev);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(ms, a, b);
    return (int)cudaGetLastError();
}
