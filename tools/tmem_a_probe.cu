// tmem_a_probe.cu — verifies the TMEM A-operand layout of tcgen05.mma kind::f16 (A from TMEM, B from smem)
// and the 16x256b.xN store mapping + K permutation used by the halo kernel.  Standalone probe (tools/).
//
// mode 0: A row m written by thread m with tcgen05.st.32x32b.x32: column j = bf16 pair (2j, 2j+1);
//         B image in natural K order.  Expect D = A · Bᵀ.
// mode 1: A written with tcgen05.st.16x256b.x4 as the halo kernel does (thread t0 = t&3 of a 4-thread row
//         group holds channels 8·c(t0,j) + 0..7 for loads j = 0,1 with c = 2·t0 + j); B image packed with
//         the matching permutation π(k) (host).  Expect D = A · Bᵀ.
#include <cuda_bf16.h>
#include <stdint.h>

#include "../paper_2407_01781_b200/csrc/tc_ptx.cuh"

using namespace fvdb::tc;

__device__ __forceinline__ uint32_t swz128(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

__device__ __forceinline__ void st32x32(uint32_t ta, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,"
        "%29,%30,%31,%32};" ::"r"(ta),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
__device__ __forceinline__ void st16x256x4(uint32_t ta, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}

__global__ void __launch_bounds__(128, 1) k_probe(const uint16_t* A, const uint8_t* bimg, float* out, int mode) {
    __shared__ __align__(1024) uint8_t sB[8192];
    __shared__ __align__(8) uint64_t done;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 8192 / 16; i += 128)
        reinterpret_cast<uint4*>(sB)[i] = reinterpret_cast<const uint4*>(bimg)[i];
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&done), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(smem_u32(&slot), 128);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot, ta = tmem + 64;  // D: cols 0..63, A: cols 64..95
    const uint32_t qlane = (uint32_t)(warp * 32) << 16;
    const uint32_t* A32 = reinterpret_cast<const uint32_t*>(A);  // row-major [128][64] bf16 = [128][32] words
    if (mode == 0) {
        uint32_t v[32];
        const int m = warp * 32 + lane;
        for (int j = 0; j < 32; ++j) v[j] = A32[m * 32 + j];
        st32x32(ta + qlane, v);
    } else {
        const int t0 = lane & 3, t1 = lane >> 2;
        for (int g = 0; g < 2; ++g) {
            uint32_t v[16];
            for (int hi = 0; hi < 2; ++hi) {
                const int row = warp * 32 + g * 16 + t1 + 8 * hi;
                for (int i = 0; i < 8; ++i) {
                    const int j = i >> 2, e = i & 3, c = 2 * t0 + j;
                    v[4 * (i >> 1) + (i & 1) + 2 * hi] = A32[row * 32 + 4 * c + e];
                }
            }
            st16x256x4(ta + qlane + ((uint32_t)(g * 16) << 16), v);
        }
    }
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_bf16_f32(128, 64, false, false);
        for (int ks = 0; ks < 4; ++ks) {
            uint64_t bd = smem_desc(smem_u32(sB) + ks * 32, 16, 1024, kSwizzle128B);
            mma_ts(tmem, ta + ks * 8, bd, idesc, ks > 0);
        }
        mma_commit(smem_u32(&done));
    }
    __syncwarp();
    mbar_wait(smem_u32(&done), 0);
    tc_fence_after();
    for (int c0 = 0; c0 < 64; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + qlane + c0, v);
        tmem_ld_wait();
        for (int j = 0; j < 32; ++j) out[(warp * 32 + lane) * 64 + c0 + j] = __uint_as_float(v[j]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 128);
    }
}

extern "C" int probe_tmem_a(const void* A, const void* bimg, float* out, int mode) {
    k_probe<<<1, 128>>>((const uint16_t*)A, (const uint8_t*)bimg, out, mode);
    cudaError_t e = cudaDeviceSynchronize();
    return (int)e;
}

// whole-warp issue: one elected lane executes the MMA (no compiler-generated uniformity loop)
__device__ __forceinline__ void mma_ts_elect(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_ss_elect(uint32_t d, uint64_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}

// ---- issue rate: M=128, N=64, K=16 MMAs back to back (mode 0 SS, 1 TS, 2 TS + zero mask, 3 TS + half mask)
template <int N>
__global__ void __launch_bounds__(128, 1) k_rate(int iters, int mode, long long* cycles) {
    __shared__ __align__(1024) uint8_t sm[32768];
    __shared__ __align__(8) uint64_t done;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&done), (mode == 6 || mode == 8) ? 2 : ((mode == 7 || mode == 9) ? 4 : 1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(smem_u32(&slot), 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (mode >= 6) {  // modes 6/7: 2 / 4 warps, lane 0 of each issues SS MMAs into its own accumulator
        const int nw = (mode == 6 || mode == 8) ? 2 : 4;
        if (4 * N + nw * 32 > 512) {
            if (threadIdx.x == 0) cycles[blockIdx.x] = 0;
        } else if (warp < nw && (threadIdx.x & 31) == 0) {
            const uint32_t idesc = idesc_bf16_f32(128, N, false, false);
            const uint32_t sA = smem_u32(sm), sB = sA;
            const uint32_t dcol = tmem + warp * N;
            long long t0 = clock64();
            const bool ts = mode >= 8;
            const uint32_t acol = tmem + 4 * N + warp * 32;  // A (TS): 32 columns per warp after the D regions
            for (int i = 0; i < iters / nw; ++i)
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    if (ts)
                        mma_ts(dcol, acol + ks * 8, smem_desc(sB + ks * 32, 16, 1024, kSwizzle128B), idesc, (i | ks) != 0);
                    else
                        mma_bf16(dcol, smem_desc(sA + ks * 32, 16, 1024, kSwizzle128B),
                                 smem_desc(sB + ks * 32, 16, 1024, kSwizzle128B), idesc, (i | ks) != 0);
                }
            mma_commit(smem_u32(&done));
            if (warp == 0) {
                mbar_wait(smem_u32(&done), 0);
                cycles[blockIdx.x] = clock64() - t0;
            }
        }
    } else if (mode >= 4) {  // whole warp 0, elect.sync inside the asm
        if (warp == 0) {
            const uint32_t idesc = idesc_bf16_f32(128, N, false, false);
            const uint32_t sA = smem_u32(sm), sB = sA;
            long long t0 = clock64();
            for (int i = 0; i < iters; ++i)
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    uint64_t bd = smem_desc(sB + ks * 32, 16, 1024, kSwizzle128B);
                    if (mode == 4) {
                        mma_ss_elect(tmem, smem_desc(sA + ks * 32, 16, 1024, kSwizzle128B), bd, idesc, (i | ks) != 0);
                    } else {
                        mma_ts_elect(tmem, tmem + 256 + ks * 8, bd, idesc, (i | ks) != 0);
                    }
                }
            if ((threadIdx.x & 31) == 0) mma_commit(smem_u32(&done));
            __syncwarp();
            mbar_wait(smem_u32(&done), 0);
            if ((threadIdx.x & 31) == 0) cycles[blockIdx.x] = clock64() - t0;
        }
    } else if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_bf16_f32(128, N, false, false);
        const uint32_t sA = smem_u32(sm), sB = sA;  // operand values are irrelevant here
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                uint64_t bd = smem_desc(sB + ks * 32, 16, 1024, kSwizzle128B);
                if (mode == 0) {
                    uint64_t ad = smem_desc(sA + ks * 32, 16, 1024, kSwizzle128B);
                    mma_bf16(tmem, ad, bd, idesc, (i | ks) != 0);
                } else if (mode == 1) {
                    mma_ts(tmem, tmem + 256 + ks * 8, bd, idesc, (i | ks) != 0);
                } else {
                    const uint32_t h = mode == 3 ? 0xffffffffu : 0u;
                    mma_bf16_ts_masked(tmem, tmem + 256 + ks * 8, bd, idesc, (i | ks) != 0, 0u, h, 0u, h);
                }
            }
        mma_commit(smem_u32(&done));
        mbar_wait(smem_u32(&done), 0);
        cycles[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

extern "C" int probe_rate(int n, int iters, int mode, long long* cycles, float* ms) {
    void (*kr)(int, int, long long*) = n == 64 ? k_rate<64> : (n == 128 ? k_rate<128> : k_rate<256>);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kr<<<148, 128>>>(iters, mode, cycles);
    cudaEventRecord(a);
    kr<<<148, 128>>>(iters, mode, cycles);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(ms, a, b);
    return (int)cudaGetLastError();
}

// ---- cost of waiting on an already-completed mbarrier phase: try_wait vs test_wait (mbar_test: tc_ptx.cuh)
__global__ void k_wait_cost(int iters, long long* out) {
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_arrive(smem_u32(&bar));  // phase 0 complete
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const uint32_t b = smem_u32(&bar);
        uint32_t acc = 0;
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) acc += mbar_try_wait(b, 0) ? 1u : 0u;
        long long t1 = clock64();
        for (int i = 0; i < iters; ++i) acc += mbar_test(b, 0) ? 1u : 0u;
        long long t2 = clock64();
        for (int i = 0; i < iters; ++i) mbar_wait(b, 0);
        long long t3 = clock64();
        if (threadIdx.x == 0) {
            out[0] = t1 - t0;
            out[1] = t2 - t1;
            out[2] = t3 - t2;
            out[3] = acc;
        }
    }
}
extern "C" int probe_wait_cost(int iters, long long* out) {
    k_wait_cost<<<1, 32>>>(iters, out);
    return (int)cudaDeviceSynchronize();
}

// ---- cta_group::2 issue rate: 2-CTA cluster, leader thread issues M=256 (128 rows per CTA) N=64 K=16 MMAs
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_rate2(int iters, int ts, long long* cycles) {
    __shared__ __align__(1024) uint8_t sm[32768];
    __shared__ __align__(8) uint64_t done;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    const uint32_t rank = cluster_rank();
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&done), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    tc_fence_after();
    const uint32_t tmem = slot;
    if (rank == 0 && threadIdx.x == 0) {
        const uint32_t idesc = idesc_bf16_f32(256, 64, false, false);
        const uint32_t sA = smem_u32(sm), sB = sA;
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const uint64_t bd = smem_desc(sB + ks * 32, 16, 1024, kSwizzle128B);
                const uint32_t acc = (i | ks) != 0;
                if (ts) {
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                                 "r"(tmem + 256 + ks * 8), "l"(bd), "r"(idesc), "r"(acc)
                                 : "memory");
                } else {
                    const uint64_t ad = smem_desc(sA + ks * 32, 16, 1024, kSwizzle128B);
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                 "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
                                 : "memory");
                }
            }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     ::"r"(smem_u32(&done)), "h"((uint16_t)3)
                     : "memory");
        mbar_wait(smem_u32(&done), 0);
        cycles[blockIdx.x / 2] = clock64() - t0;
    } else if (rank == 1 && threadIdx.x == 0) {
        mbar_wait(smem_u32(&done), 0);
    }
    tc_fence_before();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    }
}
extern "C" int probe_rate2(int iters, int ts, long long* cycles, float* ms) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_rate2<<<148, 128>>>(iters, ts, cycles);
    cudaEventRecord(a);
    k_rate2<<<148, 128>>>(iters, ts, cycles);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(ms, a, b);
    return (int)cudaGetLastError();
}
