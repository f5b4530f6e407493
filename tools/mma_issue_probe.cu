// Issue-rate probe for tcgen05.mma (M=128, N=64, K=16, bf16 -> f32), 148 CTAs, cycles per MMA.
// Tells whether single-thread issue is bound by operand set-up (R2UR chains) or by the hardware:
//   mode 0: one thread, TS, loop-invariant operands (same D, A, B every MMA)
//   mode 1: one thread, TS, A/B advance per K-step (as a K=64 stage: a + 8ks, b + 2ks)
//   mode 2: one thread, TS, one asm block issuing a whole K=64 stage (4 MMAs) from base registers
//   mode 3: whole warp, elect inside the asm, loop-invariant operands
//   mode 4: one thread, SS, loop-invariant operands
//   mode 5: two threads (warps 0, 1), TS, loop-invariant operands, separate accumulators
// per-iteration cost of the issue loop's synchronisation (whole warp 0; "cycles_per_mma" = per iteration):
//   mode 6: tcgen05.commit (elect) to an mbarrier;  mode 7: tcgen05.fence::after_thread_sync
//   mode 8: mbar_wait on an already-completed phase;  mode 9: 2 waits + fence + commit (a batch skeleton)
//   mode 10: mode 9 + one 4-MMA stage (mma_ts_x4_elect)
//   mode 11: lane-0 wait + __syncwarp;  mode 12: fence by lane 0 only
//   mode 13: batch skeleton with lane-0 waits, lane-0 fence, commit;  mode 14: mode 13 + one 4-MMA stage
#include <cstdint>
#include <cstdio>
#include "../paper_2407_01781_b200/csrc/tc_ptx.cuh"

using namespace fvdb::tc;

__device__ __forceinline__ void stage4_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc) {
    asm volatile(
        "{\n\t.reg .b32 a1, a2, a3;\n\t.reg .b64 b1, b2, b3;\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, 1, 0;\n\t"
        "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
        "add.u64 b1, %2, 2;\n\tadd.u64 b2, %2, 4;\n\tadd.u64 b3, %2, 6;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, p;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], b2, %3, p;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], b3, %3, p;\n\t}"
        ::"r"(d), "r"(a), "l"(b), "r"(idesc) : "memory");
}

__global__ void __launch_bounds__(128, 1) k_issue(int iters, int mode, long long* cycles) {
    __shared__ __align__(1024) uint8_t sm[32768];
    __shared__ __align__(8) uint64_t done[2];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&done[0]), 1);
        mbar_init(smem_u32(&done[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(smem_u32(&slot), 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t idesc = idesc_bf16_f32(128, 64, false, false);
    const uint32_t s = smem_u32(sm);
    const uint64_t bd = smem_desc(s, 16, 1024, kSwizzle128B);
    long long t0 = 0;
    bool timer = false;
    if (mode >= 6) {
        __shared__ __align__(8) uint64_t ready, sink;
        if (threadIdx.x == 0) {
            mbar_init(smem_u32(&ready), 1);
            mbar_init(smem_u32(&sink), 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            mbar_arrive(smem_u32(&ready));  // phase 0 complete
        }
        __syncthreads();
        if (warp == 0) {
            const uint32_t R = smem_u32(&ready), S = smem_u32(&sink);
            t0 = clock64();
            for (int i = 0; i < iters; ++i) {
                if (mode == 6) mma_commit_elect(S);
                if (mode == 7) tc_fence_after();
                if (mode == 8) mbar_wait(R, 0);
                if (mode == 11) {
                    if (lane == 0) mbar_wait(R, 0);
                    __syncwarp();
                }
                if (mode == 12 && lane == 0) tc_fence_after();
                if (mode >= 13) {
                    if (lane == 0) {
                        mbar_wait(R, 0);
                        mbar_wait(R, 0);
                        tc_fence_after();
                    }
                    __syncwarp();
                    if (mode == 14) mma_ts_x4_elect<8, 16, 24, 2, 4, 6>(tmem, tmem + 256, bd, idesc);
                    mma_commit_elect(S);
                }
                if (mode == 9 || mode == 10) {
                    mbar_wait(R, 0);
                    mbar_wait(R, 0);
                    tc_fence_after();
                    if (mode == 10) mma_ts_x4_elect<8, 16, 24, 2, 4, 6>(tmem, tmem + 256, bd, idesc);
                    mma_commit_elect(S);
                }
            }
            timer = lane == 0;
        }
    } else if (mode == 3) {
        if (warp == 0) {
            t0 = clock64();
            for (int i = 0; i < iters; ++i) mma_bf16_ts_elect(tmem, tmem + 256, bd, idesc, 1u);
            mma_commit_elect(smem_u32(&done[0]));
            mbar_wait(smem_u32(&done[0]), 0);
            timer = lane == 0;
        }
    } else if (mode == 5) {
        if (warp < 2 && lane == 0) {
            t0 = clock64();
            for (int i = 0; i < iters / 2; ++i) mma_bf16_ts(tmem + warp * 64, tmem + 256 + warp * 32, bd, idesc, 1u);
            mma_commit(smem_u32(&done[warp]));
            mbar_wait(smem_u32(&done[warp]), 0);
            timer = warp == 0;
        }
    } else if (threadIdx.x == 0) {
        t0 = clock64();
        if (mode == 0) {
            for (int i = 0; i < iters; ++i) mma_bf16_ts(tmem, tmem + 256, bd, idesc, 1u);
        } else if (mode == 1) {
            for (int i = 0; i < iters / 4; ++i)
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) mma_bf16_ts(tmem, tmem + 256 + 8 * ks, bd + 2 * ks, idesc, 1u);
        } else if (mode == 2) {
            for (int i = 0; i < iters / 4; ++i) stage4_ts(tmem, tmem + 256, bd, idesc);
        } else {
            for (int i = 0; i < iters; ++i) mma_bf16(tmem, bd, bd, idesc, 1u);
        }
        mma_commit(smem_u32(&done[0]));
        mbar_wait(smem_u32(&done[0]), 0);
        timer = true;
    }
    if (timer) cycles[blockIdx.x] = clock64() - t0;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

extern "C" int probe_issue(int iters, int mode, long long* cycles) {
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    k_issue<<<148, 128>>>(iters, mode, d);
    k_issue<<<148, 128>>>(iters, mode, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(cycles, d, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
    cudaFree(d);
    return (int)e;
}
