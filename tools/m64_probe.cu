// Probe of the M=64 tcgen05.mma TMEM layouts (cta_group::1, kind::f16, A in TMEM): where A's 64 rows must
// sit in TMEM and which lanes hold D's 64 rows.  A[m][0] = m + 1 (other K zero), B[0][n] = 1 (other K
// zero), so D[m][n] = m + 1; the host reads D from all 128 lanes.  Standalone probe (tools/).
//   layout 0: A row m in lane m (lanes 0-63);  layout 1: A row m in lane (m / 16) * 32 + m % 16
#include <cuda_bf16.h>
#include <stdint.h>

#include "../paper_2407_01781_b200/csrc/tc_ptx.cuh"

using namespace fvdb::tc;

__global__ void __launch_bounds__(128, 1) k_m64(int layout, float* out) {
    __shared__ __align__(1024) uint8_t sB[64 * 128];
    __shared__ __align__(8) uint64_t done;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = threadIdx.x;
    for (int i = t; i < 64 * 128 / 4; i += 128) reinterpret_cast<uint32_t*>(sB)[i] = 0u;
    __syncthreads();
    if (t < 64) {  // B image row n (K-major, 128B swizzle): k = 0 lives in chunk 0 ^ (n % 8)
        __nv_bfloat16 one = __float2bfloat16(1.0f);
        *reinterpret_cast<__nv_bfloat16*>(sB + t * 128 + ((t % 8) * 16)) = one;
    }
    if (t == 0) {
        mbar_init(smem_u32(&done), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(smem_u32(&slot), 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    // A at columns 256..263 (8 columns = 16 bf16 of K), D at columns 0..63
    {
        int m = -1;
        if (layout == 0) m = t < 64 ? t : -1;
        else m = (t % 32) < 16 ? (t / 32) * 16 + (t % 32) : -1;
        uint32_t v[32];
        for (int j = 0; j < 32; ++j) v[j] = 0u;
        if (m >= 0) {
            __nv_bfloat162 p = __floats2bfloat162_rn((float)(m + 1), 0.0f);  // (k=0, k=1)
            v[0] = *reinterpret_cast<uint32_t*>(&p);
        }
        const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + 256;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
            "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
            "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
            "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
            "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
            : "memory");
        // D columns 0..63 poisoned with -1 so untouched lanes are visible
        for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(-1.0f);
        const uint32_t td = tmem + ((uint32_t)(warp * 32) << 16);
        for (int c = 0; c < 64; c += 32)
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(td + c),
                "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
                "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
                "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
                : "memory");
        tmem_st_wait();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (t == 0) {
        const uint64_t bd = smem_desc(smem_u32(sB), 16, 1024, kSwizzle128B);
        mma_bf16_ts(tmem, tmem + 256, bd, idesc_bf16_f32(64, 64, false, false), 0u);
        mma_commit(smem_u32(&done));
    }
    mbar_wait(smem_u32(&done), 0);
    tc_fence_after();
    uint32_t r[32];
    for (int c = 0; c < 64; c += 32) {
        tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
        tmem_ld_wait();
        for (int j = 0; j < 32; ++j) out[t * 64 + c + j] = __uint_as_float(r[j]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

extern "C" int probe_m64(int layout, float* host_out) {
    float* d;
    cudaMalloc(&d, 128 * 64 * sizeof(float));
    k_m64<<<1, 128>>>(layout, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(host_out, d, 128 * 64 * sizeof(float), cudaMemcpyDeviceToHost);
    cudaFree(d);
    return (int)e;
}
