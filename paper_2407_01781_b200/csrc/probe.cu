// probe.cu — measurement probes for bench.py's roofline denominators (not on the product path).
//
// fvdb_probe_ffma: the FP32 CUDA-core FMA peak, which MEASURED_PEAKS.json does not carry and which bounds the
// exact-precision (fp32) gather conv of cfg1.  Every thread runs 8 independent FFMA chains
// (enough in flight to cover the FMA latency) for `iters` rounds; 8 blocks of 256 threads per SM.
#include "common.cuh"

namespace fvdb {
namespace {

__global__ void __launch_bounds__(256) k_probe_ffma(int iters, float* __restrict__ out, int64_t n) {
    float a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = (float)(threadIdx.x + j) * 1e-3f;
    const float b = 0.999f, c = 1e-6f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], b, c);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += a[j];
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < n) out[t] = s;  // keeps the chains live
}

}  // namespace
}  // namespace fvdb

using namespace fvdb;

extern "C" int fvdb_probe_ffma(int iters, float* out, int64_t n, double* flops, void* stream) {
    const int sms = device_sm_count();
    const int blocks = sms * 8, threads = 256;
    k_probe_ffma<<<blocks, threads, 0, as_stream(stream)>>>(iters, out, n);
    FVDB_LAUNCH_CHECK();
    *flops = 2.0 * 16 * 8 * (double)iters * blocks * threads;
    return FVDB_OK;
}
