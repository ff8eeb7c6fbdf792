// FP32 FMA-pipe throughput probe: the measured denominator of the raster
// kernels' roofline ("measure sustained FP32 FMA on the box").
// Every thread runs 8 independent fma.rn.f32 chains (enough ILP to cover the
// FMA latency at any occupancy); bench.py times the launch with CUDA events
// on its stream.  flops per launch = blocks * 256 threads * iters * 16 * 8 * 2.
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace isg {

__global__ void __launch_bounds__(256) ffma_probe_kernel(int32_t iters, float b, float c,
                                                         float *__restrict__ out) {
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = (float)threadIdx.x * 1e-3f + (float)k;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int u = 0; u < 16; u++) {
#pragma unroll
            for (int k = 0; k < 8; k++) a[k] = __fmaf_rn(a[k], b, c);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; k++) s += a[k];
    if (s == -1.2345f) out[blockIdx.x] = s;  // never true; keeps the chains live
}

}  // namespace isg

extern "C" int isg_probe_ffma(int32_t blocks, int32_t iters, float *out, void *stream) {
    if (blocks <= 0 || iters <= 0 || !out) return (int)cudaErrorInvalidValue;
    isg::ffma_probe_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(iters, 0.99999994f, 1e-7f,
                                                                     out);
    ISG_CHECK_LAUNCH();
    return 0;
}
