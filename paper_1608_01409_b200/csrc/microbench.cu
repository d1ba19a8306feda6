// microbench.cu -- calibration kernels for the B200 roofline: the
// CUDA-core FP32 FMA rate and the shared-memory word rate.  They play the role of the
// paper's SGEMM / STREAM calibration: measured "achievable"
// peaks rather than data-sheet numbers.
#include "skc_internal.h"

namespace skc {
namespace {

constexpr int kChains = 16;

// 16 independent FFMA chains per thread, no memory traffic in the loop.
__global__ void __launch_bounds__(256) ffma_kernel(float *out, int iters, float a, float b) {
    float x[kChains];
#pragma unroll
    for (int i = 0; i < kChains; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int i = 0; i < kChains; ++i) x[i] = fmaf(x[i], a, b);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < kChains; ++i) s += x[i];
    if (s == 1234.5f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;  // defeat DCE
}

// Conflict-free LDS.32: lane l of warp w reads word (w*32 + l + 32*k) mod 8192.
__global__ void __launch_bounds__(256) lds_kernel(float *out, int iters) {
    __shared__ float buf[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = float(i & 7);
    __syncthreads();
    float s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    int idx = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            s0 += buf[(idx + 0 * 256) & 8191];
            s1 += buf[(idx + 1 * 256) & 8191];
            s2 += buf[(idx + 2 * 256) & 8191];
            s3 += buf[(idx + 3 * 256) & 8191];
            idx += 1024 + 32;
        }
    }
    const float s = s0 + s1 + s2 + s3;
    if (s == 1234.5f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class F>
cudaError_t timed(F &&launch, float *ms) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();  // warm-up
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    if (e == cudaSuccess) e = cudaGetLastError();
    cudaEventElapsedTime(ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return e;
}

}  // namespace

cudaError_t bench_ffma(void *scratch, int blocks, int iters, float *ms, double *flops) {
    *flops = 2.0 * blocks * 256.0 * iters * 8.0 * kChains;
    return timed([&] { ffma_kernel<<<blocks, 256>>>((float *)scratch, iters, 1.0001f, 1e-7f); },
                 ms);
}

cudaError_t bench_lds(void *scratch, int blocks, int iters, float *ms, double *bytes) {
    *bytes = 4.0 * blocks * 256.0 * iters * 8.0 * 4.0;
    return timed([&] { lds_kernel<<<blocks, 256>>>((float *)scratch, iters); }, ms);
}

}  // namespace skc
