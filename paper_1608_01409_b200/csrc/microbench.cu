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

// 16 independent packed FFMA2 chains per thread (fma.rn.f32x2: two FP32 FMAs per
// instruction, the JIT kernel's inner instruction), no memory traffic in the loop.
__device__ __forceinline__ unsigned long long ffma2(unsigned long long x, unsigned long long a,
                                                   unsigned long long b) {
    unsigned long long d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x), "l"(a), "l"(b));
    return d;
}

__global__ void __launch_bounds__(256) ffma2_kernel(float *out, int iters, float a, float b) {
    unsigned long long x[kChains];
    unsigned long long aa, bb;
    asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
    asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(b));
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
        const float v = threadIdx.x * 1e-3f + i;
        asm("mov.b64 %0, {%1, %2};" : "=l"(x[i]) : "f"(v), "f"(v + 0.5f));
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int i = 0; i < kChains; ++i) x[i] = ffma2(x[i], aa, bb);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[i]));
        s += lo + hi;
    }
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

// Conflict-free LDS.64: lane l reads the 8-byte word (w*32 + l + 32*k) mod 4096 (a warp's
// load is 256 contiguous bytes = 2 wavefronts, like the JIT kernel's window loads).
__global__ void __launch_bounds__(256) lds64_kernel(float *out, int iters) {
    __shared__ float2 buf[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = make_float2(float(i & 7), 1.0f);
    __syncthreads();
    float2 s0 = {0, 0}, s1 = {0, 0}, s2 = {0, 0}, s3 = {0, 0};
    int idx = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float2 a = buf[(idx + 0 * 256) & 4095], b = buf[(idx + 1 * 256) & 4095];
            const float2 c = buf[(idx + 2 * 256) & 4095], d = buf[(idx + 3 * 256) & 4095];
            s0.x += a.x; s0.y += a.y; s1.x += b.x; s1.y += b.y;
            s2.x += c.x; s2.y += c.y; s3.x += d.x; s3.y += d.y;
            idx += 1024 + 32;
        }
    }
    const float s = s0.x + s0.y + s1.x + s1.y + s2.x + s2.y + s3.x + s3.y;
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

cudaError_t bench_ffma2(void *scratch, int blocks, int iters, float *ms, double *flops) {
    *flops = 4.0 * blocks * 256.0 * iters * 8.0 * kChains;  // 2 FMAs of 2 FLOP per FFMA2
    return timed([&] { ffma2_kernel<<<blocks, 256>>>((float *)scratch, iters, 1.0001f, 1e-7f); },
                 ms);
}

cudaError_t bench_lds64(void *scratch, int blocks, int iters, float *ms, double *bytes) {
    *bytes = 8.0 * blocks * 256.0 * iters * 8.0 * 4.0;
    return timed([&] { lds64_kernel<<<blocks, 256>>>((float *)scratch, iters); }, ms);
}

cudaError_t bench_lds(void *scratch, int blocks, int iters, float *ms, double *bytes) {
    *bytes = 4.0 * blocks * 256.0 * iters * 8.0 * 4.0;
    return timed([&] { lds_kernel<<<blocks, 256>>>((float *)scratch, iters); }, ms);
}

}  // namespace skc
