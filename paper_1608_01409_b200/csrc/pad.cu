// pad.cu -- row a2: NCHW -> zero-padded [N][C][Hp][Wp] (R1).
//
// HBM-bound copy.  Algorithmic bytes per image: read C*H*W*4, write C*Hp*Wp*4.
// grid.y = image, grid.x strides over the image's C*Hp*Wp outputs, 4 per thread, with
// float4 stores when the per-image element count allows it.  Index math uses 32-bit
// magic-number division (C*Hp*Wp < 2^31 is checked at pack time).
#include "ptx.cuh"
#include "skc_internal.h"

#include <cstdlib>

namespace skc {
namespace {

// Programmatic dependent launch (launched with the programmatic-serialization attribute):
// wait until the preceding grid has completed and its writes are visible (this pass may read
// the previous layer's output), then let the next grid's CTAs be scheduled as SMs free up.
// Both are no-ops for a plain launch.
__device__ __forceinline__ void pdl_wait_and_trigger() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

constexpr int kPadVec = 4;    // outputs per vector (float4 store)
constexpr int kPadUnroll = 4; // vectors per thread per iteration: 16 loads in flight

__global__ void __launch_bounds__(256) pad_kernel(const float *__restrict__ in,
                                                  float *__restrict__ out, int C, int H, int W,
                                                  int pad, int Wp, uint32_t per_img,
                                                  FastDiv div_plane, FastDiv div_wp, int vec4) {
    pdl_wait_and_trigger();
    const int64_t n = blockIdx.y;
    const float *src = in + n * int64_t(C) * H * W;
    float *dst = out + n * int64_t(per_img);
    const uint32_t span = blockDim.x * kPadVec;  // outputs covered by one vector round
    const uint32_t stride = gridDim.x * span * kPadUnroll;
    for (uint32_t base = blockIdx.x * span * kPadUnroll + threadIdx.x * kPadVec; base < per_img;
         base += stride) {
        float v[kPadUnroll][kPadVec];
        // all loads first (independent), then the stores
#pragma unroll
        for (int u = 0; u < kPadUnroll; ++u) {
            const uint32_t i0 = base + u * span;
#pragma unroll
            for (int k = 0; k < kPadVec; ++k) {
                const uint32_t i = i0 + k;
                v[u][k] = 0.0f;
                if (i < per_img) {
                    const uint32_t plane = fdiv(i, div_plane);
                    const uint32_t rem = i - plane * div_plane.d;
                    const uint32_t yy = fdiv(rem, div_wp);
                    const int y = int(yy) - pad;
                    const int x = int(rem - yy * uint32_t(Wp)) - pad;
                    if (y >= 0 && y < H && x >= 0 && x < W)
                        v[u][k] = __ldg(src + (int64_t(plane) * H + y) * W + x);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kPadUnroll; ++u) {
            const uint32_t i0 = base + u * span;
            if (vec4 && i0 + 3 < per_img) {
                *reinterpret_cast<float4 *>(dst + i0) =
                    make_float4(v[u][0], v[u][1], v[u][2], v[u][3]);
            } else {
#pragma unroll
                for (int k = 0; k < kPadVec; ++k)
                    if (i0 + k < per_img) dst[i0 + k] = v[u][k];
            }
        }
    }
}

// Row f3: lowering (im2col) for the comparison baseline.
// L[n][(c*R + r)*S + s][y][x] = in[n][c][y*stride + r - pad][x*stride + s - pad] (0 outside).
// HBM-bound (the R*S-fold replicated write stream).  One WARP per lowered row (unit, crs) at a
// time, rows dealt warp-strided over a grid of whole waves: (c, r, s) and the row's source
// base are warp-uniform, so a lane does one division per element (y = pix / Wo), each warp
// store is a contiguous run, and a CTA does many rows (one CTA or one element per thread per
// row made the pass CTA-launch bound: 0.43-1.2 ms for AlexNet conv2-5 at batch 256).
// PAIRS: the image-pair interleaved layout of a JIT 1x1 plan (pad 0): out[p][crs][y][x][j] =
// L[2p+j][crs][y][x], one float2 per element, zero for a missing second image of an odd N.
template <bool PAIRS>
__global__ void __launch_bounds__(256) im2col_kernel(const float *__restrict__ in,
                                                     float *__restrict__ out, int C, int H,
                                                     int W, int R, int S, int stride, int pad,
                                                     int Wo, uint32_t howo, FastDiv div_wo,
                                                     uint32_t CRS, uint64_t rows, int64_t N) {
    constexpr int U = 4;  // elements per lane in flight
    const int lane = threadIdx.x & 31;
    const uint64_t nwarps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    const int64_t img = int64_t(C) * H * W;
    const int RS = R * S;
    for (uint64_t row = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; row < rows;
         row += nwarps) {
        const uint64_t unit = row / CRS;  // image (NCHW) or pair (PAIRS)
        const int crs = int(row - unit * CRS);
        const int c = crs / RS, rs = crs - c * RS;
        const int r = rs / S, s = rs - r * S;
        const float *src = in + int64_t(PAIRS ? 2 * unit : unit) * img + int64_t(c) * H * W;
        const bool hb = PAIRS && int64_t(2 * unit + 1) < N;
        const uint64_t base = row * howo;
        for (uint32_t p0 = lane; p0 < howo; p0 += 32 * U) {
            float2 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t pix = p0 + 32 * u;
                v[u] = make_float2(0.0f, 0.0f);
                const uint32_t y = fdiv(pix, div_wo), x = pix - y * uint32_t(Wo);
                const int yi = int(y) * stride + r - pad, xi = int(x) * stride + s - pad;
                if (pix < howo && yi >= 0 && yi < H && xi >= 0 && xi < W) {
                    const int64_t o = int64_t(yi) * W + xi;
                    v[u].x = __ldg(src + o);
                    if (hb) v[u].y = __ldg(src + img + o);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t pix = p0 + 32 * u;
                if (pix >= howo) break;
                if (PAIRS)
                    reinterpret_cast<float2 *>(out)[base + pix] = v[u];
                else
                    out[base + pix] = v[u].x;
            }
        }
    }
}

// Image-pair interleaved variant (the padded layout of JIT plans; a layout function in the
// sense of PAPER.md:289-292 -- f(n, c, y, x) = (((n/2)*C + c)*Hp + y)*Wp + x)*2 + n%2 keeps
// f(c, y+r, x+s) = f(c, y, x) + f(0, r, s) per image): out[p][c][y][x][j] = in[2p+j][c][y-pad]
// [x-pad], zero in the halo and for a missing second image.  grid.y = pair; each thread
// writes two consecutive (A, B) elements as one float4.
__global__ void __launch_bounds__(256) pad_pairs_kernel(const float *__restrict__ in,
                                                        float *__restrict__ out, int C, int H,
                                                        int W, int pad, int Wp, uint32_t per_img,
                                                        FastDiv div_plane, FastDiv div_wp,
                                                        int has_b) {
    pdl_wait_and_trigger();
    const int64_t p = blockIdx.y;
    const int64_t img = int64_t(C) * H * W;
    const float *srcA = in + 2 * p * img;
    const float *srcB = srcA + img;
    const bool hb = has_b || p + 1 < gridDim.y;
    float *dst = out + p * int64_t(per_img) * 2;
    const uint32_t span = blockDim.x * 2;
    const uint32_t stride = gridDim.x * span * kPadUnroll;
    for (uint32_t base = blockIdx.x * span * kPadUnroll + threadIdx.x * 2; base < per_img;
         base += stride) {
        float v[kPadUnroll][4];
#pragma unroll
        for (int u = 0; u < kPadUnroll; ++u) {
            const uint32_t i0 = base + u * span;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const uint32_t i = i0 + k;
                v[u][2 * k] = v[u][2 * k + 1] = 0.0f;
                if (i < per_img) {
                    const uint32_t plane = fdiv(i, div_plane);
                    const uint32_t rem = i - plane * div_plane.d;
                    const uint32_t yy = fdiv(rem, div_wp);
                    const int y = int(yy) - pad;
                    const int x = int(rem - yy * uint32_t(Wp)) - pad;
                    if (y >= 0 && y < H && x >= 0 && x < W) {
                        const int64_t o = (int64_t(plane) * H + y) * W + x;
                        v[u][2 * k] = __ldg(srcA + o);
                        if (hb) v[u][2 * k + 1] = __ldg(srcB + o);
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kPadUnroll; ++u) {
            const uint32_t i0 = base + u * span;
            if (i0 + 1 < per_img) {
                *reinterpret_cast<float4 *>(dst + 2 * size_t(i0)) =
                    make_float4(v[u][0], v[u][1], v[u][2], v[u][3]);
            } else if (i0 < per_img) {
                *reinterpret_cast<float2 *>(dst + 2 * size_t(i0)) = make_float2(v[u][0], v[u][1]);
            }
        }
    }
}

// Flat variant: one grid-stride loop over every (pair, element) of the batch with a grid of
// whole waves (SMs x 8 CTAs), so the pass has no partly filled last wave per image and no
// per-image grid dimension; otherwise as pad_pairs_kernel.  i < 2^31 (checked by the launcher).
__global__ void __launch_bounds__(256) pad_pairs_flat_kernel(const float *__restrict__ in,
                                                             float *__restrict__ out, int C, int H,
                                                             int W, int pad, int Wp, uint32_t per_img,
                                                             uint32_t total, int64_t N,
                                                             FastDiv div_img, FastDiv div_plane,
                                                             FastDiv div_wp) {
    pdl_wait_and_trigger();
    const int64_t img = int64_t(C) * H * W;
    const uint32_t span = gridDim.x * blockDim.x * 2;
    for (uint32_t base = (blockIdx.x * blockDim.x + threadIdx.x) * 2; base < total;
         base += span * kPadUnroll) {
        float v[kPadUnroll][4];
#pragma unroll
        for (int u = 0; u < kPadUnroll; ++u) {
            const uint32_t i0 = base + u * span;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const uint32_t i = i0 + k;
                v[u][2 * k] = v[u][2 * k + 1] = 0.0f;
                if (i < total) {
                    const uint32_t p = fdiv(i, div_img);
                    const uint32_t r0 = i - p * per_img;
                    const uint32_t plane = fdiv(r0, div_plane);
                    const uint32_t rem = r0 - plane * div_plane.d;
                    const uint32_t yy = fdiv(rem, div_wp);
                    const int y = int(yy) - pad;
                    const int x = int(rem - yy * uint32_t(Wp)) - pad;
                    if (y >= 0 && y < H && x >= 0 && x < W) {
                        const float *a = in + 2 * int64_t(p) * img + (int64_t(plane) * H + y) * W + x;
                        v[u][2 * k] = __ldg(a);
                        if (2 * int64_t(p) + 1 < N) v[u][2 * k + 1] = __ldg(a + img);
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kPadUnroll; ++u) {
            const uint32_t i0 = base + u * span;
            if (i0 + 1 < total) {
                *reinterpret_cast<float4 *>(out + 2 * size_t(i0)) =
                    make_float4(v[u][0], v[u][1], v[u][2], v[u][3]);
            } else if (i0 < total) {
                *reinterpret_cast<float2 *>(out + 2 * size_t(i0)) = make_float2(v[u][0], v[u][1]);
            }
        }
    }
}

}  // namespace

namespace {
cudaError_t im2col_launch(bool pairs, const float *in, float *out, int64_t N, int C, int H, int W,
                          int R, int S, int stride, int pad, int Ho, int Wo, cudaStream_t st) {
    static int nsm = 0;
    if (!nsm) {
        int dev = 0, v = 0;
        nsm = (cudaGetDevice(&dev) == cudaSuccess &&
               cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
                  ? v
                  : 148;
    }
    const uint32_t howo = uint32_t(Ho) * uint32_t(Wo);
    const uint32_t crs = uint32_t(C * R * S);
    const uint64_t rows = uint64_t(pairs ? (N + 1) / 2 : N) * crs;
    // whole waves: 8 CTAs of 8 warps per SM, fewer for a small pass
    const uint64_t need = (rows + 7) / 8;
    const unsigned grid = unsigned(need < uint64_t(nsm) * 8 ? need : uint64_t(nsm) * 8);
    if (pairs)
        im2col_kernel<true><<<grid, 256, 0, st>>>(in, out, C, H, W, R, S, stride, pad, Wo, howo,
                                                  make_fastdiv(uint32_t(Wo)), crs, rows, N);
    else
        im2col_kernel<false><<<grid, 256, 0, st>>>(in, out, C, H, W, R, S, stride, pad, Wo, howo,
                                                   make_fastdiv(uint32_t(Wo)), crs, rows, N);
    return cudaGetLastError();
}
}  // namespace

cudaError_t launch_im2col(const float *in, float *out, int64_t N, int C, int H, int W, int R,
                          int S, int stride, int pad, int Ho, int Wo, cudaStream_t st) {
    return im2col_launch(false, in, out, N, C, H, W, R, S, stride, pad, Ho, Wo, st);
}

cudaError_t launch_im2col_pairs(const float *in, float *out, int64_t N, int C, int H, int W,
                                int R, int S, int stride, int pad, int Ho, int Wo, cudaStream_t st) {
    return im2col_launch(true, in, out, N, C, H, W, R, S, stride, pad, Ho, Wo, st);
}

namespace {
// Launch with programmatic stream serialization (PDL) when SKC_PDL=1.
template <typename... KArgs, typename... Args>
cudaError_t pdl_launch(void (*k)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args... args) {
    static const bool on = [] {
        // off by default: measured no gain on the AlexNet step (profiles/r01_jit_order.txt)
        const char *e = std::getenv("SKC_PDL");
        return e && e[0] == '1';
    }();
    cudaLaunchConfig_t lc{};
    cudaLaunchAttribute at[1];
    lc.gridDim = grid;
    lc.blockDim = block;
    lc.dynamicSmemBytes = 0;
    lc.stream = st;
    if (on) {
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
    }
    return cudaLaunchKernelEx(&lc, k, static_cast<KArgs>(args)...);
}
}  // namespace

cudaError_t launch_pad(const float *in, float *out, int64_t N, int C, int H, int W, int pad,
                       cudaStream_t st) {
    const int Hp = H + 2 * pad, Wp = W + 2 * pad;
    const uint32_t per_img = uint32_t(int64_t(C) * Hp * Wp);
    const int threads = 256;
    int64_t bx = (int64_t(per_img) + threads * 16 - 1) / (threads * 16);
    bx = bx > 4096 ? 4096 : bx;
    for (int64_t n0 = 0; n0 < N; n0 += 65535) {
        const int64_t nn = (N - n0) < 65535 ? (N - n0) : 65535;
        const dim3 grid{static_cast<unsigned>(bx), static_cast<unsigned>(nn), 1u};
        cudaError_t e = pdl_launch(pad_kernel, grid, dim3(threads), st,
                                   in + n0 * int64_t(C) * H * W, out + n0 * int64_t(per_img), C,
                                   H, W, pad, Wp, per_img, make_fastdiv(uint32_t(Hp * Wp)),
                                   make_fastdiv(uint32_t(Wp)), int(per_img % 4 == 0));
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

cudaError_t launch_pad_pairs(const float *in, float *out, int64_t N, int C, int H, int W,
                             int pad, cudaStream_t st) {
    const int Hp = H + 2 * pad, Wp = W + 2 * pad;
    const uint32_t per_img = uint32_t(int64_t(C) * Hp * Wp);
    const int threads = 256;
    const int64_t P = (N + 1) / 2;
    // SKC_PAD_FLAT=1: one whole-wave grid over the batch -- measured SLOWER than the per-pair
    // grid (conv2-5 pads 0.038/0.027/0.037/0.038 vs 0.0325/0.024/0.031/0.032 ms,
    // profiles/r02_pad_flat.txt), kept as an option
    const char *flat_env = std::getenv("SKC_PAD_FLAT");
    const bool flat = flat_env && flat_env[0] == '1';
    if (flat && P * int64_t(per_img) < (int64_t(1) << 31)) {
        static int nsm = 0;
        if (!nsm) {
            int dev = 0, v = 0;
            if (cudaGetDevice(&dev) == cudaSuccess &&
                cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
                nsm = v;
            else
                nsm = 148;
        }
        const uint32_t total = uint32_t(P * int64_t(per_img));
        const int64_t need = (int64_t(total) + threads * 2 * kPadUnroll - 1) / (threads * 2 * kPadUnroll);
        const int64_t grid = need < int64_t(nsm) * 8 ? need : int64_t(nsm) * 8;
        cudaError_t e = pdl_launch(pad_pairs_flat_kernel, dim3(unsigned(grid)), dim3(threads), st, in, out,
                                   C, H, W, pad, Wp, per_img, total, N, make_fastdiv(per_img),
                                   make_fastdiv(uint32_t(Hp * Wp)), make_fastdiv(uint32_t(Wp)));
        if (e != cudaSuccess) return e;
        return cudaGetLastError();
    }
    int64_t bx = (int64_t(per_img) + threads * 8 - 1) / (threads * 8);
    bx = bx > 4096 ? 4096 : bx;
    for (int64_t p0 = 0; p0 < P; p0 += 65535) {
        const int64_t np = (P - p0) < 65535 ? (P - p0) : 65535;
        // the last pair of an odd batch has no second image (has_b = 0 for that launch's
        // last pair: the kernel checks p + 1 < gridDim.y)
        const int has_b = (p0 + np < P) || (N % 2 == 0);
        const dim3 grid{static_cast<unsigned>(bx), static_cast<unsigned>(np), 1u};
        cudaError_t e = pdl_launch(pad_pairs_kernel, grid, dim3(threads), st,
                                   in + 2 * p0 * int64_t(C) * H * W,
                                   out + 2 * p0 * int64_t(per_img), C, H, W, pad, Wp, per_img,
                                   make_fastdiv(uint32_t(Hp * Wp)), make_fastdiv(uint32_t(Wp)),
                                   int(has_b));
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

}  // namespace skc
