// pad.cu -- row a2: NCHW -> zero-padded [N][C][Hp][Wp] (R1).
//
// HBM-bound copy.  Algorithmic bytes per image: read C*H*W*4, write C*Hp*Wp*4.
// grid.y = image, grid.x strides over the image's C*Hp*Wp outputs, 4 per thread, with
// float4 stores when the per-image element count allows it.  Index math uses 32-bit
// magic-number division (C*Hp*Wp < 2^31 is checked at pack time).
#include "ptx.cuh"
#include "skc_internal.h"

namespace skc {
namespace {

constexpr int kPadVec = 4;    // outputs per vector (float4 store)
constexpr int kPadUnroll = 4; // vectors per thread per iteration: 16 loads in flight

__global__ void __launch_bounds__(256) pad_kernel(const float *__restrict__ in,
                                                  float *__restrict__ out, int C, int H, int W,
                                                  int pad, int Wp, uint32_t per_img,
                                                  FastDiv div_plane, FastDiv div_wp, int vec4) {
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
        pad_kernel<<<grid, threads, 0, st>>>(in + n0 * int64_t(C) * H * W,
                                             out + n0 * int64_t(per_img), C, H, W, pad, Wp,
                                             per_img, make_fastdiv(uint32_t(Hp * Wp)),
                                             make_fastdiv(uint32_t(Wp)), per_img % 4 == 0);
    }
    return cudaGetLastError();
}

}  // namespace skc
