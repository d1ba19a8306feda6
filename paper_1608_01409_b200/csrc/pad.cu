// pad.cu -- row a2: NCHW -> zero-padded [N][C][Hp][Wp] (R1).
//
// HBM-bound copy.  Algorithmic bytes per image: read C*H*W*4, write C*Hp*Wp*4.
// One warp per padded row (row = (n*C + c)*Hp + y): one magic-number division per row, lanes
// walk x with coalesced loads and stores; halo rows and columns are plain zero stores.
// Row indices are 64-bit (N*C*Hp may exceed 2^31); in-plane indices are 32-bit.
#include "ptx.cuh"
#include "skc_internal.h"

namespace skc {
namespace {

template <bool WIDE>
__global__ void __launch_bounds__(256) pad_kernel(const float *__restrict__ in,
                                                  float *__restrict__ out, int64_t rows, int H,
                                                  int W, int pad, int Hp, int Wp, FastDiv div_hp) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t r = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows;
         r += warps) {
        // r = plane * Hp + y with plane = n*C + c: 32-bit magic division unless rows >= 2^31
        const int64_t pl = WIDE ? r / Hp : int64_t(fdiv(uint32_t(r), div_hp));
        const int y = int(r - pl * Hp) - pad;
        float *o = out + r * Wp;
        if (y < 0 || y >= H) {
            for (int x = lane; x < Wp; x += 32) o[x] = 0.0f;
        } else {
            const float *src = in + (pl * H + y) * W;
            for (int x = lane; x < Wp; x += 32) {
                const int xi = x - pad;
                o[x] = (xi >= 0 && xi < W) ? __ldg(src + xi) : 0.0f;
            }
        }
    }
}

}  // namespace

cudaError_t launch_pad(const float *in, float *out, int64_t N, int C, int H, int W, int pad,
                       cudaStream_t st) {
    const int Hp = H + 2 * pad, Wp = W + 2 * pad;
    const int64_t rows = N * int64_t(C) * Hp;
    const int threads = 256;
    int64_t blocks = (rows + 7) / 8;
    blocks = blocks > 148 * 32 ? 148 * 32 : blocks;
    const FastDiv dh = make_fastdiv(uint32_t(Hp));
    if (rows < (int64_t(1) << 31))
        pad_kernel<false><<<unsigned(blocks), threads, 0, st>>>(in, out, rows, H, W, pad, Hp, Wp, dh);
    else
        pad_kernel<true><<<unsigned(blocks), threads, 0, st>>>(in, out, rows, H, W, pad, Hp, Wp, dh);
    return cudaGetLastError();
}

}  // namespace skc
