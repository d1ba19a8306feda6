// sconv_direct.cu -- rows a3..a6: direct sparse convolution, the Fig. 2 statement per lane.
//
// PAPER.md:198-208 (Fig. 2):
//     for each output channel n { for j in row n { off = colidx[j]; coeff = value[j];
//         for y, x: out[n][y][x] += coeff * in[off + f(0,y,x)] } }
// B200 mapping:
//   - CTA = (image n, band of BH output rows, block of NW*M output channels of one group);
//     NW compute warps + 1 producer warp.
//   - a3: the producer warp stages the group's input channels CB at a time (column
//     blocking) into a ring of NS shared-memory stages with TMA bulk copies
//     (cp.async.bulk ... mbarrier::complete_tx); consumers release a stage with an mbarrier
//     arrive.  Padding is already materialised (skc_pad_input) so the loop is branch-free.
//   - a4: a warp owns M output channels (perm order, interleaved across warps so that the
//     nnz-sorted channels balance); for each stage it walks its channels' nonzeros of that
//     channel block, 32 at a time: one coalesced 8-byte load of {w, off} per lane, then the
//     pair is broadcast with __shfl_sync (reused for every pixel).
//   - a5: each lane keeps T output pixels of the band in registers and performs
//     acc[t] = fma(w, stage[off + q_t], acc[t]), q_t = (y*stride)*Wp + x*stride -- exactly
//     in[off + f(0,y,x)] of Fig. 2, in shared memory.  One shared-memory word per MAC.
//     Two lane mappings (chosen per shape by plan.cpp's bank-conflict model):
//       PITCH = false: pixel p = t*32 + lane over the Ho x Wo outputs (no junk lanes, but
//                      32 consecutive outputs can span > 32 words -> 2-way bank conflicts);
//       PITCH = true : (stride 1) lane slot p = t*32 + lane over the band in PADDED-row
//                      coordinates, q_t = p: 32 consecutive words, conflict-free, and the
//                      T loads use immediate offsets t*128 B; x >= Wo slots are junk (never
//                      stored).
//   - a6: coalesced stores of the band rows into out[n][k][y][x] (original channel index).
// Accumulation order per output element: CSR order (c ascending, then r, s), fixed ->
// results are bitwise deterministic.
#include "ptx.cuh"
#include "skc_internal.h"

namespace skc {
namespace {

constexpr int kFull = 0xffffffff;

template <int T, int M, bool PITCH>
__global__ void __launch_bounds__(288, 1) sconv_direct_kernel(const DirectParams p) {
    extern __shared__ __align__(128) float smem[];
    const StageGeom &g = p.g;
    uint64_t *full =
        reinterpret_cast<uint64_t *>(smem + size_t(g.NS) * g.stage_floats + g.tail_floats);
    uint64_t *empty = full + kMaxStages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int NW = p.NW;

    // work item: channel block fastest, then group, band, image
    const int groups = g.K / g.Kg;
    int rest = blockIdx.x;
    const int cb = rest % p.cblocks;
    rest /= p.cblocks;
    const int gi = rest % groups;
    rest /= groups;
    const int band = rest % g.nbands;
    const int n = rest / g.nbands;

    if (threadIdx.x == 0) {
        for (int s = 0; s < g.NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        mbar_fence_init();
    }
    __syncthreads();

    const int row0 = band * g.BH * g.stride;  // first padded input row of the band
    const int BHcur = min(g.BH, g.Ho - band * g.BH);
    const int64_t plane = int64_t(g.Hp) * g.Wp;

    if (warp == NW) {
        // ---------------- producer warp: a3 slab staging ----------------
        const float *src = p.in + (int64_t(n) * g.C + int64_t(gi) * g.Cg) * plane +
                           int64_t(row0) * g.Wp;
        const int rows = min(g.BHin, g.Hp - row0);
        const int chan_floats = g.BHin * g.Wp;
        for (int i = 0; i < g.nchunks; ++i) {
            const int s = i % g.NS;
            if (i >= g.NS) mbar_wait(&empty[s], uint32_t((i / g.NS) - 1) & 1u);
            const int c0 = i * g.CB;
            const int cn = min(g.CB, g.Cg - c0);
            float *dst = smem + size_t(s) * g.stage_floats;
            const float *csrc = src + int64_t(c0) * plane;
            if (g.bulk) {
                if (g.whole) {
                    if (lane == 0) {
                        const uint32_t bytes = uint32_t(cn) * uint32_t(plane) * 4u;
                        mbar_arrive_expect_tx(&full[s], bytes);
                        bulk_g2s(dst, csrc, bytes, &full[s]);
                    }
                } else {
                    const uint32_t per = uint32_t(rows) * uint32_t(g.Wp) * 4u;
                    if (lane == 0) mbar_arrive_expect_tx(&full[s], per * uint32_t(cn));
                    __syncwarp();
                    for (int c = lane; c < cn; c += 32)
                        bulk_g2s(dst + c * chan_floats, csrc + int64_t(c) * plane, per, &full[s]);
                }
            } else {
                const int cnt = rows * g.Wp;
                for (int c = 0; c < cn; ++c)
                    for (int e = lane; e < cnt; e += 32)
                        dst[c * chan_floats + e] = __ldg(csrc + int64_t(c) * plane + e);
                __threadfence_block();
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[s]);
            }
        }
        return;
    }

    // ---------------- compute warps ----------------
    const int npix = BHcur * g.Wo;
    int q[PITCH ? 1 : T];
    if constexpr (!PITCH) {
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const int px = t * 32 + lane;
            const int yl = px / g.Wo, x = px - yl * g.Wo;
            q[t] = (px < npix) ? (yl * g.stride * g.Wp + x * g.stride) : 0;
        }
    }
    float acc[M][T];
#pragma unroll
    for (int m = 0; m < M; ++m)
#pragma unroll
        for (int t = 0; t < T; ++t) acc[m][t] = 0.0f;

    const int cpc = NW * M;
    const int local0 = cb * cpc + warp;           // channel index inside the group
    const int kp0 = gi * g.Kg + local0;           // perm position of slot m = 0
    const int stride_cp = g.nchunks + 1;
    const int2 *nz = reinterpret_cast<const int2 *>(p.nz);

    for (int i = 0; i < g.nchunks; ++i) {
        const int s = i % g.NS;
        mbar_wait(&full[s], uint32_t(i / g.NS) & 1u);
        const float *sm = smem + size_t(s) * g.stage_floats;
#pragma unroll
        for (int m = 0; m < M; ++m) {
            if (local0 + m * NW < g.Kg) {
                const int kp = kp0 + m * NW;
                const int b = __ldg(p.chunkptr + kp * stride_cp + i);
                const int e = __ldg(p.chunkptr + kp * stride_cp + i + 1);
                for (int j0 = b; j0 < e; j0 += 32) {
                    const int cnt = min(32, e - j0);
                    int2 pr = make_int2(0, 0);
                    if (lane < cnt) pr = __ldg(nz + j0 + lane);
#pragma unroll 4
                    for (int j = 0; j < cnt; ++j) {
                        const float w = __int_as_float(__shfl_sync(kFull, pr.x, j));
                        const int off = __shfl_sync(kFull, pr.y, j);
                        if constexpr (PITCH) {
                            const float *base = sm + off + lane;
#pragma unroll
                            for (int t = 0; t < T; ++t)
                                acc[m][t] = fmaf(w, base[t * 32], acc[m][t]);
                        } else {
                            const float *base = sm + off;
#pragma unroll
                            for (int t = 0; t < T; ++t)
                                acc[m][t] = fmaf(w, base[q[t]], acc[m][t]);
                        }
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }

    // a6: epilogue -- store the band rows of each owned channel
#pragma unroll
    for (int m = 0; m < M; ++m) {
        if (local0 + m * NW < g.Kg) {
            const int k = __ldg(p.perm + kp0 + m * NW);
            float *o = p.out + ((int64_t(n) * g.K + k) * g.Ho + int64_t(band) * g.BH) * g.Wo;
#pragma unroll
            for (int t = 0; t < T; ++t) {
                const int px = t * 32 + lane;
                if constexpr (PITCH) {
                    const int yl = px / g.Wp, x = px - yl * g.Wp;
                    if (yl < BHcur && x < g.Wo) o[yl * g.Wo + x] = acc[m][t];
                } else {
                    if (px < npix) o[px] = acc[m][t];
                }
            }
        }
    }
}

template <int T, int M, bool PITCH>
cudaError_t launch_tm(const DirectParams &p, size_t smem, cudaStream_t st) {
    static bool attr_set = false;
    auto fn = sconv_direct_kernel<T, M, PITCH>;
    if (!attr_set) {
        cudaError_t e =
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int groups = p.g.K / p.g.Kg;
    const int64_t grid = int64_t(p.g.N) * p.g.nbands * groups * p.cblocks;
    if (grid > 0x7fffffff) return cudaErrorInvalidConfiguration;
    fn<<<unsigned(grid), (p.NW + 1) * 32, smem, st>>>(p);
    return cudaGetLastError();
}

#define SKC_DIRECT_CASES(X)                                                              \
    X(2, 1) X(2, 2) X(2, 4) X(4, 1) X(4, 2) X(4, 4) X(6, 1) X(6, 2) X(6, 4) X(7, 1) X(7, 2) \
    X(7, 4) X(8, 1) X(8, 2) X(8, 4) X(12, 1) X(12, 2) X(14, 1) X(14, 2) X(16, 1) X(16, 2)

}  // namespace

bool direct_supported(int T, int M) {
#define X(t, m) if (T == t && M == m) return true;
    SKC_DIRECT_CASES(X)
#undef X
    return false;
}

cudaError_t launch_direct(const DirectParams &p, int T, bool pitch, size_t smem,
                          cudaStream_t st) {
    if (p.NW != 8) return cudaErrorInvalidValue;
#define X(t, m)                                                      \
    if (T == t && p.M == m)                                          \
        return pitch ? launch_tm<t, m, true>(p, smem, st) : launch_tm<t, m, false>(p, smem, st);
    SKC_DIRECT_CASES(X)
#undef X
    return cudaErrorInvalidValue;
}

}  // namespace skc
