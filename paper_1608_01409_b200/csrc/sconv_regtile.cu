// sconv_regtile.cu -- rows a3..a6, register-tiled variant of direct sparse convolution.
//
// Same computation as Fig. 2: out[k][y][x] += w * in[f(c,r,s) + f(0,y,x)]
// for every nonzero w = W(k,c,r,s), accumulated in CSR order.  What changes is where the
// input operand comes from.  The direct kernel reads one shared-memory word per MAC, which
// caps it at 32 MAC/clk/SM against 128 FP32 lanes (the B200 analogue of the paper's
// "1 unaligned load per cycle vs 2 FMA per cycle").  Here each lane keeps
// a (TY+R-1) x (TX+S-1) window of ONE input channel c in registers -- the register blocking
// on the y,x loops of PAPER.md:309-310 -- and applies every nonzero of the warp's M output
// channels at that c to its TY x TX output tile straight from registers:
//
//     acc[m][ty][tx] += w * win[ty + r][tx + s]         (TY*TX FMAs per nonzero)
//
// The tap (r, s) and the channel slot m are warp-uniform (all lanes walk the same nonzero
// stream), so each nonzero is dispatched through a switch on case = (m*R + r)*S + s to a
// block whose register operands are compile-time constants.  Shared-memory words per MAC
// drop from 1 to (window loads + 1 per nonzero) / (nonzeros * TY*TX).
//
// Pipeline: input channels are staged CB at a time (column blocking) for NI
// images by TMA bulk copies, together with the op-stream segment of the chunk, into a ring
// of NS stages.  There is no producer warp: the last warp to release a stage (an atomic
// counter) refills it with chunk i+NS.
#include <atomic>

#include "ptx.cuh"
#include "skc_internal.h"
#include "regtile_gen.inc"

namespace skc {
namespace {

// Issue the TMA copies of chunk `i` into stage `s` (one thread).
__device__ __forceinline__ void fill_stage(const RegtileParams &p, float *stage, uint64_t *bar,
                                           int i, int n0, int gi, int bidx) {
    const int64_t plane = int64_t(p.Hp) * p.Wp;
    const int c0 = i * p.CB;
    const int cn = min(p.CB, p.Cg - c0);
    const uint32_t in_bytes = uint32_t(cn) * uint32_t(plane) * 4u;
    const int nimg = min(p.NI, p.N - n0);
    const int32_t *so = p.segoff + (int64_t(bidx) * p.nchunks + i) * (p.NT + 1);
    const int32_t s0 = so[0];
    const int32_t len = (so[p.NT] - s0 + 1) & ~1;  // regions are padded to 16 B
    const uint32_t st_bytes = uint32_t(len) * 8u;
    mbar_arrive_expect_tx(bar, in_bytes * uint32_t(nimg) + st_bytes);
    for (int j = 0; j < nimg; ++j)
        bulk_g2s(stage + j * p.img_stride,
                 p.in + ((int64_t(n0 + j) * p.C + int64_t(gi) * p.Cg + c0) * plane), in_bytes,
                 bar);
    if (st_bytes) bulk_g2s(stage + p.slab_floats, p.stream + s0, st_bytes, bar);
}

template <int R, int S, int TY, int TX, int M, int NWMAX, int MINB>
__global__ void __launch_bounds__(NWMAX * 32, MINB) sconv_regtile_kernel(const RegtileParams p) {
    constexpr int WR = TY + R - 1, WC = TX + S - 1;
    extern __shared__ __align__(128) float smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + size_t(p.NS) * p.stage_floats);
    int *relcnt = reinterpret_cast<int *>(full + kMaxStages);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int NW = p.NG * p.NT;

    int rest = blockIdx.x;
    const int blk = rest % p.nblocks;
    rest /= p.nblocks;
    const int gi = rest % p.groups;
    const int n0 = (rest / p.groups) * p.NI;
    const int bidx = gi * p.nblocks + blk;

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.NS; ++s) {
            mbar_init(&full[s], 1);
            relcnt[s] = 0;
        }
        mbar_fence_init();
        for (int s = 0; s < p.NS && s < p.nchunks; ++s)
            fill_stage(p, smem + size_t(s) * p.stage_floats, &full[s], s, n0, gi, bidx);
    }
    __syncthreads();

    const int lg = warp % p.NG, t = warp / p.NG;
    // lanemap: (img << 24) | (y0 << 12) | x0; bit 30 marks an idle lane (it mirrors an
    // active lane's tile so its loads broadcast instead of conflicting, and stores nothing)
    const int lm = __ldg(p.lanemap + lg * 32 + lane);
    const bool idle = (lm >> 30) & 1;
    const int img = (lm >> 24) & 0x3f;
    const int y0 = (lm >> 12) & 0xfff;
    const int x0 = lm & 0xfff;
    const int lbase = img * p.img_stride + y0 * p.Wp + x0;

    float acc[M][TY][TX];
#pragma unroll
    for (int m = 0; m < M; ++m)
#pragma unroll
        for (int ty = 0; ty < TY; ++ty)
#pragma unroll
            for (int tx = 0; tx < TX; ++tx) acc[m][ty][tx] = 0.0f;
    float win[WR][WC];
#pragma unroll
    for (int r = 0; r < WR; ++r)
#pragma unroll
        for (int c = 0; c < WC; ++c) win[r][c] = 0.0f;
    const uint32_t wp4 = uint32_t(p.Wp) * 4u;

    for (int i = 0; i < p.nchunks; ++i) {
        const int s = i % p.NS;
        float *stage = smem + size_t(s) * p.stage_floats;
        mbar_wait(&full[s], uint32_t(i / p.NS) & 1u);
        // staged segment table: region-relative entry offset of this warp's task
        const int32_t off = reinterpret_cast<const int32_t *>(stage + p.slab_floats)[t];
        // the warp's segment: HDR / FMA ops ... EXIT, dispatched in registers (regtile_gen.inc)
        rt_dispatch<R, S, TY, TX, M>(acc, win, smem_u32(stage + p.slab_floats) + uint32_t(off) * 8u,
                                     smem_u32(stage + lbase), wp4);
        // release the stage; the last warp out refills it with chunk i + NS
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            const int old = atomicAdd(&relcnt[s], 1);
            if (old == NW - 1) {
                relcnt[s] = 0;
                if (i + p.NS < p.nchunks) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    fill_stage(p, stage, &full[s], i + p.NS, n0, gi, bidx);
                }
            }
        }
    }

    // a6: epilogue (optionally fused bias + ReLU into the next layer's padded layout)
    if (idle || n0 + img >= p.N) return;
    const int opad = p.epi.opad;
    const int Hop = p.Ho + 2 * opad, Wop = p.Wo + 2 * opad;
    const int *ch = p.chan + (int64_t(bidx) * p.NT + t) * M;
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const int k = __ldg(ch + m);
        if (k < 0) continue;
        const float bias = p.epi.bias ? __ldg(p.epi.bias + k) : 0.0f;
#pragma unroll
        for (int ty = 0; ty < TY; ++ty)
#pragma unroll
            for (int tx = 0; tx < TX; ++tx) {
                const int y = y0 + ty, x = x0 + tx;
                float v = acc[m][ty][tx] + bias;
                if (p.epi.relu) v = fmaxf(v, 0.0f);
                if (y < p.Ho && x < p.Wo)
                    p.out[out_index(n0 + img, k, y + opad, x + opad, p.K, Hop, Wop, p.epi.olay)] = v;
            }
    }
}

template <int R, int S, int TY, int TX, int M, int NWMAX, int MINB>
cudaError_t launch_shape(const RegtileParams *pp, size_t smem, cudaStream_t st) {
    // the opt-in shared-memory limit is a per-device function attribute: skc_plan_upload sets
    // it (pp == nullptr: prepare only); a launch on a device no upload prepared sets it too
    static std::atomic<uint64_t> attr_set{0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    auto fn = sconv_regtile_kernel<R, S, TY, TX, M, NWMAX, MINB>;
    if (!(attr_set.load(std::memory_order_acquire) >> dev & 1u)) {
        cudaError_t e =
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        attr_set.fetch_or(uint64_t(1) << dev, std::memory_order_acq_rel);
    }
    if (!pp) return cudaSuccess;
    const RegtileParams &p = *pp;
    const int64_t grid = int64_t((p.N + p.NI - 1) / p.NI) * p.groups * p.nblocks;
    if (grid > 0x7fffffff || p.NG * p.NT > NWMAX) return cudaErrorInvalidConfiguration;
    fn<<<unsigned(grid), p.NG * p.NT * 32, smem, st>>>(p);
    return cudaGetLastError();
}

}  // namespace

int regtile_shapes(RegtileShape *out, int max) {
    int n = 0;
#define X(r, s, ty, tx, m, nw, mb) \
    if (n < max) out[n] = RegtileShape{r, s, ty, tx, m, nw, mb}; \
    ++n;
    SKC_REGTILE_SHAPES(X)
#undef X
    return n;
}

cudaError_t launch_regtile(const RegtileParams &p, const RegtileShape &sh, size_t smem,
                           cudaStream_t st) {
#define X(r, s, ty, tx, m, nw, mb)                                                    \
    if (sh.R == r && sh.S == s && sh.TY == ty && sh.TX == tx && sh.M == m &&          \
        sh.nwmax == nw && sh.minb == mb)                                               \
        return launch_shape<r, s, ty, tx, m, nw, mb>(&p, smem, st);
    SKC_REGTILE_SHAPES(X)
#undef X
    return cudaErrorInvalidValue;
}

cudaError_t prepare_regtile(const RegtileShape &sh) {
#define X(r, s, ty, tx, m, nw, mb)                                                    \
    if (sh.R == r && sh.S == s && sh.TY == ty && sh.TX == tx && sh.M == m &&          \
        sh.nwmax == nw && sh.minb == mb)                                               \
        return launch_shape<r, s, ty, tx, m, nw, mb>(nullptr, 0, nullptr);
    SKC_REGTILE_SHAPES(X)
#undef X
    return cudaErrorInvalidValue;
}

}  // namespace skc
