// sconv_direct.cu -- rows a3..a6: direct sparse convolution, the Fig. 2 statement per lane.
//
// PAPER.md:198-208 (Fig. 2):
//     for each output channel n { for j in row n { off = colidx[j]; coeff = value[j];
//         for y, x: out[n][y][x] += coeff * in[off + f(0,y,x)] } }
// B200 mapping:
//   - CTA = (group of NI images, band of BH output rows, block of NW*M output channels of one
//     conv group); NW compute warps + 1 producer warp.
//   - a3: the producer warp stages CB input channels of the band for the NI images, and the
//     block's (w, off) stream for that chunk, into a ring of NS shared-memory stages with TMA
//     bulk copies (cp.async.bulk ... mbarrier::complete_tx) -- column blocking.
//     Consumers release a stage with an mbarrier arrive.  Planes that are not 16-byte
//     multiples fall back to 4-byte cp.async copies that complete on the same barrier.
//     Padding is already materialised (skc_pad_input).
//   - a4: warp w owns channel slots j = m*NW + w (perm order, so nnz-sorted channels
//     interleave across warps); per nonzero ONE broadcast LDS.64 of {w, off} from the staged
//     stream ("reused for every pixel").  Each staged region starts with
//     its segment table (region-relative entry offsets of every slot).
//   - a5: each lane owns T pixel slots; slot (t, lane) sits at shared word slotq[t][lane],
//     chosen on the host so that slotq[t][lane] == lane (mod 32): acc[m][t] += w *
//     stage[off + slotq[t]] touches 32 distinct banks for ANY off -- in[off + f(0,y,x)] of
//     Fig. 2 at one shared-memory wavefront per 32 MACs, without junk columns.
//   - a6: stores to out[n][k][y][x] at the original channel index (slotout tables); with
//     the fused epilogue (f1) out = act(acc + bias[k]) lands in the interior of the next
//     layer's zero-padded layout.
// Accumulation order per output element: CSR order (c ascending, then r, s) -> bitwise
// deterministic results.
#include <atomic>

#include "ptx.cuh"
#include "skc_internal.h"

namespace skc {
namespace {

__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

// Producer: stage chunk i (input band of NI images + the block's stream region) into `dst`.
__device__ __forceinline__ void produce(const DirectParams &p, float *dst, uint64_t *bar, int i,
                                        int n0, int gi, int gb, int row0, int lane) {
    const int64_t plane = int64_t(p.Hp) * p.Wp;
    const int c0 = i * p.CB;
    const int cn = min(p.CB, p.Cg - c0);
    const int nimg = min(p.NI, p.N - n0);
    const int rows = min(p.BHin, p.Hp - row0);
    const int32_t *sp = p.segptr + (int64_t(gb) * p.nchunks + i) * (p.NW * p.M + 1);
    const int32_t s0 = sp[0];
    const int32_t len = (sp[p.NW * p.M] - s0 + 1) & ~1;  // regions are padded to 16 B
    float *sdst = dst + p.slab_floats;
    if (p.bulk) {
        const uint32_t per = uint32_t(rows) * uint32_t(p.Wp) * 4u;
        const uint32_t in_bytes = p.whole ? uint32_t(cn) * uint32_t(plane) * 4u : per * uint32_t(cn);
        if (lane == 0) mbar_arrive_expect_tx(bar, in_bytes * uint32_t(nimg) + uint32_t(len) * 8u);
        __syncwarp();
        for (int j = 0; j < nimg; ++j) {
            const float *src = p.in + (int64_t(n0 + j) * p.C + int64_t(gi) * p.Cg + c0) * plane +
                               int64_t(row0) * p.Wp;
            float *d = dst + j * p.img_stride;
            if (p.whole) {
                if (lane == 0) bulk_g2s(d, src, in_bytes, bar);
            } else {
                for (int c = lane; c < cn; c += 32)
                    bulk_g2s(d + c * p.chan_stride, src + int64_t(c) * plane, per, bar);
            }
        }
        if (lane == 0 && len) bulk_g2s(sdst, p.stream + s0, uint32_t(len) * 8u, bar);
    } else {
        // planes not 16-byte aligned: 4-byte cp.async copies by all 32 lanes, each lane's
        // completion arriving on the stage barrier (initial count 33 = 32 lanes + lane 0's
        // expect_tx for the stream region, which is always 16-byte aligned)
        if (lane == 0) {
            mbar_arrive_expect_tx(bar, uint32_t(len) * 8u);
            if (len) bulk_g2s(sdst, p.stream + s0, uint32_t(len) * 8u, bar);
        }
        const int cnt = rows * p.Wp;
        for (int j = 0; j < nimg; ++j) {
            const float *src = p.in + (int64_t(n0 + j) * p.C + int64_t(gi) * p.Cg + c0) * plane +
                               int64_t(row0) * p.Wp;
            float *d = dst + j * p.img_stride;
            for (int c = 0; c < cn; ++c)
                for (int e = lane; e < cnt; e += 32)
                    cp_async4(d + c * p.chan_stride + e, src + int64_t(c) * plane + e);
        }
        cp_async_mbar_arrive(bar);
    }
}

template <int T, int M>
__global__ void __launch_bounds__(544, 1) sconv_direct_kernel(const DirectParams p) {
    extern __shared__ __align__(128) float smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + size_t(p.NS) * p.stage_floats);
    uint64_t *empty = full + kMaxStages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int NW = p.NW;

    // work item: channel block fastest, then conv group, band, image group
    int rest = blockIdx.x;
    const int cb = rest % p.cblocks;
    rest /= p.cblocks;
    const int gi = rest % p.groups;
    rest /= p.groups;
    const int band = rest % p.nbands;
    const int n0 = (rest / p.nbands) * p.NI;
    const int gb = gi * p.cblocks + cb;
    const int row0 = band * p.BH * p.stride;

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.NS; ++s) {
            mbar_init(&full[s], p.bulk ? 1 : 33);
            mbar_init(&empty[s], NW);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == NW) {
        // ---------------- producer warp: a3 staging ----------------
        for (int i = 0; i < p.nchunks; ++i) {
            const int s = i % p.NS;
            if (i >= p.NS) mbar_wait(&empty[s], uint32_t((i / p.NS) - 1) & 1u);
            produce(p, smem + size_t(s) * p.stage_floats, &full[s], i, n0, gi, gb, row0, lane);
        }
        return;
    }

    // ---------------- compute warps ----------------
    int q[T];
    const int32_t *sq = p.slotq + (int64_t(band) * T) * 32 + lane;
#pragma unroll
    for (int t = 0; t < T; ++t) q[t] = __ldg(sq + t * 32);
    // accumulators as float2 pairs of slots: one packed FFMA2 (fma.rn.f32x2, sm_100) per two
    // slots -- two independent round-to-nearest FMAs, bit-identical to two fmaf()
    constexpr int T2 = (T + 1) / 2;
    float2 acc[M][T2];
#pragma unroll
    for (int m = 0; m < M; ++m)
#pragma unroll
        for (int t = 0; t < T2; ++t) acc[m][t] = make_float2(0.0f, 0.0f);
    const int nslot = NW * M;

    for (int i = 0; i < p.nchunks; ++i) {
        const int s = i % p.NS;
        mbar_wait(&full[s], uint32_t(i / p.NS) & 1u);
        const float *sm = smem + size_t(s) * p.stage_floats;
        const uint2 *st = reinterpret_cast<const uint2 *>(sm + p.slab_floats);
        uint32_t qb[T];  // shared byte address of every slot in this stage
        const uint32_t sbase = smem_u32(sm);
#pragma unroll
        for (int t = 0; t < T; ++t) qb[t] = sbase + uint32_t(q[t]) * 4u;
        const int *seg = reinterpret_cast<const int *>(st);  // staged segment table
#pragma unroll
        for (int m = 0; m < M; ++m) {
            const int j = m * NW + warp;
            const int b = seg[j], e = seg[j + 1];
#pragma unroll 2
            for (int idx = b; idx < e; ++idx) {
                const uint2 pr = st[idx];  // same address in every lane: broadcast
                const float w = __uint_as_float(pr.x);
                const float2 w2 = make_float2(w, w);
                const uint32_t ob = pr.y;  // byte offset of (c, r, s) in the stage
#pragma unroll
                for (int u = 0; u < T2; ++u) {
                    const float a = lds_f32(qb[2 * u] + ob);
                    const float b = (2 * u + 1 < T) ? lds_f32(qb[2 * u + 1] + ob) : 0.0f;
                    acc[m][u] = __ffma2_rn(w2, make_float2(a, b), acc[m][u]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }

    // a6: epilogue (optionally fused bias + ReLU into the next layer's padded layout)
    const int nimg = min(p.NI, p.N - n0);
    const int opad = p.epi.opad;
    const int Hop = p.Ho + 2 * opad, Wop = p.Wo + 2 * opad;
    const int32_t *so = p.slotout + (int64_t(band) * T) * 32 + lane;
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const int k = __ldg(p.chan + int64_t(gb) * nslot + m * NW + warp);
        if (k < 0) continue;
        const float bias = p.epi.bias ? __ldg(p.epi.bias + k) : 0.0f;
        const int yb = band * p.BH + opad;
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const int code = __ldg(so + t * 32);
            float v = (t & 1) ? acc[m][t / 2].y : acc[m][t / 2].x;
            v += bias;
            if (p.epi.relu) v = fmaxf(v, 0.0f);
            const int img = code >> 24;
            if (code >= 0 && img < nimg)
                p.out[out_index(n0 + img, k, yb + ((code >> 12) & 0xfff), opad + (code & 0xfff),
                                p.K, Hop, Wop, p.epi.olay)] = v;
        }
    }
}

template <int T, int M>
cudaError_t launch_tm(const DirectParams *pp, size_t smem, cudaStream_t st) {
    // the opt-in shared-memory limit is a per-device function attribute: skc_plan_upload sets
    // it (pp == nullptr: prepare only); a launch on a device no upload prepared sets it too
    static std::atomic<uint64_t> attr_set{0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    auto fn = sconv_direct_kernel<T, M>;
    if (!(attr_set.load(std::memory_order_acquire) >> dev & 1u)) {
        cudaError_t e =
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        attr_set.fetch_or(uint64_t(1) << dev, std::memory_order_acq_rel);
    }
    if (!pp) return cudaSuccess;
    const DirectParams &p = *pp;
    const int64_t grid =
        int64_t((p.N + p.NI - 1) / p.NI) * p.nbands * p.groups * p.cblocks;
    if (grid > 0x7fffffff || p.NW < 1 || p.NW > 16) return cudaErrorInvalidConfiguration;
    fn<<<unsigned(grid), (p.NW + 1) * 32, smem, st>>>(p);
    return cudaGetLastError();
}

#define SKC_DIRECT_CASES(X) \
    X(1, 1) X(1, 2) X(1, 4) X(2, 1) X(2, 2) X(2, 4) X(3, 1) X(3, 2) X(3, 4) X(4, 1) \
    X(4, 2) X(4, 4) X(5, 1) X(5, 2) X(5, 4) X(6, 1) X(6, 2) X(6, 4) X(7, 1) X(7, 2) \
    X(7, 4) X(8, 1) X(8, 2) X(8, 4) X(9, 1) X(9, 2) X(9, 4) X(10, 1) X(10, 2) X(10, 4) \
    X(11, 1) X(11, 2) X(11, 4) X(12, 1) X(12, 2) X(12, 4) X(13, 1) X(13, 2) X(13, 4) \
    X(14, 1) X(14, 2) X(14, 4) X(15, 1) X(15, 2) X(15, 4) X(16, 1) X(16, 2) X(16, 4)

}  // namespace

bool direct_supported(int T, int M) {
#define X(t, m) if (T == t && M == m) return true;
    SKC_DIRECT_CASES(X)
#undef X
    return false;
}

cudaError_t launch_direct(const DirectParams &p, int T, size_t smem, cudaStream_t st) {
#define X(t, m) if (T == t && p.M == m) return launch_tm<t, m>(&p, smem, st);
    SKC_DIRECT_CASES(X)
#undef X
    return cudaErrorInvalidValue;
}

cudaError_t prepare_direct(int T, int M) {
#define X(t, m) if (T == t && M == m) return launch_tm<t, m>(nullptr, 0, nullptr);
    SKC_DIRECT_CASES(X)
#undef X
    return cudaErrorInvalidValue;
}

}  // namespace skc
