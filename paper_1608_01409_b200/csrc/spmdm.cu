// spmdm.cu -- row f2: sparse FC layers as SpMDM, Y[M x B] = W[M x K] X[K x B]
// with X, Y batch-minor (the batch is the fast axis, SpMDM's dense operand).  Also any 1x1,
// stride-1, pad-0, single-group convolution: per image, Y[m][p] = sum_k W[m][k] X[k][p] over the
// plane's pixels p (plane = H*W plays the batch).
//
// Why a kernel of its own: with B = 256 columns there are too few pixels per weight for the
// compiled-weights kernel (its code would be ~nnz instructions run by 4 warps), and the conv
// kernels' CTA items assume many pixels per channel.  Here a lane owns LC consecutive columns,
// a warp owns up to RWM rows, and a CTA owns a tile of rows x a block of BC = 32*LC columns:
//   * X is staged in chunks of KC rows (TMA bulk copies by a producer warp into an NS-deep
//     ring of full/empty mbarriers -- no CTA-wide barrier per chunk), so
//     each X element a warp reads comes from shared memory, at a pitch of BC (or B) floats;
//   * the chunk's nonzeros of the tile's rows travel with it: a header of per-row entry
//     offsets, then (x byte offset in the stage, w) pairs, in CSR order per row;
//   * per nonzero a lane does LC/4 LDS.128 of its columns (column groups 4*lane + 128*q, so
//     each warp load is one contiguous 512 B segment) and LC/2 packed FFMA2 with w.
// Every output element is accumulated by one lane in CSR order (ascending k) with fma.rn,
// so results are bitwise those of the direct kernel on the same plan.  Bound: shared-memory
// wavefronts (LC per nonzero per warp for X + 1 for the broadcast entry), i.e. about a quarter
// of the FP32 FMA peak when every X element is used once -- random 90% sparsity has no
// reuse of a staged X element across a warp's rows to exploit.
#include "ptx.cuh"
#include "skc_internal.h"

namespace skc {
namespace {

__device__ __forceinline__ void ffma2(float2 &acc, float w, float2 x) {
    uint64_t a = *reinterpret_cast<uint64_t *>(&acc);
    const uint64_t xx = *reinterpret_cast<const uint64_t *>(&x);
    const uint32_t wb = __float_as_uint(w);
    const uint64_t ww = (uint64_t(wb) << 32) | wb;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(ww), "l"(xx));
    acc = *reinterpret_cast<float2 *>(&a);
}

// a lane's q-th group of 4 columns is 128 columns after its (q-1)-th: each LDS.128 of the
// warp then reads one contiguous 512 B row segment (4 wavefronts, no bank conflict; with the
// lane's 8 columns adjacent, the 32 B lane stride made every LDS.128 a 2-way conflict)
template <int LC>
__device__ __forceinline__ void load_x(float2 (&x)[LC / 2], const uint8_t *p) {
#pragma unroll
    for (int q = 0; q < LC / 4; ++q) {
        const float4 v = *reinterpret_cast<const float4 *>(p + 512 * q);
        x[2 * q] = make_float2(v.x, v.y);
        x[2 * q + 1] = make_float2(v.z, v.w);
    }
}

template <int LC, int RWM>
__global__ void __launch_bounds__(544, 1) spmdm_kernel(const SpmdmParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);  // NS "stage filled" barriers
    uint64_t *empty = full + 8;                           // NS "stage consumed" barriers
    uint8_t *xs0 = smem + 128;
    uint8_t *ms0 = xs0 + size_t(p.NS) * p.xstage;
    const int t = blockIdx.x, cb = blockIdx.y;
    const int64_t n = blockIdx.z;
    // NW consumer warps + 1 producer warp (the last)
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, NW = (blockDim.x >> 5) - 1;
    const int col0 = cb * 32 * LC;
    const int bcols = min(32 * LC, p.plane - col0);
    const bool active = lane * 4 < bcols;  // lane owns columns q*128 + 4*lane + {0..3}
    const float *X = p.X + n * int64_t(p.C) * p.plane;
    const int r0 = p.trow[t], rows = p.trow[t + 1] - r0;
    const int64_t *blk = p.blk + int64_t(t) * p.nch;

    // stage chunk j into slot s: lane 0 announces the bytes, the warp's lanes issue the copies
    auto issue = [&](int j, int s) {
        const int k0 = j * p.KC, kr = min(p.KC, p.C - k0);
        const uint32_t mbytes = uint32_t(blk[j + 1] - blk[j]);
        const uint32_t xrow = uint32_t(bcols) * 4u;
        if (lane == 0) {
            mbar_arrive_expect_tx(&full[s], uint32_t(kr) * xrow + mbytes);
            bulk_g2s(ms0 + size_t(s) * p.mstage, p.meta + blk[j], mbytes, &full[s]);
            if (p.xcontig)  // the chunk's rows are contiguous in global and in the stage
                bulk_g2s(xs0 + size_t(s) * p.xstage, X + int64_t(k0) * p.plane, uint32_t(kr) * xrow,
                         &full[s]);
        }
        __syncwarp();
        if (!p.xcontig)
            for (int r = lane; r < kr; r += 32)
                bulk_g2s(xs0 + size_t(s) * p.xstage + size_t(r) * p.xpitch,
                         X + int64_t(k0 + r) * p.plane + col0, xrow, &full[s]);
    };

    if (tid == 0) {
        for (int s = 0; s < p.NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], uint32_t(NW));
        }
        mbar_fence_init();
    }
    __syncthreads();
    if (wid == NW) {
        // producer: refill a stage once every consumer warp has released it, so a warp that
        // finishes a chunk early runs ahead (up to NS - 1 chunks) instead of waiting at a
        // CTA barrier for the slowest warp of every chunk
        for (int j = 0; j < p.nch; ++j) {
            const int s = j % p.NS;
            if (j >= p.NS) mbar_wait(&empty[s], uint32_t(j / p.NS - 1) & 1u);
            issue(j, s);
        }
        return;
    }

    float2 acc[RWM][LC / 2];
#pragma unroll
    for (int rr = 0; rr < RWM; ++rr)
#pragma unroll
        for (int q = 0; q < LC / 2; ++q) acc[rr][q] = make_float2(0.0f, 0.0f);

    for (int j = 0; j < p.nch; ++j) {
        const int s = j % p.NS;
        mbar_wait(&full[s], uint32_t(j / p.NS) & 1u);
        const uint8_t *xs = xs0 + size_t(s) * p.xstage + lane * 16;
        const uint8_t *ms = ms0 + size_t(s) * p.mstage;
        const uint32_t *off = reinterpret_cast<const uint32_t *>(ms);
        const uint2 *ent = reinterpret_cast<const uint2 *>(ms + p.hbytes);
        if (active) {
#pragma unroll
            for (int rr = 0; rr < RWM; ++rr) {
                const int lr = wid + rr * NW;
                if (lr >= rows) break;
                int i = off[lr];
                const int e = off[lr + 1];
                // two nonzeros per iteration: both entries, both X loads, then the FMAs
                for (; i + 1 < e; i += 2) {
                    const uint2 a = ent[i], b = ent[i + 1];
                    float2 xa[LC / 2], xb[LC / 2];
                    load_x<LC>(xa, xs + a.x);
                    load_x<LC>(xb, xs + b.x);
#pragma unroll
                    for (int q = 0; q < LC / 2; ++q) ffma2(acc[rr][q], __uint_as_float(a.y), xa[q]);
#pragma unroll
                    for (int q = 0; q < LC / 2; ++q) ffma2(acc[rr][q], __uint_as_float(b.y), xb[q]);
                }
                if (i < e) {
                    const uint2 a = ent[i];
                    float2 xa[LC / 2];
                    load_x<LC>(xa, xs + a.x);
#pragma unroll
                    for (int q = 0; q < LC / 2; ++q) ffma2(acc[rr][q], __uint_as_float(a.y), xa[q]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s
    }

    // a6 epilogue: bias, ReLU, store to the original row index in the output layout
    if (!active) return;
    const Epilogue &E = p.epi;
#pragma unroll
    for (int rr = 0; rr < RWM; ++rr) {
        const int lr = wid + rr * NW;
        if (lr >= rows) break;
        const int m = r0 + lr;
        float v[LC];
#pragma unroll
        for (int q = 0; q < LC / 2; ++q) {
            v[2 * q] = acc[rr][q].x;
            v[2 * q + 1] = acc[rr][q].y;
        }
        if (E.bias) {
            const float b = E.bias[m];
#pragma unroll
            for (int q = 0; q < LC; ++q) v[q] += b;
        }
        if (E.relu) {
#pragma unroll
            for (int q = 0; q < LC; ++q) v[q] = fmaxf(v[q], 0.0f);
        }
        const int cend = col0 + bcols;  // a multiple of 4
        if (E.opad == 0 && E.olay == 0) {
            float *y = p.Y + (n * p.K + m) * int64_t(p.plane) + col0 + 4 * lane;
#pragma unroll
            for (int q = 0; q < LC / 4; ++q)
                if (col0 + 128 * q + 4 * lane < cend)
                    *reinterpret_cast<float4 *>(y + 128 * q) =
                        make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else {
            const int Hop = p.H + 2 * E.opad, Wop = p.W + 2 * E.opad;
#pragma unroll
            for (int q = 0; q < LC; ++q) {
                const int c = col0 + 128 * (q / 4) + 4 * lane + (q % 4);
                if (c >= cend) continue;
                const int yy = c / p.W, xx = c - yy * p.W;
                p.Y[out_index(n, m, yy + E.opad, xx + E.opad, p.K, Hop, Wop, E.olay)] = v[q];
            }
        }
    }
}

template <int LC, int RWM>
cudaError_t set_attr(size_t smem) {
    return cudaFuncSetAttribute(spmdm_kernel<LC, RWM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(smem));
}

}  // namespace

#define SKC_SPMDM_CASES(X) X(4, 4) X(4, 8) X(8, 4) X(8, 8)

cudaError_t prepare_spmdm(int LC, int RWM, size_t smem) {
#define SKC_CASE(lc, rw) \
    if (LC == lc && RWM == rw) return set_attr<lc, rw>(smem);
    SKC_SPMDM_CASES(SKC_CASE)
#undef SKC_CASE
    return cudaErrorInvalidValue;
}

cudaError_t launch_spmdm(const SpmdmParams &p, int LC, int RWM, int NW, int N, size_t smem,
                         cudaStream_t st) {
    const dim3 grid{unsigned(p.ntiles), unsigned(p.ncb), unsigned(N)};
#define SKC_CASE(lc, rw)                                                            \
    if (LC == lc && RWM == rw) {                                                    \
        spmdm_kernel<lc, rw><<<grid, unsigned(32 * (NW + 1)), smem, st>>>(p);       \
        return cudaGetLastError();                                                  \
    }
    SKC_SPMDM_CASES(SKC_CASE)
#undef SKC_CASE
    return cudaErrorInvalidValue;
}

}  // namespace skc
