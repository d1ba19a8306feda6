/*
 * oracle_conv.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU
 * evaluation of the convolution that direct sparse convolution computes.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this.  It shares no code, header, table or helper with the CUDA path
 * (paper_1608_01409_b200/), and never calls into it.
 *
 * What it computes -- PAPER.md:237-242 (Sec. 2.1, Eq. 1):
 *
 *     O(n,y,x) = sum_c sum_r sum_s  W(n,c,r,s) * I(c, y+r, x+s)
 *
 * with the build's conventions:
 *   - the paper's output-channel index "n" is called k here; n is the image index;
 *   - stride and zero padding enter only through the input index
 *     yi = y*stride + r - pad, xi = x*stride + s - pad; taps outside [0,H)x[0,W)
 *     read zero (bounds checks -- NOT a padded copy, so this is independent of
 *     skc_pad_input);
 *   - groups: output channel k belongs to group g_k = k / (K/groups) and reads the
 *     input channels g_k*(C/groups) + cl, cl < C/groups  (reading R3);
 *   - Ho = (H + 2*pad - R)/stride + 1 (floor), likewise Wo (reading R7).
 *
 * The weights are DENSE and zero-filled: pruned entries are simply 0 and contribute
 * 0 (BASELINE.json north_star: "a plain CPU seven-loop direct convolution over dense
 * zero-filled weights").  Accumulation is in fp64 (double), rounded never; the caller
 * gets the fp64 sum.  Alongside it, bound(n,k,y,x) = sum |W * I| over the same terms,
 * the scale the parity tolerance is stated in (north_star: "max |err| <= 1e-4 times the
 * sum of |w*x| per output element").
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC (no -ffast-math: fp64 semantics must hold).
 */
#include <stdint.h>
#include <math.h>

/* Returns 0 on success, -1 on invalid geometry (nothing written). */
int oracle_conv2d(const float *in,   /* [N][C][H][W] fp32          */
                  const float *w,    /* [K][C/groups][R][S] fp32    */
                  int64_t N, int C, int H, int W,
                  int K, int R, int S,
                  int stride, int pad, int groups,
                  double *out,       /* [N][K][Ho][Wo] fp64 sums    */
                  double *bound)     /* [N][K][Ho][Wo] sum |w*x|, may be NULL */
{
    if (N < 0 || C < 1 || H < 1 || W < 1 || K < 1 || R < 1 || S < 1 || stride < 1 ||
        pad < 0 || groups < 1 || C % groups != 0 || K % groups != 0)
        return -1;
    const int Ho = (H + 2 * pad - R) / stride + 1;
    const int Wo = (W + 2 * pad - S) / stride + 1;
    if (H + 2 * pad - R < 0 || W + 2 * pad - S < 0 || Ho < 1 || Wo < 1)
        return -1;
    const int Cg = C / groups;   /* input channels per group  */
    const int Kg = K / groups;   /* output channels per group */

    int64_t nk;
#pragma omp parallel for schedule(dynamic, 1)
    for (nk = 0; nk < N * (int64_t)K; ++nk) {
        const int64_t n = nk / K;
        const int k = (int)(nk % K);
        const int g = k / Kg;
        for (int y = 0; y < Ho; ++y) {
            for (int x = 0; x < Wo; ++x) {
                double acc = 0.0, mag = 0.0;
                for (int cl = 0; cl < Cg; ++cl) {
                    const int c = g * Cg + cl;
                    for (int r = 0; r < R; ++r) {
                        for (int s = 0; s < S; ++s) {
                            const int yi = y * stride + r - pad;
                            const int xi = x * stride + s - pad;
                            double v = 0.0;
                            if (yi >= 0 && yi < H && xi >= 0 && xi < W)
                                v = (double)in[((n * C + c) * (int64_t)H + yi) * W + xi];
                            const double wt =
                                (double)w[(((int64_t)k * Cg + cl) * R + r) * S + s];
                            acc += wt * v;
                            mag += fabs(wt * v);
                        }
                    }
                }
                const int64_t o = ((n * K + k) * (int64_t)Ho + y) * Wo + x;
                out[o] = acc;
                if (bound) bound[o] = mag;
            }
        }
    }
    return 0;
}
