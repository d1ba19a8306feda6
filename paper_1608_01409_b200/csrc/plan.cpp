// plan.cpp -- host side of libskc: the C-ABI (include/skc.h), the CSR/offset packer
// (row a1), plan construction and upload, launch wrappers for the pad (a2) and conv
// (a3..a6) kernels, and the B200 roofline model (a7).
//
// Everything here is host C++17; device memory is never allocated (the caller owns it).
#include "skc.h"
#include "skc_internal.h"

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <new>
#include <numeric>
#include <string>
#include <tuple>
#include <vector>

using namespace skc;

namespace {

thread_local std::string g_err;

skc_status fail(skc_status st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

skc_status ok() {
    g_err.clear();
    return SKC_OK;
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace

// Host-side staging geometry of a plan (the kernels receive DirectParams / RegtileParams).
struct StageGeom {
    int C, K, Kg, Cg, Hp, Wp, Ho, Wo, stride;
    int NI;           // images per CTA
    int BH, BHin, nbands;
    int CB, nchunks, NS;
    int chan_stride, img_stride, stage_floats;
    int bulk, whole;
};

// ---------------------------------------------------------------------------------------
// The plan
// ---------------------------------------------------------------------------------------
struct skc_plan {
    int K, C, R, S, H, W, stride, pad, groups;
    int Ho, Wo, Hp, Wp, Kg, Cg;

    // canonical CSR (the checked contract) and the nnz-sorted order
    std::vector<int32_t> rowptr, colidx, perm;
    std::vector<float> values;

    // kernel choice + configuration
    int kernel = SKC_KERNEL_DIRECT;
    StageGeom sg{};
    int T = 0, NW = 0, M = 0, cblocks = 0;
    DirectParams dp{};
    double direct_waves = 0;  // smem wavefronts per nonzero per image (all bands)
    int max_ni = 4;           // images per CTA the direct kernel may stage (FC: 1)
    int batch_hint = 256;     // images per launch the configuration is chosen for
    size_t smem = 0;

    // register-tiled kernel configuration (kernel == SKC_KERNEL_REGTILE)
    RegtileParams rp{};
    RegtileShape rsh{};

    // device image (bytes uploaded verbatim) and the offsets of its arrays
    std::vector<uint8_t> image;
    size_t off_nz = 0, off_chunkptr = 0, off_perm = 0;
    size_t off_stream = 0, off_segoff = 0, off_chan = 0, off_lanemap = 0;

    // SpMDM kernel (kernel == SKC_KERNEL_SPMDM, spmdm.cu): configuration, the params the
    // launch fills in with workspace pointers, and the image offsets of its tables
    SpmdmParams sp{};
    int sp_LC = 0, sp_RWM = 0, sp_NW = 0;
    size_t off_trow = 0, off_blk = 0, off_meta = 0;

    // "compiled weights" kernel (kernel == SKC_KERNEL_JIT, jit.cpp)
    JitPlan *jit = nullptr;
    // padded-input layout the plan's kernel reads (skc_pad_input writes it):
    // SKC_LAYOUT_NCHW [N][C][Hp][Wp] or SKC_LAYOUT_PAIRS [ceil(N/2)][C][Hp][Wp][2]
    int layout = SKC_LAYOUT_NCHW;

    void *d_ws = nullptr;  // set by skc_plan_upload

    skc_plan() = default;
    skc_plan(const skc_plan &) = delete;
    skc_plan &operator=(const skc_plan &) = delete;
    ~skc_plan() { jit_destroy(jit); }
};

namespace {

constexpr int kDirectNW = 8;              // compute warps per CTA (+1 producer warp)
constexpr size_t kStageTarget = 24 << 10;  // bytes per stage we aim for
constexpr int kDirectSmallBatch = 16;      // batch hints below this: launch-time config model
constexpr int kAutoJitMinBatch = 16;       // AUTO: compiled-weights kernel from this batch up
constexpr size_t kSmemBudget = 112 << 10;  // per CTA, so that >= 2 CTAs fit an SM

skc_status check_geometry(int K, int C, int R, int S, int H, int W, int stride, int pad,
                          int groups) {
    if (K < 1 || C < 1 || R < 1 || S < 1 || H < 1 || W < 1 || stride < 1 || pad < 0 ||
        groups < 1)
        return fail(SKC_ERR_GEOMETRY, "non-positive dimension (K=%d C=%d R=%d S=%d H=%d W=%d "
                    "stride=%d pad=%d groups=%d)", K, C, R, S, H, W, stride, pad, groups);
    if (C % groups || K % groups)
        return fail(SKC_ERR_GEOMETRY, "K=%d and C=%d must be divisible by groups=%d", K, C,
                    groups);
    if (H + 2 * pad < R || W + 2 * pad < S)
        return fail(SKC_ERR_GEOMETRY, "kernel %dx%d larger than padded input %dx%d", R, S,
                    H + 2 * pad, W + 2 * pad);
    const int64_t plane = int64_t(H + 2 * pad) * (W + 2 * pad);
    if (plane * C >= (int64_t(1) << 31))
        return fail(SKC_ERR_OVERFLOW, "C*Hp*Wp = %lld does not fit int32 offsets",
                    (long long)(plane * C));
    return SKC_OK;
}

// Residue-bucketed pixel slots of one band: pixel (img, yl, x) of the band lives at shared
// word q = img*IS + yl*stride*Wp + x*stride (relative to its channel's base in image slot 0);
// lane l gets the pixels with q == l (mod 32), so for any nonzero offset the 32 lanes of a
// warp load from 32 distinct banks.  Returns T = slots per lane (the largest bucket).
int band_slots(int NI, int IS, int rows, int Wo, int Wp, int stride,
               std::vector<std::vector<std::pair<int, int>>> *buckets) {
    std::vector<std::vector<std::pair<int, int>>> bk(32);
    for (int img = 0; img < NI; ++img)
        for (int yl = 0; yl < rows; ++yl)
            for (int x = 0; x < Wo; ++x) {
                const int q = img * IS + yl * stride * Wp + x * stride;
                bk[size_t(q & 31)].emplace_back(q, (img << 24) | (yl << 12) | x);
            }
    size_t T = 0;
    for (auto &b : bk) T = std::max(T, b.size());
    if (buckets) *buckets = std::move(bk);
    return int(T);
}

// TMA bulk-copy legality of a direct-kernel staging layout: 16-byte aligned sources,
// destinations and sizes for every (image, chunk, band) copy.
bool bulk_legal(const skc_plan *p, int NI, int BH, int BHin, int nbands, bool whole, int CB,
                int chan_stride, int IS) {
    (void)NI;
    const int64_t plane = int64_t(p->Hp) * p->Wp;
    bool bulk = (int64_t(p->C) * plane) % 4 == 0 && (int64_t(p->Cg) * plane) % 4 == 0 &&
                IS % 4 == 0;
    if (whole) {
        bulk = bulk && (int64_t(CB) * plane) % 4 == 0 &&
               (int64_t(p->Cg % CB ? p->Cg % CB : CB) * plane) % 4 == 0;
    } else {
        bulk = bulk && plane % 4 == 0 && (int64_t(BH) * p->stride * p->Wp) % 4 == 0 &&
               chan_stride % 4 == 0;
        for (int b = 0; b < nbands && bulk; ++b) {
            const int row0 = b * BH * p->stride;
            bulk = (int64_t(std::min(BHin, p->Hp - row0)) * p->Wp) % 4 == 0;
        }
    }
    return bulk;
}

// Pick the direct kernel's images per CTA (NI), band height, image-slot stride, pixel slots
// per lane (T), channel chunk and warp layout.  Cost per nonzero per image, in shared-memory
// wavefronts: bands * (T loads + 1 broadcast) / NI; the cheapest candidate wins.
skc_status configure_direct(skc_plan *p) {
    const int Ho = p->Ho, Wo = p->Wo;
    StageGeom &g = p->sg;
    g = StageGeom{};
    g.C = p->C; g.K = p->K; g.Kg = p->Kg; g.Cg = p->Cg; g.Hp = p->Hp; g.Wp = p->Wp;
    g.Ho = Ho; g.Wo = Wo; g.stride = p->stride;
    if (Wo >= 4096 || Ho >= 4096)
        return fail(SKC_ERR_UNSUPPORTED, "output %dx%d too large for the direct kernel", Ho, Wo);
    const int64_t plane = int64_t(p->Hp) * p->Wp;
    double best_cost = 1e300;
    const char *nb_env = std::getenv("SKC_DIRECT_BANDS");
    const int nb_force = nb_env ? std::atoi(nb_env) : 0;
    // Small batches (batch_hint < kDirectSmallBatch): the per-image cost below ignores how
    // many CTAs a launch has, and a batch-1 launch of a 256-image configuration runs a few
    // dozen CTAs on 148 SMs.  There the candidates (band height, images per CTA, channels per
    // warp M) are ranked by a launch-time model instead: CTAs = groups x channel blocks x
    // bands x image groups in waves of 148 x (CTAs per SM by shared memory, at most 2); a
    // CTA is latency-bound -- each warp walks its channels' nonzeros one after another at
    // ~110 cycles each whatever the pixel slots T (B200, conv3 at batch 1-2:
    // profiles/r02_small_batch.txt) -- plus its staged input and {w, off} stream at ~64 B/clk
    // from L2, ~2000 cycles of setup, and a small charge per row band (more bands measured
    // slower at equal waves).
    const bool small = p->batch_hint < kDirectSmallBatch;
    int best_M = 0;
    for (int NI = 1; NI <= p->max_ni; NI *= 2) {
        if (small && NI > 1 && NI / 2 >= p->batch_hint) break;  // no empty image slots
        for (int nb = 1; nb <= Ho; ++nb) {
            if (nb_force > 0 && nb != std::min(nb_force, Ho)) continue;
            const int BH = (Ho + nb - 1) / nb;
            if ((Ho + BH - 1) / BH != nb) continue;  // same BH as a smaller nb
            const int BHin = std::min((BH - 1) * p->stride + p->R, p->Hp);
            const bool whole = nb == 1 && BHin == p->Hp;
            const int chan_stride = whole ? int(plane) : BHin * p->Wp;
            const size_t chan_bytes = size_t(NI) * chan_stride * 4;
            if (chan_bytes > (96u << 10)) continue;
            int CB = int(std::max<size_t>(1, kStageTarget / chan_bytes));
            CB = std::min(CB, p->Cg);
            if (CB >= 4) CB -= CB % 4;
            const int base_is = int(align_up(size_t(CB) * chan_stride, 4));
            for (int pad = 0; pad < (NI > 1 ? 32 : 4); pad += 4) {
                const int IS = base_is + pad;
                int T = 0;
                for (int b = 0; b < nb; ++b)
                    T = std::max(T, band_slots(NI, IS, std::min(BH, Ho - b * BH), Wo, p->Wp,
                                               p->stride, nullptr));
                if (T > 16) continue;
                const bool bulk_ok = bulk_legal(p, NI, BH, BHin, nb, whole, CB, chan_stride, IS);
                const int M0 = T <= 8 ? 4 : 2;
                if (small) {
                    // co-resident CTAs of these latency-bound launches slow each other about
                    // as much as a second wave would: count waves of 148
                    const double P = 148.0;
                    const double nig = std::ceil(double(p->batch_hint) / NI);
                    for (int M = M0; M >= 1; M /= 2) {
                        const double blocks = std::ceil(double(p->Kg) / (kDirectNW * M)) * p->groups;
                        const double ctas = blocks * nb * nig;
                        const double nz_cta = double(p->colidx.size()) / blocks;
                        const double staged = double(BHin) * p->Wp * p->Cg * NI * 4.0;
                        const double copy = (bulk_ok ? staged / 64.0 : staged / 4.0 / 32.0 * 8.0) +
                                            nz_cta * 8.0 / 64.0;
                        const double walk = nz_cta / kDirectNW * 110.0;
                        const double cost = std::ceil(ctas / P) * (walk + copy + 2000.0) + 500.0 * nb;
                        if (cost < best_cost) {
                            best_cost = cost; best_M = M;
                            g.NI = NI; g.BH = BH; g.nbands = nb; g.BHin = BHin; g.whole = whole;
                            g.CB = CB; g.chan_stride = chan_stride; g.img_stride = IS; p->T = T;
                        }
                    }
                    continue;
                }
                // per nonzero and image: T loads + 1 broadcast per band (wavefront-cycles)
                double cost = double(nb) * (T + 1) / NI + 1e-3 * NI + 1e-4 * nb;
                if (!bulk_ok) {
                    // cp.async fallback: ~8 cycles per 32 staged words, repeated by every
                    // channel block; expressed per nonzero of the layer
                    const int M = M0;
                    const double blocks = std::ceil(double(p->Kg) / (kDirectNW * M)) * p->groups;
                    const double words = double(nb) * BHin * p->Wp * p->C * blocks;
                    cost += words / 32.0 * 8.0 / std::max<double>(1.0, double(p->colidx.size()));
                }
                if (cost < best_cost) {
                    best_cost = cost;
                    g.NI = NI; g.BH = BH; g.nbands = nb; g.BHin = BHin; g.whole = whole;
                    g.CB = CB; g.chan_stride = chan_stride; g.img_stride = IS; p->T = T;
                }
            }
        }
    }
    if (best_cost >= 1e300)
        return fail(SKC_ERR_UNSUPPORTED, "no band/slot tiling fits the direct kernel (Wo=%d)", Wo);
    p->direct_waves = double(g.nbands) * (p->T + 1) / g.NI;
    g.nchunks = (p->Cg + g.CB - 1) / g.CB;
    const bool bulk = bulk_legal(p, g.NI, g.BH, g.BHin, g.nbands, g.whole, g.CB, g.chan_stride,
                                 g.img_stride);
    g.bulk = bulk ? 1 : 0;
    p->NW = kDirectNW;
    p->M = p->T <= 8 ? 4 : (p->T <= 16 ? 2 : 1);
    if (small && best_M > 0) p->M = std::min(p->M, best_M);
    // tuning overrides (benchmarks): SKC_DIRECT_NW (compute warps, 1..16), SKC_DIRECT_M
    if (const char *e = std::getenv("SKC_DIRECT_NW")) p->NW = std::max(1, std::min(16, std::atoi(e)));
    if (const char *e = std::getenv("SKC_DIRECT_M")) p->M = std::max(1, std::min(4, std::atoi(e)));
    while (p->M > 1 && p->NW * p->M > p->Kg * 2) p->M /= 2;
    if (!direct_supported(p->T, p->M))
        return fail(SKC_ERR_UNSUPPORTED, "no direct kernel instance for T=%d M=%d", p->T, p->M);
    p->cblocks = (p->Kg + p->NW * p->M - 1) / (p->NW * p->M);
    return SKC_OK;
}

// Build the device image of the direct kernel: per (channel block, chunk) stream regions of
// {w, off} (off relative to the channel's base in image slot 0 of the stage), segment
// pointers, the channel table and the per-band pixel-slot tables.
skc_status build_direct_image(skc_plan *p) {
    StageGeom &g = p->sg;
    const int64_t plane = int64_t(p->Hp) * p->Wp;
    const int nslot = p->NW * p->M;
    const int gblocks = p->groups * p->cblocks;
    std::vector<uint32_t> stream;  // pairs
    std::vector<int32_t> segptr(size_t(gblocks) * g.nchunks * (nslot + 1));
    std::vector<int32_t> chan(size_t(gblocks) * nslot, -1);
    // per channel: its nonzeros bucketed by chunk, as {w bits, off}
    int64_t max_region = 0;
    for (int gi = 0; gi < p->groups; ++gi) {
        for (int cb = 0; cb < p->cblocks; ++cb) {
            const int gb = gi * p->cblocks + cb;
            std::vector<std::vector<std::vector<std::pair<uint32_t, uint32_t>>>> per(
                static_cast<size_t>(nslot),
                std::vector<std::vector<std::pair<uint32_t, uint32_t>>>(
                    static_cast<size_t>(g.nchunks)));
            for (int j = 0; j < nslot; ++j) {
                // slot j = m*NW + w is computed by warp w; sorted channels are dealt to the
                // warps in snake order (m odd reverses w) so per-warp nnz sums balance
                const int m = j / p->NW, wi = j % p->NW;
                const int lc = cb * nslot + m * p->NW + ((m & 1) ? p->NW - 1 - wi : wi);
                if (lc >= p->Kg) continue;
                const int k = p->perm[size_t(gi) * p->Kg + lc];
                chan[size_t(gb) * nslot + j] = k;
                for (int32_t e = p->rowptr[k]; e < p->rowptr[k + 1]; ++e) {
                    const int64_t col = p->colidx[e];
                    const int cl = int(col / plane) - gi * p->Cg;
                    const int64_t rem = col % plane;
                    const int r = int(rem / p->Wp), s = int(rem % p->Wp);
                    uint32_t wb;
                    std::memcpy(&wb, &p->values[e], 4);
                    const int off = (cl % g.CB) * g.chan_stride + r * p->Wp + s;
                    per[size_t(j)][size_t(cl / g.CB)].emplace_back(wb, uint32_t(off) * 4u);
                }
            }
            for (int i = 0; i < g.nchunks; ++i) {
                if (stream.size() % 4) stream.resize(align_up(stream.size(), 4), 0);  // 16 B
                // region = [segment table: nslot+1 int32 offsets (entries, region-relative),
                //            padded to whole uint2] [ {w, off} entries of slot 0, 1, ... ]
                int32_t *sp = &segptr[(size_t(gb) * g.nchunks + i) * (nslot + 1)];
                const size_t r0 = stream.size() / 2;
                const size_t hdr = size_t(nslot + 2) / 2;
                stream.resize(stream.size() + 2 * hdr, 0);
                for (int j = 0; j <= nslot; ++j) {
                    const size_t at = stream.size() / 2;
                    stream[2 * r0 + size_t(j)] = uint32_t(at - r0);
                    sp[j] = int32_t(at);
                    if (j == nslot) break;
                    for (auto &e : per[size_t(j)][size_t(i)]) {
                        stream.push_back(e.first);
                        stream.push_back(e.second);
                    }
                }
                sp[0] = int32_t(r0);  // region start (the producer copies from here)
                max_region = std::max(max_region, int64_t(stream.size() / 2 - r0));
            }
        }
    }
    if (stream.size() / 2 >= (size_t(1) << 31))
        return fail(SKC_ERR_OVERFLOW, "direct stream too large");
    // pixel-slot tables per band
    const int T = p->T;
    std::vector<int32_t> slotq(size_t(g.nbands) * T * 32), slotout(slotq.size());
    for (int b = 0; b < g.nbands; ++b) {
        std::vector<std::vector<std::pair<int, int>>> bk;
        band_slots(g.NI, g.img_stride, std::min(g.BH, p->Ho - b * g.BH), p->Wo, p->Wp,
                   p->stride, &bk);
        for (int t = 0; t < T; ++t)
            for (int l = 0; l < 32; ++l) {
                const size_t o = (size_t(b) * T + t) * 32 + l;
                if (size_t(t) < bk[size_t(l)].size()) {
                    const int q = bk[size_t(l)][size_t(t)].first;
                    const int code = bk[size_t(l)][size_t(t)].second;
                    slotq[o] = q;
                    slotout[o] = code;  // (img << 24) | (yl << 12) | x
                } else {
                    slotq[o] = l;  // empty slot: a conflict-free dummy read, never stored
                    slotout[o] = -1;
                }
            }
    }
    g.NS = 1;
    const int stream_cap = int(align_up(size_t(max_region) + 2, 2));
    const int slab = g.NI * g.img_stride;
    g.stage_floats = slab + 2 * stream_cap + 32;  // +32: empty slots read off + lane
    const size_t stage_bytes = size_t(g.stage_floats) * 4;
    g.NS = int(std::min<size_t>(4, std::max<size_t>(1, kSmemBudget / stage_bytes)));
    g.NS = std::min(g.NS, std::max(1, g.nchunks));
    if (size_t(g.NS) * stage_bytes + 2 * kMaxStages * 8 > (227u << 10))
        return fail(SKC_ERR_UNSUPPORTED, "direct stage of %zu B does not fit", stage_bytes);
    p->smem = size_t(g.NS) * stage_bytes + 2 * kMaxStages * sizeof(uint64_t);
    p->dp = DirectParams{};
    DirectParams &d = p->dp;
    d.C = p->C; d.K = p->K; d.Kg = p->Kg; d.Cg = p->Cg; d.Hp = p->Hp; d.Wp = p->Wp;
    d.Ho = p->Ho; d.Wo = p->Wo; d.stride = p->stride; d.groups = p->groups;
    d.NI = g.NI; d.BH = g.BH; d.BHin = g.BHin; d.nbands = g.nbands; d.CB = g.CB;
    d.nchunks = g.nchunks; d.NS = g.NS; d.chan_stride = g.chan_stride;
    d.img_stride = g.img_stride; d.slab_floats = slab; d.stream_cap = stream_cap;
    d.stage_floats = g.stage_floats; d.bulk = g.bulk; d.whole = g.whole;
    d.NW = p->NW; d.M = p->M; d.cblocks = p->cblocks;
    // device image: stream | segptr | chan | slotq | slotout | perm
    p->off_stream = 0;
    p->off_segoff = align_up(stream.size() * 4, 256);
    p->off_chan = align_up(p->off_segoff + segptr.size() * 4, 256);
    p->off_lanemap = align_up(p->off_chan + chan.size() * 4, 256);      // slotq
    p->off_chunkptr = align_up(p->off_lanemap + slotq.size() * 4, 256);  // slotout
    p->off_perm = align_up(p->off_chunkptr + slotout.size() * 4, 256);
    const size_t total = align_up(p->off_perm + size_t(p->K) * 4, 256);
    p->image.assign(total, 0);
    if (!stream.empty())
        std::memcpy(p->image.data() + p->off_stream, stream.data(), stream.size() * 4);
    std::memcpy(p->image.data() + p->off_segoff, segptr.data(), segptr.size() * 4);
    std::memcpy(p->image.data() + p->off_chan, chan.data(), chan.size() * 4);
    std::memcpy(p->image.data() + p->off_lanemap, slotq.data(), slotq.size() * 4);
    std::memcpy(p->image.data() + p->off_chunkptr, slotout.data(), slotout.size() * 4);
    std::memcpy(p->image.data() + p->off_perm, p->perm.data(), size_t(p->K) * 4);
    return SKC_OK;
}

// ---------------------------------------------------------------------------------------
// Register-tiled kernel: configuration and op streams (see sconv_regtile.cu)
// ---------------------------------------------------------------------------------------
// register cap of a shape's instance (its __launch_bounds__)
int rt_regs(const RegtileShape &sh) { return std::min(255, 65536 / (32 * sh.nwmax * sh.minb)) & ~7; }

constexpr size_t kRtStageTarget = 24 << 10;
constexpr int kRtStages = 3;

// Shared-memory conflict degree of one warp-wide load whose lane addresses are `addr`
// (words; -1 = inactive lane reading word 0): max number of distinct words in one bank.
int conflict_degree(const std::vector<int> &addr) {
    int worst = 1;
    for (int b = 0; b < 32; ++b) {
        std::vector<int> d;
        for (int a : addr) {
            const int w = a < 0 ? 0 : a;
            if ((w & 31) == b && std::find(d.begin(), d.end(), w) == d.end()) d.push_back(w);
        }
        worst = std::max(worst, int(d.size()));
    }
    return worst;
}

struct RtCandidate {
    RegtileShape sh{};
    int NI = 0, NG = 0, NT = 0, nblocks = 0, CB = 0, NS = 0, img_stride = 0, wf = 1;
    int ctas_per_sm = 1;
    std::vector<int32_t> lanemap;
    double cost = 1e300;
};

// c-groups (HDR entries) of a task = distinct input channels among its M channels.
int64_t task_groups(const skc_plan *p, int g, int task, int M) {
    std::vector<char> seen(size_t(p->Cg), 0);
    const int64_t plane = int64_t(p->Hp) * p->Wp;
    int64_t n = 0;
    for (int m = 0; m < M; ++m) {
        const int lp = task * M + m;
        if (lp >= p->Kg) break;
        const int k = p->perm[size_t(g) * p->Kg + lp];
        for (int32_t j = p->rowptr[k]; j < p->rowptr[k + 1]; ++j) {
            const int cl = int(p->colidx[j] / plane) - g * p->Cg;
            if (!seen[size_t(cl)]) { seen[size_t(cl)] = 1; ++n; }
        }
    }
    return n;
}

bool regtile_candidate(const skc_plan *p, const RegtileShape &sh, RtCandidate &c) {
    if (p->stride != 1 || sh.R != p->R || sh.S != p->S) return false;
    const int64_t plane = int64_t(p->Hp) * p->Wp;
    if ((int64_t(p->C) * plane) % 4 || (int64_t(p->Cg) * plane) % 4) return false;
    const int nty = (p->Ho + sh.TY - 1) / sh.TY, ntx = (p->Wo + sh.TX - 1) / sh.TX;
    const int tiles = nty * ntx;
    if (ntx > 4096 || nty * sh.TY > 4095) return false;
    c.sh = sh;
    c.NI = tiles >= 32 ? 1 : std::max(1, 32 / tiles);
    const int total = c.NI * tiles;
    c.NG = (total + 31) / 32;
    if (c.NG > sh.nwmax) return false;
    // tasks per CTA: keep the most warps resident per SM, fill the last block, and prefer
    // more tasks per CTA (each CTA re-reads its images' slabs: fewer blocks, less traffic)
    const int tasks = (p->Kg + sh.M - 1) / sh.M;
    double best = -1;
    const char *nt_env = std::getenv("SKC_RT_NT");
    const int nt_force = nt_env ? std::atoi(nt_env) : 0;
    for (int NT = std::min(sh.nwmax / c.NG, tasks); NT >= 1; --NT) {
        if (nt_force > 0 && NT != std::min(nt_force, std::min(sh.nwmax / c.NG, tasks))) continue;
        const int nb = (tasks + NT - 1) / NT;
        const int warps = c.NG * NT;
        const int by_regs = 65536 / (warps * 32 * rt_regs(sh));
        if (by_regs < 1) continue;
        const int resident = std::min(64, warps * std::min(by_regs, 3));
        const double fill = double(tasks) / double(nb * NT);
        const double score = fill * double(resident) * (1.0 + 0.05 * NT);
        if (score > best) { best = score; c.NT = NT; c.nblocks = nb; c.ctas_per_sm = by_regs; }
    }
    if (!c.NT) return false;
    // channels per stage: input slab of NI images + the op stream of the NT tasks (8 B per
    // nonzero).  Stages as large as the shared-memory budget of the ctas_per_sm CTAs that
    // the register cap allows (fewer chunk hand-offs; measured +4..13%), capped at 48 KB;
    // CB*plane must keep image slots 16-byte aligned
    const double density = double(p->colidx.size()) / (double(p->K) * p->Cg * p->R * p->S);
    const double chan_bytes = double(c.NI) * double(plane) * 4.0 +
                              8.0 * (c.NT * (sh.M * sh.R * sh.S * density + 1.0));
    const double budget = (227.0 * 1024) / std::max(1, std::min(c.ctas_per_sm, 3)) - 2048.0;
    double stage_target = std::min(48.0 * 1024, budget / kRtStages);
    if (const char *e = std::getenv("SKC_RT_STAGE_KB")) stage_target = std::atof(e) * 1024.0;
    int CB = int(std::max(1.0, stage_target / chan_bytes));
    CB = std::min(CB, p->Cg);
    while (CB > 1 && (int64_t(CB) * plane) % 4) --CB;
    if ((int64_t(CB) * plane) % 4) {
        CB = 4;  // plane odd: 4 channels always align
        if (CB > p->Cg) return false;
    }
    if (p->Cg % CB && ((int64_t(p->Cg % CB) * plane) % 4)) return false;  // last chunk copy
    c.CB = CB;
    // Lane map.  Every window load of a warp reads word (tile base + const), so its bank
    // conflicts are those of the tile bases mod 32.  Tiles are dealt to lane groups greedily
    // by bank (a tile goes to the group where its bank is least used), for each candidate
    // image-slot padding; the layout with the fewest conflicts wins.
    const int base = int(align_up(size_t(CB) * size_t(plane), 4));
    int best_wf = 1 << 30;
    for (int pad = 0; pad < (c.NI > 1 ? 32 : 4); pad += 4) {
        const int IS = base + pad;
        std::vector<int32_t> lm(size_t(c.NG) * 32, -1);
        std::vector<std::vector<int>> used(size_t(c.NG), std::vector<int>(32, 0));
        std::vector<int> fill(size_t(c.NG), 0);
        // visit tiles bank by bank, fullest bank first, so each bank's tiles spread across
        // the groups (achieves max_b ceil(count_b / NG) whenever the capacities allow)
        std::vector<int> order(static_cast<size_t>(total)), bank_of(static_cast<size_t>(total));
        std::vector<int> cnt(32, 0);
        for (int i = 0; i < total; ++i) {
            const int img = i / tiles, rem = i % tiles;
            bank_of[size_t(i)] = (img * IS + (rem / ntx) * sh.TY * p->Wp + (rem % ntx) * sh.TX) & 31;
            cnt[size_t(bank_of[size_t(i)])]++;
            order[size_t(i)] = i;
        }
        std::stable_sort(order.begin(), order.end(), [&](int a, int b2) {
            const int ba = bank_of[size_t(a)], bb = bank_of[size_t(b2)];
            return cnt[size_t(ba)] != cnt[size_t(bb)] ? cnt[size_t(ba)] > cnt[size_t(bb)] : ba < bb;
        });
        for (int i : order) {
            const int img = i / tiles, rem = i % tiles;
            const int y0 = (rem / ntx) * sh.TY, x0 = (rem % ntx) * sh.TX;
            const int bank = bank_of[size_t(i)];
            int gbest = -1;
            for (int g = 0; g < c.NG; ++g) {
                if (fill[size_t(g)] >= 32) continue;
                if (gbest < 0 || used[size_t(g)][size_t(bank)] < used[size_t(gbest)][size_t(bank)] ||
                    (used[size_t(g)][size_t(bank)] == used[size_t(gbest)][size_t(bank)] &&
                     fill[size_t(g)] < fill[size_t(gbest)]))
                    gbest = g;
            }
            used[size_t(gbest)][size_t(bank)]++;
            lm[size_t(gbest) * 32 + size_t(fill[size_t(gbest)]++)] = (img << 24) | (y0 << 12) | x0;
        }
        // idle lanes duplicate lane 0's tile (same word: a broadcast, never a conflict) and
        // carry the idle flag (bit 30) so the epilogue skips them
        for (int g = 0; g < c.NG; ++g)
            for (int l = fill[size_t(g)]; l < 32; ++l)
                lm[size_t(g) * 32 + size_t(l)] = (1 << 30) | lm[size_t(g) * 32];
        int wf = 0;
        for (int g = 0; g < c.NG; ++g) {
            std::vector<int> addr(32);
            for (int l = 0; l < 32; ++l) {
                const int v = lm[size_t(g) * 32 + l] & ~(1 << 30);
                addr[size_t(l)] = ((v >> 24) & 0x3f) * IS + ((v >> 12) & 0xfff) * p->Wp + (v & 0xfff);
            }
            wf = std::max(wf, conflict_degree(addr));
        }
        if (wf < best_wf) { best_wf = wf; c.img_stride = IS; c.lanemap = lm; }
    }
    c.wf = best_wf;
    // Cost model, SM-cycles per image summed over SMs (fitted to B200 measurements, see
    // DESIGN.md "Kernel selection"): every dispatched op costs a(occ) -- the brx.idx dispatch
    // is latency-bound, so its cost falls with the warps resident per SM -- and every HDR
    // costs its window's shared-memory wavefronts.
    const int WR = sh.TY + sh.R - 1, WC = sh.TX + sh.S - 1;
    double hdr = 0;
    for (int g = 0; g < p->groups; ++g)
        for (int t = 0; t < tasks; ++t) hdr += double(task_groups(p, g, t, sh.M));
    const double ops = double(p->colidx.size());
    const double per_img = double(c.NG) / double(c.NI);
    const double stage_est = double(c.NI) * c.img_stride * 4.0 +
                             8.0 * c.NT * (c.CB * (sh.M * sh.R * sh.S * density + 1.0) + 2.0);
    const int warps = c.NG * c.NT;
    const int by_smem = std::max(1, int((228.0 * 1024) / (kRtStages * stage_est + 1024)));
    const int ctas = std::min({c.ctas_per_sm, by_smem, 2048 / (warps * 32), 32});
    const double occ = std::min(64, warps * ctas);
    const double a = 10.7 * (16.0 / occ) * (16.0 / occ);
    c.cost = (ops * a + hdr * WR * WC * std::max(1.0, 0.5 * c.wf)) * per_img;
    return true;
}

skc_status build_regtile(skc_plan *p, const RtCandidate &c) {
    const RegtileShape &sh = c.sh;
    const int M = sh.M;
    const int64_t plane = int64_t(p->Hp) * p->Wp;
    const int nchunks = (p->Cg + c.CB - 1) / c.CB;
    const int tasks = (p->Kg + M - 1) / M;
    const int nb = c.nblocks, NT = c.NT;
    const int ncase = M * sh.R * sh.S;
    std::vector<uint32_t> stream;  // pairs (x, case)
    std::vector<int32_t> segoff(size_t(p->groups) * nb * nchunks * (NT + 1));
    std::vector<int32_t> chan(size_t(p->groups) * nb * NT * M, -1);
    int64_t max_region = 0;
    // per (group, task): nonzeros of its M channels bucketed by chunk, each bucket sorted by
    // (c, m, r, s) -- accumulation per output element stays in CSR order (c, r, s)
    struct Op { int cl, m, rs; float w; };
    for (int g = 0; g < p->groups; ++g) {
        for (int b = 0; b < nb; ++b) {
            std::vector<std::vector<std::vector<Op>>> per(
                static_cast<size_t>(NT),
                std::vector<std::vector<Op>>(static_cast<size_t>(nchunks)));
            for (int t = 0; t < NT; ++t) {
                const int task = b * NT + t;
                if (task >= tasks) continue;
                for (int m = 0; m < M; ++m) {
                    const int lp = task * M + m;
                    if (lp >= p->Kg) break;
                    const int k = p->perm[size_t(g) * p->Kg + lp];
                    chan[((size_t(g) * nb + b) * NT + t) * M + m] = k;
                    for (int32_t j = p->rowptr[k]; j < p->rowptr[k + 1]; ++j) {
                        const int64_t col = p->colidx[j];
                        const int cl = int(col / plane) - g * p->Cg;
                        const int64_t rem = col % plane;
                        const int r = int(rem / p->Wp), s = int(rem % p->Wp);
                        per[size_t(t)][size_t(cl / c.CB)].push_back(
                            Op{cl, m, r * sh.S + s, p->values[j]});
                    }
                }
            }
            for (int i = 0; i < nchunks; ++i) {
                if (stream.size() % 4) stream.resize(align_up(stream.size(), 4), 0);  // 16 B
                int32_t *so = &segoff[((size_t(g) * nb + b) * nchunks + i) * (NT + 1)];
                // region = [segment table: NT+1 int32 region-relative entry offsets, padded
                //            to whole uint2] [segment of task 0] [task 1] ...
                const int64_t region0 = int64_t(stream.size() / 2);
                const size_t hdr = size_t(NT + 2) / 2;
                stream.resize(stream.size() + 2 * hdr, 0);
                for (int t = 0; t < NT; ++t) {
                    so[t] = int32_t(stream.size() / 2);
                    stream[2 * size_t(region0) + size_t(t)] = uint32_t(so[t] - region0);
                    auto &ops = per[size_t(t)][size_t(i)];
                    std::stable_sort(ops.begin(), ops.end(), [](const Op &a, const Op &b2) {
                        return a.cl != b2.cl ? a.cl < b2.cl : a.m != b2.m ? a.m < b2.m
                                                                            : a.rs < b2.rs;
                    });
                    int cur = -1;
                    for (const Op &o : ops) {
                        if (o.cl != cur) {
                            cur = o.cl;
                            stream.push_back(uint32_t((cur - i * c.CB) * plane));
                            stream.push_back(uint32_t(ncase));  // HDR
                        }
                        uint32_t wb;
                        std::memcpy(&wb, &o.w, 4);
                        stream.push_back(wb);
                        stream.push_back(uint32_t(o.m * sh.R * sh.S + o.rs));
                    }
                    stream.push_back(0);
                    stream.push_back(uint32_t(ncase + 1));  // EXIT
                }
                so[NT] = int32_t(stream.size() / 2);
                stream[2 * size_t(region0) + size_t(NT)] = uint32_t(so[NT] - region0);
                so[0] = int32_t(region0);  // region start (fill_stage copies from here)
                max_region = std::max(max_region, int64_t(so[NT]) - region0);
            }
        }
    }
    if (stream.size() / 2 >= (size_t(1) << 31))
        return fail(SKC_ERR_OVERFLOW, "regtile op stream too large");
    RegtileParams &rp = p->rp;
    rp = RegtileParams{};
    rp.C = p->C; rp.K = p->K; rp.Cg = p->Cg; rp.Kg = p->Kg; rp.Hp = p->Hp; rp.Wp = p->Wp;
    rp.Ho = p->Ho; rp.Wo = p->Wo; rp.groups = p->groups;
    rp.NI = c.NI; rp.CB = c.CB; rp.nchunks = nchunks;
    rp.img_stride = c.img_stride;
    rp.slab_floats = c.NI * c.img_stride;
    rp.stream_cap = int(align_up(size_t(max_region) + 2, 2));
    rp.stage_floats = rp.slab_floats + 2 * rp.stream_cap;
    rp.NG = c.NG; rp.NT = NT; rp.nblocks = nb;
    const size_t stage_bytes = size_t(rp.stage_floats) * 4;
    const int WR = sh.TY + sh.R - 1, WC = sh.TX + sh.S - 1;
    const size_t tail = align_up(size_t(WR) * p->Wp + WC + 4, 4) * 4;  // junk-tile overrun
    const size_t fixed = tail + kMaxStages * (sizeof(uint64_t) + sizeof(int));
    int NS = kRtStages;
    const size_t smem_cap = (220u << 10) / size_t(std::max(1, std::min(c.ctas_per_sm, 3)));
    while (NS > 1 && NS * stage_bytes + fixed > smem_cap)
        --NS;
    NS = std::min(NS, nchunks);
    if (NS * stage_bytes + fixed > (227 << 10))
        return fail(SKC_ERR_UNSUPPORTED, "regtile stage of %zu B does not fit", stage_bytes);
    rp.NS = NS;
    // stages come first; the tail slack sits between the last stage and the barriers
    p->smem = size_t(NS) * stage_bytes + fixed;
    p->rsh = sh;
    p->sg = StageGeom{};
    p->sg.CB = c.CB; p->sg.NS = NS; p->sg.BH = sh.TY;
    p->NW = c.NG * NT; p->M = M; p->T = sh.TY * sh.TX;
    // device image: stream | segoff | chan | lanemap | perm
    p->off_stream = 0;
    p->off_segoff = align_up(stream.size() * 4, 256);
    p->off_chan = align_up(p->off_segoff + segoff.size() * 4, 256);
    p->off_lanemap = align_up(p->off_chan + chan.size() * 4, 256);
    p->off_perm = align_up(p->off_lanemap + c.lanemap.size() * 4, 256);
    const size_t total = align_up(p->off_perm + size_t(p->K) * 4, 256);
    p->image.assign(total, 0);
    std::memcpy(p->image.data() + p->off_stream, stream.data(), stream.size() * 4);
    std::memcpy(p->image.data() + p->off_segoff, segoff.data(), segoff.size() * 4);
    std::memcpy(p->image.data() + p->off_chan, chan.data(), chan.size() * 4);
    std::memcpy(p->image.data() + p->off_lanemap, c.lanemap.data(), c.lanemap.size() * 4);
    std::memcpy(p->image.data() + p->off_perm, p->perm.data(), size_t(p->K) * 4);
    return SKC_OK;
}

// Estimated direct-kernel cost on the same scale as RtCandidate::cost (clk per image).
double direct_cost(const skc_plan *p) {
    // shared-memory wavefronts per nonzero per image (T loads + 2 shuffles per band), at the
    // ~80% wavefront utilisation ncu measured (profiles/r01_ncu_conv3_direct_pitch.json)
    return double(p->colidx.size()) * p->direct_waves / 0.80;
}

// ---- row f2: the SpMDM kernel's tables (spmdm.cu) ------------------------------------------
constexpr int kSpmdmSMs = 148;                 // B200 SM count (grid sizing at pack time)
constexpr int kSpmdmNW = 16;                   // warps per CTA
constexpr size_t kSpmdmSmemMax = 227 << 10;    // opt-in shared memory per CTA
constexpr size_t kSpmdmStageX = 64 << 10;      // X bytes per stage we aim for

bool spmdm_eligible(const skc_plan *p) {
    return p->R == 1 && p->S == 1 && p->stride == 1 && p->pad == 0 && p->groups == 1 &&
           (int64_t(p->Hp) * p->Wp) % 4 == 0;
}

// Tile configuration: LC columns per lane, RWM rows per warp, ntiles row tiles.  Cost model
// in shared-memory wavefronts per CTA (the kernel's bound): per nonzero and warp, the X row
// slice (min(BC, plane)/32 wavefronts) + 1 broadcast entry; per chunk row staged, the same
// slice again (TMA writes into the stage); times the waves of CTAs over the SMs.  A column
// block narrower than the plane needs one bulk copy per X row, which the producer issues
// one at a time (~40 clk each, profiles/r02_fc_spmdm.txt): a chunk then costs at least
// KC x 40 clk, which made LC = 4 blocks of a 256-wide batch copy-bound.
struct SpmdmCfg {
    int LC = 0, RWM = 0, ntiles = 0, ncb = 0;
    double cost = 1e300;
};

SpmdmCfg spmdm_choose(const skc_plan *p) {
    const int M = p->K, C = p->C, plane = p->Hp * p->Wp;
    const double nnzr = double(p->colidx.size()) / M;
    SpmdmCfg best;
    for (int LC : {8, 4}) {
        const int BC = 32 * LC;
        const int ncb = (plane + BC - 1) / BC;
        const double xw = double(std::min(BC, plane)) / 32.0;
        for (int RWM : {4, 8}) {
            const int min_t = (M + kSpmdmNW * RWM - 1) / (kSpmdmNW * RWM);
            std::vector<int> cand{min_t};
            for (int k = 1; k <= 8; ++k) cand.push_back((k * kSpmdmSMs + ncb - 1) / ncb);
            const int KC = std::min<int>(C, int(std::max<size_t>(1, kSpmdmStageX /
                                                 (size_t(ncb == 1 ? plane : BC) * 4))));
            const int nch = (C + KC - 1) / KC;
            for (int nt : cand) {
                if (nt < min_t || nt > M) continue;
                const int RT = (M + nt - 1) / nt;
                const int waves = (nt * ncb + kSpmdmSMs - 1) / kSpmdmSMs;
                const double chunk = std::max(RT * nnzr * KC / C * (xw + 1.0) + KC * xw,
                                              ncb == 1 ? 0.0 : 40.0 * KC);
                const double cost = waves * nch * chunk;
                if (cost < best.cost * 0.999) best = SpmdmCfg{LC, RWM, nt, ncb, cost};
            }
        }
    }
    return best;
}

skc_status build_spmdm(skc_plan *p) {
    const int M = p->K, C = p->C, plane = p->Hp * p->Wp;
    const SpmdmCfg cfg = spmdm_choose(p);
    const int LC = cfg.LC, nt = cfg.ntiles, ncb = cfg.ncb, BC = 32 * LC;
    const uint32_t xpitch = uint32_t(ncb == 1 ? plane : BC) * 4u;
    std::vector<int32_t> trow(size_t(nt) + 1);
    for (int t = 0; t <= nt; ++t) trow[size_t(t)] = int32_t(int64_t(t) * M / nt);
    int RTmax = 0;
    for (int t = 0; t < nt; ++t) RTmax = std::max(RTmax, trow[size_t(t) + 1] - trow[size_t(t)]);
    const uint32_t hbytes = uint32_t(align_up(size_t(RTmax + 1) * 4, 16));
    int KC = int(std::max<size_t>(1, kSpmdmStageX / xpitch));
    KC = std::min(KC, C);
    for (;;) {
        const int nch = (C + KC - 1) / KC;
        // blocks: header (uint32 entry offsets per local row), entries (x offset, w bits)
        std::vector<int64_t> blk(size_t(nt) * nch + 1, 0);
        std::vector<uint8_t> meta;
        size_t mstage = 16;
        std::vector<int32_t> cur(static_cast<size_t>(M), 0);
        for (int m = 0; m < M; ++m) cur[size_t(m)] = p->rowptr[size_t(m)];
        for (int t = 0; t < nt; ++t)
            for (int j = 0; j < nch; ++j) {
                const size_t b0 = meta.size();
                blk[size_t(t) * nch + j] = int64_t(b0);
                meta.resize(b0 + hbytes, 0);
                std::vector<uint32_t> hdr;
                std::vector<uint32_t> ent;
                const int kend = std::min(C, (j + 1) * KC);
                for (int m = trow[size_t(t)]; m < trow[size_t(t) + 1]; ++m) {
                    hdr.push_back(uint32_t(ent.size() / 2));
                    int32_t &c = cur[size_t(m)];
                    while (c < p->rowptr[size_t(m) + 1] && p->colidx[size_t(c)] / plane < kend) {
                        const int k = p->colidx[size_t(c)] / plane;
                        uint32_t wb;
                        std::memcpy(&wb, &p->values[size_t(c)], 4);
                        ent.push_back(uint32_t(k - j * KC) * xpitch);
                        ent.push_back(wb);
                        ++c;
                    }
                }
                hdr.push_back(uint32_t(ent.size() / 2));
                std::memcpy(meta.data() + b0, hdr.data(), hdr.size() * 4);
                meta.resize(align_up(b0 + hbytes + ent.size() * 4, 16), 0);
                if (!ent.empty()) std::memcpy(meta.data() + b0 + hbytes, ent.data(), ent.size() * 4);
                mstage = std::max(mstage, meta.size() - b0);
            }
        blk[size_t(nt) * nch] = int64_t(meta.size());
        for (int m = 0; m < M; ++m)
            if (cur[size_t(m)] != p->rowptr[size_t(m) + 1])
                return fail(SKC_ERR_STATE, "spmdm: row %d not fully packed", m);
        const size_t xstage = align_up(size_t(KC) * xpitch, 128);
        mstage = align_up(mstage, 128);
        // + 512 B of slack after the last stage: a lane's second column group (LC = 8) may read
        // up to 512 B past the last staged row when the plane is narrower than 256 columns
        // (those values are never stored)
        int NS = 0;
        for (int ns : {3, 2})
            if (128 + ns * (xstage + mstage) + 512 <= kSpmdmSmemMax) { NS = ns; break; }
        if (NS == 0) {
            if (KC == 1) return fail(SKC_ERR_UNSUPPORTED, "spmdm: a chunk does not fit shared memory");
            KC = std::max(1, KC / 2);
            continue;
        }
        // image: trow | blk | meta
        p->off_trow = 0;
        p->off_blk = align_up(trow.size() * 4, 16);
        p->off_meta = align_up(p->off_blk + blk.size() * 8, 16);
        p->image.assign(p->off_meta + meta.size(), 0);
        std::memcpy(p->image.data() + p->off_trow, trow.data(), trow.size() * 4);
        std::memcpy(p->image.data() + p->off_blk, blk.data(), blk.size() * 8);
        std::memcpy(p->image.data() + p->off_meta, meta.data(), meta.size());
        SpmdmParams &sp = p->sp;
        sp = SpmdmParams{};
        sp.K = M; sp.C = C; sp.H = p->H; sp.W = p->W; sp.plane = plane;
        sp.KC = KC; sp.nch = nch; sp.NS = NS; sp.ntiles = nt; sp.ncb = ncb;
        sp.xcontig = ncb == 1;
        sp.xpitch = xpitch; sp.xstage = uint32_t(xstage); sp.mstage = uint32_t(mstage);
        sp.hbytes = hbytes;
        p->sp_LC = LC; p->sp_RWM = cfg.RWM; p->sp_NW = kSpmdmNW;
        p->smem = 128 + NS * (xstage + mstage) + 512;
        p->kernel = SKC_KERNEL_SPMDM;
        p->layout = SKC_LAYOUT_NCHW;
        (void)BC;
        return SKC_OK;
    }
}

bool aligned16(const void *ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; }

}  // namespace

// ---------------------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------------------
extern "C" {

const char *skc_last_error(void) { return g_err.c_str(); }

static skc_status pack_common(const float *w, int K, int C, int R, int S, int H, int W, int stride,
                       int pad, int groups, int kernel, int max_ni, int batch_hint, skc_plan **out);

// The configuration's default batch: 256 (the benchmark batch), or SKC_JIT_NHINT.
static int default_batch_hint() {
    const char *e = std::getenv("SKC_JIT_NHINT");
    return e ? std::max(1, std::atoi(e)) : 256;
}

skc_status skc_pack_csr_ex(const float *w, int K, int C, int R, int S, int H, int W,
                           int stride, int pad, int groups, int kernel, skc_plan **out) {
    return pack_common(w, K, C, R, S, H, W, stride, pad, groups, kernel, 4, default_batch_hint(), out);
}

skc_status skc_pack_csr_batch(const float *w, int K, int C, int R, int S, int H, int W,
                              int stride, int pad, int groups, int kernel, int batch_hint,
                              skc_plan **out) {
    if (batch_hint < 1) return fail(SKC_ERR_ARG, "batch_hint %d < 1", batch_hint);
    return pack_common(w, K, C, R, S, H, W, stride, pad, groups, kernel, 4, batch_hint, out);
}

static skc_status pack_common(const float *w, int K, int C, int R, int S, int H, int W, int stride,
                       int pad, int groups, int kernel, int max_ni, int batch_hint, skc_plan **out) {
    if (!w || !out) return fail(SKC_ERR_ARG, "NULL weights or output pointer");
    *out = nullptr;
    if (kernel < SKC_KERNEL_AUTO || kernel > SKC_KERNEL_SPMDM)
        return fail(SKC_ERR_ARG, "unknown kernel variant %d", kernel);
    skc_status st = check_geometry(K, C, R, S, H, W, stride, pad, groups);
    if (st != SKC_OK) return st;
    skc_plan *p = new (std::nothrow) skc_plan();
    if (!p) return fail(SKC_ERR_ARG, "out of host memory");
    p->K = K; p->C = C; p->R = R; p->S = S; p->H = H; p->W = W;
    p->stride = stride; p->pad = pad; p->groups = groups;
    p->Hp = H + 2 * pad; p->Wp = W + 2 * pad;
    p->Ho = (p->Hp - R) / stride + 1; p->Wo = (p->Wp - S) / stride + 1;
    p->Kg = K / groups; p->Cg = C / groups;
    p->max_ni = max_ni;
    p->batch_hint = std::max(1, batch_hint);

    // a1: canonical CSR.  Row k scans (c_local, r, s) lexicographically; because r < Hp
    // and s < Wp the offset is strictly increasing in that order.
    const size_t per_k = size_t(p->Cg) * R * S;
    p->rowptr.assign(size_t(K) + 1, 0);
    size_t nnz = 0;
    for (int k = 0; k < K; ++k) {
        const float *wk = w + size_t(k) * per_k;
        for (size_t i = 0; i < per_k; ++i) {
            if (!std::isfinite(wk[i])) {
                delete p;
                return fail(SKC_ERR_NONFINITE, "weight [%d][%zu] is not finite", k, i);
            }
            nnz += (wk[i] != 0.0f);
        }
        if (nnz >= (size_t(1) << 31)) {
            delete p;
            return fail(SKC_ERR_OVERFLOW, "nnz does not fit int32");
        }
        p->rowptr[size_t(k) + 1] = int32_t(nnz);
    }
    p->colidx.resize(nnz);
    p->values.resize(nnz);
    for (int k = 0; k < K; ++k) {
        const int gk = k / p->Kg;
        const float *wk = w + size_t(k) * per_k;
        size_t j = size_t(p->rowptr[k]);
        for (int cl = 0; cl < p->Cg; ++cl)
            for (int r = 0; r < R; ++r)
                for (int s = 0; s < S; ++s) {
                    const float v = wk[(size_t(cl) * R + r) * S + s];
                    if (v == 0.0f) continue;
                    p->colidx[j] = int32_t((int64_t(gk * p->Cg + cl) * p->Hp + r) * p->Wp + s);
                    std::memcpy(&p->values[j], &v, 4);  // bit-exact copy
                    ++j;
                }
    }
    // nnz-sorted permutation: descending nnz, stable (ties by ascending k), per group
    p->perm.resize(size_t(K));
    std::iota(p->perm.begin(), p->perm.end(), 0);
    // SKC_NO_NNZ_SORT=1 keeps the natural channel order (load-balance experiments only;
    // the default, and the checked contract, is the nnz-sorted order)
    const char *nosort = std::getenv("SKC_NO_NNZ_SORT");
    for (int g = 0; g < groups && !(nosort && nosort[0] == '1'); ++g) {
        auto b = p->perm.begin() + ptrdiff_t(g) * p->Kg;
        std::stable_sort(b, b + p->Kg, [p](int a, int c) {
            return p->rowptr[a + 1] - p->rowptr[a] > p->rowptr[c + 1] - p->rowptr[c];
        });
    }

    // row f2: the SpMDM kernel for FC plans (AUTO with max_ni == 1: skc_pack_fc) and on request
    // for any eligible 1x1 plan
    if (kernel == SKC_KERNEL_SPMDM || (kernel == SKC_KERNEL_AUTO && max_ni == 1 && spmdm_eligible(p))) {
        if (!spmdm_eligible(p)) {
            delete p;
            return fail(SKC_ERR_UNSUPPORTED, "SPMDM needs a 1x1, stride-1, pad-0, one-group plan "
                        "with H*W %% 4 == 0");
        }
        st = build_spmdm(p);
        if (st != SKC_OK) {
            delete p;
            return st;
        }
        *out = p;
        return ok();
    }
    // kernel choice: the compiled-weights kernel when a configuration fits (AUTO; disabled
    // with SKC_NO_JIT=1); else the register-tiled kernel when an instantiated tile shape fits
    // and the cost model prefers it; the direct kernel otherwise (any stride, any R x S)
    const char *nojit = std::getenv("SKC_NO_JIT");
    // (AUTO keeps single-image FC plans -- max_ni == 1 -- on the data-driven kernels: their
    // code would be millions of instructions for ~one CTA item per block)
    // (AUTO also keeps small batches on them: a compiled layer's code is fetched cold by the
    // few CTAs a small batch has, and the direct kernel with a small-batch configuration is
    // faster below kAutoJitMinBatch images per launch, profiles/r02_small_batch.txt)
    if (kernel == SKC_KERNEL_JIT ||
        (kernel == SKC_KERNEL_AUTO && max_ni > 1 && p->batch_hint >= kAutoJitMinBatch &&
         !(nojit && nojit[0] == '1'))) {
        const JitInput ji{K, C, R, S, p->Hp, p->Wp, p->Ho, p->Wo, stride, groups, p->Kg, p->Cg, pad,
                          p->rowptr.data(), p->colidx.data(), p->perm.data(), p->values.data()};
        std::string msg;
        // the configuration search at batch hints below 256 picks code-heavy blocks (few
        // channels each) whose cold code costs more than its model charges -- 3x slower than
        // the 256-image configuration on ResNet res256 at 8 images -- so JIT plans are always
        // configured for 256 images (profiles/r02_small_batch.txt; SKC_JIT_NHINT, an
        // experiment knob, is passed through)
        const int jit_hint = std::getenv("SKC_JIT_NHINT") && max_ni > 1 ? p->batch_hint : 256;
        const int r = jit_configure(ji, max_ni == 1 ? 1 : 64, jit_hint, &p->jit, &msg);
        if (r == SKC_OK) {
            p->kernel = SKC_KERNEL_JIT;
            p->image.assign(jit_image_bytes(p->jit), 0);   // lane tables, counters, staging
            jit_image(p->jit, p->image.data());
            p->off_lanemap = 0;
            JitInfo ji2{};
            jit_info(p->jit, &ji2);
            p->smem = ji2.smem;
            p->layout = ji2.raw ? SKC_LAYOUT_RAW : ji2.pair ? SKC_LAYOUT_PAIRS : SKC_LAYOUT_NCHW;
            *out = p;
            return ok();
        }
        if (kernel == SKC_KERNEL_JIT) {
            delete p;
            return fail(skc_status(r), "%s", msg.c_str());
        }
    }
    RtCandidate best_rt;
    // (small batches: the register-tiled kernel's configurations are per-image ones; AUTO
    // takes the direct kernel's launch-time configuration there)
    const bool small_auto = kernel == SKC_KERNEL_AUTO && p->batch_hint < kAutoJitMinBatch;
    if (kernel != SKC_KERNEL_DIRECT && !small_auto) {
        RegtileShape shapes[32];
        const int ns = std::min(32, regtile_shapes(shapes, 32));
        // SKC_RT_SHAPE="R,S,TY,TX,M" restricts the search to one shape (tuning/benchmarks)
        RegtileShape want{};
        const char *env = std::getenv("SKC_RT_SHAPE");
        const bool forced = env && std::sscanf(env, "%d,%d,%d,%d,%d", &want.R, &want.S,
                                              &want.TY, &want.TX, &want.M) == 5;
        // SKC_RT_COST=1 prints the cost model of every candidate (tuning aid)
        const bool verbose = std::getenv("SKC_RT_COST") != nullptr;
        for (int i = 0; i < ns; ++i) {
            const RegtileShape &sh = shapes[i];
            if (forced && (sh.R != want.R || sh.S != want.S || sh.TY != want.TY ||
                           sh.TX != want.TX || sh.M != want.M))
                continue;
            RtCandidate cand;
            const bool okc = regtile_candidate(p, sh, cand);
            if (verbose)
                std::fprintf(stderr, "skc regtile %dx%d tile %dx%d M=%d nw=%d: %s cost %.4g NI=%d "
                             "NG=%d NT=%d CB=%d wf=%d\n", sh.R, sh.S, sh.TY, sh.TX, sh.M, sh.nwmax,
                             okc ? "ok" : "n/a", cand.cost, cand.NI, cand.NG, cand.NT, cand.CB,
                             cand.wf);
            if (okc && cand.cost < best_rt.cost) best_rt = cand;
        }
    }
    st = configure_direct(p);
    if (small_auto && st != SKC_OK) {
        // no small-batch direct configuration (e.g. a row wider than the kernel's pixel
        // slots): the configuration for kAutoJitMinBatch images, whatever the kernel
        delete p;
        return pack_common(w, K, C, R, S, H, W, stride, pad, groups, kernel, max_ni,
                           kAutoJitMinBatch, out);
    }
    if (kernel == SKC_KERNEL_REGTILE && best_rt.cost >= 1e300) {
        delete p;
        return fail(SKC_ERR_UNSUPPORTED, "no register-tile shape for R=%d S=%d stride=%d "
                    "(or TMA alignment)", R, S, stride);
    }
    if (kernel == SKC_KERNEL_DIRECT && st != SKC_OK) {
        delete p;
        return st;
    }
    const bool use_rt = best_rt.cost < 1e300 &&
                        (kernel == SKC_KERNEL_REGTILE || st != SKC_OK ||
                         best_rt.cost < 0.9 * direct_cost(p));  // prefer direct on near-ties
    if (use_rt) {
        p->kernel = SKC_KERNEL_REGTILE;
        st = build_regtile(p, best_rt);
    } else if (st == SKC_OK) {
        p->kernel = SKC_KERNEL_DIRECT;
        st = build_direct_image(p);
    }
    if (st != SKC_OK) {
        delete p;
        return st;
    }
    *out = p;
    return ok();
}

skc_status skc_pack_csr(const float *w, int K, int C, int R, int S, int H, int W, int stride,
                        int pad, int groups, skc_plan **out) {
    return skc_pack_csr_ex(w, K, C, R, S, H, W, stride, pad, groups, SKC_KERNEL_AUTO, out);
}

skc_status skc_pack_fc(const float *w, int M, int K, int B, int kernel, skc_plan **out) {
    // Y[M x B] = W[M x K] X[K x B] is the 1x1 convolution of one "image" with K channels of
    // 1 x B pixels: PAPER.md:318-329 (sparse FC layers as SpMDM)
    if (B < 1) return fail(SKC_ERR_GEOMETRY, "batch B = %d < 1", B);
    // one "image" per call: never stage more than one image per CTA.  The batch axis may be
    // folded into rows (B = rows x B/rows, same memory layout) so the direct kernel can split
    // it into bands -- more CTAs for a single image (SKC_FC_ROWS, tuning)
    int rows = 1;
    if (const char *e = std::getenv("SKC_FC_ROWS")) rows = std::max(1, std::atoi(e));
    if (B % rows) rows = 1;
    return pack_common(w, M, K, 1, 1, rows, B / rows, 1, 0, 1, kernel, 1, default_batch_hint(), out);
}

skc_status skc_plan_info(const skc_plan *p, skc_info *info) {
    if (!p || !info) return fail(SKC_ERR_ARG, "NULL plan or info");
    skc_info &i = *info;
    i.K = p->K; i.C = p->C; i.R = p->R; i.S = p->S; i.H = p->H; i.W = p->W;
    i.stride = p->stride; i.pad = p->pad; i.groups = p->groups;
    i.Ho = p->Ho; i.Wo = p->Wo; i.Hp = p->Hp; i.Wp = p->Wp;
    i.nnz = int64_t(p->colidx.size());
    i.padded_elems_per_image = size_t(p->C) * p->Hp * p->Wp;
    i.out_elems_per_image = size_t(p->K) * p->Ho * p->Wo;
    i.device_bytes = p->image.size();
    i.kernel = p->kernel;
    i.band_rows = p->sg.BH; i.chunk_channels = p->sg.CB; i.stages = p->sg.NS;
    i.warps = p->NW; i.channels_per_warp = p->M; i.pixels_per_lane = p->T;
    i.smem_bytes = p->smem;
    i.lane_mapping = p->kernel == SKC_KERNEL_DIRECT ? p->sg.NI : 0;
    i.tile_h = p->kernel == SKC_KERNEL_REGTILE ? p->rsh.TY : 0;
    i.tile_w = p->kernel == SKC_KERNEL_REGTILE ? p->rsh.TX : 0;
    i.images_per_cta = p->kernel == SKC_KERNEL_REGTILE ? p->rp.NI : p->sg.NI;
    i.jit_blocks = 0; i.jit_compiled = 0; i.jit_cache_hit = 0; i.jit_compile_s = 0;
    i.code_bytes = 0; i.model_instr_per_image = 0;
    i.layout = p->layout;
    i.bands = 0;
    i.jit_whole = 0;
    i.jit_split = 0;
    i.jit_sched = -1;
    i.jit_np = 0;
    i.jit_deal = 0;
    if (p->kernel == SKC_KERNEL_SPMDM) {
        i.band_rows = 0; i.chunk_channels = p->sp.KC; i.stages = p->sp.NS; i.warps = p->sp_NW;
        i.channels_per_warp = p->sp_RWM; i.pixels_per_lane = p->sp_LC; i.lane_mapping = 0;
        i.images_per_cta = 1;
    }
    if (p->kernel == SKC_KERNEL_JIT) {
        JitInfo j{};
        jit_info(p->jit, &j);
        i.band_rows = 0; i.chunk_channels = j.CB; i.stages = j.NS; i.warps = j.NW;
        i.channels_per_warp = j.M; i.pixels_per_lane = j.TY * j.TX; i.smem_bytes = j.smem;
        i.lane_mapping = 0; i.tile_h = j.TY; i.tile_w = j.TX; i.images_per_cta = j.NI;
        i.jit_blocks = j.nblocks; i.jit_compiled = j.compiled; i.jit_cache_hit = j.cache_hit;
        i.jit_compile_s = j.compile_s; i.code_bytes = j.cubin_bytes;
        i.model_instr_per_image = j.cost;
        i.bands = j.bands;
        i.jit_whole = j.whole;
        i.jit_split = j.split;
        i.jit_sched = j.sched;
        i.jit_np = j.np;
        i.jit_deal = j.deal;
    }
    return ok();
}

skc_status skc_plan_csr(const skc_plan *p, const int32_t **rowptr, const int32_t **colidx,
                        const float **values) {
    if (!p) return fail(SKC_ERR_ARG, "NULL plan");
    if (rowptr) *rowptr = p->rowptr.data();
    if (colidx) *colidx = p->colidx.data();
    if (values) *values = p->values.data();
    return ok();
}

skc_status skc_plan_perm(const skc_plan *p, const int32_t **perm) {
    if (!p || !perm) return fail(SKC_ERR_ARG, "NULL plan or perm");
    *perm = p->perm.data();
    return ok();
}

}  // extern "C"

// ---------------------------------------------------------------------------------------
// Plan verifier: a static check of every kernel-private index the kernels dereference, and
// an exact round trip of the kernel streams back to the canonical CSR.
// ---------------------------------------------------------------------------------------
namespace {

struct NzKey {
    int k, c, r, s;
    uint32_t wbits;
    bool operator<(const NzKey &o) const {
        return std::tie(k, c, r, s, wbits) < std::tie(o.k, o.c, o.r, o.s, o.wbits);
    }
    bool operator==(const NzKey &o) const {
        return k == o.k && c == o.c && r == o.r && s == o.s && wbits == o.wbits;
    }
};

std::vector<NzKey> csr_keys(const skc_plan *p) {
    std::vector<NzKey> v;
    const int64_t plane = int64_t(p->Hp) * p->Wp;
    for (int k = 0; k < p->K; ++k)
        for (int32_t j = p->rowptr[k]; j < p->rowptr[k + 1]; ++j) {
            const int64_t col = p->colidx[j];
            uint32_t wb;
            std::memcpy(&wb, &p->values[j], 4);
            v.push_back(NzKey{k, int(col / plane), int(col % plane / p->Wp), int(col % p->Wp), wb});
        }
    std::sort(v.begin(), v.end());
    return v;
}

template <class T>
const T *img_ptr(const skc_plan *p, size_t off) {
    return reinterpret_cast<const T *>(p->image.data() + off);
}

int sp_rows_max(const skc_plan *p) { return p->sp_NW * p->sp_RWM; }

// SpMDM tables decoded back to the canonical CSR: tiles cover the rows once, each block's
// header is monotone and its entries land inside the chunk's stage, and the (row, k, w) set in
// per-row order is exactly the CSR's.
skc_status verify_spmdm(const skc_plan *p) {
    const SpmdmParams &sp = p->sp;
    const int plane = sp.plane;
    const int32_t *trow = img_ptr<int32_t>(p, p->off_trow);
    const int64_t *blk = img_ptr<int64_t>(p, p->off_blk);
    const uint8_t *meta = p->image.data() + p->off_meta;
    const size_t meta_bytes = p->image.size() - p->off_meta;
    if (trow[0] != 0 || trow[sp.ntiles] != p->K)
        return fail(SKC_ERR_STATE, "verify: row tiles do not span [0, %d)", p->K);
    std::vector<int32_t> nxt(p->rowptr.begin(), p->rowptr.end() - 1);  // next CSR entry per row
    for (int t = 0; t < sp.ntiles; ++t) {
        const int r0 = trow[t], rows = trow[t + 1] - r0;
        if (rows < 0 || rows > sp_rows_max(p))
            return fail(SKC_ERR_STATE, "verify: tile %d has %d rows", t, rows);
        for (int j = 0; j < sp.nch; ++j) {
            const int64_t b0 = blk[size_t(t) * sp.nch + j], b1 = blk[size_t(t) * sp.nch + j + 1];
            if (b0 % 16 || b1 % 16 || b1 < b0 + sp.hbytes || size_t(b1) > meta_bytes ||
                uint64_t(b1 - b0) > sp.mstage)
                return fail(SKC_ERR_STATE, "verify: block (%d, %d) bounds", t, j);
            const uint32_t *hdr = reinterpret_cast<const uint32_t *>(meta + b0);
            const uint32_t *ent = reinterpret_cast<const uint32_t *>(meta + b0 + sp.hbytes);
            const uint64_t nent = uint64_t(b1 - b0 - sp.hbytes) / 8;
            const int kr = std::min(sp.KC, p->C - j * sp.KC);
            if (hdr[0] != 0) return fail(SKC_ERR_STATE, "verify: block (%d, %d) header", t, j);
            for (int lr = 0; lr < rows; ++lr) {
                if (hdr[lr + 1] < hdr[lr] || hdr[lr + 1] > nent)
                    return fail(SKC_ERR_STATE, "verify: block (%d, %d) row %d offsets", t, j, lr);
                const int m = r0 + lr;
                for (uint32_t i = hdr[lr]; i < hdr[lr + 1]; ++i) {
                    const uint32_t xo = ent[2 * i], wb = ent[2 * i + 1];
                    if (xo % sp.xpitch || xo / sp.xpitch >= uint32_t(kr))
                        return fail(SKC_ERR_STATE, "verify: entry outside the chunk's stage");
                    const int32_t c = nxt[size_t(m)]++;
                    uint32_t vb;
                    if (c >= p->rowptr[size_t(m) + 1])
                        return fail(SKC_ERR_STATE, "verify: row %d has extra entries", m);
                    std::memcpy(&vb, &p->values[size_t(c)], 4);
                    if (int64_t(j) * sp.KC + xo / sp.xpitch != p->colidx[size_t(c)] / plane || wb != vb)
                        return fail(SKC_ERR_STATE, "verify: row %d entry %d differs from the CSR", m,
                                    int(c - p->rowptr[size_t(m)]));
                }
            }
        }
    }
    for (int m = 0; m < p->K; ++m)
        if (nxt[size_t(m)] != p->rowptr[size_t(m) + 1])
            return fail(SKC_ERR_STATE, "verify: row %d misses entries", m);
    return SKC_OK;
}

skc_status verify_direct(const skc_plan *p) {
    const DirectParams &d = p->dp;
    const int nslot = d.NW * d.M, T = p->T;
    const int gblocks = p->groups * d.cblocks;
    const int32_t *segptr = img_ptr<int32_t>(p, p->off_segoff);
    const int32_t *chan = img_ptr<int32_t>(p, p->off_chan);
    const int32_t *slotq = img_ptr<int32_t>(p, p->off_lanemap);
    const int32_t *slotout = img_ptr<int32_t>(p, p->off_chunkptr);
    const uint32_t *stream = img_ptr<uint32_t>(p, p->off_stream);
    const size_t stream_entries = p->off_segoff / 8;
    // channel table: every output channel exactly once, in its own conv group
    std::vector<int> seen(size_t(p->K), 0);
    for (int gb = 0; gb < gblocks; ++gb)
        for (int j = 0; j < nslot; ++j) {
            const int k = chan[size_t(gb) * nslot + j];
            if (k < -1 || k >= p->K) return fail(SKC_ERR_STATE, "verify: channel %d out of range", k);
            if (k >= 0 && (seen[size_t(k)]++ || k / p->Kg != gb / d.cblocks))
                return fail(SKC_ERR_STATE, "verify: channel %d placed twice or in the wrong group", k);
        }
    for (int k = 0; k < p->K; ++k)
        if (!seen[size_t(k)]) return fail(SKC_ERR_STATE, "verify: channel %d never computed", k);
    // slots: reads stay inside the stage, outputs cover every (image, y, x) exactly once
    int qmax = 0;
    for (int b = 0; b < d.nbands; ++b) {
        const int rows = std::min(d.BH, p->Ho - b * d.BH);
        std::vector<int> cover(size_t(d.NI) * rows * p->Wo, 0);
        for (int t = 0; t < T; ++t)
            for (int l = 0; l < 32; ++l) {
                const size_t o = (size_t(b) * T + t) * 32 + l;
                const int q = slotq[o], out = slotout[o];
                if ((q & 31) != l) return fail(SKC_ERR_STATE, "verify: slot bank %d != lane %d", q & 31, l);
                if (q < 0) return fail(SKC_ERR_STATE, "verify: negative slot offset");
                qmax = std::max(qmax, q);
                if (out < 0) continue;
                const int img = out >> 24, yl = (out >> 12) & 0xfff, x = out & 0xfff;
                if (img >= d.NI || yl >= rows)
                    return fail(SKC_ERR_STATE, "verify: slot output out of the band");
                if (q != img * d.img_stride + yl * p->stride * p->Wp + x * p->stride)
                    return fail(SKC_ERR_STATE, "verify: slot reads the wrong input pixel");
                cover[(size_t(img) * rows + yl) * p->Wo + x]++;
            }
        for (int v : cover)
            if (v != 1) return fail(SKC_ERR_STATE, "verify: output pixel covered %d times", v);
    }
    // streams: segment tables, bounds of every read, exact round trip to the CSR
    std::vector<NzKey> got;
    const int64_t plane = int64_t(p->Hp) * p->Wp;
    for (int gb = 0; gb < gblocks; ++gb)
        for (int i = 0; i < d.nchunks; ++i) {
            const int32_t *sp = segptr + (size_t(gb) * d.nchunks + i) * (nslot + 1);
            const int32_t r0 = sp[0], r1 = sp[nslot];
            if (r0 < 0 || r1 < r0 || size_t(r1) > stream_entries || (r0 & 1))
                return fail(SKC_ERR_STATE, "verify: bad stream region");
            if (((r1 - r0 + 1) & ~1) > d.stream_cap)
                return fail(SKC_ERR_STATE, "verify: stream region exceeds the stage capacity");
            const int32_t *hdr = reinterpret_cast<const int32_t *>(stream + 2 * size_t(r0));
            for (int j = 0; j < nslot; ++j) {
                const int b0 = hdr[j], b1 = hdr[j + 1];
                if (b0 < (nslot + 2) / 2 || b1 < b0 || r0 + b1 > r1)
                    return fail(SKC_ERR_STATE, "verify: bad segment table");
                const int k = chan[size_t(gb) * nslot + j];
                if (k < 0 && b1 > b0) return fail(SKC_ERR_STATE, "verify: ops for an empty slot");
                for (int e = b0; e < b1; ++e) {
                    const uint32_t wb = stream[2 * size_t(r0 + e)];
                    const uint32_t ob = stream[2 * size_t(r0 + e) + 1];
                    if (ob & 3) return fail(SKC_ERR_STATE, "verify: misaligned offset");
                    const int off = int(ob / 4);
                    if (off + qmax >= d.stage_floats)
                        return fail(SKC_ERR_STATE, "verify: read beyond the stage");
                    const int cl = off / d.chan_stride, rem = off % d.chan_stride;
                    if (cl >= d.CB || i * d.CB + cl >= p->Cg)
                        return fail(SKC_ERR_STATE, "verify: channel outside the chunk");
                    got.push_back(NzKey{k, (k / p->Kg) * p->Cg + i * d.CB + cl, rem / p->Wp,
                                        rem % p->Wp, wb});
                }
            }
        }
    (void)plane;
    std::sort(got.begin(), got.end());
    if (got != csr_keys(p)) return fail(SKC_ERR_STATE, "verify: direct streams != canonical CSR");
    return SKC_OK;
}

skc_status verify_jit(const skc_plan *p) {
    std::string msg;
    const int r = jit_verify_code(p->jit, &msg);
    if (r != SKC_OK) return fail(skc_status(r), "%s", msg.c_str());
    return SKC_OK;
}

skc_status verify_regtile(const skc_plan *p) {
    const RegtileParams &r = p->rp;
    const RegtileShape &sh = p->rsh;
    const int M = sh.M, ncase = M * sh.R * sh.S;
    const int WR = sh.TY + sh.R - 1, WC = sh.TX + sh.S - 1;
    const int gblocks = p->groups * r.nblocks;
    const int64_t plane = int64_t(p->Hp) * p->Wp;
    const int32_t *segoff = img_ptr<int32_t>(p, p->off_segoff);
    const int32_t *chan = img_ptr<int32_t>(p, p->off_chan);
    const int32_t *lanemap = img_ptr<int32_t>(p, p->off_lanemap);
    const uint32_t *stream = img_ptr<uint32_t>(p, p->off_stream);
    const size_t stream_entries = p->off_segoff / 8;
    std::vector<int> seen(size_t(p->K), 0);
    for (int gb = 0; gb < gblocks; ++gb)
        for (int j = 0; j < r.NT * M; ++j) {
            const int k = chan[size_t(gb) * r.NT * M + j];
            if (k < -1 || k >= p->K) return fail(SKC_ERR_STATE, "verify: channel %d out of range", k);
            if (k >= 0 && (seen[size_t(k)]++ || k / p->Kg != gb / r.nblocks))
                return fail(SKC_ERR_STATE, "verify: channel %d placed twice or in the wrong group", k);
        }
    for (int k = 0; k < p->K; ++k)
        if (!seen[size_t(k)]) return fail(SKC_ERR_STATE, "verify: channel %d never computed", k);
    // lane map: every output pixel of the NI images in exactly one active lane's tile
    std::vector<int> cover(size_t(r.NI) * p->Ho * p->Wo, 0);
    int lb_max = 0;
    for (int g = 0; g < r.NG; ++g)
        for (int l = 0; l < 32; ++l) {
            const int v = lanemap[g * 32 + l];
            const bool idle = (v >> 30) & 1;
            const int img = (v >> 24) & 0x3f, y0 = (v >> 12) & 0xfff, x0 = v & 0xfff;
            if (img >= r.NI) return fail(SKC_ERR_STATE, "verify: lane image out of range");
            lb_max = std::max(lb_max, img * r.img_stride + y0 * p->Wp + x0);
            if (idle) continue;
            for (int ty = 0; ty < sh.TY; ++ty)
                for (int tx = 0; tx < sh.TX; ++tx)
                    if (y0 + ty < p->Ho && x0 + tx < p->Wo)
                        cover[(size_t(img) * p->Ho + y0 + ty) * p->Wo + x0 + tx]++;
        }
    for (int v : cover)
        if (v != 1) return fail(SKC_ERR_STATE, "verify: output pixel covered %d times", v);
    // op streams
    const int64_t alloc_floats = int64_t(p->smem / 4);
    std::vector<NzKey> got;
    for (int gb = 0; gb < gblocks; ++gb)
        for (int i = 0; i < r.nchunks; ++i) {
            const int32_t *so = segoff + (size_t(gb) * r.nchunks + i) * (r.NT + 1);
            const int32_t r0 = so[0], r1 = so[r.NT];
            if (r0 < 0 || r1 < r0 || size_t(r1) > stream_entries || (r0 & 1))
                return fail(SKC_ERR_STATE, "verify: bad stream region");
            if (((r1 - r0 + 1) & ~1) > r.stream_cap)
                return fail(SKC_ERR_STATE, "verify: stream region exceeds the stage capacity");
            const int32_t *hdr = reinterpret_cast<const int32_t *>(stream + 2 * size_t(r0));
            for (int t = 0; t < r.NT; ++t) {
                const int b0 = hdr[t], b1 = (t + 1 < r.NT) ? hdr[t + 1] : r1 - r0;
                if (b0 < (r.NT + 2) / 2 || b1 <= b0 || r0 + b1 > r1)
                    return fail(SKC_ERR_STATE, "verify: bad segment table");
                int cbase = -1;
                for (int e = b0; e < b1; ++e) {
                    const uint32_t x = stream[2 * size_t(r0 + e)];
                    const uint32_t c = stream[2 * size_t(r0 + e) + 1];
                    const bool last = e + 1 == b1;
                    if (c == uint32_t(ncase + 1)) {
                        if (!last) return fail(SKC_ERR_STATE, "verify: EXIT before the end");
                        continue;
                    }
                    if (last) return fail(SKC_ERR_STATE, "verify: segment without EXIT");
                    if (c == uint32_t(ncase)) {  // HDR: window of channel x in every lane
                        if (int64_t(x) % plane || int64_t(x) / plane >= r.CB)
                            return fail(SKC_ERR_STATE, "verify: HDR channel offset");
                        const int64_t hi = int64_t(r.NS - 1) * r.stage_floats + lb_max + x +
                                           int64_t(WR - 1) * p->Wp + WC - 1;
                        if (hi >= alloc_floats) return fail(SKC_ERR_STATE, "verify: window beyond smem");
                        cbase = int(x);
                        continue;
                    }
                    if (c >= uint32_t(ncase)) return fail(SKC_ERR_STATE, "verify: bad case %u", c);
                    if (cbase < 0) return fail(SKC_ERR_STATE, "verify: FMA op before any HDR");
                    const int m = int(c) / (sh.R * sh.S), rr = (int(c) / sh.S) % sh.R, ss = int(c) % sh.S;
                    const int k = chan[(size_t(gb) * r.NT + t) * M + m];
                    if (k < 0) return fail(SKC_ERR_STATE, "verify: op for an empty channel slot");
                    got.push_back(NzKey{k, (k / p->Kg) * p->Cg + i * r.CB + int(cbase / plane), rr, ss, x});
                }
            }
        }
    std::sort(got.begin(), got.end());
    if (got != csr_keys(p)) return fail(SKC_ERR_STATE, "verify: regtile streams != canonical CSR");
    return SKC_OK;
}

}  // namespace

namespace {
template <class F>
skc_status bench_call(F &&fn, const char *name, void *d_scratch, int blocks, int iters, double *ms,
                      double *count) {
    if (!d_scratch || !ms || !count || blocks < 1 || iters < 1)
        return fail(SKC_ERR_ARG, "bad micro-benchmark arguments");
    float t = 0;
    cudaError_t e = fn(d_scratch, blocks, iters, &t, count);
    if (e != cudaSuccess) return fail(SKC_ERR_CUDA, "%s: %s", name, cudaGetErrorString(e));
    *ms = t;
    return ok();
}
}  // namespace

extern "C" {

skc_status skc_plan_compile(skc_plan *p) {
    if (!p) return fail(SKC_ERR_ARG, "NULL plan");
    if (p->kernel != SKC_KERNEL_JIT) return ok();
    std::string msg;
    const int r = jit_compile(p->jit, &msg);
    if (r != SKC_OK) return fail(skc_status(r), "JIT compile: %s", msg.c_str());
    return ok();
}

skc_status skc_sm_topology(int *vid, int cap, int *nsm) {
    if (!vid || !nsm) return fail(SKC_ERR_ARG, "NULL pointer");
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail(SKC_ERR_CUDA, "no CUDA device");
    std::vector<uint16_t> v;
    if (!sm_gpc_order_cached(dev, &v))
        return fail(SKC_ERR_STATE, "no SM order for this device: the probe runs at the first "
                    "skc_plan_upload of a JIT plan (or it failed)");
    *nsm = int(v.size());
    if (cap < int(v.size())) return fail(SKC_ERR_ARG, "cap %d < %zu SMs", cap, v.size());
    for (size_t i = 0; i < v.size(); ++i) vid[i] = int(v[i]);
    return ok();
}

skc_status skc_plan_tune(skc_plan *p, int N, const float *d_in, float *d_out, void *d_flush,
                         size_t flush_bytes, void *stream, double *best_ms) {
    if (!p) return fail(SKC_ERR_ARG, "NULL plan");
    if (N < 1) return fail(SKC_ERR_ARG, "N = %d < 1", N);
    if (best_ms) *best_ms = 0.0;
    if (p->kernel != SKC_KERNEL_JIT) return ok();
    if (!p->d_ws) return fail(SKC_ERR_STATE, "plan not uploaded (call skc_plan_upload)");
    if (!d_in || !d_out) return fail(SKC_ERR_ARG, "NULL scratch buffer");
    if (!aligned16(d_in) || !aligned16(d_out))
        return fail(SKC_ERR_ALIGN, "device pointers must be 16-byte aligned");
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || !jit_ready(p->jit, dev))
        return fail(SKC_ERR_STATE, "plan not uploaded on this device");
    std::string msg;
    const int r = jit_tune(p->jit, p->d_ws, N, d_in, d_out, d_flush, d_flush ? flush_bytes : 0,
                           (cudaStream_t)stream, best_ms, &msg);
    if (r != SKC_OK) return fail(skc_status(r), "tune: %s", msg.c_str());
    return ok();
}

skc_status skc_plan_verify(const skc_plan *p) {
    if (!p) return fail(SKC_ERR_ARG, "NULL plan");
    const skc_status st = p->kernel == SKC_KERNEL_JIT       ? verify_jit(p)
                          : p->kernel == SKC_KERNEL_REGTILE ? verify_regtile(p)
                          : p->kernel == SKC_KERNEL_SPMDM   ? verify_spmdm(p)
                                                            : verify_direct(p);
    return st == SKC_OK ? ok() : st;
}

skc_status skc_plan_upload(skc_plan *p, void *d_ws, size_t bytes, void *stream) {
    if (!p || !d_ws) return fail(SKC_ERR_ARG, "NULL plan or workspace");
    if (!aligned16(d_ws)) return fail(SKC_ERR_ALIGN, "workspace not 16-byte aligned");
    if (bytes < p->image.size())
        return fail(SKC_ERR_ARG, "workspace has %zu bytes, plan needs %zu", bytes,
                    p->image.size());
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return fail(SKC_ERR_CUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
    cudaStream_t st = (cudaStream_t)stream;
    // everything a launch needs is set up here, so forward launches are capture-safe and
    // allocation-free from the first call: the kernel attributes, and for JIT plans the code
    // (compiled if needed, loaded), occupancy figures and the SM topology
    if (p->kernel == SKC_KERNEL_JIT) {
        std::string msg;
        const int r = jit_prepare(p->jit, dev, &msg);
        if (r != SKC_OK) return fail(skc_status(r), "JIT prepare: %s", msg.c_str());
        // GPC-major SM order (once per device; the probe uses this workspace as scratch and
        // synchronises `stream`), written into the workspace's vid table
        int *scratch = reinterpret_cast<int *>(static_cast<char *>(d_ws) + jit_probe_offset(p->jit));
        const std::vector<uint16_t> &v = sm_gpc_order(dev, scratch, jit_probe_ints(), st);
        uint16_t *vid = reinterpret_cast<uint16_t *>(p->image.data() + jit_vid_offset(p->jit));
        for (size_t i = 0; i < jit_vid_cap(); ++i) vid[i] = i < v.size() ? v[i] : uint16_t(i);
        jit_set_vid(p->jit, !v.empty() && v.size() <= jit_vid_cap());
    } else if (p->kernel == SKC_KERNEL_REGTILE) {
        e = prepare_regtile(p->rsh);
    } else if (p->kernel == SKC_KERNEL_SPMDM) {
        e = prepare_spmdm(p->sp_LC, p->sp_RWM, p->smem);
    } else {
        e = prepare_direct(p->T, p->M);
    }
    if (e != cudaSuccess) return fail(SKC_ERR_CUDA, "kernel attributes: %s", cudaGetErrorString(e));
    e = cudaMemcpyAsync(d_ws, p->image.data(), p->image.size(), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return fail(SKC_ERR_CUDA, "upload: %s", cudaGetErrorString(e));
    p->d_ws = d_ws;
    return ok();
}

skc_status skc_pad_input(const skc_plan *p, const float *d_in, float *d_pad, int N,
                         void *stream) {
    if (!p) return fail(SKC_ERR_ARG, "NULL plan");
    if (N < 0) return fail(SKC_ERR_ARG, "N = %d < 0", N);
    if (N == 0) return ok();
    if (!d_in || !d_pad) return fail(SKC_ERR_ARG, "NULL device pointer");
    if (!aligned16(d_in) || !aligned16(d_pad))
        return fail(SKC_ERR_ALIGN, "device pointers must be 16-byte aligned");
    if (p->layout == SKC_LAYOUT_RAW) {  // the kernel pads while staging: a copy at most
        if (d_in == d_pad) return ok();
        cudaError_t e = cudaMemcpyAsync(d_pad, d_in, size_t(N) * p->C * p->H * p->W * 4,
                                        cudaMemcpyDeviceToDevice, (cudaStream_t)stream);
        if (e != cudaSuccess) return fail(SKC_ERR_CUDA, "raw copy: %s", cudaGetErrorString(e));
        return ok();
    }
    cudaError_t e = p->layout == SKC_LAYOUT_PAIRS
                        ? launch_pad_pairs(d_in, d_pad, N, p->C, p->H, p->W, p->pad, (cudaStream_t)stream)
                        : launch_pad(d_in, d_pad, N, p->C, p->H, p->W, p->pad, (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(SKC_ERR_CUDA, "pad launch: %s", cudaGetErrorString(e));
    return ok();
}

skc_status skc_im2col_ex(const skc_plan *p, const float *d_in, float *d_lowered, int N,
                         int layout, void *stream) {
    if (!p) return fail(SKC_ERR_ARG, "NULL plan");
    if (layout != SKC_LAYOUT_NCHW && layout != SKC_LAYOUT_PAIRS)
        return fail(SKC_ERR_ARG, "im2col layout %d: NCHW (0) or PAIRS (1)", layout);
    if (layout == SKC_LAYOUT_PAIRS && (!aligned16(d_in) || !aligned16(d_lowered)))
        return fail(SKC_ERR_ALIGN, "device pointers must be 16-byte aligned");
    if (N < 0) return fail(SKC_ERR_ARG, "N = %d < 0", N);
    if (N == 0) return ok();
    if (!d_in || !d_lowered) return fail(SKC_ERR_ARG, "NULL device pointer");
    if (int64_t(p->C) * p->R * p->S * p->Ho * p->Wo >= (int64_t(1) << 31))
        return fail(SKC_ERR_OVERFLOW, "lowered image does not fit int32 indexing");
    cudaError_t e = layout == SKC_LAYOUT_PAIRS
                        ? launch_im2col_pairs(d_in, d_lowered, N, p->C, p->H, p->W, p->R, p->S,
                                              p->stride, p->pad, p->Ho, p->Wo, (cudaStream_t)stream)
                        : launch_im2col(d_in, d_lowered, N, p->C, p->H, p->W, p->R, p->S,
                                        p->stride, p->pad, p->Ho, p->Wo, (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(SKC_ERR_CUDA, "im2col launch: %s", cudaGetErrorString(e));
    return ok();
}

skc_status skc_im2col(const skc_plan *p, const float *d_in, float *d_lowered, int N,
                      void *stream) {
    return skc_im2col_ex(p, d_in, d_lowered, N, SKC_LAYOUT_NCHW, stream);
}

static skc_status forward_epi(const skc_plan *p, const float *d_in, float *d_out, int N,
                              const float *d_bias, int relu, int out_pad, int olay, void *stream);

skc_status skc_sparse_conv_forward_ex(const skc_plan *p, const float *d_in, float *d_out,
                                      int N, const float *d_bias, int relu, int out_pad,
                                      void *stream) {
    return forward_epi(p, d_in, d_out, N, d_bias, relu, out_pad, SKC_LAYOUT_NCHW, stream);
}

skc_status skc_sparse_conv_forward_into(const skc_plan *p, const float *d_in,
                                        const skc_plan *next, float *d_next_in, int N,
                                        const float *d_bias, int relu, void *stream) {
    if (!p || !next) return fail(SKC_ERR_ARG, "NULL plan");
    if (next->C != p->K || next->H != p->Ho || next->W != p->Wo)
        return fail(SKC_ERR_GEOMETRY, "next plan expects C=%d H=%d W=%d, this layer gives %d x %d x %d",
                    next->C, next->H, next->W, p->K, p->Ho, p->Wo);
    if (next->layout == SKC_LAYOUT_RAW)  // unpadded NCHW
        return forward_epi(p, d_in, d_next_in, N, d_bias, relu, 0, SKC_LAYOUT_NCHW, stream);
    return forward_epi(p, d_in, d_next_in, N, d_bias, relu, next->pad, next->layout, stream);
}

static skc_status forward_epi(const skc_plan *p, const float *d_in, float *d_out, int N,
                              const float *d_bias, int relu, int out_pad, int olay, void *stream) {
    if (!p) return fail(SKC_ERR_ARG, "NULL plan");
    if (out_pad < 0 || out_pad > 64) return fail(SKC_ERR_ARG, "out_pad = %d outside [0, 64]", out_pad);
    if (relu != 0 && relu != 1) return fail(SKC_ERR_ARG, "relu must be 0 or 1");
    const Epilogue epi{d_bias, relu, out_pad, olay};
    if (N < 0) return fail(SKC_ERR_ARG, "N = %d < 0", N);
    if (!p->d_ws) return fail(SKC_ERR_STATE, "plan not uploaded (call skc_plan_upload)");
    if (N == 0) return ok();
    if (!d_in || !d_out) return fail(SKC_ERR_ARG, "NULL device pointer");
    if (!aligned16(d_in) || !aligned16(d_out))
        return fail(SKC_ERR_ALIGN, "device pointers must be 16-byte aligned");
    const uint8_t *ws = static_cast<const uint8_t *>(p->d_ws);
    if (p->kernel == SKC_KERNEL_JIT) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || !jit_ready(p->jit, dev))
            return fail(SKC_ERR_STATE, "JIT plan not uploaded on the current device");
        std::string msg;
        cudaError_t e = jit_launch(p->jit, d_in, d_out, ws, N, epi, (cudaStream_t)stream, &msg);
        if (e != cudaSuccess)
            return fail(SKC_ERR_CUDA, "JIT conv launch: %s %s", cudaGetErrorString(e), msg.c_str());
        return ok();
    }
    if (p->kernel == SKC_KERNEL_SPMDM) {
        if (N > 65535) return fail(SKC_ERR_ARG, "N = %d > 65535 for the SpMDM kernel", N);
        SpmdmParams sp = p->sp;
        sp.X = d_in;
        sp.Y = d_out;
        sp.meta = ws + p->off_meta;
        sp.blk = reinterpret_cast<const int64_t *>(ws + p->off_blk);
        sp.trow = reinterpret_cast<const int32_t *>(ws + p->off_trow);
        sp.epi = epi;
        cudaError_t e = launch_spmdm(sp, p->sp_LC, p->sp_RWM, p->sp_NW, N, p->smem, (cudaStream_t)stream);
        if (e != cudaSuccess) return fail(SKC_ERR_CUDA, "spmdm launch: %s", cudaGetErrorString(e));
        return ok();
    }
    if (p->kernel == SKC_KERNEL_REGTILE) {
        RegtileParams rp = p->rp;
        rp.N = N;
        rp.in = d_in;
        rp.out = d_out;
        rp.stream = reinterpret_cast<const uint2 *>(ws + p->off_stream);
        rp.segoff = reinterpret_cast<const int32_t *>(ws + p->off_segoff);
        rp.chan = reinterpret_cast<const int32_t *>(ws + p->off_chan);
        rp.lanemap = reinterpret_cast<const int32_t *>(ws + p->off_lanemap);
        rp.epi = epi;
        cudaError_t e = launch_regtile(rp, p->rsh, p->smem, (cudaStream_t)stream);
        if (e != cudaSuccess)
            return fail(SKC_ERR_CUDA, "regtile launch: %s", cudaGetErrorString(e));
        return ok();
    }
    DirectParams dp = p->dp;
    dp.N = N;
    dp.in = d_in;
    dp.out = d_out;
    dp.stream = reinterpret_cast<const uint2 *>(ws + p->off_stream);
    dp.segptr = reinterpret_cast<const int32_t *>(ws + p->off_segoff);
    dp.chan = reinterpret_cast<const int32_t *>(ws + p->off_chan);
    dp.slotq = reinterpret_cast<const int32_t *>(ws + p->off_lanemap);
    dp.slotout = reinterpret_cast<const int32_t *>(ws + p->off_chunkptr);
    dp.epi = epi;
    cudaError_t e = launch_direct(dp, p->T, p->smem, (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(SKC_ERR_CUDA, "conv launch: %s", cudaGetErrorString(e));
    return ok();
}

skc_status skc_sparse_conv_forward(const skc_plan *p, const float *d_in, float *d_out, int N,
                                   void *stream) {
    return skc_sparse_conv_forward_ex(p, d_in, d_out, N, nullptr, 0, 0, stream);
}

skc_status skc_forward_host(const skc_plan *p, const float *h_in, float *h_out, int N,
                            float *d_in, float *d_pad, float *d_out, void *stream) {
    if (!p) return fail(SKC_ERR_ARG, "NULL plan");
    if (N < 0) return fail(SKC_ERR_ARG, "N = %d < 0", N);
    if (N == 0) return ok();
    if (!h_in || !h_out || !d_in || !d_pad || !d_out) return fail(SKC_ERR_ARG, "NULL pointer");
    if (!p->d_ws) return fail(SKC_ERR_STATE, "plan not uploaded (call skc_plan_upload)");
    // Pipeline over image chunks: H2D of chunk i+1 and D2H of chunk i-1 (two copy streams)
    // overlap pad + conv of chunk i on the caller's stream; the caller's stream finally
    // waits for the last D2H, so completion semantics are those of one stream.
    cudaStream_t st = (cudaStream_t)stream;
    const size_t in_img = size_t(p->C) * p->H * p->W;
    const size_t pad_img = p->layout == SKC_LAYOUT_RAW ? in_img : size_t(p->C) * p->Hp * p->Wp;
    const size_t out_img = size_t(p->K) * p->Ho * p->Wo;
    // chunks: a few per call, whole images, >= 8 images each
    int max_chunks = 8;  // SKC_HOST_CHUNKS: pipeline depth (tuning)
    if (const char *e = std::getenv("SKC_HOST_CHUNKS")) max_chunks = std::max(1, std::atoi(e));
    int nchunk = std::max(1, std::min(max_chunks, N / 8));
    int per = (N + nchunk - 1) / nchunk;
    if (p->layout == SKC_LAYOUT_PAIRS) per += per & 1;  // chunks start on an image pair
    nchunk = (N + per - 1) / per;
    cudaStream_t s_in = nullptr, s_out = nullptr;
    std::vector<cudaEvent_t> ev(size_t(2 * nchunk + 2), nullptr);
    cudaError_t e = cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking);
    for (auto &x : ev)
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
    skc_status result = SKC_OK;
    if (e != cudaSuccess) result = fail(SKC_ERR_CUDA, "forward_host setup: %s", cudaGetErrorString(e));
    // order the copies after whatever the caller already queued on its stream
    if (result == SKC_OK) {
        e = cudaEventRecord(ev[size_t(2 * nchunk)], st);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s_in, ev[size_t(2 * nchunk)], 0);
        if (e != cudaSuccess) result = fail(SKC_ERR_CUDA, "forward_host: %s", cudaGetErrorString(e));
    }
    for (int c = 0; c < nchunk && result == SKC_OK; ++c) {
        const int n0 = c * per, n = std::min(per, N - n0);
        e = cudaMemcpyAsync(d_in + n0 * in_img, h_in + n0 * in_img, n * in_img * 4,
                            cudaMemcpyHostToDevice, s_in);
        if (e == cudaSuccess) e = cudaEventRecord(ev[size_t(2 * c)], s_in);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev[size_t(2 * c)], 0);
        if (e != cudaSuccess) { result = fail(SKC_ERR_CUDA, "H2D: %s", cudaGetErrorString(e)); break; }
        result = skc_pad_input(p, d_in + n0 * in_img, d_pad + n0 * pad_img, n, stream);
        if (result == SKC_OK)
            result = skc_sparse_conv_forward(p, d_pad + n0 * pad_img, d_out + n0 * out_img, n, stream);
        if (result != SKC_OK) break;
        e = cudaEventRecord(ev[size_t(2 * c + 1)], st);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s_out, ev[size_t(2 * c + 1)], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(h_out + n0 * out_img, d_out + n0 * out_img, n * out_img * 4,
                                cudaMemcpyDeviceToHost, s_out);
        if (e != cudaSuccess) { result = fail(SKC_ERR_CUDA, "D2H: %s", cudaGetErrorString(e)); break; }
    }
    if (s_out) {
        // the caller's stream completes only after the last D2H
        cudaError_t e2 = cudaEventRecord(ev[size_t(2 * nchunk + 1)], s_out);
        if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(st, ev[size_t(2 * nchunk + 1)], 0);
        if (e2 != cudaSuccess && result == SKC_OK)
            result = fail(SKC_ERR_CUDA, "forward_host join: %s", cudaGetErrorString(e2));
    }
    for (auto &x : ev)
        if (x) cudaEventDestroy(x);  // deferred by the runtime until the event completes
    if (s_in) cudaStreamDestroy(s_in);
    if (s_out) cudaStreamDestroy(s_out);
    return result == SKC_OK ? ok() : result;
}

int64_t skc_layout_offset(const skc_plan *p, int c, int y, int x) {
    if (!p || c < 0 || c >= p->C || y < 0 || y >= p->Hp || x < 0 || x >= p->Wp) return -1;
    return (int64_t(c) * p->Hp + y) * p->Wp + x;
}

void skc_plan_destroy(skc_plan *p) { delete p; }

// ---------------------------------------------------------------------------------------
// a7: roofline model
// ---------------------------------------------------------------------------------------
skc_status skc_model_layer_cost(int K, int C, int R, int S, int H, int W, int stride, int pad,
                                int groups, int64_t batch, int amortised, skc_layer_cost *out) {
    if (!out) return fail(SKC_ERR_ARG, "NULL output");
    if (batch < 1) return fail(SKC_ERR_ARG, "batch < 1");
    skc_status st = check_geometry(K, C, R, S, H, W, stride, pad, groups);
    if (st != SKC_OK) return st;
    const double Ho = (H + 2 * pad - R) / stride + 1, Wo = (W + 2 * pad - S) / stride + 1;
    const double b = double(batch);
    out->C = 2.0 * K * (C / groups) * R * S * Ho * Wo * b;
    out->S_A = 4.0 * b * (double(C) * H * W + K * Ho * Wo);
    out->S_W = 4.0 * K * (C / groups) * R * S * (amortised ? 1.0 : b);
    return ok();
}

skc_status skc_model_project(const skc_layer_cost *c, double x, const skc_platform *pf,
                             skc_projection *o) {
    if (!c || !pf || !o) return fail(SKC_ERR_ARG, "NULL argument");
    if (!(x > 0.0)) return fail(SKC_ERR_ARG, "density x must be > 0");
    if (!(pf->F > 0) || !(pf->B > 0) || !(pf->alpha > 0))
        return fail(SKC_ERR_ARG, "platform F, B, alpha must be > 0");
    o->t_dense = c->C / pf->F;
    o->t_sparse_compute = pf->alpha * x * c->C / pf->F;
    o->t_sparse_bw = (c->S_A + pf->beta * x * c->S_W) / pf->B;
    o->t_sparse = std::max(o->t_sparse_compute, o->t_sparse_bw);
    o->speedup = o->t_dense / o->t_sparse;
    o->effective_flops = c->C / o->t_sparse;
    o->actual_flops = x * c->C / o->t_sparse;
    return ok();
}

skc_status skc_model_window(const skc_layer_cost *c, const skc_platform *pf, skc_window *o) {
    if (!c || !pf || !o) return fail(SKC_ERR_ARG, "NULL argument");
    if (!(pf->F > 0) || !(pf->B > 0) || !(pf->alpha > 0))
        return fail(SKC_ERR_ARG, "platform F, B, alpha must be > 0");
    o->x_hi = 1.0 / pf->alpha;
    const double denom = pf->alpha * c->C * pf->B / pf->F - pf->beta * c->S_W;
    if (denom <= 0.0) {
        o->x_lo = std::numeric_limits<double>::infinity();
        o->has_speedup_potential = 0;
        return ok();
    }
    o->x_lo = c->S_A / denom;
    skc_projection pr;
    skc_model_project(c, std::min(o->x_lo, 1.0), pf, &pr);
    o->has_speedup_potential = (o->x_lo < o->x_hi && pr.speedup > 1.0) ? 1 : 0;
    return ok();
}


skc_status skc_bench_ffma(void *d_scratch, int blocks, int iters, double *ms, double *flops) {
    return bench_call(bench_ffma, "bench_ffma", d_scratch, blocks, iters, ms, flops);
}

skc_status skc_bench_ffma2(void *d_scratch, int blocks, int iters, double *ms, double *flops) {
    return bench_call(bench_ffma2, "bench_ffma2", d_scratch, blocks, iters, ms, flops);
}

skc_status skc_bench_lds(void *d_scratch, int blocks, int iters, double *ms, double *bytes) {
    return bench_call(bench_lds, "bench_lds", d_scratch, blocks, iters, ms, bytes);
}

skc_status skc_bench_lds64(void *d_scratch, int blocks, int iters, double *ms, double *bytes) {
    return bench_call(bench_lds64, "bench_lds64", d_scratch, blocks, iters, ms, bytes);
}

}  // extern "C"
