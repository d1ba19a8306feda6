// jit.cpp -- rows a3..a6, "compiled weights" variant of direct sparse convolution.
//
// Same computation as Fig. 2:  out[k][y][x] += w * in[f(c,r,s) + f(0,y,x)]
// for every nonzero w = W(k,c,r,s), accumulated in CSR order.  The sparse matrix is known
// before the layer runs ("pre-computed"), so instead of walking a (w, off)
// stream at run time, the plan emits the walk itself as straight-line sm_100a code:
//
//   for each input channel c (ascending; staged CB at a time in shared memory by TMA):
//       load the lane's input-window positions that the block's nonzeros at c touch:
//           ld.shared [lane base + f(c, y, x)]        -- f folded into an immediate
//       for each nonzero (m, r, s, w) of the block's M output channels at c, in CSR order:
//           acc[m][ty][tx] += w * win[ty + r][tx + s]  -- FFMA2 (fma.rn.f32x2) with w as an
//                                                         immediate, two pixels per instruction
//
// Each lane owns a TY x TX output tile (register blocking of the y, x loops,
// PAPER.md:309-310) for M output channels; pixels tx and tx + PX share one packed FFMA2, so
// the window is held as register pairs (win[u], win[u + PX]) and every (r, s) shift of the
// tile is an aligned pair.  There is no per-nonzero dispatch, no weight or offset load and
// no address arithmetic in the inner code: the instruction stream is FFMA2 + window loads.
// Straight-line code does not fit the instruction cache, so B200 runs it at the
// instruction-fetch rate; the design therefore minimises instructions per MAC: packed pairs
// (64 MACs per warp instruction), needed-only window loads, volatile (CSE-free) pair loads
// so no register moves are needed to build pairs.
//
// Code layout: one PTX module per channel block (a .func holding the block's whole walk and
// its epilogue), compiled in parallel with the PTX compiler library and linked by nvJitLink
// with an entry module (stage setup, lane tables, dispatch on the CTA's block) -- or, for
// moderate code, all of it as one whole-program module.  Loaded with cudaLibraryLoadData at
// the first launch, launched with cudaLaunchKernelExC.
//
// Map of this file (DESIGN.md Sec. 7.4 has the measurements behind each choice):
//   emit_block   a block's code: image-pair window loads in position-major order, immediate-
//                weight FFMA2, the staging ring's waits / last-warp-out TMA refills (or raw
//                cp.async staging), bias-free and general epilogues, the dry-run entry points
//   emit_entry   the persistent CTA loop: item numbering (cluster rank or GPC-major via the
//                topology table), work order (first round spread / block-major), static or
//                dynamic (counter) scheduling, per-item barrier / slot-table setup, dispatch
//   jit_configure  the configuration search (tile, channels per block, warps, bands, staging)
//                under the cost model, whole-round costing, block partition / tail split
//   jit_verify   decodes the emitted PTX back to the CSR (independent of the generator)
//   jit_compile / jit_launch / jit_tune  build (cached), launch, and launch-schedule tuning
#include "skc.h"
#include "skc_internal.h"

#include <dlfcn.h>
#include <nvJitLink.h>
#include <nvPTXCompiler.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <queue>
#include <string>
#include <sys/stat.h>
#include <thread>
#include <unistd.h>
#include <vector>

namespace skc {

namespace {

constexpr int kMaxSmem = 227 * 1024;
constexpr int kStageTarget = 72 * 1024;
constexpr int kStage2Max = 108 * 1024;    // stage bytes when only 2 stages are used
constexpr double kChunkInstr = 1000.0;   // minimum instructions per warp per chunk
constexpr double kWholeMaxInstr = 1.2e5; // largest code compiled as one whole program
// cost model (clk per image): unique-code fetch ~0.12 instr/clk/SM, shared by the CTA's warps;
// issue ~1.6 warp-instr/clk/SM (fitted to the B200 sweeps in profiles/r01_jit_*.jsonl)
constexpr double kFetchInv = 1.0 / 0.12;
constexpr double kIssue = 1.6;
// ... times a penalty for the number of distinct block codes the 148 SMs run at once (the
// L1.5 instruction cache is per GPC; microbenchmarks: 1 code 33 TF, 2-4 codes 22-24 TF), plus
// a fixed cost per CTA work item (stage set-up, first TMA round trip, epilogue); fitted to
// profiles/r01_jit_cfg_sweep.jsonl
constexpr double kItemCycles = 4000.0;
constexpr int kSMs = 148;
// position-major code keeps few window positions live: registers the configuration reserves
// for them (pair layout; profiles/r01_jit_pmajor.txt)
constexpr int kPmajorWregs = 8;
double conc_penalty(int conc) {
    static const double pen[] = {1.0, 1.0, 1.2, 1.45, 1.5};
    return conc < 5 ? pen[conc] : 1.6;
}
constexpr int kJitVersion = 21;  // bump when the generated code changes (cache key)
// workspace regions after the lane / staging tables: the GPC-major SM order (vid[smid],
// kVidCap u16, written by skc_plan_upload), the first-item claim table (kVidCap u32, zero
// between launches), and scratch for the SM-topology probe (kProbeInts int32)
constexpr int kVidCap = 1024;
constexpr int kProbeInts = 4096;

// Fast appender for the (large) generated PTX.
struct Out {
    std::string s;
    void operator()(const char *fmt, ...) __attribute__((format(printf, 2, 3))) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        const int n = vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        if (n >= int(sizeof buf)) {  // long line (e.g. a parameter list): format again
            std::vector<char> big(size_t(n) + 1);
            va_start(ap, fmt);
            vsnprintf(big.data(), big.size(), fmt, ap);
            va_end(ap);
            s.append(big.data(), size_t(n));
        } else {
            s.append(buf, size_t(std::max(0, n)));
        }
        s.push_back('\n');
    }
};

uint32_t fbits(float v) {
    uint32_t u;
    std::memcpy(&u, &v, 4);
    return u;
}

uint64_t fnv1a(const void *data, size_t n, uint64_t h = 1469598103934665603ull) {
    const uint8_t *p = static_cast<const uint8_t *>(data);
    for (size_t i = 0; i < n; ++i) h = (h ^ p[i]) * 1099511628211ull;
    return h;
}

// One nonzero of a block at one input channel: output-channel slot m, tap (r, s), weight.
struct JNz {
    int m, r, s;
    float w;
};

}  // namespace

struct JitPlan {
    JitInput in{};
    // configuration
    int TY = 0, TX = 0, PX = 0;  // lane tile; pixel pairs (tx, tx + PX) for tx < PX
    int pair = 0;                // 1: image-pair interleaved input layout, FFMA2 over 2 images
    int M = 0, NW = 0, NI = 0, CB = 0, NS = 0, nchunks = 0;
    int tiles_y = 0, tiles_x = 0;
    int NB = 1;                  // row bands: a work item covers tile rows of one band
                                 // (lane table per band) -- pair mode on large images
    int plane = 0, img_stride = 0, stage_bytes = 0;
    int off_bar = 0, off_cnt = 0, off_info = 0, off_item = 0;
    size_t smem = 0;
    int maxreg = 255;          // register cap of the block functions (NW warps per SM)
    int sync_every = 0;        // FMA instructions between CTA barriers in the code (0: none)
    int l2hint = 3;            // bit 0: streaming (.cs) output stores, bit 1: evict-first TMA
                               // loads -- the activations do not push the code out of L2
    // work-item order: 0 block-major, 1 spread (blocks interleaved), 2 first round spread then
    // block-major.  2: every block's (cold, DRAM-resident) code is fetched in parallel by the
    // first round, later rounds share one code stream chip-wide (profiles/r01_jit_order.txt)
    int order = 2;
    int dry = 1;               // 1: instruction prefetch by dry-running code segments at start
    int pmajor = 1;            // 1: position-major FMA order within a channel (pair layout)
    int lookahead = 0;         // position-major: window loads issued this many positions ahead
    // 1: an item's last chunks stage the next item's first chunks (rotated stages, barriers
    // live across items).  Measured -1..-2% on conv3/4 (profiles/r01_jit_xpf.txt): the item
    // start was not waiting on its first stage; off by default
    int xpf = 0;
    // raw staging (SKC_JIT_RAW): the kernel reads the unpadded NCHW input; every thread
    // cp.async-copies its fixed input positions (stab) of each chunk into the padded,
    // pair-interleaved stage, whose halo is zeroed once -- no pad pass
    int raw = 0;
    int kmax = 0;                  // staged positions per thread per (slot, channel)
    std::vector<uint32_t> stab;    // [NB][NW*32][kmax][2]: raw offset (img*C*H*W + y*W + x, or
                                   // ~0 = none), stage offset (((y+pad)*Wp + x+pad)*2 + img)
    // launch schedule chosen by jit_tune (-1: default): first round block-major (order 3),
    // GPC-major item numbers, cluster size
    std::atomic<int> t_order3{-1}, t_vid{-1}, t_cs{-1}, t_nodry{-1}, t_lanes{-1}, t_dryall{-1};
    int dyn = 1;               // dynamic item scheduling (global counter in the workspace):
                               // 1 per CTA, 2 per cluster; 0: static (t += grid)
    int whole = 0;             // 1: whole-program compile (no ABI saves at block calls)
    // 1: non-persistent kernel (one work item per CTA, block functions .noreturn and compiled
    // as separate modules in parallel -- no ABI saves either, seconds to build) plus a
    // separate dry-run prefetch kernel (skc_jit_dry)
    int np = 0;
    int np_ret = 0;            // debug (SKC_JIT_NP_RET=1): np, but block functions return
    double code_instr = 0;     // modelled instructions of all blocks' code
    int nbg = 0, nblocks = 0;  // blocks per group (even partition), total blocks
    // block b: conv group, first index into the group's nnz-sorted channels, channel count.
    // Blocks are numbered longest-first; the last ones may be halves of an even block (tail
    // split: the short items fill the last round of the persistent grid)
    std::vector<int> bgrp;
    std::vector<std::vector<int>> bidx;  // positions in the group's nnz-sorted channel list
    int split = 0;             // even blocks (per group) split into halves
    int deal = 0;              // 1: channels dealt to blocks in snake order (skewed masks)
    double cost = 0;           // modelled warp-instructions per image
    int conflict = 0;          // extra wavefronts per warp-wide window load, summed over warps
    std::vector<int32_t> chan; // [nblocks][M] original output channel or -1
    std::vector<uint32_t> lanemap;  // [NB][NW*32][4]: lane smem byte base, pos, store mask, idle
    // second lane table, tiles dealt to lanes row-major (a warp stores runs of consecutive
    // pixels; bank conflicts accepted): chosen per launch by skc_plan_tune (sched bit 3)
    std::vector<uint32_t> lanemap_c;
    // compiled code
    std::vector<char> cubin;
    uint64_t key = 0;
    bool compiled = false;
    double compile_s = 0;
    int cache_hit = 0;
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kern = nullptr;
    cudaKernel_t kern_dry = nullptr;  // np mode: the dry-run prefetch kernel
    // device state taken by jit_prepare (skc_plan_upload)
    int prep_dev = -1;
    int nsm = 0, per_sm = 1;
    int ncl[17] = {0};         // max active clusters per cluster size 2/4/8/16
    bool vid_ok = false;       // the workspace holds a GPC-major SM order (topology probe)
    std::mutex mu;
};

namespace {

// ---------------------------------------------------------------------------------------
// nonzeros per block and channel
// ---------------------------------------------------------------------------------------

// Block q of group g: sorted channels perm[g*Kg + q*M ...] (nnz-descending, PAPER.md:313-314
// load balance via the plan's permutation).
void block_channels(const JitInput &in, int M, int g, int q, std::vector<int> &ks) {
    ks.clear();
    for (int m = 0; m < M; ++m) {
        const int idx = q * M + m;
        if (idx < in.Kg) ks.push_back(in.perm[size_t(g) * in.Kg + size_t(idx)]);
    }
}

// Block b of a plan (explicit partition, see JitPlan::bgrp / bidx).
void plan_block_channels(const JitInput &in, int g, const std::vector<int> &idx,
                         std::vector<int> &ks) {
    ks.clear();
    for (int i : idx) ks.push_back(in.perm[size_t(g) * in.Kg + size_t(i)]);
}

// A block's nonzeros per local input channel, in CSR order per output channel.
void block_nz(const JitInput &in, const std::vector<int> &ks,
              std::vector<std::vector<JNz>> &per_c) {
    per_c.assign(size_t(in.Cg), {});
    const int64_t plane = int64_t(in.Hp) * in.Wp;
    for (size_t m = 0; m < ks.size(); ++m) {
        const int k = ks[m];
        const int64_t gbase = int64_t(k / in.Kg) * in.Cg * plane;
        for (int32_t j = in.rowptr[k]; j < in.rowptr[k + 1]; ++j) {
            const int64_t off = in.colidx[j] - gbase;
            const int cl = int(off / plane);
            const int rem = int(off % plane);
            per_c[size_t(cl)].push_back(JNz{int(m), rem / in.Wp, rem % in.Wp, in.values[j]});
        }
    }
}

// Window positions (wy * WCw + wx, relative to the lane's tile origin) a channel's
// nonzeros touch.  Canonical layout (sw = 1): `pairs` are loaded as (win[u], win[u + PX*st])
// register pairs (pixels tx, tx + PX share an FFMA2), `scalars` (the odd column of an
// odd-width tile) only where no pair half already holds them.  Pair layout (sw = 2): every
// position u is one 8-byte load of (image A, image B), `pairs` lists them.
struct Need {
    std::vector<int> pairs, scalars;
    std::vector<uint32_t> stamp_p, stamp_s;
    uint32_t gen = 0;
    void reset(size_t n) {
        if (stamp_p.size() < n) {
            stamp_p.assign(n, 0);
            stamp_s.assign(n, 0);
            gen = 0;
        }
        ++gen;
        pairs.clear();
        scalars.clear();
    }
};

void window_need(const std::vector<JNz> &nz, int TY, int TX, int PX, int st, int WRw, int WCw,
                 bool pairmode, Need &nd) {
    nd.reset(size_t(WRw) * WCw);
    for (const JNz &z : nz)
        for (int ty = 0; ty < TY; ++ty) {
            const int row = (ty * st + z.r) * WCw;
            const int np = pairmode ? TX : PX;
            for (int q = 0; q < np; ++q) {
                const int u = row + q * st + z.s;
                if (nd.stamp_p[size_t(u)] != nd.gen) {
                    nd.stamp_p[size_t(u)] = nd.gen;
                    nd.pairs.push_back(u);
                }
            }
            if (pairmode) continue;
            for (int tx = 2 * PX; tx < TX; ++tx) {
                const int v = row + tx * st + z.s;
                if (nd.stamp_s[size_t(v)] != nd.gen) {
                    nd.stamp_s[size_t(v)] = nd.gen;
                    nd.scalars.push_back(v);
                }
            }
        }
    std::sort(nd.pairs.begin(), nd.pairs.end());
    std::sort(nd.scalars.begin(), nd.scalars.end());
    // scalars already held as the low or high half of a loaded pair need no load
    std::vector<int> keep;
    for (int v : nd.scalars) {
        const bool lo = nd.stamp_p[size_t(v)] == nd.gen;
        const bool hi = (v % WCw) >= PX * st && nd.stamp_p[size_t(v - PX * st)] == nd.gen;
        if (!lo && !hi) keep.push_back(v);
    }
    nd.scalars.swap(keep);
}

int window_regs(int TY, int TX, int PX, int R, int S, int st, bool pairmode) {
    const int rows = (TY - 1) * st + R;
    if (pairmode) return rows * ((TX - 1) * st + S) * 2;
    if (PX == 0) return rows * ((TX - 1) * st + S);
    const int npc = (PX - 1) * st + S;
    return rows * (2 * npc + (TX > 2 * PX ? st + 1 : 0));
}

// Register cap per thread for NW warps on one SM: warps are spread over the 4 SM
// sub-partitions, each with a 16K-register file, so ceil(NW/4) * regs * 32 <= 16384.
int reg_cap(int NW) {
    const int per = 16384 / (32 * ((NW + 3) / 4));
    return per >= 256 ? 255 : (per & ~7);
}

// FMA instructions per nonzero for one lane's tile.
int fma_per_nz(int TY, int TX, int PX, bool pairmode) {
    return pairmode ? TY * TX : TY * (PX + (TX - 2 * PX));
}

// Modelled warp-instructions of one block's code (per CTA pass).
double block_instr(const JitInput &in, const std::vector<std::vector<JNz>> &per_c, int TY,
                   int TX, int PX, bool pairmode, int CB, int Mb, Need &nd) {
    const int st = in.stride, WRw = (TY - 1) * st + in.R, WCw = (TX - 1) * st + in.S;
    double n = 0;
    for (int c = 0; c < in.Cg; ++c) {
        const auto &nz = per_c[size_t(c)];
        if (nz.empty()) continue;
        window_need(nz, TY, TX, PX, st, WRw, WCw, pairmode, nd);
        n += double(nz.size()) * fma_per_nz(TY, TX, PX, pairmode);
        n += (pairmode ? 1.0 : 2.0) * double(nd.pairs.size()) + double(nd.scalars.size());
    }
    n += ((in.Cg + CB - 1) / CB) * 14.0;
    n += Mb * (TY * TX * (pairmode ? 9.0 : 5.0) + TY * 3.0);
    return n;
}

// ---------------------------------------------------------------------------------------
// lane assignment: the tiles of the slots (images, or image pairs in pair mode) onto NW
// warps x 32 lanes, first fit by shared-memory bank residue of the lane base, so that a
// warp's window load (one immediate offset for all lanes) touches distinct banks: 32 lanes x
// 4-byte words, or (pair mode) each half-warp's 16 lanes x 8-byte words
// ---------------------------------------------------------------------------------------
struct Tile {
    int slot, y0, x0, ry0, rx0;  // origin (shifted back inside the image), nominal origin
};

// Tile rows of band b of NB: [b*tiles_y/NB, (b+1)*tiles_y/NB).
int band_lo(int tiles_y, int NB, int b) { return int((int64_t(b) * tiles_y) / NB); }

int assign_lanes(const JitPlan &jp, int IS, int band, uint32_t *lanemap, int lanes_mode = 0) {
    const JitInput &in = jp.in;
    const int st = in.stride, sw = jp.pair ? 2 : 1;
    const int nslot = jp.NI / sw;
    std::vector<Tile> tiles;
    const int iy0 = band_lo(jp.tiles_y, jp.NB, band), iy1 = band_lo(jp.tiles_y, jp.NB, band + 1);
    for (int j = 0; j < nslot; ++j)
        for (int iy = iy0; iy < iy1; ++iy)
            for (int ix = 0; ix < jp.tiles_x; ++ix) {
                const int ry = iy * jp.TY, rx = ix * jp.TX;
                tiles.push_back(
                    Tile{j, std::min(ry, in.Ho - jp.TY), std::min(rx, in.Wo - jp.TX), ry, rx});
            }
    // lane base in floats, and its bank residue in units of the load width
    std::vector<int> base(tiles.size()), res(tiles.size());
    const int groups = jp.pair ? 2 : 1, glanes = 32 / groups, nres = 32 / sw;
    for (size_t i = 0; i < tiles.size(); ++i) {
        base[i] = tiles[i].slot * IS + (tiles[i].y0 * st * in.Wp + tiles[i].x0 * st) * sw;
        res[i] = (base[i] / sw) % nres;
    }
    std::vector<char> used(tiles.size(), 0);
    std::vector<int> lane_tile(size_t(jp.NW) * 32, -1);
    size_t left = tiles.size();
    int extra = 0;
    const int ngroups = jp.NW * groups;
    if (lanes_mode == 1 && tiles.size() <= size_t(jp.NW) * 32) {
        // contiguous: lane l takes tile l (row-major), so a warp's output stores are runs of
        // consecutive pixels; the bank conflicts this costs are counted, not avoided
        for (size_t i = 0; i < tiles.size(); ++i) {
            lane_tile[i] = int(i);
            used[i] = 1;
        }
        left = 0;
        for (int gi = 0; gi < ngroups; ++gi) {
            int cnt[32] = {0}, mx = 0;
            for (int l = 0; l < glanes; ++l) {
                const int ti = lane_tile[size_t(gi) * glanes + size_t(l)];
                if (ti >= 0) mx = std::max(mx, ++cnt[res[size_t(ti)]]);
            }
            extra += std::max(0, mx - 1);
        }
    }
    for (int gi = 0; gi < ngroups && left; ++gi) {
        int cnt[32] = {0};
        int filled = 0;
        // pass 0: distinct residues only; pass 1: any tile, when the remaining lane groups
        // could not take the rest conflict-free anyway
        for (int pass = 0; pass < 2 && filled < glanes && left; ++pass) {
            if (pass == 1 && int(left) <= (ngroups - gi - 1) * glanes) break;
            for (size_t i = 0; i < tiles.size() && filled < glanes; ++i) {
                if (used[i]) continue;
                if (pass == 0 && cnt[res[i]]) continue;
                used[i] = 1;
                --left;
                ++cnt[res[i]];
                lane_tile[size_t(gi) * glanes + size_t(filled++)] = int(i);
                if (pass == 1 && int(left) <= (ngroups - gi - 1) * glanes) break;
            }
        }
        int mx = 0;
        for (int r = 0; r < nres; ++r) mx = std::max(mx, cnt[r]);
        extra += std::max(0, mx - 1);
    }
    if (left) return -1;  // does not fit
    if (lanemap) {
        std::fill(lanemap, lanemap + size_t(jp.NW) * 32 * 4, 0u);
        for (int l = 0; l < jp.NW * 32; ++l) {
            int ti = lane_tile[size_t(l)];
            const bool idle = ti < 0;
            if (idle) ti = lane_tile[size_t(l / glanes) * glanes];  // mirror the group's lane 0
            if (ti < 0) ti = lane_tile[size_t(l / 32) * 32];
            if (ti < 0) ti = 0;                                      // whole warp idle
            const Tile &t = tiles[size_t(ti)];
            uint32_t mask = 0;
            if (!idle)
                for (int ty = 0; ty < jp.TY; ++ty)
                    for (int tx = 0; tx < jp.TX; ++tx) {
                        const int y = t.y0 + ty, x = t.x0 + tx;
                        // pixels of a shifted-back tile that an earlier tile owns are
                        // computed twice but stored once
                        if (y >= t.ry0 && x >= t.rx0 && y < in.Ho && x < in.Wo)
                            mask |= 1u << (ty * jp.TX + tx);
                    }
            uint32_t *e = lanemap + size_t(l) * 4;
            e[0] = uint32_t(base[size_t(ti)]) * 4u;
            e[1] = (uint32_t(t.slot) << 24) | (uint32_t(t.y0) << 12) | uint32_t(t.x0);
            e[2] = mask;
            e[3] = idle ? 1u : 0u;
        }
    }
    return extra;
}

// ---------------------------------------------------------------------------------------
// PTX emission
// ---------------------------------------------------------------------------------------
const char *kHdr = ".version 8.8\n.target sm_100a\n.address_size 64\n";
// block function parameters: lane smem base, smem base, lane output base (image A), store
// mask (bit 31: image B valid, pair mode), slots in this item, bias, relu, output row /
// channel / pixel strides, byte offset of image B's output from image A's, dry-run chunk
// (0: a real run; k + 1: execute only chunk k's code, no waits, no stores -- instruction
// prefetch, see emit_entry), stage phase/rotation (bits 0-7: parity base of logical stage s,
// bits 8-15: rotation -- logical stage s is physical stage (s + rot) % NS), smem offsets of
// this item's and the next item's slot-source tables, the next item's slot count (0: none;
// else the last chunks' releases stage the next item's first chunks)
const char *kBlkParams =
    "(.param .b32 q_lb, .param .b32 q_sm, .param .b64 q_out, .param .b32 q_mask, "
    ".param .b32 q_nsl, .param .b64 q_bias, .param .b32 q_relu, .param .b32 q_rs, "
    ".param .b64 q_cs, .param .b32 q_ps, .param .b64 q_bo, .param .b32 q_dry, "
    ".param .b32 q_ph, .param .b32 q_info, .param .b32 q_ninfo, .param .b32 q_nnsl, "
    ".param .b64 q_gin, .param .b32 q_nimg, .param .b64 q_stab)";

int chunk_channels(const JitPlan &jp, int i) { return std::min(jp.CB, jp.in.Cg - i * jp.CB); }

// Raw staging of chunk i into (logical) stage s: every thread copies its kmax positions of
// every (slot, channel) with 4-byte cp.async (zero-filled when the image is past the batch),
// then arrives on the stage's barrier once its copies land (count = all threads).
void emit_raw_fill(Out &o, const JitPlan &jp, int i, int s) {
    const JitInput &in = jp.in;
    const int H = in.Hp - 2 * in.pad, W = in.Wp - 2 * in.pad, NSL = jp.NI / 2;
    const int cn = chunk_channels(jp, i);
    for (int j = 0; j < NSL; ++j)
        for (int cl = 0; cl < cn; ++cl)
            for (int k = 0; k < jp.kmax; ++k) {
                const long long goff =
                    ((long long)(i * jp.CB + cl) * H * W + (long long)j * 2 * in.C * H * W) * 4;
                const long long soff = ((long long)j * jp.img_stride + (long long)cl * jp.plane * 2) * 4;
                o("cp.async.ca.shared.global [%%rak%d+%lld], [%%rgk%d+%lld], 4, %%rz%d;",
                  s * jp.kmax + k, soff, k, goff, j * jp.kmax + k);
            }
    o("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%%rw%d];", s);
}

std::string emit_block(const JitPlan &jp, int b, const std::vector<int> &ks,
                       const std::vector<std::vector<JNz>> &per_c) {
    const JitInput &in = jp.in;
    const bool pm = jp.pair;
    const int sw = pm ? 2 : 1;
    const int st = in.stride, TY = jp.TY, TX = jp.TX, PX = pm ? 0 : jp.PX;
    const int WRw = (TY - 1) * st + in.R, WCw = (TX - 1) * st + in.S;
    const int NWIN = WRw * WCw;
    const int Mb = int(ks.size());
    // accumulators: pair mode -- one .b64 (image A, image B) per pixel; canonical -- pairs
    // (tx, tx + PX) as .b64 and the odd column as .f32
    const int NPT = pm ? TY * TX : TY * PX, NST = pm ? 0 : TY * (TX - 2 * PX);
    Out o;
    o.s.reserve(1 << 20);
    o("%s", kHdr);
    // np (non-persistent per-block modules): the function never returns -- it ends the thread
    // (`exit`), so a separately compiled block saves no callee-saved registers
    o(".visible .func skc_b%d%s%s", b, kBlkParams, jp.np && !jp.np_ret ? " .noreturn" : "");
    o("{");
    o(".reg .pred %%p<10>;");
    o(".reg .b32 %%r<32>;");
    o(".reg .b64 %%rd<12>;");
    o(".reg .b32 %%rb<%d>;", jp.NS);
    o(".reg .b32 %%rs<%d>;", jp.NS);
    o(".reg .b32 %%rw<%d>;", jp.NS);
    o(".reg .b32 %%rq<%d>;", 2 * jp.NS);
    o(".reg .b64 %%a<%d>;", std::max(1, Mb * NPT));
    o(".reg .f32 %%f<%d>;", std::max(1, Mb * NST));
    o(".reg .f32 %%wl<%d>;", NWIN);
    o(".reg .f32 %%wh<%d>;", NWIN);
    o(".reg .f32 %%ws<%d>;", NWIN);
    o(".reg .b64 %%wp<%d>;", NWIN);
    o(".reg .b64 %%wt;");
    o(".reg .pred %%pe<8>;");
    o(".reg .b64 %%rdp<4>;");
    if (jp.raw) {
        o(".reg .b64 %%rgin, %%rstab;");
        o(".reg .b64 %%rgk<%d>;", jp.kmax);
        o(".reg .b32 %%rgo<%d>;", jp.kmax);
        o(".reg .b32 %%rso<%d>;", jp.kmax);
        o(".reg .b32 %%rz<%d>;", (jp.NI / 2) * jp.kmax);
        o(".reg .b32 %%rak<%d>;", jp.NS * jp.kmax);
        o(".reg .b32 %%rnimg, %%rimg, %%rtt;");
        o(".reg .pred %%ppk, %%ppt;");
    }
    o(".reg .f32 %%e<4>;");
    o("ld.param.b32 %%r0, [q_lb];");
    o("ld.param.b32 %%r1, [q_sm];");
    o("ld.param.b64 %%rd0, [q_out];");
    o("ld.param.b32 %%r2, [q_mask];");
    o("ld.param.b32 %%r3, [q_nsl];");
    o("ld.param.b64 %%rd1, [q_bias];");
    o("ld.param.b32 %%r4, [q_relu];");
    o("ld.param.b32 %%r5, [q_rs];");
    o("ld.param.b64 %%rd2, [q_cs];");
    o("ld.param.b32 %%r16, [q_ps];");
    o("ld.param.b64 %%rd7, [q_bo];");
    o("mov.u32 %%r6, %%laneid;");
    o("setp.eq.u32 %%p0, %%r6, 0;");
    o("mov.u32 %%r7, 0;");
    o("mov.u32 %%r8, 1;");
    // activations stream through L2 (evict first) so the straight-line code stays resident
    if (jp.l2hint & 2) o("createpolicy.fractional.L2::evict_first.b64 %%rd10, 1.0;");
    // logical stage s = physical stage (s + rot) % NS: stage base (rs), lane base (rb),
    // barrier (rw), wait parities (rq: base, base ^ 1)
    o("ld.param.b32 %%r18, [q_ph];");
    o("ld.param.b32 %%r19, [q_info];");
    o("add.u32 %%r19, %%r19, %%r1;");
    o("ld.param.b32 %%r20, [q_ninfo];");
    o("add.u32 %%r20, %%r20, %%r1;");
    o("ld.param.b32 %%r21, [q_nnsl];");
    o("bfe.u32 %%r22, %%r18, 8, 8;");
    for (int s = 0; s < jp.NS; ++s) {
        o("add.u32 %%r23, %%r22, %d;", s);
        o("rem.u32 %%r23, %%r23, %d;", jp.NS);
        o("mad.lo.u32 %%rs%d, %%r23, %d, %%r1;", s, jp.stage_bytes);
        o("add.u32 %%rb%d, %%rs%d, %%r0;", s, s);
        o("mad.lo.u32 %%rw%d, %%r23, 8, %%r1;", s);
        o("add.u32 %%rw%d, %%rw%d, %d;", s, s, jp.off_bar);
        o("bfe.u32 %%rq%d, %%r18, %d, 1;", 2 * s, s);
        o("xor.b32 %%rq%d, %%rq%d, 1;", 2 * s + 1, 2 * s);
    }
    for (int i = 0; i < Mb * NPT; ++i) o("mov.b64 %%a%d, 0;", i);
    for (int i = 0; i < Mb * NST; ++i) o("mov.f32 %%f%d, 0f00000000;", i);
    // dry run: jump straight to chunk k's code (no barrier wait), return after it
    o("ld.param.b32 %%r17, [q_dry];");
    o("setp.ne.u32 %%p8, %%r17, 0;");
    o("@!%%p8 bra $REAL;");
    for (int i = 0; i < jp.nchunks; ++i) {
        o("setp.eq.u32 %%p9, %%r17, %d;", i + 1);
        o("@%%p9 bra $B%d;", i);
    }
    o("bra.uni $DRYRET;");
    o("$REAL:");
    if (jp.raw) {
        // this thread's staged positions (raw offset, stage offset) and per-slot copy sizes
        o("ld.param.b64 %%rgin, [q_gin];");
        o("ld.param.b32 %%rnimg, [q_nimg];");
        o("ld.param.b64 %%rstab, [q_stab];");
        for (int k = 0; k < jp.kmax; ++k) {
            o("ld.global.nc.v2.u32 {%%rgo%d, %%rso%d}, [%%rstab+%d];", k, k, 8 * k);
            o("setp.ne.u32 %%ppk, %%rgo%d, -1;", k);
            o("mul.wide.u32 %%rgk%d, %%rgo%d, 4;", k, k);
            o("add.u64 %%rgk%d, %%rgk%d, %%rgin;", k, k);
            o("and.b32 %%rimg, %%rso%d, 1;", k);
            for (int j = 0; j < jp.NI / 2; ++j) {
                o("add.u32 %%rtt, %%rimg, %d;", 2 * j);
                o("setp.lt.u32 %%ppt, %%rtt, %%rnimg;");
                o("and.pred %%ppt, %%ppt, %%ppk;");
                o("selp.u32 %%rz%d, 4, 0, %%ppt;", j * jp.kmax + k);
            }
            o("shl.b32 %%rso%d, %%rso%d, 2;", k, k);
            for (int s = 0; s < jp.NS; ++s) o("add.u32 %%rak%d, %%rs%d, %%rso%d;", s * jp.kmax + k, s, k);
        }
        for (int i = 0; i < std::min(jp.NS, jp.nchunks); ++i) emit_raw_fill(o, jp, i, i);
    }

    Need nd;
    int since_sync = 0;
    for (int i = 0; i < jp.nchunks; ++i) {
        const int s = i % jp.NS;
        const int par = (i / jp.NS) & 1;
        o("$W%d:", i);
        o("mbarrier.try_wait.parity.shared::cta.b64 %%p4, [%%rw%d], %%rq%d;", s, 2 * s + par);
        o("@!%%p4 bra $W%d;", i);
        o("$B%d:", i);
        const int cn = chunk_channels(jp, i);
        bool cn_done = false;
        if (pm && jp.pmajor && jp.lookahead > 0 && jp.sync_every == 0) {
            // position-major with software-pipelined window loads: the chunk's (channel,
            // position) sequence is flattened and position j + D is loaded before the FMAs of
            // position j, into a rotating pool of D + 1 window registers (each warp keeps D + 1
            // loads in flight).  Per accumulator the FMA order is unchanged (bitwise equal).
            struct Pos { int c, u; };
            std::vector<Pos> seq;
            for (int cl = 0; cl < cn; ++cl) {
                const int c = i * jp.CB + cl;
                const auto &nz = per_c[size_t(c)];
                if (nz.empty()) continue;
                window_need(nz, TY, TX, PX, st, WRw, WCw, pm, nd);
                for (int u : nd.pairs) seq.push_back(Pos{cl, u});
            }
            const int D = std::min(jp.lookahead, NWIN - 1);
            auto off_of = [&](const Pos &p) {
                return (p.c * jp.plane + (p.u / WCw) * in.Wp + (p.u % WCw)) * 4 * sw;
            };
            for (int j = 0; j < std::min(D, int(seq.size())); ++j)
                o("ld.volatile.shared.b64 %%wp%d, [%%rb%d+%d];", j % (D + 1), s, off_of(seq[size_t(j)]));
            for (int j = 0; j < int(seq.size()); ++j) {
                if (j + D < int(seq.size()))
                    o("ld.volatile.shared.b64 %%wp%d, [%%rb%d+%d];", (j + D) % (D + 1), s,
                      off_of(seq[size_t(j + D)]));
                const Pos &p = seq[size_t(j)];
                for (const JNz &z : per_c[size_t(i * jp.CB + p.c)])
                    for (int ty = 0; ty < TY; ++ty)
                        for (int tx = 0; tx < TX; ++tx) {
                            if ((ty * st + z.r) * WCw + tx * st + z.s != p.u) continue;
                            const uint32_t wb = fbits(z.w);
                            const int a = z.m * NPT + ty * TX + tx;
                            o("mov.b64 %%wt, 0x%08X%08X;", wb, wb);
                            o("fma.rn.f32x2 %%a%d, %%wt, %%wp%d, %%a%d;", a, j % (D + 1), a);
                        }
            }
            cn_done = true;
        }
        for (int cl = 0; cl < cn && !cn_done; ++cl) {
            const int c = i * jp.CB + cl;
            const auto &nz = per_c[size_t(c)];
            if (nz.empty()) continue;
            // optional: keep the CTA's warps in lockstep on the straight-line code
            if (jp.sync_every > 0 && since_sync >= jp.sync_every) {
                o("bar.sync 1, %d;", jp.NW * 32);
                since_sync = 0;
            }
            since_sync += int(nz.size()) * fma_per_nz(TY, TX, PX, pm);
            window_need(nz, TY, TX, PX, st, WRw, WCw, pm, nd);
            const int cbase = cl * jp.plane;
            auto off = [&](int u) { return (cbase + (u / WCw) * in.Wp + (u % WCw)) * 4 * sw; };
            if (pm && jp.pmajor) {
                // position-major: load window position u, then every FMA reading it (per
                // accumulator the (r, s) order is unchanged: u grows with (r, s) for a fixed
                // pixel), so only a few window registers are live
                for (int u : nd.pairs) {
                    o("ld.volatile.shared.b64 %%wp%d, [%%rb%d+%d];", u, s, off(u));
                    for (const JNz &z : nz)
                        for (int ty = 0; ty < TY; ++ty)
                            for (int tx = 0; tx < TX; ++tx) {
                                if ((ty * st + z.r) * WCw + tx * st + z.s != u) continue;
                                const uint32_t wb = fbits(z.w);
                                const int a = z.m * NPT + ty * TX + tx;
                                o("mov.b64 %%wt, 0x%08X%08X;", wb, wb);
                                o("fma.rn.f32x2 %%a%d, %%wt, %%wp%d, %%a%d;", a, u, a);
                            }
                }
                continue;
            }
            if (pm) {
                // one aligned 8-byte load = the same input element of images A and B
                for (int u : nd.pairs) o("ld.volatile.shared.b64 %%wp%d, [%%rb%d+%d];", u, s, off(u));
            } else {
                for (int u : nd.pairs) {
                    o("ld.volatile.shared.f32 %%wl%d, [%%rb%d+%d];", u, s, off(u));
                    o("ld.volatile.shared.f32 %%wh%d, [%%rb%d+%d];", u, s, off(u + PX * st));
                    o("mov.b64 %%wp%d, {%%wl%d, %%wh%d};", u, u, u);
                }
                for (int v : nd.scalars)
                    o("ld.volatile.shared.f32 %%ws%d, [%%rb%d+%d];", v, s, off(v));
            }
            // which register holds scalar position v (canonical layout, odd column)
            auto sreg = [&](int v, char *buf) {
                if (nd.stamp_p[size_t(v)] == nd.gen)
                    std::snprintf(buf, 32, "%%wl%d", v);
                else if ((v % WCw) >= PX * st && nd.stamp_p[size_t(v - PX * st)] == nd.gen)
                    std::snprintf(buf, 32, "%%wh%d", v - PX * st);
                else
                    std::snprintf(buf, 32, "%%ws%d", v);
            };
            char src[32];
            for (const JNz &z : nz) {
                const uint32_t wb = fbits(z.w);
                if (NPT) o("mov.b64 %%wt, 0x%08X%08X;", wb, wb);
                for (int ty = 0; ty < TY; ++ty) {
                    const int row = (ty * st + z.r) * WCw;
                    if (pm) {
                        for (int tx = 0; tx < TX; ++tx) {
                            const int a = z.m * NPT + ty * TX + tx;
                            o("fma.rn.f32x2 %%a%d, %%wt, %%wp%d, %%a%d;", a, row + tx * st + z.s, a);
                        }
                        continue;
                    }
                    for (int q = 0; q < PX; ++q) {
                        const int a = z.m * NPT + ty * PX + q;
                        o("fma.rn.f32x2 %%a%d, %%wt, %%wp%d, %%a%d;", a, row + q * st + z.s, a);
                    }
                    for (int tx = 2 * PX; tx < TX; ++tx) {
                        const int f = z.m * NST + ty * (TX - 2 * PX) + (tx - 2 * PX);
                        sreg(row + tx * st + z.s, src);
                        o("fma.rn.f32 %%f%d, %s, 0f%08X, %%f%d;", f, src, wb, f);
                    }
                }
            }
        }
        o("@%%p8 bra $DRYRET;");
        if (jp.raw) {
            // every warp is done with the stage: all threads stage chunk i + NS into it
            if (i + jp.NS < jp.nchunks) {
                o("bar.sync 1, %d;", jp.NW * 32);
                emit_raw_fill(o, jp, i + jp.NS, s);
            }
            continue;
        }
        // release the stage; the last warp out refills it with chunk i + NS
        if (i + jp.NS < jp.nchunks) {
            const int nxt = i + jp.NS;
            const int bytes = chunk_channels(jp, nxt) * jp.plane * 4 * sw;
            o("bar.warp.sync -1;");
            o("@!%%p0 bra $R%d;", i);
            o("fence.acq_rel.cta;");
            o("atom.shared.add.u32 %%r10, [%%r1+%d], 1;", jp.off_cnt + 4 * s);
            o("setp.ne.u32 %%p5, %%r10, %d;", jp.NW * (i / jp.NS + 1) - 1);
            o("@%%p5 bra $R%d;", i);
            o("fence.proxy.async.shared::cta;");
            o("mov.u32 %%r15, %%rw%d;", s);
            o("mul.lo.u32 %%r11, %%r3, %d;", bytes);
            o("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%%r15], %%r11;");
            o("mov.u32 %%r12, 0;");
            o("$L%d:", i);
            o("shl.b32 %%r13, %%r12, 3;");
            o("add.u32 %%r13, %%r13, %%r19;");
            o("ld.shared.u64 %%rd6, [%%r13];");
            o("add.u64 %%rd6, %%rd6, %lld;", (long long)nxt * jp.CB * jp.plane * 4 * sw);
            o("mad.lo.u32 %%r14, %%r12, %d, %%rs%d;", jp.img_stride * 4, s);
            if (jp.l2hint & 2)
                o("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
                  "[%%r14], [%%rd6], %d, [%%r15], %%rd10;", bytes);
            else
                o("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%%r14], [%%rd6], "
                  "%d, [%%r15];", bytes);
            o("add.u32 %%r12, %%r12, 1;");
            o("setp.lt.u32 %%p6, %%r12, %%r3;");
            o("@%%p6 bra $L%d;", i);
            o("$R%d:", i);
        } else if (jp.xpf) {
            // the stage's last use in this item: the last warp out stages the NEXT item's
            // chunk i + NS - nchunks into it (same physical stage by the rotation), so the
            // next item starts on data already in shared memory
            const int nxt = i + jp.NS - jp.nchunks;
            const int bytes = chunk_channels(jp, nxt) * jp.plane * 4 * sw;
            o("bar.warp.sync -1;");
            o("@!%%p0 bra $R%d;", i);
            o("fence.acq_rel.cta;");
            o("atom.shared.add.u32 %%r10, [%%r1+%d], 1;", jp.off_cnt + 4 * s);
            o("setp.ne.u32 %%p5, %%r10, %d;", jp.NW * (i / jp.NS + 1) - 1);
            o("@%%p5 bra $R%d;", i);
            o("setp.eq.u32 %%p5, %%r21, 0;");
            o("@%%p5 bra $R%d;", i);
            o("fence.proxy.async.shared::cta;");
            o("mov.u32 %%r15, %%rw%d;", s);
            o("mul.lo.u32 %%r11, %%r21, %d;", bytes);
            o("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%%r15], %%r11;");
            o("mov.u32 %%r12, 0;");
            o("$LN%d:", i);
            o("shl.b32 %%r13, %%r12, 3;");
            o("add.u32 %%r13, %%r13, %%r20;");
            o("ld.shared.u64 %%rd6, [%%r13];");
            o("add.u64 %%rd6, %%rd6, %lld;", (long long)nxt * jp.CB * jp.plane * 4 * sw);
            o("mad.lo.u32 %%r14, %%r12, %d, %%rs%d;", jp.img_stride * 4, s);
            if (jp.l2hint & 2)
                o("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
                  "[%%r14], [%%rd6], %d, [%%r15], %%rd10;", bytes);
            else
                o("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%%r14], [%%rd6], "
                  "%d, [%%r15];", bytes);
            o("add.u32 %%r12, %%r12, 1;");
            o("setp.lt.u32 %%p6, %%r12, %%r21;");
            o("@%%p6 bra $LN%d;", i);
            o("$R%d:", i);
        }
    }

    // a6: epilogue -- out = act(acc + bias[k]) at the original channel index; stores only
    // the pixels this lane owns (mask), image B only if it exists (mask bit 31, pair mode).
    // Address = lane base + k*cs + ty*rs + tx*ps (+ bo for image B): canonical or pair-
    // interleaved output, with or without a halo, chosen at run time by the strides.
    o("setp.ne.u64 %%p1, %%rd1, 0;");
    o("setp.ne.u32 %%p2, %%r4, 0;");
    if (pm) {
        o("and.b32 %%r9, %%r2, %u;", 0x80000000u);
        o("setp.ne.u32 %%p7, %%r9, 0;");
    }
    const int T = TY * TX;
    const bool fast_epi = pm && T <= 3;
    if (fast_epi) {
        // without bias (the common case) the epilogue is address + store per accumulator:
        // the pixel predicates and offsets are hoisted out of the channel loop and the relu /
        // no-relu variants are separate code (one runs), so no predicated-off add / max issues
        for (int i = 0; i < T; ++i) {
            const int ty = i / TX, tx = i % TX;
            o("and.b32 %%r9, %%r2, %u;", 1u << i);
            o("setp.ne.u32 %%pe%d, %%r9, 0;", 2 * i);
            o("and.pred %%pe%d, %%pe%d, %%p7;", 2 * i + 1, 2 * i);
            if (i == 0) continue;
            o("mul.wide.u32 %%rdp%d, %%r5, %d;", i, ty);
            o("mul.wide.u32 %%rd6, %%r16, %d;", tx);
            o("add.u64 %%rdp%d, %%rdp%d, %%rd6;", i, i);
        }
        if (std::getenv("SKC_JIT_NOSTORE")) {
            // measurement only: the stores stay in the code (so nothing is dead) but are
            // predicated off by a runtime-false predicate (relu flag == 77): no output traffic
            o("setp.eq.u32 %%p9, %%r4, 77;");
            for (int i = 0; i < 2 * T; ++i) o("and.pred %%pe%d, %%pe%d, %%p9;", i, i);
        }
        o("@%%p1 bra $EPI_B;");
        for (int relu = 0; relu < 2; ++relu) {
            o("$EPI_%c:", relu ? 'R' : 'N');
            if (!relu) o("@%%p2 bra $EPI_R;");
            for (int m = 0; m < Mb; ++m) {
                const int k = ks[size_t(m)];
                o("mul.lo.u64 %%rd3, %%rd2, %d;", k);
                o("add.u64 %%rd3, %%rd0, %%rd3;");
                for (int i = 0; i < T; ++i) {
                    const char *ad = "%rd3";
                    if (i) {
                        o("add.u64 %%rd5, %%rd3, %%rdp%d;", i);
                        ad = "%rd5";
                    }
                    o("mov.b64 {%%e0, %%e1}, %%a%d;", m * NPT + i);
                    if (relu) {
                        o("max.f32 %%e0, %%e0, 0f00000000;");
                        o("max.f32 %%e1, %%e1, 0f00000000;");
                    }
                    o("@%%pe%d st.global%s.f32 [%s], %%e0;", 2 * i, (jp.l2hint & 1) ? ".cs" : "", ad);
                    o("add.u64 %%rd6, %s, %%rd7;", ad);
                    o("@%%pe%d st.global%s.f32 [%%rd6], %%e1;", 2 * i + 1, (jp.l2hint & 1) ? ".cs" : "");
                }
            }
            o("bra.uni $EPI_END;");
        }
        o("$EPI_B:");
    }
    for (int m = 0; m < Mb; ++m) {
        const int k = ks[size_t(m)];
        o("mov.f32 %%e2, 0f00000000;");
        o("@%%p1 ld.global.nc.f32 %%e2, [%%rd1+%d];", 4 * k);
        o("mul.lo.u64 %%rd3, %%rd2, %d;", k);
        o("add.u64 %%rd3, %%rd0, %%rd3;");
        for (int ty = 0; ty < TY; ++ty) {
            if (ty == 0) {
                o("mov.b64 %%rd4, %%rd3;");
            } else {
                o("mul.wide.u32 %%rd5, %%r5, %d;", ty);
                o("add.u64 %%rd4, %%rd3, %%rd5;");
            }
            for (int tx = 0; tx < TX; ++tx) {
                const uint32_t bit = 1u << (ty * TX + tx);
                if (tx == 0) {
                    o("mov.b64 %%rd5, %%rd4;");
                } else {
                    o("mul.wide.u32 %%rd6, %%r16, %d;", tx);
                    o("add.u64 %%rd5, %%rd4, %%rd6;");
                }
                o("and.b32 %%r9, %%r2, %u;", bit);
                o("setp.ne.u32 %%p3, %%r9, 0;");
                if (pm) {
                    o("mov.b64 {%%e0, %%e1}, %%a%d;", m * NPT + ty * TX + tx);
                    o("add.f32 %%e3, %%e0, %%e2;");
                    o("@%%p2 max.f32 %%e3, %%e3, 0f00000000;");
                    o((jp.l2hint & 1) ? "@%%p3 st.global.cs.f32 [%%rd5], %%e3;" : "@%%p3 st.global.f32 [%%rd5], %%e3;");
                    o("add.f32 %%e3, %%e1, %%e2;");
                    o("@%%p2 max.f32 %%e3, %%e3, 0f00000000;");
                    o("and.pred %%p3, %%p3, %%p7;");
                    o("add.u64 %%rd6, %%rd5, %%rd7;");
                    o((jp.l2hint & 1) ? "@%%p3 st.global.cs.f32 [%%rd6], %%e3;" : "@%%p3 st.global.f32 [%%rd6], %%e3;");
                    continue;
                }
                if (tx < 2 * PX) {
                    o("mov.b64 {%%e0, %%e1}, %%a%d;", m * NPT + ty * PX + (tx < PX ? tx : tx - PX));
                    o("add.f32 %%e3, %s, %%e2;", tx < PX ? "%e0" : "%e1");
                } else {
                    o("add.f32 %%e3, %%f%d, %%e2;", m * NST + ty * (TX - 2 * PX) + tx - 2 * PX);
                }
                o("@%%p2 max.f32 %%e3, %%e3, 0f00000000;");
                o((jp.l2hint & 1) ? "@%%p3 st.global.cs.f32 [%%rd5], %%e3;" : "@%%p3 st.global.f32 [%%rd5], %%e3;");
            }
        }
    }
    if (fast_epi) o("$EPI_END:");
    o(jp.np && !jp.np_ret ? "exit;" : "ret;");
    o("$DRYRET:");
    o(jp.np && !jp.np_ret ? "exit;" : "ret;");
    o("}");
    return std::move(o.s);
}

// Entry: a persistent loop over work items t = b * NIG + ig (block-major: channel block b,
// image group ig of NI images = NI / sw slots), CTA j taking items j, j + G, j + 2G, ...  At
// any moment the CTAs of the grid therefore run the SAME block's code, started together, so
// the straight-line code is fetched once for many SMs (instruction fetch is the limit).
// item t (register tr) -> block (rb) and image group x band index (rc), the work order of
// jp.order; NIG in %r5, grid size G in %r31; ta/tb/tc are scratch registers
void emit_decode(Out &o, const JitPlan &jp, const char *tr, const char *rb, const char *rc,
                 const char *ta, const char *tb, const char *tc, const char *tag) {
    if (jp.order == 1) {
        // spread: consecutive items are different blocks (every block's code is fetched
        // in parallel from the first round on)
        o("rem.u32 %s, %s, %d;", rb, tr, jp.nblocks);
        o("div.u32 %s, %s, %d;", rc, tr, jp.nblocks);
    } else if (jp.order == 2 || jp.order == 3) {
        // first round spread (image groups 0..F-1 of every block, F = floor(G / nblocks):
        // all blocks' code is pulled from DRAM in parallel), then block-major over the rest.
        // Order 3: the first round is block-major too (item t < F*nb: block t / F), so with
        // GPC-major item numbers the CTAs of a GPC start on one or two blocks
        o("div.u32 %s, %%r31, %d;", ta, jp.nblocks);   // F
        o("min.u32 %s, %s, %%r5;", ta, ta);
        o("mul.lo.u32 %s, %s, %d;", tb, ta, jp.nblocks); // F * nblocks
        o("setp.lt.u32 %%p3, %s, %s;", tr, tb);
        o("@!%%p3 bra $ORD_REST%s;", tag);
        // p8: first round block-major (order 3, a launch-time choice: p_sched bit 0)
        o("@%%p8 bra $FR3%s;", tag);
        o("rem.u32 %s, %s, %d;", rb, tr, jp.nblocks);
        o("div.u32 %s, %s, %d;", rc, tr, jp.nblocks);
        o("bra.uni $ORD_DONE%s;", tag);
        o("$FR3%s:", tag);
        o("div.u32 %s, %s, %s;", rb, tr, ta);
        o("rem.u32 %s, %s, %s;", rc, tr, ta);
        o("bra.uni $ORD_DONE%s;", tag);
        o("$ORD_REST%s:", tag);
        o("sub.u32 %s, %s, %s;", rc, tr, tb);           // t' = t - F*nb
        o("sub.u32 %s, %%r5, %s;", rb, ta);             // NIG - F (> 0 here)
        o("rem.u32 %s, %s, %s;", tc, rc, rb);
        o("div.u32 %s, %s, %s;", rb, rc, rb);           // block
        o("add.u32 %s, %s, %s;", rc, tc, ta);           // image group
        o("$ORD_DONE%s:", tag);
    } else {
        o("rem.u32 %s, %s, %%r5;", rc, tr);             // image group
        o("div.u32 %s, %s, %%r5;", rb, tr);             // block
    }
}

const char *kEntryParams =
    ".param .u64 p_in, .param .u64 p_out, .param .u64 p_lm, .param .u64 p_bias, .param .u32 p_N, "
    ".param .u32 p_relu, .param .u32 p_opad, .param .u32 p_olay, .param .u64 p_vid, "
    ".param .u32 p_sched, .param .u32 p_G";

// np mode: the instruction prefetch as its own kernel (launched just before the items): CTA j
// executes chunk segment j mod (blocks x chunks) of the blocks' code once, with no waits and no
// stores, so the layer's cold code is pulled into L2 by many fetch streams at once (the
// persistent kernel does this before its first item, see emit_entry)
void emit_dry_entry(Out &o, const JitPlan &jp) {
    o(".visible .entry skc_jit_dry(%s)", kEntryParams);
    o("{");
    o(".reg .pred %%p<4>;");
    o(".reg .b32 %%r<16>;");
    o(".reg .b64 %%rd<8>;");
    o("griddepcontrol.launch_dependents;");   // the items may start as dry CTAs retire
    o("ld.param.u64 %%rd2, [p_lm];");
    o("cvta.to.global.u64 %%rd2, %%rd2;");
    o("mov.u32 %%r3, %%tid.x;");
    o("mul.wide.u32 %%rd4, %%r3, 16;");
    o("add.u64 %%rd4, %%rd2, %%rd4;");
    o("ld.global.nc.u32 %%r10, [%%rd4];");        // a valid lane base (band 0)
    o("mov.u32 %%r11, skc_smem;");
    o("mov.u32 %%r4, %%ctaid.x;");
    o("rem.u32 %%r4, %%r4, %d;", jp.nblocks * jp.nchunks);
    o("div.u32 %%r5, %%r4, %d;", jp.nchunks);      // block
    o("rem.u32 %%r6, %%r4, %d;", jp.nchunks);
    o("add.u32 %%r6, %%r6, 1;");                    // chunk + 1
    for (int b = 0; b < jp.nblocks; ++b) {
        o("setp.eq.u32 %%p0, %%r5, %d;", b);
        o("@%%p0 bra $DC%d;", b);
    }
    o("ret;");
    for (int b = 0; b < jp.nblocks; ++b) {
        o("$DC%d:", b);
        o("{");
        o(".param .b32 t0;\n.param .b32 t1;\n.param .b64 t2;\n.param .b32 t3;\n.param .b32 t4;");
        o(".param .b64 t5;\n.param .b32 t6;\n.param .b32 t7;\n.param .b64 t8;\n.param .b32 t9;");
        o(".param .b64 t10;\n.param .b32 t11;\n.param .b32 t12;\n.param .b32 t13;");
        o(".param .b32 t14;\n.param .b32 t15;");
        o("st.param.b32 [t0], %%r10;\nst.param.b32 [t1], %%r11;\nst.param.b64 [t2], 0;");
        o("st.param.b32 [t3], 0;\nst.param.b32 [t4], 0;\nst.param.b64 [t5], 0;");
        o("st.param.b32 [t6], 0;\nst.param.b32 [t7], 0;\nst.param.b64 [t8], 0;");
        o("st.param.b32 [t9], 0;\nst.param.b64 [t10], 0;\nst.param.b32 [t11], %%r6;");
        o("st.param.b32 [t12], 0;\nst.param.b32 [t13], %d;", jp.off_info);
        o("st.param.b32 [t14], %d;\nst.param.b32 [t15], 0;", jp.off_info);
        o(".param .b64 t16;\n.param .b32 t17;\n.param .b64 t18;");
        o("st.param.b64 [t16], 0;\nst.param.b32 [t17], 0;\nst.param.b64 [t18], 0;");
        o("call.uni skc_b%d, (t0, t1, t2, t3, t4, t5, t6, t7, t8, t9, t10, t11, t12, t13, "
          "t14, t15, t16, t17, t18);", b);
        o("}");
    }
    o("ret;");
    o("}");
}

std::string emit_entry(const JitPlan &jp) {
    const JitInput &in = jp.in;
    const int sw = jp.pair ? 2 : 1;
    Out o;
    o("%s", kHdr);
    for (int b = 0; b < jp.nblocks; ++b)
        o(".extern .func skc_b%d%s%s;", b, kBlkParams, jp.np && !jp.np_ret ? " .noreturn" : "");
    o(".extern .shared .align 128 .b8 skc_smem[];");
    if (jp.np) emit_dry_entry(o, jp);
    o(".visible .entry skc_jit_kernel(%s)", kEntryParams);
    o("{");
    o(".reg .pred %%p<10>;");
    o(".reg .b32 %%r<80>;");
    o(".reg .b64 %%rd<24>;");
    o("ld.param.u64 %%rd0, [p_in];");
    o("cvta.to.global.u64 %%rd0, %%rd0;");
    o("ld.param.u64 %%rd1, [p_out];");
    o("cvta.to.global.u64 %%rd1, %%rd1;");
    o("ld.param.u64 %%rd2, [p_lm];");
    o("cvta.to.global.u64 %%rd2, %%rd2;");
    o("ld.param.u64 %%rd3, [p_bias];");
    o("setp.eq.u64 %%p7, %%rd3, 0;");
    o("@!%%p7 cvta.to.global.u64 %%rd3, %%rd3;");
    o("ld.param.u32 %%r0, [p_N];");
    o("ld.param.u32 %%r1, [p_relu];");
    o("ld.param.u32 %%r2, [p_opad];");
    o("ld.param.u32 %%r39, [p_olay];");
    o("mov.u32 %%r3, %%tid.x;");
    // item t = u * CS + rank for cluster-level items u = clusterid, clusterid + nclusters, ...
    // (CS = cluster size; 1 without clusters)
    o("mov.u32 %%r35, %%cluster_ctarank;");
    o("mov.u32 %%r36, %%cluster_nctarank;");
    o("mov.u32 %%r37, %%clusterid.x;");
    o("mov.u32 %%r38, %%nclusterid.x;");
    o("mad.lo.u32 %%r4, %%r37, %%r36, %%r35;");  // item t
    if (jp.np) {
        // one work item per CTA (the grid is all items); G = the CTAs resident at once, which
        // the first-round order and the GPC-major first items refer to
        o("ld.param.u32 %%r31, [p_G];");
    } else {
        o("mul.lo.u32 %%r31, %%r38, %%r36;");    // stride G
    }
    // GPC-major item numbering (one CTA per SM, grid = all SMs): the first item of the CTA on
    // SM s is vid[s], the SM's position in a GPC-major order (topo.cu), so the CTAs of one GPC
    // take neighbouring items -- the same channel block -- and share the GPC's instruction
    // cache.  p_vid = 0: item t = cluster-major CTA rank.
    o("ld.param.u32 %%r63, [p_sched];");
    o("mov.u32 %%r61, %%r63;");                    // (the whole sched word, for the dry run)
    {
        // sched bit 3: read the contiguous lane table (after counters and staging tables)
        const long long lc_off = (long long)jp.lanemap.size() * 4 + 16 + (long long)jp.stab.size() * 4;
        o("and.b32 %%r62, %%r63, 8;");
        o("setp.ne.u32 %%p0, %%r62, 0;");
        o("selp.u64 %%rd19, %lld, 0, %%p0;", jp.lanemap_c.empty() ? 0LL : lc_off);
    }
    o("and.b32 %%r62, %%r63, 4;");
    o("setp.ne.u32 %%p9, %%r62, 0;");              // p9: skip the dry-run prefetch
    o("and.b32 %%r63, %%r63, 1;");
    o("setp.ne.u32 %%p8, %%r63, 0;");
    // The launch is not cooperative, so nothing guarantees one CTA per SM: the first item is
    // CLAIMED, not assumed.  Thread 0 starts at vid[smid] (smid clamped to the table) and
    // probes the claim table (in the workspace after the vid table, one word per first-round
    // item, zero between launches) linearly with compare-and-swap; each of the G CTAs claims
    // exactly one of the G first items, whatever SMs they landed on.  The last CTA to exit
    // clears the table ($EXIT).
    o("ld.param.u64 %%rd21, [p_vid];");
    o("setp.eq.u64 %%p0, %%rd21, 0;");
    if (jp.np) o("setp.ge.or.u32 %%p0, %%r4, %%r31, %%p0;");  // np: only the first G items
    o("@%%p0 bra $VID_DONE;");
    o("cvta.to.global.u64 %%rd21, %%rd21;");
    o("mov.u32 %%r78, skc_smem;");
    o("add.u32 %%r78, %%r78, %d;", jp.off_item + 8);
    o("setp.ne.u32 %%p1, %%r3, 0;");
    o("@%%p1 bra $VID_WAIT;");
    o("mov.u32 %%r79, %%smid;");
    o("min.u32 %%r79, %%r79, %d;", kVidCap - 1);
    o("mul.wide.u32 %%rd22, %%r79, 2;");
    o("add.u64 %%rd22, %%rd21, %%rd22;");
    o("ld.global.nc.u16 %%r79, [%%rd22];");
    o("rem.u32 %%r79, %%r79, %%r31;");
    o("add.u64 %%rd23, %%rd21, %d;", 2 * kVidCap);  // claim table
    o("$VID_PROBE:");
    o("mul.wide.u32 %%rd22, %%r79, 4;");
    o("add.u64 %%rd22, %%rd23, %%rd22;");
    o("atom.global.cas.b32 %%r77, [%%rd22], 0, 1;");
    o("setp.eq.u32 %%p1, %%r77, 0;");
    o("@%%p1 bra $VID_GOT;");
    o("add.u32 %%r79, %%r79, 1;");
    o("setp.ge.u32 %%p1, %%r79, %%r31;");
    o("@%%p1 mov.u32 %%r79, 0;");
    o("bra.uni $VID_PROBE;");
    o("$VID_GOT:");
    o("st.shared.u32 [%%r78], %%r79;");
    if (jp.np) {
        // np: the G-th CTA to claim clears the table (every claim is made by then; CTAs of
        // items >= G never touch it)
        o("add.u64 %%rd22, %%rd2, %d;", jp.NB * jp.NW * 32 * 16 + 4);
        o("fence.acq_rel.gpu;");
        o("atom.global.add.u32 %%r77, [%%rd22], 1;");
        o("sub.u32 %%r76, %%r31, 1;");
        o("setp.ne.u32 %%p1, %%r77, %%r76;");
        o("@%%p1 bra $VID_WAIT;");
        o("mov.u32 %%r76, 0;");
        o("$VID_CLR:");
        o("mul.wide.u32 %%rd20, %%r76, 4;");
        o("add.u64 %%rd20, %%rd23, %%rd20;");
        o("st.global.u32 [%%rd20], 0;");
        o("add.u32 %%r76, %%r76, 1;");
        o("setp.lt.u32 %%p1, %%r76, %%r31;");
        o("@%%p1 bra $VID_CLR;");
        o("st.global.u32 [%%rd22], 0;");
    }
    o("$VID_WAIT:");
    o("bar.sync 0;");
    o("ld.shared.u32 %%r4, [%%r78];");
    o("$VID_DONE:");
    o("add.u32 %%r5, %%r0, %d;", jp.NI - 1);
    o("div.u32 %%r5, %%r5, %d;", jp.NI);        // image groups
    o("mul.lo.u32 %%r5, %%r5, %d;", jp.NB);     // NIG = image groups x bands
    o("mul.lo.u32 %%r32, %%r5, %d;", jp.nblocks);  // items
    o("mov.u32 %%r11, skc_smem;");
    o("mov.u32 %%r34, 1;");
    if (jp.l2hint & 2) o("createpolicy.fractional.L2::evict_first.b64 %%rd13, 1.0;");                      // first item: barriers not yet initialised
    o("add.u32 %%r24, %%r2, %%r2;");
    o("add.u32 %%r25, %%r24, %d;", in.Ho);       // Hop
    o("add.u32 %%r26, %%r24, %d;", in.Wo);       // Wop
    o("mul.lo.u32 %%r27, %%r25, %%r26;");        // Hop*Wop
    // output strides: canonical [N][K][Hop][Wop] (olay 0) or pair-interleaved
    // [N/2][K][Hop][Wop][2] (olay 1): element width ew = 4 or 8 bytes
    o("setp.ne.u32 %%p6, %%r39, 0;");
    o("selp.u32 %%r40, 8, 4, %%p6;");            // ew
    o("mul.lo.u32 %%r30, %%r26, %%r40;");         // row stride bytes
    o("mul.wide.u32 %%rd10, %%r27, %%r40;");      // channel stride bytes
    o("mul.lo.u64 %%rd11, %%rd10, %d;", in.K);    // image stride bytes (canonical)
    o("selp.u64 %%rd12, 4, %%rd11, %%p6;");       // image B offset: 4 (interleaved) or K*Hop*Wop*4
    // PDL: the next grid may be scheduled as our CTAs retire; the dry run below needs no data,
    // so it overlaps the previous grid's tail; wait for the previous grid before the first item
    o("griddepcontrol.launch_dependents;");
    if (jp.dry && !jp.np) {  // (np: the dry run is its own kernel, skc_jit_dry)
        // Instruction prefetch: the code of a layer is cold in DRAM at launch and fetching it
        // is latency-bound per code stream.  Before the first item every CTA dry-runs a few
        // (block, chunk) code segments -- pairs ctaid, ctaid + G, ... of nblocks x nchunks --
        // so the whole layer's code is pulled into L2 by many parallel streams at once.
        o("mul.wide.u32 %%rd14, %%r3, 16;");
        o("add.u64 %%rd14, %%rd2, %%rd14;");
        o("add.u64 %%rd14, %%rd14, %%rd19;");
        o("ld.global.nc.u32 %%r50, [%%rd14];");     // a valid lane base (band 0)
        o("mov.u32 %%r51, %%r4;");
        // sched bit 9: every CTA dry-runs segment t mod (blocks x chunks), so each segment is
        // run by several CTAs spread over the GPCs (their instruction caches warm too)
        o("and.b32 %%r62, %%r61, 512;");
        o("setp.ne.u32 %%p0, %%r62, 0;");
        o("@%%p0 rem.u32 %%r51, %%r51, %d;", jp.nblocks * jp.nchunks);
        o("@%%p9 bra $DRY_DONE;");
        o("$DRY_LOOP:");
        o("setp.ge.u32 %%p0, %%r51, %d;", jp.nblocks * jp.nchunks);
        o("@%%p0 bra $DRY_DONE;");
        o("div.u32 %%r52, %%r51, %d;", jp.nchunks);  // block
        o("rem.u32 %%r53, %%r51, %d;", jp.nchunks);
        o("add.u32 %%r53, %%r53, 1;");               // chunk + 1
        for (int b = 0; b < jp.nblocks; ++b) {
            o("setp.eq.u32 %%p3, %%r52, %d;", b);
            o("@%%p3 bra $DC%d;", b);
        }
        o("bra.uni $DRY_NEXT;");
        for (int b = 0; b < jp.nblocks; ++b) {
            o("$DC%d:", b);
            o("{");
            o(".param .b32 t0;\n.param .b32 t1;\n.param .b64 t2;\n.param .b32 t3;\n.param .b32 t4;");
            o(".param .b64 t5;\n.param .b32 t6;\n.param .b32 t7;\n.param .b64 t8;\n.param .b32 t9;");
            o(".param .b64 t10;\n.param .b32 t11;\n.param .b32 t12;\n.param .b32 t13;");
            o(".param .b32 t14;\n.param .b32 t15;");
            o("st.param.b32 [t0], %%r50;\nst.param.b32 [t1], %%r11;\nst.param.b64 [t2], %%rd1;");
            o("st.param.b32 [t3], 0;\nst.param.b32 [t4], 0;\nst.param.b64 [t5], 0;");
            o("st.param.b32 [t6], 0;\nst.param.b32 [t7], 0;\nst.param.b64 [t8], 0;");
            o("st.param.b32 [t9], 0;\nst.param.b64 [t10], 0;\nst.param.b32 [t11], %%r53;");
            o("st.param.b32 [t12], 0;\nst.param.b32 [t13], %d;", jp.off_info);
            o("st.param.b32 [t14], %d;\nst.param.b32 [t15], 0;", jp.off_info);
            o(".param .b64 t16;\n.param .b32 t17;\n.param .b64 t18;");
            o("st.param.b64 [t16], 0;\nst.param.b32 [t17], 0;\nst.param.b64 [t18], 0;");
            o("call.uni skc_b%d, (t0, t1, t2, t3, t4, t5, t6, t7, t8, t9, t10, t11, t12, t13, "
              "t14, t15, t16, t17, t18);", b);
            o("}");
            o("bra.uni $DRY_NEXT;");
        }
        o("$DRY_NEXT:");
        o("add.u32 %%r51, %%r51, %%r31;");
        o("bra.uni $DRY_LOOP;");
        o("$DRY_DONE:");
    }
    // (sched bit 10: launched programmatically right after the np dry-run kernel, which this
    // kernel does not depend on -- its inputs were complete before that kernel started)
    o("and.b32 %%r62, %%r61, 1024;");
    o("setp.ne.u32 %%p0, %%r62, 0;");
    o("@%%p0 bra $NO_PDL_WAIT;");
    o("griddepcontrol.wait;");
    o("$NO_PDL_WAIT:");
    // dynamic scheduling: thread 0 takes the next item from a global counter in the plan
    // workspace (after the lane tables); items are numbered longest-first, so CTAs that
    // finish early take the short tail items.  The last CTA to exit resets the counters.
    const int ctr_off = jp.NB * jp.NW * 32 * 16;
    // A cluster takes CS consecutive items u .. u+CS-1 (rank r: item u + r), so the CTAs of a
    // cluster (one TPC) run the same block's code side by side, as in the static order.
    // Thread 0 of rank 0 fetches one cluster item ahead (the atomic's latency overlaps the
    // current item) and writes u into every rank's slot (two slots, alternating); a cluster
    // barrier publishes it.  u >= items ends every rank of the cluster together.
    // dyn 1: every CTA fetches its own items; dyn 2: per cluster (see above).  The first
    // item is the static one (t = cluster item * CS + rank); the counter numbers the items
    // after the first round (fetched value + grid size G).
    const bool cl = jp.dyn == 2;
    if (jp.dyn) {
        o("add.u64 %%rd20, %%rd2, %d;", ctr_off);
        o("mov.u32 %%r58, 0;");                        // slot parity
        o("mov.u32 %%r60, 1;");                        // first item
        o("setp.eq.u32 %%p0, %%r3, 0;");
        if (cl) o("setp.eq.and.u32 %%p0, %%r35, 0, %%p0;");
        o("@%%p0 atom.global.add.u32 %%r56, [%%rd20], %s;", cl ? "%r36" : "1");
    }
    const int NSL = jp.NI / sw;
    if (jp.raw) {
        // the stages' halo (and every position no thread stages) stays zero for the whole
        // kernel: zero all stage memory once
        o("shl.b32 %%r62, %%r3, 4;");
        o("$ZERO:");
        o("setp.ge.u32 %%p0, %%r62, %d;", jp.NS * jp.stage_bytes);
        o("@%%p0 bra $ZERO_DONE;");
        o("add.u32 %%r61, %%r11, %%r62;");
        o("st.shared.v4.u32 [%%r61], {0, 0, 0, 0};");
        o("add.u32 %%r62, %%r62, %d;", jp.NW * 32 * 16);
        o("bra.uni $ZERO;");
        o("$ZERO_DONE:");
        o("bar.sync 0;");
    }
    if (jp.xpf) {
        // cross-item staging: the barriers live for the whole kernel (phases continue from
        // item to item), so they are initialised once here
        o("setp.ne.u32 %%p0, %%r3, 0;");
        o("@%%p0 bra $BINIT_DONE;");
        for (int s = 0; s < jp.NS; ++s) o("mbarrier.init.shared::cta.b64 [%%r11+%d], 1;", jp.off_bar + 8 * s);
        o("fence.mbarrier_init.release.cluster;");
        o("$BINIT_DONE:");
        o("mov.u32 %%r64, 0;");                      // item ordinal k of this CTA
    }
    o("$ITEM:");
    if (jp.dyn) {
        o("mad.lo.u32 %%r57, %%r58, 4, %%r11;");
        o("add.u32 %%r57, %%r57, %d;", jp.off_item);   // this item's slot
        o("xor.b32 %%r58, %%r58, 1;");
        o("setp.ne.u32 %%p0, %%r3, 0;");
        if (cl) o("setp.ne.or.u32 %%p0, %%r35, 0, %%p0;");
        o("setp.ne.or.u32 %%p0, %%r60, 0, %%p0;");
        o("@%%p0 bra $FETCHED;");
        o("add.u32 %%r61, %%r56, %%r31;");
        o("st.shared.u32 [%%r57], %%r61;");
        if (cl) {
            o("mov.u32 %%r59, 1;");
            o("$PEERS:");
            o("setp.ge.u32 %%p1, %%r59, %%r36;");
            o("@%%p1 bra $PEERS_DONE;");
            o("mapa.shared::cluster.u32 %%r54, %%r57, %%r59;");
            o("st.shared::cluster.u32 [%%r54], %%r61;");
            o("add.u32 %%r59, %%r59, 1;");
            o("bra.uni $PEERS;");
            o("$PEERS_DONE:");
        }
        o("atom.global.add.u32 %%r56, [%%rd20], %s;", cl ? "%r36" : "1");
        o("$FETCHED:");
        if (cl) {
            o("barrier.cluster.arrive.release;");
            o("barrier.cluster.wait.acquire;");
        } else {
            o("bar.sync 0;");
        }
        o("setp.eq.u32 %%p1, %%r60, 0;");
        o("@%%p1 ld.shared.u32 %%r4, [%%r57];");
        if (cl) o("@%%p1 add.u32 %%r4, %%r4, %%r35;");   // t = u + rank
        o("mov.u32 %%r60, 0;");
        if (cl) {
            o("sub.u32 %%r54, %%r4, %%r35;");            // u
            o("setp.ge.u32 %%p0, %%r54, %%r32;");
            o("@%%p0 bra $EXIT;");                       // the whole cluster ends
            o("setp.ge.u32 %%p0, %%r4, %%r32;");
            o("@%%p0 bra $NEXT;");                       // past the end: idle, stay in step
        } else {
            o("setp.ge.u32 %%p0, %%r4, %%r32;");
            o("@%%p0 bra $EXIT;");
        }
    } else {
        o("setp.ge.u32 %%p0, %%r4, %%r32;");
        o("@%%p0 bra $EXIT;");
    }
    emit_decode(o, jp, "%r4", "%r7", "%r6", "%r46", "%r47", "%r14", "");
    // image group x band -> band, image group; the lane table of the band:
    // {smem byte base, (slot<<24)|(y0<<12)|x0, store mask, idle}
    o("rem.u32 %%r48, %%r6, %d;", jp.NB);        // band
    o("div.u32 %%r6, %%r6, %d;", jp.NB);         // image group
    o("mad.lo.u32 %%r49, %%r48, %d, %%r3;", jp.NW * 32);
    o("mul.wide.u32 %%rd7, %%r49, 16;");
    o("add.u64 %%rd7, %%rd2, %%rd7;");
    o("add.u64 %%rd7, %%rd7, %%rd19;");
    o("ld.global.nc.v4.u32 {%%r17, %%r18, %%r33, %%r20}, [%%rd7];");
    o("shr.u32 %%r21, %%r18, 24;");              // slot
    o("shr.u32 %%r22, %%r18, 12;");
    o("and.b32 %%r22, %%r22, 4095;");            // y0
    o("and.b32 %%r23, %%r18, 4095;");            // x0
    o("add.u32 %%r29, %%r22, %%r2;");
    o("mad.lo.u32 %%r29, %%r29, %%r26, %%r23;");
    o("add.u32 %%r29, %%r29, %%r2;");            // (y0+opad)*Wop + x0+opad
    o("mul.lo.u32 %%r8, %%r6, %d;", jp.NI);      // n0
    o("sub.u32 %%r9, %%r0, %%r8;");
    o("min.u32 %%r9, %%r9, %d;", jp.NI);        // images in this item
    o("add.u32 %%r41, %%r9, %d;", sw - 1);
    o("shr.u32 %%r41, %%r41, %d;", sw - 1);      // slots in this item
    o("mov.u32 %%r10, 0;");                      // conv group of the block
    for (int b = 0; b < jp.nblocks; ++b)
        if (jp.bgrp[size_t(b)] != 0) {
            o("setp.eq.u32 %%p3, %%r7, %d;", b);
            o("@%%p3 mov.u32 %%r10, %d;", jp.bgrp[size_t(b)]);
        }
    if (jp.raw) {
        // raw input of image n0, channel g*Cg: in + (n0*C + g*Cg)*H*W*4; this thread's
        // staging entries: after the lane tables and counters, [band][thread][kmax]
        const long long HW = (long long)(in.Hp - 2 * in.pad) * (in.Wp - 2 * in.pad);
        o("cvt.u64.u32 %%rd16, %%r8;");
        o("mul.lo.u64 %%rd16, %%rd16, %lld;", (long long)in.C * HW * 4);
        o("cvt.u64.u32 %%rd18, %%r10;");
        o("mul.lo.u64 %%rd18, %%rd18, %lld;", (long long)in.Cg * HW * 4);
        o("add.u64 %%rd16, %%rd16, %%rd18;");
        o("add.u64 %%rd16, %%rd0, %%rd16;");
        o("mad.lo.u32 %%r62, %%r48, %d, %%r3;", jp.NW * 32);
        o("mul.wide.u32 %%rd17, %%r62, %d;", jp.kmax * 8);
        o("add.u64 %%rd17, %%rd17, %%rd2;");
        o("add.u64 %%rd17, %%rd17, %d;", jp.NB * jp.NW * 32 * 16 + 16);
    } else {
        o("mov.u64 %%rd16, 0;");
        o("mov.u64 %%rd17, 0;");
    }
    if (!jp.dyn) o("bar.sync 0;");               // every warp is done with the previous item
                                                 // (dynamic: the fetch barrier already is)
    o("setp.ne.u32 %%p0, %%r3, 0;");
    o("@%%p0 bra $INIT_DONE;");
    const long long slot_bytes = (long long)in.C * jp.plane * 4 * sw;
    // per-slot source base of image n0 in conv group g: in + ((n0/sw + j) * C + g * Cg) *
    // plane * sw * 4, written to the slot table at smem offset `tab`
    auto emit_info = [&](const char *n0, const char *g, const char *nsl, const char *tab,
                         const char *tag) {
        o("shr.u32 %%r42, %s, %d;", n0, sw - 1);
        o("cvt.u64.u32 %%rd4, %%r42;");
        o("mul.lo.u64 %%rd4, %%rd4, %lld;", slot_bytes);
        o("cvt.u64.u32 %%rd5, %s;", g);
        o("mul.lo.u64 %%rd5, %%rd5, %lld;", (long long)in.Cg * jp.plane * 4 * sw);
        o("add.u64 %%rd4, %%rd4, %%rd5;");
        o("add.u64 %%rd4, %%rd0, %%rd4;");
        o("mov.u32 %%r12, 0;");
        o("add.u32 %%r13, %%r11, %s;", tab);
        o("$INFO%s:", tag);
        o("st.shared.u64 [%%r13], %%rd4;");
        o("add.u64 %%rd4, %%rd4, %lld;", slot_bytes);
        o("add.u32 %%r13, %%r13, 8;");
        o("add.u32 %%r12, %%r12, 1;");
        o("setp.lt.u32 %%p1, %%r12, %s;", nsl);
        o("@%%p1 bra $INFO%s;", tag);
    };
    char tab0[32];
    std::snprintf(tab0, sizeof tab0, "%d", jp.off_info);
    if (jp.xpf) {
        for (int s = 0; s < jp.NS; ++s) o("st.shared.u32 [%%r11+%d], 0;", jp.off_cnt + 4 * s);
        // the first item stages its own first chunks; later items find them staged
        o("setp.ne.u32 %%p4, %%r64, 0;");
        o("@%%p4 bra $FILLS_DONE;");
    } else {
        // barriers of the previous item have completed every phase and have no pending
        // transfers: invalidate and re-initialise them (phase parity restarts at 0)
        o("setp.eq.u32 %%p4, %%r34, 0;");
        for (int s = 0; s < jp.NS; ++s) {
            o("@%%p4 mbarrier.inval.shared::cta.b64 [%%r11+%d];", jp.off_bar + 8 * s);
            // raw staging: every thread arrives once per fill (cp.async ... arrive.noinc)
            o("mbarrier.init.shared::cta.b64 [%%r11+%d], %d;", jp.off_bar + 8 * s, jp.raw ? jp.NW * 32 : 1);
            o("st.shared.u32 [%%r11+%d], 0;", jp.off_cnt + 4 * s);
        }
        o("mov.u32 %%r34, 0;");
    }
    if (jp.raw) {
        o("fence.mbarrier_init.release.cluster;");
        o("bra.uni $INIT_DONE;");                   // the block stages its own chunks
    }
    emit_info("%r8", "%r10", "%r41", tab0, "");
    o("fence.mbarrier_init.release.cluster;");
    o("fence.proxy.async.shared::cta;");
    for (int i = 0; i < std::min(jp.NS, jp.nchunks); ++i) {
        const int bytes = chunk_channels(jp, i) * jp.plane * 4 * sw;
        o("add.u32 %%r15, %%r11, %d;", jp.off_bar + 8 * i);
        o("mul.lo.u32 %%r14, %%r41, %d;", bytes);
        o("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%%r15], %%r14;");
        o("mov.u32 %%r12, 0;");
        o("$F%d:", i);
        o("shl.b32 %%r13, %%r12, 3;");
        o("add.u32 %%r13, %%r13, %%r11;");
        o("ld.shared.u64 %%rd6, [%%r13+%d];", jp.off_info);
        o("add.u64 %%rd6, %%rd6, %lld;", (long long)i * jp.CB * jp.plane * 4 * sw);
        o("mad.lo.u32 %%r16, %%r12, %d, %%r11;", jp.img_stride * 4);
        o("add.u32 %%r16, %%r16, %d;", i * jp.stage_bytes);
        if (jp.l2hint & 2)
            o("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
              "[%%r16], [%%rd6], %d, [%%r15], %%rd13;", bytes);
        else
            o("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%%r16], [%%rd6], "
              "%d, [%%r15];", bytes);
        o("add.u32 %%r12, %%r12, 1;");
        o("setp.lt.u32 %%p1, %%r12, %%r41;");
        o("@%%p1 bra $F%d;", i);
    }
    if (jp.xpf) {
        o("$FILLS_DONE:");
        // the next item of this CTA (t + G): its slot table into the other buffer and its
        // slot count for the block (0: none)
        o("add.u32 %%r65, %%r4, %%r31;");
        o("mov.u32 %%r67, 0;");
        o("setp.ge.u32 %%p4, %%r65, %%r32;");
        o("@%%p4 bra $NX_DONE;");
        emit_decode(o, jp, "%r65", "%r68", "%r69", "%r70", "%r71", "%r72", "_NX");
        o("div.u32 %%r69, %%r69, %d;", jp.NB);       // image group
        o("mul.lo.u32 %%r70, %%r69, %d;", jp.NI);    // n0
        o("sub.u32 %%r71, %%r0, %%r70;");
        o("min.u32 %%r71, %%r71, %d;", jp.NI);
        o("add.u32 %%r67, %%r71, %d;", sw - 1);
        o("shr.u32 %%r67, %%r67, %d;", sw - 1);      // slots of the next item
        o("mov.u32 %%r72, 0;");                      // its conv group
        for (int b = 0; b < jp.nblocks; ++b)
            if (jp.bgrp[size_t(b)] != 0) {
                o("setp.eq.u32 %%p3, %%r68, %d;", b);
                o("@%%p3 mov.u32 %%r72, %d;", jp.bgrp[size_t(b)]);
            }
        o("and.b32 %%r73, %%r64, 1;");
        o("xor.b32 %%r73, %%r73, 1;");
        o("mad.lo.u32 %%r73, %%r73, %d, %d;", NSL * 8, jp.off_info);
        emit_info("%r70", "%r72", "%r67", "%r73", "_NX");
        o("$NX_DONE:");
        o("st.shared.u32 [%%r11+%d], %%r67;", jp.off_item);
    }
    o("$INIT_DONE:");
    o("bar.sync 0;");
    // stage phases (r74), slot tables (r76 this item, r77 next), next item's slots (r75)
    if (jp.xpf) {
        // global chunk g = k * nchunks + j runs on physical stage g % NS, fill ordinal g / NS:
        // logical stage s of item k has parity base ((k*nchunks + s) / NS) & 1 and rotation
        // (k * nchunks) % NS
        o("mov.u32 %%r74, 0;");
        for (int s = 0; s < jp.NS; ++s) {
            o("mad.lo.u32 %%r78, %%r64, %d, %d;", jp.nchunks, s);
            o("div.u32 %%r78, %%r78, %d;", jp.NS);
            o("and.b32 %%r78, %%r78, 1;");
            o("shl.b32 %%r78, %%r78, %d;", s);
            o("or.b32 %%r74, %%r74, %%r78;");
        }
        o("mul.lo.u32 %%r78, %%r64, %d;", jp.nchunks);
        o("rem.u32 %%r78, %%r78, %d;", jp.NS);
        o("shl.b32 %%r78, %%r78, 8;");
        o("or.b32 %%r74, %%r74, %%r78;");
        o("and.b32 %%r76, %%r64, 1;");
        o("xor.b32 %%r77, %%r76, 1;");
        o("mad.lo.u32 %%r76, %%r76, %d, %d;", NSL * 8, jp.off_info);
        o("mad.lo.u32 %%r77, %%r77, %d, %d;", NSL * 8, jp.off_info);
        o("ld.shared.u32 %%r75, [%%r11+%d];", jp.off_item);
    } else {
        o("mov.u32 %%r74, 0;");
        o("mov.u32 %%r76, %d;", jp.off_info);
        o("mov.u32 %%r77, %d;", jp.off_info);
        o("mov.u32 %%r75, 0;");
    }
    // store mask: none for a slot past the batch; pair mode: bit 31 = image B exists
    o("mov.u32 %%r19, %%r33;");
    o("setp.ge.u32 %%p2, %%r21, %%r41;");
    o("@%%p2 mov.u32 %%r19, 0;");
    // image A of this lane: n = n0 + slot * sw
    o("mad.lo.u32 %%r28, %%r21, %d, %%r8;", sw);
    if (jp.pair) {
        o("add.u32 %%r43, %%r28, 1;");
        o("setp.lt.u32 %%p5, %%r43, %%r0;");
        o("@%%p5 or.b32 %%r19, %%r19, %u;", 0x80000000u);
    }
    // output lane base: canonical out + (n*K*Hop*Wop + (y0+opad)*Wop + x0+opad) * 4;
    // interleaved out + ((n/2)*K*Hop*Wop + ...) * 8 + (n&1) * 4
    o("shr.u32 %%r44, %%r28, 1;");
    o("selp.u32 %%r44, %%r44, %%r28, %%p6;");
    o("cvt.u64.u32 %%rd8, %%r44;");
    o("mul.lo.u64 %%rd8, %%rd8, %d;", in.K);
    o("cvt.u64.u32 %%rd9, %%r27;");
    o("mul.lo.u64 %%rd8, %%rd8, %%rd9;");
    o("cvt.u64.u32 %%rd9, %%r29;");
    o("add.u64 %%rd8, %%rd8, %%rd9;");
    o("cvt.u64.u32 %%rd9, %%r40;");
    o("mul.lo.u64 %%rd8, %%rd8, %%rd9;");
    o("and.b32 %%r45, %%r28, 1;");
    o("selp.u32 %%r45, %%r45, 0, %%p6;");
    o("mul.wide.u32 %%rd9, %%r45, 4;");
    o("add.u64 %%rd8, %%rd8, %%rd9;");
    o("add.u64 %%rd8, %%rd1, %%rd8;");
    for (int b = 0; b < jp.nblocks; ++b) {
        o("setp.eq.u32 %%p3, %%r7, %d;", b);
        o("@%%p3 bra $C%d;", b);
    }
    o("bra.uni $NEXT;");
    for (int b = 0; b < jp.nblocks; ++b) {
        o("$C%d:", b);
        o("{");
        o(".param .b32 t0;\n.param .b32 t1;\n.param .b64 t2;\n.param .b32 t3;\n.param .b32 t4;");
        o(".param .b64 t5;\n.param .b32 t6;\n.param .b32 t7;\n.param .b64 t8;\n.param .b32 t9;");
        o(".param .b64 t10;\n.param .b32 t11;\n.param .b32 t12;\n.param .b32 t13;");
        o(".param .b32 t14;\n.param .b32 t15;");
        o("st.param.b32 [t0], %%r17;\nst.param.b32 [t1], %%r11;\nst.param.b64 [t2], %%rd8;");
        o("st.param.b32 [t3], %%r19;\nst.param.b32 [t4], %%r41;\nst.param.b64 [t5], %%rd3;");
        o("st.param.b32 [t6], %%r1;\nst.param.b32 [t7], %%r30;\nst.param.b64 [t8], %%rd10;");
        o("st.param.b32 [t9], %%r40;\nst.param.b64 [t10], %%rd12;\nst.param.b32 [t11], 0;");
        o("st.param.b32 [t12], %%r74;\nst.param.b32 [t13], %%r76;");
        o("st.param.b32 [t14], %%r77;\nst.param.b32 [t15], %%r75;");
        o(".param .b64 t16;\n.param .b32 t17;\n.param .b64 t18;");
        o("st.param.b64 [t16], %%rd16;\nst.param.b32 [t17], %%r9;\nst.param.b64 [t18], %%rd17;");
        o("call.uni skc_b%d, (t0, t1, t2, t3, t4, t5, t6, t7, t8, t9, t10, t11, t12, t13, "
          "t14, t15, t16, t17, t18);", b);
        o("}");
        o("bra.uni $NEXT;");
    }
    o("$NEXT:");
    if (jp.np) {
        // one item per CTA; the block function ends the thread (unreachable)
        o("$EXIT:");
        o("ret;");
        o("}");
        return std::move(o.s);
    }
    if (!jp.dyn) o("add.u32 %%r4, %%r4, %%r31;");
    if (jp.xpf) o("add.u32 %%r64, %%r64, 1;");
    o("bra.uni $ITEM;");
    o("$EXIT:");
    // launch-scoped state in the workspace (the dynamic item counter, the first-item claim
    // table): the last CTA to exit resets it for the next launch (graph replays included)
    o("setp.ne.u32 %%p0, %%r3, 0;");
    o("@%%p0 bra $DONE;");
    o("setp.ne.u64 %%p1, %%rd21, 0;");            // first items were claimed
    if (!jp.dyn) o("@!%%p1 bra $DONE;");
    o("add.u64 %%rd20, %%rd2, %d;", ctr_off);
    o("fence.acq_rel.gpu;");          // our item fetches / claims are performed before `done`
    o("atom.global.add.u32 %%r57, [%%rd20+4], 1;");
    o("mov.u32 %%r56, %%nctaid.x;");
    o("sub.u32 %%r56, %%r56, 1;");
    o("setp.ne.u32 %%p0, %%r57, %%r56;");
    o("@%%p0 bra $DONE;");
    if (jp.dyn) o("st.global.u32 [%%rd20], 0;");   // every CTA has taken its last item: reset
    o("@!%%p1 bra $RESET_DONE;");
    o("add.u64 %%rd23, %%rd21, %d;", 2 * kVidCap);
    o("mov.u32 %%r56, 0;");
    o("$CLAIM_CLR:");
    o("st.global.u32 [%%rd23], 0;");
    o("add.u64 %%rd23, %%rd23, 4;");
    o("add.u32 %%r56, %%r56, 1;");
    o("setp.lt.u32 %%p0, %%r56, %%r31;");
    o("@%%p0 bra $CLAIM_CLR;");
    o("$RESET_DONE:");
    o("st.global.u32 [%%rd20+4], 0;");
    o("$DONE:");
    o("ret;");
    o("}");
    return std::move(o.s);
}

// ---------------------------------------------------------------------------------------
// compile + link (PTX compiler library in a thread pool, nvJitLink), with an on-disk cache
// ---------------------------------------------------------------------------------------
// nvJitLink (only the per-block build links modules) is loaded from the toolkit at first use,
// privately (RTLD_LOCAL) by path: PyTorch maps its own, older libnvJitLink.so.12 into the
// process, whose versioned symbols do not match this header's, so the library can neither
// link the shared one at build time nor rely on the one already loaded; linking the static
// archive instead would add ~90 MB to libskc.so.  Without it, plans compile as one whole
// program (nvPTXCompiler alone).
struct JitLinkApi {
    bool ok = false;
    nvJitLinkResult (*create)(nvJitLinkHandle *, uint32_t, const char **) = nullptr;
    nvJitLinkResult (*destroy)(nvJitLinkHandle *) = nullptr;
    nvJitLinkResult (*add_data)(nvJitLinkHandle, nvJitLinkInputType, const void *, size_t, const char *) = nullptr;
    nvJitLinkResult (*complete)(nvJitLinkHandle) = nullptr;
    nvJitLinkResult (*cubin_size)(nvJitLinkHandle, size_t *) = nullptr;
    nvJitLinkResult (*cubin)(nvJitLinkHandle, void *) = nullptr;
    nvJitLinkResult (*log_size)(nvJitLinkHandle, size_t *) = nullptr;
    nvJitLinkResult (*log)(nvJitLinkHandle, char *) = nullptr;
};

const JitLinkApi &jitlink() {
    static JitLinkApi api = [] {
        JitLinkApi a;
        std::vector<std::string> paths;
        if (const char *e = std::getenv("SKC_NVJITLINK")) paths.push_back(e);
        for (const char *h : {"CUDA_HOME", "CUDA_PATH"})
            if (const char *e = std::getenv(h)) paths.push_back(std::string(e) + "/lib64/libnvJitLink.so.12");
        paths.push_back("/usr/local/cuda/lib64/libnvJitLink.so.12");
        paths.push_back("/usr/local/cuda-12.9/lib64/libnvJitLink.so.12");
        void *h = nullptr;
        for (const auto &p : paths)
            if ((h = dlopen(p.c_str(), RTLD_NOW | RTLD_LOCAL))) break;
        if (!h) return a;
        auto sym = [&](const char *n) { return dlsym(h, n); };
        a.create = reinterpret_cast<decltype(a.create)>(sym("__nvJitLinkCreate_12_9"));
        a.destroy = reinterpret_cast<decltype(a.destroy)>(sym("__nvJitLinkDestroy_12_9"));
        a.add_data = reinterpret_cast<decltype(a.add_data)>(sym("__nvJitLinkAddData_12_9"));
        a.complete = reinterpret_cast<decltype(a.complete)>(sym("__nvJitLinkComplete_12_9"));
        a.cubin_size = reinterpret_cast<decltype(a.cubin_size)>(sym("__nvJitLinkGetLinkedCubinSize_12_9"));
        a.cubin = reinterpret_cast<decltype(a.cubin)>(sym("__nvJitLinkGetLinkedCubin_12_9"));
        a.log_size = reinterpret_cast<decltype(a.log_size)>(sym("__nvJitLinkGetErrorLogSize_12_9"));
        a.log = reinterpret_cast<decltype(a.log)>(sym("__nvJitLinkGetErrorLog_12_9"));
        a.ok = a.create && a.destroy && a.add_data && a.complete && a.cubin_size && a.cubin &&
               a.log_size && a.log;
        return a;
    }();
    return api;
}

bool compile_ptx(const std::string &ptx, const char *opt, int maxreg, std::vector<char> &obj,
                 std::string *msg, bool relocatable = true) {
    nvPTXCompilerHandle h = nullptr;
    if (nvPTXCompilerCreate(&h, ptx.size(), ptx.c_str()) != NVPTXCOMPILE_SUCCESS) {
        *msg = "nvPTXCompilerCreate failed";
        return false;
    }
    const std::string mr = "--maxrregcount=" + std::to_string(maxreg);
    // `opt` may hold several space-separated ptxas options (e.g. "-O1 -Ofc=min")
    std::vector<std::string> words;
    for (const char *p = opt; *p;) {
        while (*p == ' ') ++p;
        const char *q = p;
        while (*q && *q != ' ') ++q;
        if (q > p) words.emplace_back(p, size_t(q - p));
        p = q;
    }
    std::vector<const char *> opts = {"--gpu-name=sm_100a", mr.c_str()};
    for (const auto &w : words) opts.push_back(w.c_str());
    if (relocatable) opts.push_back("--compile-only");
    const nvPTXCompileResult r = nvPTXCompilerCompile(h, int(opts.size()), opts.data());
    bool okr = r == NVPTXCOMPILE_SUCCESS;
    if (!okr) {
        size_t n = 0;
        nvPTXCompilerGetErrorLogSize(h, &n);
        std::string log(n, '\0');
        if (n) nvPTXCompilerGetErrorLog(h, &log[0]);
        *msg = "PTX compile failed (" + std::to_string(int(r)) + "): " + log.substr(0, 800);
    } else {
        size_t n = 0;
        nvPTXCompilerGetCompiledProgramSize(h, &n);
        obj.resize(n);
        nvPTXCompilerGetCompiledProgram(h, obj.data());
    }
    nvPTXCompilerDestroy(&h);
    return okr;
}

std::string cache_dir() {
    if (const char *d = std::getenv("SKC_JIT_CACHE")) return d;
    const char *home = std::getenv("HOME");
    return std::string(home ? home : "/tmp") + "/.cache/skc_jit";
}

bool cache_read(uint64_t key, std::vector<char> &out) {
    if (std::getenv("SKC_JIT_NOCACHE")) return false;
    char name[64];
    std::snprintf(name, sizeof name, "/%016llx.cubin", (unsigned long long)key);
    FILE *f = std::fopen((cache_dir() + name).c_str(), "rb");
    if (!f) return false;
    std::fseek(f, 0, SEEK_END);
    const long n = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    out.resize(size_t(std::max(0L, n)));
    const bool okr = n > 0 && std::fread(out.data(), 1, out.size(), f) == out.size();
    std::fclose(f);
    return okr;
}

void cache_write(uint64_t key, const std::vector<char> &data) {
    if (std::getenv("SKC_JIT_NOCACHE")) return;
    const std::string dir = cache_dir();
    // mkdir -p (two levels is enough for $HOME/.cache/skc_jit)
    std::string acc;
    for (size_t i = 0; i <= dir.size(); ++i)
        if (i == dir.size() || (dir[i] == '/' && i > 0)) {
            acc = dir.substr(0, i);
            mkdir(acc.c_str(), 0755);
        }
    char name[96];
    std::snprintf(name, sizeof name, "/%016llx.cubin", (unsigned long long)key);
    const std::string tmp = dir + name + ".tmp" + std::to_string(getpid());
    FILE *f = std::fopen(tmp.c_str(), "wb");
    if (!f) return;
    const bool okw = std::fwrite(data.data(), 1, data.size(), f) == data.size();
    std::fclose(f);
    if (okw) std::rename(tmp.c_str(), (dir + name).c_str());
    else std::remove(tmp.c_str());
}


// ---------------------------------------------------------------------------------------
// static verification: tables + the emitted code decoded back to the CSR
// ---------------------------------------------------------------------------------------
int jit_verify(const JitPlan *jp, std::string *msg) {
    const JitInput &in = jp->in;
    const int st = in.stride, TY = jp->TY, TX = jp->TX, PX = jp->pair ? 0 : jp->PX;
    const int sw = jp->pair ? 2 : 1, NSL = jp->NI / sw;
    auto bad = [&](const std::string &m) {
        *msg = "verify (jit): " + m;
        return int(SKC_ERR_STATE);
    };
    // channel table: every output channel exactly once, in its own group's blocks
    std::vector<int> seen(size_t(in.K), 0);
    for (int b = 0; b < jp->nblocks; ++b)
        for (int m = 0; m < jp->M; ++m) {
            const int k = jp->chan[size_t(b) * jp->M + m];
            if (k < 0) continue;
            if (k >= in.K || k / in.Kg != jp->bgrp[size_t(b)]) return bad("channel in the wrong block");
            ++seen[size_t(k)];
        }
    for (int k = 0; k < in.K; ++k)
        if (seen[size_t(k)] != 1) return bad("output channel not covered exactly once");
    // lane table: tiles inside the output (so every window read stays inside its channel
    // plane of its image slot), lane base consistent, every output pixel of every image slot
    // stored by exactly one (lane, pixel)
    // (a slot is an image, or an image pair in the pair-interleaved layout; both images of
    // a pair share the lane's tile and mask)
    // (both lane tables: bank-residue first fit and the contiguous one)
    for (const std::vector<uint32_t> *tab : {&jp->lanemap, &jp->lanemap_c}) {
    if (tab == &jp->lanemap_c && tab->empty()) continue;
    std::vector<int> cover(size_t(NSL) * in.Ho * in.Wo, 0);
    if (tab->size() != size_t(jp->NB) * jp->NW * 32 * 4) return bad("lane table size");
    for (int l = 0; l < jp->NB * jp->NW * 32; ++l) {
        const uint32_t *e = tab->data() + size_t(l) * 4;
        const int img = int(e[1] >> 24), y0 = int((e[1] >> 12) & 4095), x0 = int(e[1] & 4095);
        if (img >= NSL || y0 + TY > in.Ho || x0 + TX > in.Wo) return bad("lane tile out of range");
        if (e[0] != uint32_t(img * jp->img_stride + (y0 * st * in.Wp + x0 * st) * sw) * 4u)
            return bad("lane base inconsistent with its tile");
        if (jp->img_stride < jp->CB * jp->plane * sw) return bad("image slots overlap");
        if (jp->pair && (e[2] >> 31)) return bad("mask bit 31 is reserved for image B");
        for (int b = 0; b < TY * TX; ++b)
            if (e[2] >> b & 1u) ++cover[(size_t(img) * in.Ho + y0 + b / TX) * in.Wo + x0 + b % TX];
    }
    for (int v : cover)
        if (v != 1) return bad("output pixel stored " + std::to_string(v) + " times");
    }
    if (size_t(jp->off_info) + size_t(NSL) * 8 > jp->smem ||
        size_t(jp->NS) * jp->stage_bytes > size_t(jp->off_bar) || jp->smem > size_t(kMaxSmem))
        return bad("shared-memory layout");
    // code: decode every window load and FMA of every block back to (k, c, r, s, w) per pixel
    const int NPT = jp->pair ? TY * TX : TY * PX, NST = jp->pair ? 0 : TY * (TX - 2 * PX);
    std::vector<int> ks;
    std::vector<std::vector<JNz>> per_c;
    for (int b = 0; b < jp->nblocks; ++b) {
        plan_block_channels(in, jp->bgrp[size_t(b)], jp->bidx[size_t(b)], ks);
        block_nz(in, ks, per_c);
        const std::string code = emit_block(*jp, b, ks, per_c);
        const int Mb = int(ks.size());
        const size_t NWIN = size_t((TY - 1) * st + in.R) * size_t((TX - 1) * st + in.S);
        std::vector<int> lo_off(NWIN, -1), hi_off(NWIN, -1), sc_off(NWIN, -1);
        std::vector<int> wp_lo(NWIN, -1), wp_hi(NWIN, -1);
        uint64_t wt = 0;
        bool wt_ok = false;
        int chunk = -1;
        // per (m, pixel): decoded sequence of (c, r, s, bits)
        struct Op { int c, r, s; uint32_t w; };
        std::vector<std::vector<Op>> seq(size_t(Mb) * TY * TX);
        auto decode = [&](int off, int ty, int tx, Op &op) -> bool {
            if (off < 0 || off % (4 * sw)) return false;
            const int wv = off / (4 * sw);
            const int cl = wv / jp->plane, rem = wv % jp->plane;
            const int wy = rem / in.Wp, wx = rem % in.Wp;
            op.c = chunk * jp->CB + cl;
            op.r = wy - ty * st;
            op.s = wx - tx * st;
            return cl < chunk_channels(*jp, chunk) && op.r >= 0 && op.r < in.R && op.s >= 0 &&
                   op.s < in.S;
        };
        size_t pos = 0;
        while (pos < code.size()) {
            size_t eol = code.find('\n', pos);
            if (eol == std::string::npos) eol = code.size();
            const std::string ln = code.substr(pos, eol - pos);
            pos = eol + 1;
            int a0, a1, a2, a3;
            unsigned u0, u1;
            char rn[4];
            if (std::sscanf(ln.c_str(), "$W%d:", &a0) == 1) {
                if (a0 != chunk + 1) return bad("chunks out of order");
                chunk = a0;
                continue;
            }
            if (std::sscanf(ln.c_str(), "ld.volatile.shared.f32 %%w%1[lhs]%d, [%%rb%d+%d];", rn, &a0,
                            &a1, &a2) == 4) {
                if (a1 != chunk % jp->NS || a0 < 0 || size_t(a0) >= NWIN) return bad("load stage");
                (rn[0] == 'l' ? lo_off : rn[0] == 'h' ? hi_off : sc_off)[size_t(a0)] = a2;
                continue;
            }
            if (jp->pair &&
                std::sscanf(ln.c_str(), "ld.volatile.shared.b64 %%wp%d, [%%rb%d+%d];", &a0, &a1, &a2) == 3) {
                if (a1 != chunk % jp->NS || a0 < 0 || size_t(a0) >= NWIN) return bad("load stage");
                wp_lo[size_t(a0)] = a2;  // the same element of images A and B
                continue;
            }
            if (std::sscanf(ln.c_str(), "mov.b64 %%wp%d, {%%wl%d, %%wh%d};", &a0, &a1, &a2) == 3) {
                if (a0 != a1 || a0 != a2 || size_t(a0) >= NWIN) return bad("pair build");
                wp_lo[size_t(a0)] = lo_off[size_t(a0)];
                wp_hi[size_t(a0)] = hi_off[size_t(a0)];
                continue;
            }
            if (std::sscanf(ln.c_str(), "mov.b64 %%wt, 0x%08X%08X;", &u0, &u1) == 2) {
                if (u0 != u1) return bad("weight pair halves differ");
                wt = u0;
                wt_ok = true;
                continue;
            }
            if (std::sscanf(ln.c_str(), "fma.rn.f32x2 %%a%d, %%wt, %%wp%d, %%a%d;", &a0, &a1, &a2) == 3) {
                if (a0 != a2 || !wt_ok || size_t(a1) >= NWIN || a0 >= Mb * NPT) return bad("pair fma");
                if (jp->pair) {  // accumulator pair = one pixel of images A and B
                    const int m = a0 / NPT, ty = (a0 % NPT) / TX, tx = (a0 % NPT) % TX;
                    Op op{};
                    if (!decode(wp_lo[size_t(a1)], ty, tx, op))
                        return bad("pair operand does not decode to a tap");
                    op.w = uint32_t(wt);
                    seq[(size_t(m) * TY + ty) * TX + tx].push_back(op);
                    continue;
                }
                const int m = a0 / NPT, ty = (a0 % NPT) / PX, q = (a0 % NPT) % PX;
                Op lo{}, hi{};
                if (!decode(wp_lo[size_t(a1)], ty, q, lo) || !decode(wp_hi[size_t(a1)], ty, q + PX, hi))
                    return bad("pair operand does not decode to a tap");
                lo.w = hi.w = uint32_t(wt);
                seq[(size_t(m) * TY + ty) * TX + q].push_back(lo);
                seq[(size_t(m) * TY + ty) * TX + q + PX].push_back(hi);
                continue;
            }
            if (std::sscanf(ln.c_str(), "fma.rn.f32 %%f%d, %%w%1[lhs]%d, 0f%08X, %%f%d;", &a0, rn, &a1,
                            &u0, &a3) == 5) {
                if (a0 != a3 || size_t(a1) >= NWIN || a0 >= Mb * NST) return bad("scalar fma");
                const int m = a0 / NST, rest = a0 % NST, w1 = TX - 2 * PX;
                const int ty = rest / w1, tx = 2 * PX + rest % w1;
                const int off = (rn[0] == 'l' ? wp_lo : rn[0] == 'h' ? wp_hi : sc_off)[size_t(a1)];
                Op op{};
                if (!decode(rn[0] == 's' ? off : off, ty, tx, op))
                    return bad("scalar operand does not decode to a tap");
                op.w = u0;
                seq[(size_t(m) * TY + ty) * TX + tx].push_back(op);
                continue;
            }
        }
        if (chunk != jp->nchunks - 1) return bad("missing chunks");
        // compare with the canonical CSR rows, in order, for every pixel of the tile
        const int64_t plane = int64_t(in.Hp) * in.Wp;
        for (int m = 0; m < Mb; ++m) {
            const int k = ks[size_t(m)];
            const int64_t gbase = int64_t(k / in.Kg) * in.Cg * plane;
            for (int px = 0; px < TY * TX; ++px) {
                const auto &sq = seq[size_t(m) * TY * TX + size_t(px)];
                if (int64_t(sq.size()) != in.rowptr[k + 1] - in.rowptr[k])
                    return bad("channel " + std::to_string(k) + ": nonzero count differs");
                for (size_t t = 0; t < sq.size(); ++t) {
                    const int32_t j = in.rowptr[k] + int32_t(t);
                    const int64_t off = in.colidx[j] - gbase;
                    const int cl = int(off / plane), rem = int(off % plane);
                    if (sq[t].c != cl || sq[t].r != rem / in.Wp || sq[t].s != rem % in.Wp ||
                        sq[t].w != fbits(in.values[j]))
                        return bad("channel " + std::to_string(k) + ": code differs from the CSR");
                }
            }
        }
    }
    return SKC_OK;
}

}  // namespace

// ---------------------------------------------------------------------------------------
// public (library-internal) interface
// ---------------------------------------------------------------------------------------
// Block partition.  The even partition (nbg blocks of M channels per group) gives items of
// equal length, so a batch whose item count is not a multiple of the persistent grid leaves a
// partly filled last round (conv5 at N=256: 344 items on 148 CTAs, 2.32 rounds -> 3).  With
// dynamic scheduling, splitting the last `split` blocks of every group into halves puts short
// items at the end of the queue where they fill that round.  `split` minimises the makespan
// of a list-scheduling simulation of the item queue at the hint batch (per-item time from the
// same model as the configuration cost; SKC_JIT_SPLIT forces it).
namespace {
double item_time(const JitPlan &jp, double instr) {
    return instr * std::max(kFetchInv, jp.NW / kIssue) + kItemCycles;
}

// item t -> block, the mapping emit_entry generates for jp.order (G = grid size)
int item_block(const JitPlan &jp, int64_t t, int64_t nig, int64_t G) {
    const int64_t nb = jp.nblocks;
    if (jp.order == 1) return int(t % nb);
    if (jp.order == 2 || jp.order == 3) {
        const int64_t F = std::min<int64_t>(G / nb, nig);
        if (t < F * nb) return int(jp.order == 3 ? t / F : t % nb);
        return int((t - F * nb) / (nig - F));
    }
    return int(t / nig);
}

double simulate_makespan(const JitPlan &jp, const std::vector<double> &tb, int64_t nig, int64_t P) {
    const int64_t items = nig * jp.nblocks;
    std::priority_queue<double, std::vector<double>, std::greater<double>> free_at;
    for (int64_t i = 0; i < std::min(P, items); ++i) free_at.push(0.0);
    double span = 0;
    for (int64_t t = 0; t < items; ++t) {
        const double s0 = free_at.top();
        free_at.pop();
        const double e = s0 + tb[size_t(item_block(jp, t, nig, P))];
        span = std::max(span, e);
        free_at.push(e);
    }
    return span;
}

void choose_blocks(JitPlan &jp, int n_hint) {
    const JitInput &in = jp.in;
    const int Mp = jp.M;
    int force = -1;
    if (const char *e = std::getenv("SKC_JIT_SPLIT")) force = std::atoi(e);
    // resident CTAs per SM (shared memory, registers, threads)
    const int per_sm = std::max(1, std::min({int(233472 / (jp.smem + 1024)),
                                             65536 / (jp.NW * 32 * jp.maxreg),
                                             2048 / (jp.NW * 32)}));
    const int64_t P = int64_t(kSMs) * per_sm;
    const int64_t nig = int64_t((n_hint + jp.NI - 1) / jp.NI) * jp.NB;
    std::vector<int> ks;
    std::vector<std::vector<JNz>> per_c;
    Need nd;
    struct Blk { int g; std::vector<int> idx; double instr; };
    auto instr_of = [&](int g, const std::vector<int> &idx) {
        plan_block_channels(in, g, idx, ks);
        block_nz(in, ks, per_c);
        return block_instr(in, per_c, jp.TY, jp.TX, jp.PX, jp.pair, jp.CB, int(idx.size()), nd);
    };
    // channels of even block q (of nbg): contiguous ranges of the nnz-sorted list, or dealt in
    // snake order (every block gets heavy and light channels alike).  With uniform masks the
    // two measured the same (conv2 +0.8%, conv4 -1.5%; profiles/r01_jit_deal.txt); with skewed
    // per-channel densities the contiguous ranges put the heaviest channels into one block,
    // whose items then finish last (conv4 1.72x slower than unsorted,
    // profiles/r02_skewed_masks_loadbalance.jsonl).  Snake dealing is taken when the
    // contiguous blocks are imbalanced (SKC_JIT_DEAL=0/1 forces one)
    int deal_force = -1;
    if (const char *e = std::getenv("SKC_JIT_DEAL")) deal_force = std::atoi(e) ? 1 : 0;
    double best_span = 0, snake_span = 0, imb0 = 1.0, imb1 = 1.0;
    std::vector<Blk> best, snake;
    const int smax = jp.dyn ? std::min(jp.nbg, (in.Kg + Mp - 1) / Mp) : 0;
    for (int deal = 0; deal <= 1; ++deal) {
    if (deal_force >= 0 && deal != deal_force) continue;
    std::vector<std::vector<int>> even(size_t(jp.nbg));
    for (int k = 0; k < in.Kg; ++k) {
        int q = k / Mp;
        if (deal) {
            const int r = k / jp.nbg, c = k % jp.nbg;
            q = (r & 1) ? jp.nbg - 1 - c : c;
        }
        if (q < jp.nbg) even[size_t(q)].push_back(k);
    }
    for (int sp = 0; sp <= smax; ++sp) {
        if (force >= 0 && sp != std::min(force, smax)) continue;
        std::vector<Blk> full, tail;
        for (int g = 0; g < in.groups; ++g)
            for (int q = 0; q < jp.nbg; ++q) {
                const std::vector<int> &ch = even[size_t(q)];
                const int cnt = int(ch.size());
                if (cnt <= 0) continue;
                if (q >= jp.nbg - sp && cnt >= 2) {
                    std::vector<int> h0, h1;  // alternate: both halves balanced
                    for (int m = 0; m < cnt; ++m) (m & 1 ? h1 : h0).push_back(ch[size_t(m)]);
                    tail.push_back({g, h0, instr_of(g, h0)});
                    tail.push_back({g, h1, instr_of(g, h1)});
                } else {
                    full.push_back({g, ch, instr_of(g, ch)});
                }
            }
        std::vector<Blk> blks = full;
        blks.insert(blks.end(), tail.begin(), tail.end());
        std::stable_sort(blks.begin(), blks.end(),
                         [](const Blk &a, const Blk &b) { return a.instr > b.instr; });
        std::vector<double> tb;
        for (const Blk &b : blks) tb.push_back(item_time(jp, b.instr));
        jp.nblocks = int(blks.size());
        const double span = simulate_makespan(jp, tb, nig, P);
        // block imbalance: heaviest block's modelled instructions over the mean (the model
        // charges every instruction alike, but a heavy block's code is longer than the
        // instruction caches, so contiguous ranges of a skewed nnz-sorted list measured far
        // slower than the makespan model says: decided by imbalance instead, below)
        double imax = 0, isum = 0;
        for (const Blk &b : full) {
            imax = std::max(imax, b.instr);
            isum += b.instr;
        }
        const double imb = full.empty() ? 1.0 : imax * double(full.size()) / isum;
        if (std::getenv("SKC_JIT_DEBUG"))
            std::fprintf(stderr, "skc jit: deal %d split %d blocks %d P %lld nig %lld span %.0f ideal %.0f imbalance %.3f\n",
                         deal, sp, jp.nblocks, (long long)P, (long long)nig, span,
                         [&] { double t = 0; for (double x : tb) t += x; return t * nig / P; }(), imb);
        if (sp == 0) (deal ? imb1 : imb0) = imb;
        // a split (its halves repeat the window loads) must gain >= 1%
        if (deal != (deal_force >= 0 ? deal_force : 0)) {
            // snake dealing: kept aside, taken below if the contiguous blocks are imbalanced
            if (sp == 0 && (snake.empty() || span < snake_span)) {
                snake = blks;
                snake_span = span;
            }
            continue;
        }
        if (best.empty() || span < best_span * 0.99) {
            best_span = span;
            best = blks;
            jp.split = sp;
            jp.deal = deal;
        }
    }
    }  // deal
    // contiguous ranges of a skewed list: one block holds the heavy channels (imbalance > 1.25;
    // uniform masks: 1.02-1.10) -- deal in snake order instead (no split)
    if (deal_force < 0 && !snake.empty() && imb0 > 1.25 && imb1 < imb0) {
        best = snake;
        best_span = snake_span;
        jp.split = 0;
        jp.deal = 1;
    }
    // dynamic scheduling only where it splits: with equal items the static order measured
    // as fast or faster (conv3 -2.5%: it keeps the CTAs of a TPC on the same code)
    if (jp.split == 0 && !std::getenv("SKC_JIT_DYN")) jp.dyn = 0;
    jp.nblocks = int(best.size());
    jp.bgrp.clear(); jp.bidx.clear();
    double instr = 0;
    for (const Blk &b : best) {
        jp.bgrp.push_back(b.g);
        jp.bidx.push_back(b.idx);
        instr += b.instr;
    }
    jp.code_instr = instr;
}
}  // namespace

int jit_configure(const JitInput &in, int max_ni, int batch_hint, JitPlan **out, std::string *msg) {
    *out = nullptr;
    const int plane = in.Hp * in.Wp;
    // TMA bulk copies of whole channel runs need 16-byte aligned sources and sizes: a run of
    // cb channels of one slot is cb*plane*sw floats at offset (slot*C + g*Cg + c0)*plane*sw
    auto cb_unit_for = [&](int sw) -> int {
        for (int u : {1, 2, 4})
            if ((long long)u * plane * sw % 4 == 0 && (long long)in.C * plane * sw % 4 == 0 &&
                (long long)in.Cg * plane * sw % 4 == 0)
                return u;
        return 0;
    };
    int pair_force = -1;  // SKC_JIT_PAIR=0/1 (tuning): canonical or image-pair layout only
    int band_force = 0;   // SKC_JIT_BANDS=n (tuning)
    int pmajor = 1;       // SKC_JIT_PMAJOR: position-major code (few live window registers)
    int wr_cap = kPmajorWregs;  // SKC_JIT_WREGS: window registers assumed live (position-major)
    if (const char *e = std::getenv("SKC_JIT_PMAJOR")) pmajor = std::atoi(e) ? 1 : 0;
    if (const char *e = std::getenv("SKC_JIT_WREGS")) wr_cap = std::atoi(e);
    // staging pipeline: bytes per stage and stages (SKC_JIT_STAGE_KB, SKC_JIT_NS: tuning)
    int stage_target = kStageTarget, ns_max = 3;
    if (const char *e = std::getenv("SKC_JIT_STAGE_KB")) stage_target = std::max(4, std::atoi(e)) * 1024;
    if (const char *e = std::getenv("SKC_JIT_NS")) ns_max = std::max(2, std::min(kMaxStages, std::atoi(e)));
    if (const char *e = std::getenv("SKC_JIT_BANDS")) band_force = std::max(1, std::atoi(e));
    if (const char *e = std::getenv("SKC_JIT_PAIR")) pair_force = std::atoi(e) ? 1 : 0;
    std::unique_ptr<JitPlan> best;
    std::vector<int> ks;
    std::vector<std::vector<JNz>> per_c;
    Need nd;
    const char *force = std::getenv("SKC_JIT_TILE");  // "TY,TX[,M]" (tuning)
    int fty = 0, ftx = 0, fm = 0;
    if (force) std::sscanf(force, "%d,%d,%d", &fty, &ftx, &fm);
    // warps per CTA (1 CTA per SM): more warps share each fetched instruction of the
    // straight-line code, fewer registers each (SKC_JIT_NW, tuning)
    int nw_force = 0;
    if (const char *e = std::getenv("SKC_JIT_NW")) nw_force = std::max(1, std::min(32, std::atoi(e)));
    double code_cap = 3.0e6;  // warp-instructions of all blocks' code (SKC_JIT_MAX_CODE)
    if (const char *e = std::getenv("SKC_JIT_MAX_CODE")) code_cap = std::atof(e);
    std::vector<int> nw_opts = {16, 12, 20, 24, 8};  // likely winners first (pruning)
    const int n_hint = std::max(1, batch_hint);  // batch the configuration is tuned for
    const int64_t nnz_total = in.rowptr[in.K];
    if (nw_force) nw_opts = {nw_force};
    bool any_aligned = false;
    for (int pm = 1; pm >= 0; --pm) {
        if (pair_force >= 0 && pm != pair_force) continue;
        if (pm && max_ni < 2) continue;
        const int sw = pm ? 2 : 1;
        const int cb_unit = cb_unit_for(sw);
        if (!cb_unit || cb_unit > in.Cg) continue;
        any_aligned = true;
        for (int nw_max : nw_opts) {
            const int regs = reg_cap(nw_max);
            const int reg_budget = regs - 17;
            const int lanes_max = nw_max * 32;
            for (int TY = 1; TY <= 4; ++TY)
                for (int TX = 1; TX <= 16; ++TX) {
                    if (force && (TY != fty || TX != ftx)) continue;
                    const int T = TY * TX;
                    if (TY > in.Ho || TX > in.Wo || T > (pm ? 31 : 32) || T < (pm ? 1 : 2)) continue;
                    const int PX = pm ? 0 : TX / 2;
                    int wr = window_regs(TY, TX, PX, in.R, in.S, in.stride, pm);
                    if (pm && pmajor && wr_cap > 0) wr = std::min(wr, wr_cap);
                    int M = (reg_budget - wr - 12) / (T * (pm ? 2 : 1));
                    if (fm > 0) M = fm;
                    M = std::min(M, in.Kg);
                    if (M < 1) continue;
                    const int ty_n = (in.Ho + TY - 1) / TY, tx_n = (in.Wo + TX - 1) / TX;
                    // row bands: an image (pair) too large for one CTA's lanes is split into
                    // NB bands of tile rows, one work item each (pair mode; NB = 1 otherwise)
                    for (int NB = 1; NB <= (pm ? 4 : 1); ++NB) {
                    if (NB > ty_n) break;
                    if (band_force > 0 && NB != band_force) continue;
                    const int tpi = ((ty_n + NB - 1) / NB) * tx_n;  // tiles of the largest band
                    if (NB > 1 && ty_n * tx_n <= lanes_max) break;  // a whole slot fits already
                    // slots per CTA item (no more images per item than the batch has)
                    int NSL = std::min({max_ni / sw, lanes_max / tpi, (n_hint + sw - 1) / sw});
                    if (NSL < 1) continue;
                    int CB = 0, NS = 0, IS = 0, stage = 0;
                    size_t smem = 0;
                    for (; NSL >= 1; --NSL) {
                        CB = stage_target / (NSL * plane * 4 * sw);
                        CB = std::min(in.Cg, CB / cb_unit * cb_unit);
                        if (CB < cb_unit) CB = cb_unit;
                        const int nch = (in.Cg + CB - 1) / CB;
                        NS = std::min(ns_max, nch);
                        IS = (CB * plane * sw + 3) / 4 * 4;
                        stage = NSL * IS * 4;
                        smem = size_t(NS) * stage + 264 + size_t(NSL) * 16;
                        if (smem <= size_t(kMaxSmem)) break;
                    }
                    if (NSL < 1) continue;
                    const int NI = NSL * sw;
                    const int NW = (NSL * tpi + 31) / 32;
                    if (NW > nw_max) continue;
                    // one or two more blocks than the registers need: smaller items, a
                    // different fill of the last round
                    const int M0 = M, CB0 = CB, NS0 = NS, IS0c = IS, stage0 = stage;
                    for (int xb = 0; xb <= 2; ++xb) {
                    const int nbg0 = (in.Kg + M0 - 1) / M0;
                    const int nbg = nbg0 + xb;
                    if (nbg > in.Kg || (xb > 0 && fm > 0)) continue;
                    int M = M0, CB = CB0, NS = NS0, IS = IS0c, stage = stage0;
                    // even blocks: M' = ceil(Kg / nbg) <= M (no small leftover block paying a
                    // full set of window loads for a few channels)
                    if (fm <= 0) M = (in.Kg + nbg - 1) / nbg;
                    if (xb > 0 && (in.Kg + M - 1) / M != nbg) continue;  // no real extra block
                    // distinct blocks running at once for a batch of n_hint images (an item
                    // covers NI images x 1/NB of their pixels: NIe image-equivalents)
                    const double NIe = double(std::min(NI, n_hint)) / NB;  // real images only
                    const int nig = (n_hint + NI - 1) / NI * NB;
                    const int conc = std::max(1, (kSMs + nig - 1) / nig);
                    const double share = std::max(kFetchInv, NW / kIssue) / NIe * conc_penalty(conc);
                    // lower bound (FMA instructions only; independent of the blocking) prunes
                    // most candidates before the exact count
                    if (best && double(nnz_total) * fma_per_nz(TY, TX, PX, pm) * share >= best->cost)
                        continue;
                    double instr = 0;
                    for (int g = 0; g < in.groups; ++g)
                        for (int q = 0; q < nbg; ++q) {
                            block_channels(in, M, g, q, ks);
                            block_nz(in, ks, per_c);
                            instr += block_instr(in, per_c, TY, TX, PX, pm, CB, int(ks.size()), nd);
                        }
                    // time per image (model): the straight-line code is fetched once per CTA
                    // item and shared by its NW warps; fetch-bound below ~20 warps, issue-bound
                    // above
                    if (instr > code_cap) continue;  // code size: compile time, I-fetch footprint
                    // light chunks (few instructions per warp between stage boundaries) pay
                    // the boundary (wait, release, refill) too often: use 2 large stages
                    // instead (profiles/r01_jit_stages.txt)
                    if (!std::getenv("SKC_JIT_NS") && NS == 3) {
                        const double per_ch = instr / (double(nbg) * in.groups * in.Cg);
                        if (per_ch * CB < kChunkInstr) {
                            int CB2 = kStage2Max / (NSL * plane * 4 * sw);
                            CB2 = std::min(in.Cg, CB2 / cb_unit * cb_unit);
                            if (CB2 > CB) {
                                CB = CB2;
                                NS = std::min(2, (in.Cg + CB - 1) / CB);
                                IS = (CB * plane * sw + 3) / 4 * 4;
                                stage = NSL * IS * 4;
                            }
                        }
                    }
                    // whole rounds of the persistent grid at the hint batch: items are equal
                    // (even blocks), so a partly filled last round costs a full one
                    // (profiles/r01_jit_pmajor.txt: conv3 M=43 in 2.61 rounds is slower than
                    // M=39 in 2.9)
                    const double per_img = instr * share + double(nbg * in.groups) / NIe * kItemCycles;
                    const int per_sm = std::max(1, std::min({int(233472 / (smem + 1024 + 256)),
                                                             65536 / (NW * 32 * reg_cap(nw_max)),
                                                             2048 / (NW * 32)}));
                    const double items = double(nbg) * in.groups * nig;
                    const double P = double(kSMs) * per_sm;
                    const double cost = per_img * (std::ceil(items / P) * P / items);
                    if (best && cost >= best->cost) continue;
                    std::unique_ptr<JitPlan> jp(new JitPlan());
                    jp->in = in;
                    jp->pair = pm;
                    jp->TY = TY; jp->TX = TX; jp->PX = PX; jp->M = M;
                    jp->NW = NW; jp->NI = NI; jp->CB = CB; jp->NS = NS;
                    jp->nchunks = (in.Cg + CB - 1) / CB;
                    jp->tiles_y = ty_n; jp->tiles_x = tx_n; jp->NB = NB;
                    jp->plane = plane; jp->img_stride = IS; jp->stage_bytes = stage;
                    jp->nbg = nbg; jp->nblocks = nbg * in.groups;
                    jp->cost = cost;
                    jp->code_instr = instr;
                    best = std::move(jp);
                    }  // xb
                    }  // NB
                }
        }
    }
    if (!best) {
        *msg = any_aligned ? "JIT kernel: no tile configuration fits this geometry"
                           : "JIT kernel: channel runs cannot be 16-byte aligned for TMA "
                             "(odd plane and odd C)";
        return SKC_ERR_UNSUPPORTED;
    }
    JitPlan &jp = *best;
    const int sw = jp.pair ? 2 : 1, NSL = jp.NI / sw;
    // slot stride: a multiple of 4 floats (TMA), chosen for the fewest bank conflicts
    const int IS0 = jp.img_stride;
    int best_extra = -1, best_is = IS0;
    for (int t = 0; t < 8; ++t) {
        const int IS = IS0 + 4 * t;
        const size_t smem = size_t(jp.NS) * NSL * IS * 4 + 264 + size_t(NSL) * 16;
        if (smem > size_t(kMaxSmem)) break;
        int e = 0;
        for (int b = 0; b < jp.NB && e >= 0; ++b) {
            const int eb = assign_lanes(jp, IS, b, nullptr);
            e = eb < 0 ? -1 : e + eb;
        }
        if (e >= 0 && (best_extra < 0 || e < best_extra)) {
            best_extra = e;
            best_is = IS;
        }
        if (NSL == 1 || best_extra == 0) break;
    }
    if (best_extra < 0) {
        *msg = "JIT kernel: lane assignment failed";
        return SKC_ERR_UNSUPPORTED;
    }
    jp.img_stride = best_is;
    jp.conflict = best_extra;
    jp.stage_bytes = NSL * best_is * 4;
    jp.lanemap_c.assign(size_t(jp.NB) * jp.NW * 32 * 4, 0);
    for (int b = 0; b < jp.NB; ++b)
        if (assign_lanes(jp, best_is, b, jp.lanemap_c.data() + size_t(b) * jp.NW * 32 * 4, 1) < 0) {
            jp.lanemap_c.clear();
            break;
        }
    jp.lanemap.assign(size_t(jp.NB) * jp.NW * 32 * 4, 0);
    for (int b = 0; b < jp.NB; ++b)
        assign_lanes(jp, best_is, b, jp.lanemap.data() + size_t(b) * jp.NW * 32 * 4);
    jp.off_bar = jp.NS * jp.stage_bytes;           // 128-byte aligned: stages are 16 B multiples
    jp.off_bar = (jp.off_bar + 15) / 16 * 16;
    jp.off_cnt = jp.off_bar + 8 * kMaxStages;
    jp.off_info = jp.off_cnt + 4 * kMaxStages;
    jp.off_info = (jp.off_info + 7) / 8 * 8;
    jp.off_item = jp.off_info + 2 * NSL * 8;      // two slot tables (this item, next item)
    jp.smem = size_t(jp.off_item) + 16;           // + the claimed first item (vid)
    jp.maxreg = reg_cap(jp.NW);
    if (const char *e = std::getenv("SKC_JIT_SYNC")) jp.sync_every = std::max(0, std::atoi(e));
    if (const char *e = std::getenv("SKC_JIT_L2HINT")) jp.l2hint = std::atoi(e) & 3;
    if (const char *e = std::getenv("SKC_JIT_ORDER")) jp.order = std::atoi(e);
    if (const char *e = std::getenv("SKC_JIT_DRY")) jp.dry = std::atoi(e) ? 1 : 0;
    if (const char *e = std::getenv("SKC_JIT_PMAJOR")) jp.pmajor = std::atoi(e) ? 1 : 0;
    if (const char *e = std::getenv("SKC_JIT_LOOKAHEAD")) jp.lookahead = std::max(0, std::min(8, std::atoi(e)));
    if (const char *e = std::getenv("SKC_JIT_XPF")) jp.xpf = std::atoi(e) ? 1 : 0;
    if (const char *e = std::getenv("SKC_JIT_DYN")) jp.dyn = std::max(0, std::min(2, std::atoi(e)));
    // whole-program compile (one serial ptxas run, ~10-20 s per 100k instructions) when the
    // code is moderate; parallel per-block modules otherwise (their calls pay an ABI
    // save/restore of callee-saved registers: -8-10% measured, profiles/r01_jit_whole.txt)
    choose_blocks(jp, n_hint);
    if (jp.dyn) jp.xpf = 0;  // the next item must be known an item ahead (static order)
    // raw staging (SKC_JIT_RAW=1, pair layout): per band, the padded input rows its lanes'
    // windows read; their interior positions (image, row, column) dealt to the CTA's threads
    // round-robin, (column, image) fastest so a warp's copies are consecutive stage words
    if (const char *e = std::getenv("SKC_JIT_RAW")) jp.raw = (std::atoi(e) && jp.pair) ? 1 : 0;
    if (jp.raw) {
        jp.xpf = 0;
        const int H = in.Hp - 2 * in.pad, W = in.Wp - 2 * in.pad, T = jp.NW * 32;
        std::vector<std::vector<uint32_t>> pos(size_t(jp.NB));
        for (int b = 0; b < jp.NB; ++b) {
            int lo = in.Hp, hi = 0;
            for (int l = 0; l < T; ++l) {
                const uint32_t *e = jp.lanemap.data() + (size_t(b) * T + size_t(l)) * 4;
                const int y0 = int((e[1] >> 12) & 4095);
                lo = std::min(lo, y0 * in.stride);
                hi = std::max(hi, (y0 + jp.TY - 1) * in.stride + in.R);
            }
            for (int r = std::max(lo, in.pad); r < std::min(hi, in.pad + H); ++r)
                for (int x = 0; x < W; ++x)
                    for (int img = 0; img < 2; ++img) {
                        pos[size_t(b)].push_back(uint32_t(img) * uint32_t(in.C * H * W) +
                                                 uint32_t((r - in.pad) * W + x));
                        pos[size_t(b)].push_back(uint32_t((r * in.Wp + x + in.pad) * 2 + img));
                    }
            jp.kmax = std::max(jp.kmax, int((pos[size_t(b)].size() / 2 + T - 1) / T));
        }
        jp.stab.assign(size_t(jp.NB) * T * jp.kmax * 2, 0u);
        for (int b = 0; b < jp.NB; ++b)
            for (int t = 0; t < T; ++t)
                for (int k = 0; k < jp.kmax; ++k) {
                    uint32_t *e = jp.stab.data() + ((size_t(b) * T + size_t(t)) * jp.kmax + size_t(k)) * 2;
                    const size_t q = size_t(t) + size_t(k) * T;
                    if (q < pos[size_t(b)].size() / 2) {
                        e[0] = pos[size_t(b)][2 * q];
                        e[1] = pos[size_t(b)][2 * q + 1];
                    } else {
                        e[0] = 0xffffffffu;  // no position
                        e[1] = 0;
                    }
                }
    }
    // moderate code: one whole-program module (fastest code; compile time grows ~n^1.7 with
    // the module, 20-70 s for an AlexNet layer).  Larger code: the non-persistent kernel over
    // per-block .noreturn modules compiled in parallel (seconds; 3-6% faster than the
    // persistent kernel over per-block modules, whose calls save callee-saved registers --
    // config 4 res256 / res512 -3.6% / -5.7%, profiles/r02_jit_np.txt).  SKC_JIT_NP=1 forces
    // the fast-build mode for any code (AlexNet: 3.4-4.8 s per layer, step +3.6%)
    jp.whole = jp.code_instr <= kWholeMaxInstr ? 1 : 0;
    if (const char *e = std::getenv("SKC_JIT_WHOLE")) jp.whole = std::atoi(e) ? 1 : 0;
    jp.np = jp.whole ? 0 : 1;
    if (const char *e = std::getenv("SKC_JIT_NP")) jp.np = std::atoi(e) ? 1 : 0;
    if (!jp.whole && !jitlink().ok) {  // no linker: one whole-program module, whatever its size
        jp.whole = 1;
        jp.np = 0;
    }
    if (jp.raw || jp.xpf) jp.np = 0;
    if (jp.np) {
        jp.whole = 0;  // separate modules, compiled in parallel
        jp.dyn = 0;    // items in blockIdx order: the hardware hands them out as SMs free up
        if (const char *e = std::getenv("SKC_JIT_NP_WHOLE")) jp.whole = std::atoi(e) ? 1 : 0;
        if (const char *e = std::getenv("SKC_JIT_NP_RET")) jp.np_ret = std::atoi(e) ? 1 : 0;
    }
    jp.chan.assign(size_t(jp.nblocks) * jp.M, -1);
    for (int b = 0; b < jp.nblocks; ++b) {
        plan_block_channels(in, jp.bgrp[size_t(b)], jp.bidx[size_t(b)], ks);
        for (size_t m = 0; m < ks.size(); ++m) jp.chan[size_t(b) * jp.M + m] = ks[m];
    }
    *out = best.release();
    return SKC_OK;
}

int jit_compile(JitPlan *jp, std::string *msg) {
    std::lock_guard<std::mutex> lk(jp->mu);
    if (jp->compiled) return SKC_OK;
    const JitInput &in = jp->in;
    const auto t0 = std::chrono::steady_clock::now();
    // generate every module (cheap next to compiling), then hash them for the cache key
    std::vector<std::string> mods(size_t(jp->nblocks) + 1);
    {
        std::vector<int> ks;
        std::vector<std::vector<JNz>> per_c;
        for (int b = 0; b < jp->nblocks; ++b) {
            plan_block_channels(in, jp->bgrp[size_t(b)], jp->bidx[size_t(b)], ks);
            block_nz(in, ks, per_c);
            mods[size_t(b)] = emit_block(*jp, b, ks, per_c);
        }
        mods.back() = emit_entry(*jp);
    }
    if (const char *d = std::getenv("SKC_JIT_DUMP")) {  // debugging: write the PTX modules
        for (size_t i = 0; i < mods.size(); ++i) {
            const std::string f = std::string(d) + "/m" + std::to_string(i) + ".ptx";
            if (FILE *fp = std::fopen(f.c_str(), "w")) {
                std::fwrite(mods[i].data(), 1, mods[i].size(), fp);
                std::fclose(fp);
            }
        }
    }
    // -O2: 1.2% faster steps than -O1 (fewer register moves; profiles/r02_jit_ptxas_opt.txt)
    const char *opt = std::getenv("SKC_JIT_OPT") ? std::getenv("SKC_JIT_OPT") : "-O2";
    uint64_t key = fnv1a(&kJitVersion, sizeof kJitVersion);
    key = fnv1a(opt, std::strlen(opt), key);
    key = fnv1a(&jp->maxreg, sizeof jp->maxreg, key);
    key = fnv1a(&jp->whole, sizeof jp->whole, key);
    for (const auto &m : mods) key = fnv1a(m.data(), m.size(), key);
    jp->key = key;
    if (cache_read(key, jp->cubin)) {
        jp->cache_hit = 1;
        jp->compiled = true;
        return SKC_OK;
    }
    if (jp->whole) {
        // whole-program mode: one module, one compile -- ptxas sees every call site, so the
        // block functions need no ABI save/restore of callee-saved registers (which costs a
        // burst of local-memory stores at every call of a separately compiled block)
        std::string all(kHdr);
        for (size_t i = 0; i + 1 < mods.size(); ++i) all.append(mods[i], std::strlen(kHdr), std::string::npos);
        const std::string &ent = mods.back();
        size_t pos = std::strlen(kHdr);
        for (;;) {
            while (pos < ent.size() && ent[pos] == '\n') ++pos;
            if (ent.compare(pos, 12, ".extern .fun") != 0) break;
            pos = ent.find('\n', pos) + 1;
        }
        all.append(ent, pos, std::string::npos);
        std::vector<std::string>().swap(mods);
        std::string err;
        if (!compile_ptx(all, opt, jp->maxreg, jp->cubin, &err, false)) {
            *msg = err;
            return SKC_ERR_UNSUPPORTED;
        }
        cache_write(key, jp->cubin);
        jp->compiled = true;
        jp->compile_s =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return SKC_OK;
    }
    // compile modules in parallel, then link; if the link runs out of the constant bank for
    // optimizer-generated constants (many small blocks: configurations for small batches),
    // compile again with ptxas --disable-optimizer-constants, as the linker asks
    const JitLinkApi &jl = jitlink();
    nvJitLinkHandle lh = nullptr;
    const std::string opt2 = std::string(opt) + " --disable-optimizer-constants";
    for (int attempt = 0;; ++attempt) {
        const char *o_used = attempt ? opt2.c_str() : opt;
        std::vector<std::vector<char>> objs(mods.size());
        std::vector<std::string> errs(mods.size());
        std::atomic<size_t> next{0};
        std::atomic<bool> bad{false};
        unsigned nth = std::max(1u, std::thread::hardware_concurrency());
        if (const char *e = std::getenv("SKC_JIT_THREADS")) nth = unsigned(std::max(1, std::atoi(e)));
        nth = std::min<unsigned>(nth, unsigned(mods.size()));
        // biggest modules first
        std::vector<size_t> order(mods.size());
        for (size_t i = 0; i < order.size(); ++i) order[i] = i;
        std::sort(order.begin(), order.end(),
                  [&](size_t a, size_t b) { return mods[a].size() > mods[b].size(); });
        auto work = [&]() {
            for (;;) {
                const size_t i = next.fetch_add(1);
                if (i >= order.size() || bad.load()) return;
                const size_t m = order[i];
                if (!compile_ptx(mods[m], o_used, jp->maxreg, objs[m], &errs[m])) bad.store(true);
            }
        };
        std::vector<std::thread> pool;
        for (unsigned t = 1; t < nth; ++t) pool.emplace_back(work);
        work();
        for (auto &t : pool) t.join();
        for (const auto &e : errs)
            if (!e.empty()) {
                *msg = e;
                return SKC_ERR_UNSUPPORTED;
            }
        // link
        const char *lopts[] = {"-arch=sm_100a"};
        if (!jl.ok || jl.create(&lh, 1, lopts) != NVJITLINK_SUCCESS) {
            *msg = jl.ok ? "nvJitLinkCreate failed" : "nvJitLink not found (set SKC_NVJITLINK)";
            return SKC_ERR_UNSUPPORTED;
        }
        nvJitLinkResult lr = NVJITLINK_SUCCESS;
        for (size_t i = 0; i < objs.size() && lr == NVJITLINK_SUCCESS; ++i) {
            const std::string name = "m" + std::to_string(i);
            lr = jl.add_data(lh, NVJITLINK_INPUT_CUBIN, objs[i].data(), objs[i].size(), name.c_str());
        }
        if (lr == NVJITLINK_SUCCESS) lr = jl.complete(lh);
        if (lr == NVJITLINK_SUCCESS) break;
        size_t n = 0;
        jl.log_size(lh, &n);
        std::string log(n, '\0');
        if (n) jl.log(lh, &log[0]);
        jl.destroy(&lh);
        if (attempt == 0 && log.find("disable-optimizer-constants") != std::string::npos) continue;
        *msg = "nvJitLink failed (" + std::to_string(int(lr)) + "): " + log.substr(0, 800);
        return SKC_ERR_UNSUPPORTED;
    }
    std::vector<std::string>().swap(mods);
    size_t n = 0;
    jl.cubin_size(lh, &n);
    jp->cubin.resize(n);
    jl.cubin(lh, jp->cubin.data());
    jl.destroy(&lh);
    cache_write(key, jp->cubin);
    jp->compiled = true;
    jp->compile_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return SKC_OK;
}

// device image: the lane tables, 16 bytes of (zeroed) scheduling counters, then (raw staging)
// the per-thread staging tables, the contiguous lane table, and (16-byte aligned) the vid
// table, the claim table and the topology-probe scratch
namespace {
size_t tables_bytes(const JitPlan *jp) {
    return (jp->lanemap.size() * 4 + 16 + jp->stab.size() * 4 + jp->lanemap_c.size() * 4 + 15) / 16 * 16;
}
}  // namespace
size_t jit_vid_offset(const JitPlan *jp) { return tables_bytes(jp); }
size_t jit_probe_offset(const JitPlan *jp) { return tables_bytes(jp) + 6 * size_t(kVidCap); }
size_t jit_probe_ints() { return kProbeInts; }
size_t jit_vid_cap() { return kVidCap; }
size_t jit_image_bytes(const JitPlan *jp) { return jit_probe_offset(jp) + 4 * size_t(kProbeInts); }
void jit_image(const JitPlan *jp, void *dst) {
    char *d = static_cast<char *>(dst);
    std::memset(d, 0, jit_image_bytes(jp));
    std::memcpy(d, jp->lanemap.data(), jp->lanemap.size() * 4);
    if (!jp->stab.empty()) std::memcpy(d + jp->lanemap.size() * 4 + 16, jp->stab.data(), jp->stab.size() * 4);
    if (!jp->lanemap_c.empty())
        std::memcpy(d + jp->lanemap.size() * 4 + 16 + jp->stab.size() * 4, jp->lanemap_c.data(),
                    jp->lanemap_c.size() * 4);
    uint16_t *vid = reinterpret_cast<uint16_t *>(d + jit_vid_offset(jp));
    for (int i = 0; i < kVidCap; ++i) vid[i] = uint16_t(i);  // identity until upload
}

void jit_info(const JitPlan *jp, JitInfo *o) {
    o->TY = jp->TY; o->TX = jp->TX; o->PX = jp->PX; o->M = jp->M; o->NW = jp->NW;
    o->NI = jp->NI; o->CB = jp->CB; o->NS = jp->NS; o->nblocks = jp->nblocks; o->split = jp->split; o->raw = jp->raw;
    o->sched = jp->t_order3.load() < 0 ? -1
                                       : (jp->t_order3.load() | (jp->t_vid.load() << 1) |
                                          (std::max(0, jp->t_nodry.load()) << 2) |
                                          (std::max(0, jp->t_lanes.load()) << 3) | (jp->t_cs.load() << 4) |
                                          (std::max(0, jp->t_dryall.load()) << 9));
    o->smem = jp->smem; o->cubin_bytes = jp->cubin.size(); o->cost = jp->cost;
    o->conflict = jp->conflict; o->compile_s = jp->compile_s; o->cache_hit = jp->cache_hit;
    o->pair = jp->pair;
    o->bands = jp->NB;
    o->whole = jp->whole;
    o->np = jp->np;
    o->deal = jp->deal;
    o->compiled = jp->compiled ? 1 : 0;
}

const std::vector<int32_t> &jit_chan(const JitPlan *jp) { return jp->chan; }
const std::vector<uint32_t> &jit_lanes(const JitPlan *jp) { return jp->lanemap; }

// Device-side preparation, done once by skc_plan_upload (the one synchronous call): compile
// if needed, load the cubin, set the kernel's shared-memory / cluster attributes and take the
// occupancy figures the launch needs -- so that a forward launch makes no allocation, no
// module load and no query that could fail (capture-safe from the first call).
int jit_prepare(JitPlan *jp, int dev, std::string *msg) {
    const int r = jit_compile(jp, msg);
    if (r != SKC_OK) return r;
    std::lock_guard<std::mutex> lk(jp->mu);
    auto cuda_fail = [&](const char *what, cudaError_t e) {
        *msg = std::string(what) + ": " + cudaGetErrorString(e);
        return int(SKC_ERR_CUDA);
    };
    if (!jp->lib) {
        cudaError_t e = cudaLibraryLoadData(&jp->lib, jp->cubin.data(), nullptr, nullptr, 0,
                                            nullptr, nullptr, 0);
        if (e != cudaSuccess) return cuda_fail("cudaLibraryLoadData", e);
        e = cudaLibraryGetKernel(&jp->kern, jp->lib, "skc_jit_kernel");
        if (e != cudaSuccess) return cuda_fail("cudaLibraryGetKernel", e);
        if (jp->np) {
            e = cudaLibraryGetKernel(&jp->kern_dry, jp->lib, "skc_jit_dry");
            if (e != cudaSuccess) return cuda_fail("cudaLibraryGetKernel (dry)", e);
        }
    }
    if (jp->kern_dry) {
        cudaError_t ed = cudaFuncSetAttribute(reinterpret_cast<const void *>(jp->kern_dry),
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, int(jp->smem));
        if (ed != cudaSuccess) return cuda_fail("cudaFuncSetAttribute (dry)", ed);
    }
    const void *fn = reinterpret_cast<const void *>(jp->kern);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(jp->smem));
    if (e != cudaSuccess) return cuda_fail("cudaFuncSetAttribute", e);
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return cuda_fail("cudaFuncSetAttribute (clusters)", e);
    int nsm = 0, per_sm = 0;
    e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess || nsm < 1) return cuda_fail("cudaDeviceGetAttribute", e);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, jp->NW * 32, jp->smem);
    if (e != cudaSuccess || per_sm < 1) return cuda_fail("occupancy", e);
    for (int cs = 2; cs <= 16; cs *= 2) {
        cudaLaunchConfig_t lc{};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = unsigned(cs);
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        lc.blockDim = dim3(unsigned(jp->NW * 32));
        lc.dynamicSmemBytes = jp->smem;
        lc.gridDim = dim3(unsigned(cs));
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, fn, &lc) != cudaSuccess || ncl < 1) {
            cudaGetLastError();  // (upload time) this size is not launchable: not used
            ncl = 0;
        }
        jp->ncl[cs] = ncl;
    }
    jp->nsm = nsm;
    jp->per_sm = per_sm;
    jp->prep_dev = dev;
    return SKC_OK;
}

bool jit_ready(const JitPlan *jp, int dev) { return jp->lib && jp->prep_dev == dev; }

void jit_set_vid(JitPlan *jp, bool ok) { jp->vid_ok = ok; }

namespace {
// The launch schedule (skc_info.jit_sched bits): the tuned choice, the defaults, or the
// SKC_JIT_SCHED override (testing: forces every variant the tuner can pick)
struct Sched {
    int o3, vid, nodry, lanes, cs, dryall;
};
Sched launch_sched(const JitPlan *jp) {
    Sched s{};
    if (const char *e = std::getenv("SKC_JIT_SCHED")) {
        const int v = std::atoi(e);
        s.o3 = v & 1;
        s.vid = (v >> 1) & 1;
        s.nodry = (v >> 2) & 1;
        s.lanes = (v >> 3) & 1;
        s.cs = std::max(1, (v >> 4) & 15);
        s.dryall = (v >> 9) & 1;
        return s;
    }
    s.o3 = jp->t_order3.load() >= 0 ? jp->t_order3.load() : (jp->order == 3 ? 1 : 0);
    if (jp->t_vid.load() >= 0) {
        s.vid = jp->t_vid.load();
    } else {
        const char *e = std::getenv("SKC_JIT_VID");  // GPC-major item numbers (default on)
        s.vid = !e || std::atoi(e) != 0;
    }
    s.nodry = std::max(0, jp->t_nodry.load());
    const char *le = std::getenv("SKC_JIT_LANES");  // 0/1: force the lane table (testing)
    s.lanes = le ? std::atoi(le) : std::max(0, jp->t_lanes.load());
    s.cs = jp->t_cs.load() > 0 ? jp->t_cs.load() : 2;
    if (const char *e = std::getenv("SKC_JIT_CLUSTER")) s.cs = std::max(1, std::min(16, std::atoi(e)));
    s.dryall = std::max(0, jp->t_dryall.load());
    return s;
}
}  // namespace

cudaError_t jit_launch(JitPlan *jp, const float *in, float *out, const void *d_ws, int N,
                       const Epilogue &epi, cudaStream_t st, std::string *msg) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || !jit_ready(jp, dev)) {
        *msg = "JIT plan not prepared on this device (skc_plan_upload)";
        return cudaErrorInvalidResourceHandle;
    }
    // persistent grid: one CTA per SM slot (the kernel loops over its work items)
    // work items: image groups x row bands x channel blocks (as the kernel numbers them)
    const int64_t nig = (int64_t(N) + jp->NI - 1) / jp->NI;
    const int64_t items = nig * jp->NB * jp->nblocks;
    if (items > 0x7fffffff) return cudaErrorInvalidConfiguration;
    const int nsm = jp->nsm, per_sm = jp->per_sm;
    const Sched sc = launch_sched(jp);
    // clusters of 2 CTAs: the pair is co-scheduled on one GPC and runs the same block's code
    // on neighbouring image groups, so they share instruction-cache lines (B200 packs 148 SMs
    // into 74 pairs exactly; +2-7% measured, profiles/r01_jit_cluster.txt)
    int cs = sc.cs;
    if (items < 2 * cs) cs = 1;
    int64_t grid = std::min<int64_t>(items, int64_t(nsm) * per_sm);
    if (const char *e = std::getenv("SKC_JIT_GRID")) grid = std::min<int64_t>(items, std::max(1, std::atoi(e)));
    if (std::getenv("SKC_JIT_DEBUG")) {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, reinterpret_cast<const void *>(jp->kern));
        std::fprintf(stderr, "skc jit: regs %d maxThreads %d local %zu shared %zu NW %d smem %zu per_sm %d\n",
                     fa.numRegs, fa.maxThreadsPerBlock, fa.localSizeBytes, fa.sharedSizeBytes, jp->NW,
                     jp->smem, per_sm);
    }
    cudaLaunchConfig_t lc{};
    cudaLaunchAttribute at[3];
    lc.blockDim = dim3(unsigned(jp->NW * 32));
    lc.dynamicSmemBytes = jp->smem;
    lc.stream = st;
    int nat = 0;
    if (const char *e = std::getenv("SKC_PDL"); e && e[0] == '1') {
        // off by default: measured no gain on the AlexNet step (profiles/r01_jit_order.txt)
        at[nat].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[nat].val.programmaticStreamSerializationAllowed = 1;
        ++nat;
    }
    int64_t conc = grid;  // CTAs resident at once (np: the first-round width G)
    if (cs > 1) {
        at[nat].id = cudaLaunchAttributeClusterDimension;
        at[nat].val.clusterDim.x = unsigned(cs);
        at[nat].val.clusterDim.y = 1;
        at[nat].val.clusterDim.z = 1;
        ++nat;
        int ncl = (cs == 2 || cs == 4 || cs == 8 || cs == 16) ? jp->ncl[cs] : 0;
        if (ncl < 1) ncl = std::max(1, nsm / cs);
        grid = std::min<int64_t>((items + cs - 1) / cs, ncl) * cs;
        conc = grid;
    }
    if (jp->np) {
        // one CTA per work item (a multiple of the cluster size; CTAs past the last item exit)
        grid = (items + cs - 1) / cs * cs;
        if (grid > 0x7fffffff) return cudaErrorInvalidConfiguration;
    }
    lc.gridDim = dim3(unsigned(grid));
    lc.attrs = at;
    lc.numAttrs = nat;
    const float *bias = epi.bias;
    unsigned un = unsigned(N), relu = unsigned(epi.relu), opad = unsigned(epi.opad);
    unsigned olay = unsigned(epi.olay);
    const char *ws = static_cast<const char *>(d_ws);
    // GPC-major first items (one CTA per SM, grid = all SMs; the kernel claims them, so a CTA
    // that shares an SM with another still gets a distinct item)
    const void *vid = nullptr;
    if (sc.vid && jp->vid_ok && per_sm == 1 && conc == nsm && grid >= conc && conc <= kVidCap &&
        jp->dyn != 2 && cs <= 2)
        vid = ws + jit_vid_offset(jp);
    unsigned sched = unsigned(sc.o3);
    if (sc.nodry) sched |= 4u;
    if (sc.lanes > 0 && !jp->lanemap_c.empty()) sched |= 8u;
    if (sc.dryall) sched |= 512u;
    if (std::getenv("SKC_JIT_DEBUG"))
        std::fprintf(stderr, "skc jit: grid %lld cs %d gpc-major items %s\n", (long long)grid, cs,
                     vid ? "on" : "off");
    const void *lm = d_ws;
    unsigned uG = unsigned(conc);
    void *args[] = {(void *)&in, (void *)&out, (void *)&lm, (void *)&bias,
                    (void *)&un, (void *)&relu, (void *)&opad, (void *)&olay, (void *)&vid,
                    (void *)&sched, (void *)&uG};
    if (jp->np && jp->dry && !sc.nodry) {
        // the dry-run prefetch kernel: one chunk segment per CTA (all segments; with sched
        // bit 9 at least one per resident CTA, each segment then run by several CTAs).  A plain
        // launch (it follows the producer of the input); the items kernel is launched
        // programmatically after it and skips its grid-dependency wait (sched bit 10): it
        // needs nothing from the dry run, so its CTAs take SMs as the dry CTAs retire
        const int64_t segs = int64_t(jp->nblocks) * jp->nchunks;
        cudaLaunchConfig_t ld{};
        ld.blockDim = lc.blockDim;
        ld.dynamicSmemBytes = jp->smem;
        ld.stream = st;
        ld.gridDim = dim3(unsigned(sc.dryall ? std::max<int64_t>(segs, conc) : segs));
        cudaError_t e = cudaLaunchKernelExC(&ld, reinterpret_cast<const void *>(jp->kern_dry), args);
        if (e != cudaSuccess) return e;
        if (!std::getenv("SKC_NP_NOPDL")) {
            bool has_pdl = false;
            for (int i = 0; i < nat; ++i)
                has_pdl |= at[i].id == cudaLaunchAttributeProgrammaticStreamSerialization;
            if (!has_pdl) {
                at[nat].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[nat].val.programmaticStreamSerializationAllowed = 1;
                ++nat;
                lc.numAttrs = nat;
            }
            sched |= 1024u;
        }
    }
    return cudaLaunchKernelExC(&lc, reinterpret_cast<const void *>(jp->kern), args);
}

// Launch-schedule tuning: time the variants (first round spread / block-major, GPC-major item
// numbers on / off, clusters of 2 / none, lane table, dry-run coverage) of this plan's kernel
// on the caller's scratch buffers of N images, with the L2 flushed (d_flush written) before
// every timed launch (code and data start cold, as in bench.py), and keep the fastest.  Every
// variant computes bit-identical outputs (scheduling only;
// tests/test_gpu_parity.py::test_jit_every_schedule_bitwise).  Synchronous on `st`.
int jit_tune(JitPlan *jp, const void *d_ws, int N, const float *d_in, float *d_out, void *d_flush,
             size_t flush_bytes, cudaStream_t st, double *best_ms, std::string *msg) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    auto cleanup = [&] {
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
    };
    cudaError_t ce = cudaEventCreate(&e0);
    if (ce == cudaSuccess) ce = cudaEventCreate(&e1);
    if (ce != cudaSuccess) {
        *msg = std::string("tune setup: ") + cudaGetErrorString(ce);
        cleanup();
        return SKC_ERR_CUDA;
    }
    const Epilogue epi{};
    double best = -1;
    int bo = 0, bv = 1, bc = 2, bd = 0;
    // the dry-run prefetch was never worth dropping (r01_jit_tune.txt): only tried on request
    const int nd_max = (jp->dry && std::getenv("SKC_TUNE_DRY")) ? 2 : 1;
    int bl = 0, ba = 0;
    for (int da = 0; da < (jp->dry ? 2 : 1); ++da)
    for (int ln = 0; ln < (jp->lanemap_c.empty() ? 1 : 2); ++ln)
    for (int nd = 0; nd < nd_max; ++nd)
    for (int o3 = 0; o3 < 2; ++o3)
        for (int v = 1; v >= 0; --v)
            for (int c = 2; c >= 1; --c) {
                jp->t_order3 = o3;
                jp->t_vid = v;
                jp->t_cs = c;
                jp->t_nodry = nd;
                jp->t_lanes = ln;
                jp->t_dryall = da;
                double tot = 0;
                for (int rep = 0; rep < 6; ++rep) {
                    if (d_flush && flush_bytes) cudaMemsetAsync(d_flush, rep, flush_bytes, st);
                    cudaEventRecord(e0, st);
                    cudaError_t e = jit_launch(jp, d_in, d_out, d_ws, N, epi, st, msg);
                    const char *what = "tune launch";
                    if (e == cudaSuccess) {
                        what = "tune event";
                        e = cudaEventRecord(e1, st);
                    }
                    if (e == cudaSuccess) {
                        what = "tune sync";
                        e = cudaEventSynchronize(e1);
                    }
                    if (e != cudaSuccess) {
                        *msg = std::string(what) + ": " + cudaGetErrorString(e) + " " + *msg;
                        cleanup();
                        return SKC_ERR_CUDA;
                    }
                    float ms = 0;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (rep) tot += ms;  // the first launch is a warm-up
                }
                if (best < 0 || tot < best) {
                    best = tot;
                    bo = o3; bv = v; bc = c; bd = nd; bl = ln; ba = da;
                }
            }
    jp->t_order3 = bo;
    jp->t_vid = bv;
    jp->t_cs = bc;
    jp->t_nodry = bd;
    jp->t_lanes = bl;
    jp->t_dryall = ba;
    if (best_ms) *best_ms = best / 5;
    if (std::getenv("SKC_JIT_DEBUG"))
        std::fprintf(stderr, "skc jit tune: order3 %d vid %d cluster %d: %.4f ms\n", bo, bv, bc, best / 5);
    cleanup();
    return SKC_OK;
}

int jit_verify_code(const JitPlan *jp, std::string *msg) { return jit_verify(jp, msg); }

void jit_destroy(JitPlan *jp) {
    if (!jp) return;
    if (jp->lib) cudaLibraryUnload(jp->lib);
    delete jp;
}

}  // namespace skc
