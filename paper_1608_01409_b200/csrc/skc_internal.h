// skc_internal.h -- private interface between the host library (plan.cpp) and the CUDA
// kernels (pad.cu, sconv_direct.cu, sconv_regtile.cu).  Not part of the C-ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include <string>
#include <vector>

namespace skc {

constexpr int kMaxStages = 8;

// One kernel-private nonzero: the weight and its offset relative to the base of the
// shared-memory stage that holds its input channel (colidx = f(c,r,s),
// re-encoded against the staged slab instead of the whole padded tensor).
struct Nz {
    float w;
    int32_t off;
};

// Fused epilogue (row f1): out = act(acc + bias[k]) written into an output with an opad-wide
// halo, i.e. directly in the zero-padded input layout of the next layer (the halo itself is
// never written: the caller zero-fills it once).
struct Epilogue {
    const float *bias;  // [K] or nullptr
    int relu;           // 1: max(., 0)
    int opad;           // output halo width (0: plain NCHW output)
    int olay;           // output layout: 0 [N][K][..][..]; 1 image-pair interleaved
                        // [ceil(N/2)][K][..][..][2] (the padded layout of JIT plans)
};

// Direct kernel (sconv_direct.cu).  CTA = (group of NI images, output-row band, block of
// NW*M output channels of one conv group); NW compute warps + 1 producer warp.  The
// producer stages CB input channels of the band for the NI images, plus the (w, off) stream
// of the block's channels for that chunk, per stage of an NS-deep mbarrier ring.  Each lane
// owns T output-pixel "slots" (slotq/slotout, built on the host): slot (t, lane) reads shared
// word off + slotq[t][lane], and slotq[t][lane] == lane (mod 32), so every load of a warp
// touches 32 distinct banks whatever the nonzero's offset.
struct DirectParams {
    const float *in;          // padded input [N][C][Hp][Wp]
    float *out;               // [N][K][Ho][Wo]
    const uint2 *stream;      // {w bits, off} per nonzero, regions per (block, chunk)
    const int32_t *segptr;    // [gblocks][nchunks][NW*M + 1] absolute uint2 index
    const int32_t *chan;      // [gblocks][NW*M] output channel (slot j = m*NW + warp) or -1
    const int32_t *slotq;     // [nbands][T][32] smem word offset of the slot (or lane: empty)
    const int32_t *slotout;   // [nbands][T][32] (img << 24) | (yl << 12) | x, or -1 (empty)
    int N, C, K, Kg, Cg, Hp, Wp, Ho, Wo, stride, groups;
    int NI, BH, BHin, nbands, CB, nchunks, NS;
    int chan_stride;          // floats between channels inside an image slot
    int img_stride;           // floats between image slots (multiple of 4)
    int slab_floats;          // NI * img_stride
    int stream_cap;           // uint2 entries of a stage's stream area
    int stage_floats;         // slab_floats + 2 * stream_cap
    int bulk;                 // 1: TMA bulk copies; 0: LSU copy fallback (misaligned planes)
    int whole;                // band = all Hp rows: one copy per image per chunk
    int NW, M, cblocks;
    Epilogue epi;
};

// Register-tiled kernel (sconv_regtile.cu).  A CTA = (group of NI images, block of NT
// "tasks" of one conv group); a task = M output channels.  Warps = NG lane groups x NT
// tasks: lane l of lane group q owns one TY x TX output tile (lanemap) for the task's M
// channels; the per-(block, chunk) op streams are staged into shared memory next to the
// input slab.  Stream entries (uint2): a c-group header {cbase, count} (cbase = float
// offset of the input channel inside an image slot) followed by `count` ops
// {weight bits, case}, case = (m*R + r)*S + s.
struct RegtileParams {
    const float *in;         // padded input [N][C][Hp][Wp]
    float *out;              // [N][K][Ho][Wo]
    const uint2 *stream;     // op streams
    const int32_t *segoff;   // [groups*nblocks][nchunks][NT+1] absolute uint2 index
    const int32_t *chan;     // [groups*nblocks][NT][M] output channel or -1
    const int32_t *lanemap;  // [NG][32] (img << 24) | (y0 << 12) | x0; bit 30 = idle lane
    int N, C, K, Cg, Kg, Hp, Wp, Ho, Wo, groups;
    int NI, CB, nchunks, NS;
    int img_stride;          // floats between image slots of a stage (multiple of 4)
    int slab_floats;         // NI * img_stride
    int stream_cap;          // uint2 entries per stage stream area (incl. slack)
    int stage_floats;        // slab_floats + 2 * stream_cap
    int NG, NT, nblocks;
    Epilogue epi;
};

struct RegtileShape {
    int R, S, TY, TX, M;
    int nwmax, minb;  // __launch_bounds__(nwmax*32, minb): register cap of the instance
};

// Launchers (defined in the .cu files).  Return cudaError_t of the launch.
cudaError_t launch_pad(const float *in, float *out, int64_t N, int C, int H, int W, int pad,
                       cudaStream_t st);
// NCHW -> image-pair interleaved padded layout [ceil(N/2)][C][Hp][Wp][2] (zero halo; the
// second image of an odd batch's last pair is zero).
cudaError_t launch_pad_pairs(const float *in, float *out, int64_t N, int C, int H, int W,
                             int pad, cudaStream_t st);
cudaError_t launch_im2col(const float *in, float *out, int64_t N, int C, int H, int W, int R,
                          int S, int stride, int pad, int Ho, int Wo, cudaStream_t st);
cudaError_t launch_im2col_pairs(const float *in, float *out, int64_t N, int C, int H, int W, int R,
                          int S, int stride, int pad, int Ho, int Wo, cudaStream_t st);
cudaError_t launch_direct(const DirectParams &p, int T, size_t smem, cudaStream_t st);
// set the kernel's opt-in shared-memory attribute on the current device (skc_plan_upload), so
// that launches need no attribute call (capture-safe from the first launch)
cudaError_t prepare_direct(int T, int M);
bool direct_supported(int T, int M);
// SpMDM kernel (spmdm.cu, row f2): 1x1 / stride 1 / pad 0 / one group, the plane's pixels as
// the dense operand's columns.  Row tiles t own output rows [trow[t], trow[t+1]); the chunk j
// block of tile t is meta[blk[t*nch + j] .. blk[t*nch + j + 1]): a header of per-row
// entry offsets (uint32, hbytes, 16-aligned), then uint2 entries (x byte offset in the stage, w bits).
struct SpmdmParams {
    const float *X;        // [N][C][plane]
    float *Y;              // [N][K][plane] (or the epilogue's layout)
    const uint8_t *meta;   // workspace
    const int64_t *blk;    // [ntiles*nch + 1] byte offsets into meta
    const int32_t *trow;   // [ntiles + 1]
    int K, C, H, W, plane;
    int KC, nch, NS, ntiles, ncb;
    int xcontig;           // 1: one column block spanning the plane (one copy per chunk)
    uint32_t xpitch, xstage, mstage, hbytes;
    Epilogue epi;
};
cudaError_t prepare_spmdm(int LC, int RWM, size_t smem);
cudaError_t launch_spmdm(const SpmdmParams &p, int LC, int RWM, int NW, int N, size_t smem,
                         cudaStream_t st);
cudaError_t launch_regtile(const RegtileParams &p, const RegtileShape &sh, size_t smem,
                           cudaStream_t st);
cudaError_t prepare_regtile(const RegtileShape &sh);
// Instantiated register-tile shapes (count returned, shapes written to out[0..max)).
int regtile_shapes(RegtileShape *out, int max);
// "Compiled weights" kernel (jit.cpp).  JitInput points into the plan's canonical CSR.
struct JitInput {
    int K, C, R, S, Hp, Wp, Ho, Wo, stride, groups, Kg, Cg, pad;
    const int32_t *rowptr, *colidx, *perm;
    const float *values;
};
struct JitInfo {
    int TY, TX, PX, M, NW, NI, CB, NS, nblocks;
    size_t smem, cubin_bytes;
    double cost;
    int conflict;
    double compile_s;
    int cache_hit, compiled;
    int pair;  // 1: the plan reads the image-pair interleaved padded layout
    int bands; // row bands per image (pair) -- work items per image group
    int whole; // 1: compiled as one whole program
    int split; // even blocks per group split into halves
    int sched; // tuned launch schedule (skc_info.jit_sched), -1 untuned
    int raw;   // 1: reads the unpadded NCHW input (halo filled while staging)
    int np;    // 1: non-persistent kernel (one item per CTA) + dry-run kernel
    int deal;  // 1: channels dealt to blocks in snake order
};
struct JitPlan;
// Pick the tile / channel-block / staging configuration (host, cheap; no code generated).
int jit_configure(const JitInput &in, int max_ni, int batch_hint, JitPlan **out, std::string *msg);
// Generate + compile + link the code (host; thread pool; on-disk cache).
int jit_compile(JitPlan *jp, std::string *msg);
// device image of the plan's kernel-private tables (lane tables, scheduling counters, raw
// staging tables); jit_image fills `bytes` = jit_image_bytes(jp)
size_t jit_image_bytes(const JitPlan *jp);
void jit_image(const JitPlan *jp, void *dst);
void jit_info(const JitPlan *jp, JitInfo *o);
const std::vector<int32_t> &jit_chan(const JitPlan *jp);
// device preparation at skc_plan_upload (compile if needed, load the cubin, attributes,
// occupancy); jit_ready: prepared on `dev`; jit_set_vid: the workspace holds the SM order
int jit_prepare(JitPlan *jp, int dev, std::string *msg);
bool jit_ready(const JitPlan *jp, int dev);
void jit_set_vid(JitPlan *jp, bool ok);
// workspace regions (byte offsets from the workspace base): vid table (jit_vid_cap() u16)
// followed by the claim table (jit_vid_cap() u32); probe scratch (jit_probe_ints() int32)
size_t jit_vid_offset(const JitPlan *jp);
size_t jit_probe_offset(const JitPlan *jp);
size_t jit_probe_ints();
size_t jit_vid_cap();
cudaError_t jit_launch(JitPlan *jp, const float *in, float *out, const void *d_ws, int N,
                       const Epilogue &epi, cudaStream_t st, std::string *msg);
// Static check: tables + the emitted code decoded back to the canonical CSR (host).
int jit_verify_code(const JitPlan *jp, std::string *msg);
// launch-schedule tuning on caller-owned scratch (input in the plan's layout, output, and an
// optional L2-flush buffer written before every timed launch); synchronous on `st`
int jit_tune(JitPlan *jp, const void *d_ws, int N, const float *d_in, float *d_out, void *d_flush,
             size_t flush_bytes, cudaStream_t st, double *best_ms, std::string *msg);
// GPC-major SM order (topo.cu): vid[smid].  sm_gpc_order runs the probe once per device on
// `st` with the caller's device scratch (>= scratch_ints int32; synchronous), then returns the
// cached order; empty when the probe fails.  sm_gpc_order_cached never launches.
const std::vector<uint16_t> &sm_gpc_order(int dev, int *d_scratch, size_t scratch_ints,
                                          cudaStream_t st);
bool sm_gpc_order_cached(int dev, std::vector<uint16_t> *out);
void jit_destroy(JitPlan *jp);

cudaError_t bench_ffma(void *scratch, int blocks, int iters, float *ms, double *flops);
cudaError_t bench_lds(void *scratch, int blocks, int iters, float *ms, double *bytes);
cudaError_t bench_ffma2(void *scratch, int blocks, int iters, float *ms, double *flops);
cudaError_t bench_lds64(void *scratch, int blocks, int iters, float *ms, double *bytes);

}  // namespace skc
