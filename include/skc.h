/*
 * skc.h -- C-ABI of libskc, the B200-native hot path of direct sparse convolution
 * (Park et al., "Faster CNNs with Direct Sparse Convolutions and Guided Pruning",
 * arXiv:1608.01409).  Citations "PAPER.md:<line>" refer to the paper's LaTeX source.
 *
 * The problem (Sec. 2.1, Eq. 1): a bank of K filters W [K][C/g][R][S]
 * applied to an input I [C][H][W] gives O [K][Ho][Wo],
 *      O(k,y,x) = sum_{c,r,s} W(k,c,r,s) * I(c, y*stride + r - pad, x*stride + s - pad).
 * Direct sparse convolution (Fig. 2 at :198-218) stores the pruned
 * weights in CSR, one row per output channel, with each nonzero's column index
 * pre-encoded as the layout offset f(c,r,s) into the (zero-padded) input, and computes
 * every output position as that sparse row dotted with the input vector shifted by
 * f(0,y,x): a sparse-matrix x "virtual" dense-matrix product, no lowering.
 *
 * Conventions for every entry point
 *   - Status: every function returns skc_status (0 = OK, < 0 = error); a thread-local
 *     message is available from skc_last_error().  No C++ exception crosses the ABI and
 *     nothing aborts.  Argument/geometry checks happen before any launch.
 *   - Precision: fp32 data, fp32 FMA accumulation (single precision).
 *   - Ownership: the caller owns every device buffer (activations, outputs, the plan
 *     workspace, the tuning scratch).  libskc NEVER allocates device memory (no cudaMalloc
 *     anywhere in the library).  A plan owns its host arrays and is freed by
 *     skc_plan_destroy(), which does not synchronise: the caller must make sure no launch
 *     using the plan's workspace is still running.
 *   - Streams: device work is enqueued asynchronously on the caller's stream (a
 *     cudaStream_t passed as void*; NULL = legacy default stream).  Launch errors are
 *     returned as SKC_ERR_CUDA; faults during execution surface at the caller's sync.
 *     skc_plan_upload() is the one setup call that synchronises the stream (it prepares
 *     everything a launch needs: JIT code loaded, kernel attributes, occupancy, SM topology),
 *     and skc_plan_tune() synchronises it too; every launch entry point (skc_pad_input,
 *     skc_sparse_conv_forward*, skc_im2col) only enqueues work, so it may be captured into a
 *     CUDA graph from its very first call.
 *   - Thread safety: a plan's host data is immutable after skc_plan_upload().  A JIT plan
 *     keeps launch-scoped scheduling state in its WORKSPACE (the dynamic work-item counter
 *     and the first-item claim table, reset by the last CTA of each launch), so launches that
 *     use one workspace must not overlap in time: issue them on one stream (or order them
 *     with events), or upload the plan into one workspace per concurrent stream.  Other
 *     kernels' launches may overlap freely.  skc_plan_tune() rewrites the plan's launch
 *     schedule: no launch of that plan may run concurrently with it.
 *   - Layouts (all contiguous, fp32):
 *       input  NCHW            [N][C][H][W]
 *       padded input           [N][C][Hp][Wp],  Hp = H + 2*pad, Wp = W + 2*pad
 *       output NCHW            [N][K][Ho][Wo],  Ho = (H+2*pad-R)/stride + 1 (floor), same Wo
 *   - Device pointers must be 16-byte aligned (TMA bulk copies), else SKC_ERR_ALIGN.
 */
#ifndef SKC_H_
#define SKC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SKC_OK = 0,
    SKC_ERR_ARG = -1,         /* NULL pointer, negative count, bad enum value          */
    SKC_ERR_GEOMETRY = -2,    /* Ho/Wo < 1, K or C not divisible by groups, ...         */
    SKC_ERR_NONFINITE = -3,   /* a weight is NaN or Inf                                 */
    SKC_ERR_OVERFLOW = -4,    /* an offset or size does not fit the int32 encoding      */
    SKC_ERR_UNSUPPORTED = -5, /* shape the kernels cannot tile (no CPU fallback exists) */
    SKC_ERR_ALIGN = -6,       /* device pointer not 16-byte aligned                     */
    SKC_ERR_STATE = -7,       /* e.g. forward before skc_plan_upload                    */
    SKC_ERR_CUDA = -8         /* a CUDA runtime call failed                             */
} skc_status;

typedef struct skc_plan skc_plan; /* opaque */

/* Kernel variants for the conv step.  AUTO picks per geometry. */
typedef enum {
    SKC_KERNEL_AUTO = 0,
    SKC_KERNEL_DIRECT = 1,   /* Fig. 2 statement per lane: one shared-memory read per MAC */
    SKC_KERNEL_REGTILE = 2,  /* register-tiled input window, per-nonzero dispatch        */
    SKC_KERNEL_JIT = 3,      /* "compiled weights": the CSR walk emitted as straight-line
                                sm_100a code (immediate weights, register windows, packed
                                FFMA2), compiled at plan time, see skc_plan_compile      */
    SKC_KERNEL_SPMDM = 4     /* row f2: sparse x dense matrix product for FC layers and
                                1x1 / stride 1 / pad 0 / one-group convs (plane % 4 == 0):
                                X staged by TMA in chunks of rows, a lane owns 4-8 columns,
                                the chunk's (offset, w) entries travel with it; AUTO picks it
                                for skc_pack_fc plans                                    */
} skc_kernel;

/* Padded-input layouts (the method only needs a layout function f with
 * f(c, y+r, x+s) = f(c, y, x) + f(0, r, s); the CSR colidx always encodes the canonical f).
 *   SKC_LAYOUT_NCHW   [N][C][Hp][Wp]                          (direct / regtile kernels)
 *   SKC_LAYOUT_PAIRS  [ceil(N/2)][C][Hp][Wp][2]: images 2p and 2p+1 interleaved element by
 *                     element, so one aligned 8-byte load feeds a packed FFMA2 over both
 *                     images (JIT kernel); an odd batch's last pair has a zero second image.
 *   SKC_LAYOUT_RAW    [N][C][H][W], unpadded: the JIT kernel pads and pair-interleaves while
 *                     staging (SKC_JIT_RAW=1), so no pad pass is needed; skc_pad_input copies
 *                     (or, in place, does nothing).
 * skc_info.layout says which one a plan reads; skc_pad_input writes it. */
typedef enum { SKC_LAYOUT_NCHW = 0, SKC_LAYOUT_PAIRS = 1, SKC_LAYOUT_RAW = 2 } skc_layout;

typedef struct {
    int K, C, R, S, H, W, stride, pad, groups;
    int Ho, Wo, Hp, Wp;
    int64_t nnz;                   /* realised nonzeros (the paper's x*|W|)           */
    size_t padded_elems_per_image; /* C*Hp*Wp                                           */
    size_t out_elems_per_image;    /* K*Ho*Wo                                           */
    size_t device_bytes;           /* workspace size skc_plan_upload needs              */
    int kernel;                    /* skc_kernel chosen (after AUTO resolution)         */
    int band_rows, chunk_channels, stages, warps, channels_per_warp, pixels_per_lane;
    size_t smem_bytes;             /* dynamic shared memory per CTA of the conv kernel  */
    int lane_mapping;              /* direct kernel: images sharing residue-bucketed slots */
    int tile_h, tile_w;            /* regtile kernel: register tile per lane (0: direct)  */
    int images_per_cta;            /* images staged together in one CTA                   */
    /* JIT kernel (kernel == SKC_KERNEL_JIT; zero otherwise) */
    int jit_blocks;                /* channel blocks = separately compiled code modules   */
    int jit_compiled;              /* 1 once skc_plan_compile / upload compiled the code  */
    int jit_cache_hit;             /* 1 if the linked code came from the on-disk cache    */
    double jit_compile_s;          /* wall seconds of generate + compile + link           */
    size_t code_bytes;             /* linked device code (cubin) bytes                    */
    double model_instr_per_image;  /* modelled warp-instructions per image (JIT config)   */
    int layout;                    /* skc_layout of the padded input this plan reads      */
    int bands;                     /* JIT: row bands per image (pair), one CTA item each  */
    int jit_whole;                 /* JIT: 1 = one whole-program compile (no ABI calls)   */
    int jit_split;                 /* JIT: even blocks per group split in halves (tail)   */
    int jit_sched;                 /* JIT launch schedule from skc_plan_tune: -1 untuned,
                                      else bit 0 first round block-major, bit 1 GPC-major
                                      item numbers, bit 2 no dry-run code prefetch, bit 3
                                      contiguous lane table, bits 4-7 cluster size, bit 9
                                      dry run by every CTA                                */
    int jit_np;                    /* JIT: 1 = non-persistent kernel over per-block modules
                                      (one work item per CTA); a forward then launches 2
                                      kernels: the dry-run code prefetch and the items     */
    int jit_deal;                  /* JIT: 1 = channels dealt to blocks in snake order
                                      (skewed per-channel nnz), 0 = contiguous ranges     */
} skc_info;

/* a1 -- CSR/offset packer (PAPER.md:210-216 Fig. 2 caption; :251-256 mode-1 matricisation).
 * w_host: dense pruned weights, host memory, [K][C/groups][R][S] row-major fp32, read only.
 * A nonzero is any w != 0.0f.  Canonical CSR: rows k = 0..K-1 in natural order, nonzeros in
 * ascending (c_local, r, s) == ascending colidx, colidx = ((g_k*(C/g) + c_local)*Hp + r)*Wp + s
 * with g_k = k / (K/groups) (global input channel; R1-R3).  Also builds the
 * nnz-sorted channel permutation (descending nnz, stable, within each group) and the kernel-
 * private streams.  *out receives a new plan (host memory only; upload before use).
 * Errors: SKC_ERR_ARG (NULL), SKC_ERR_GEOMETRY, SKC_ERR_NONFINITE, SKC_ERR_OVERFLOW
 * (C*Hp*Wp >= 2^31 or nnz >= 2^31), SKC_ERR_UNSUPPORTED (no kernel tiling fits). */
skc_status skc_pack_csr(const float *w_host, int K, int C, int R, int S, int H, int W,
                        int stride, int pad, int groups, skc_plan **out);

/* Same as skc_pack_csr, forcing a kernel variant (testing both paths on one shape). */
skc_status skc_pack_csr_ex(const float *w_host, int K, int C, int R, int S, int H, int W,
                           int stride, int pad, int groups, int kernel, skc_plan **out);

/* Same as skc_pack_csr_ex, with the number of images per forward call the plan is configured
 * for.  skc_pack_csr / _ex assume 256 (the benchmark batch; SKC_JIT_NHINT overrides).  The
 * configuration (kernel, images per CTA, channel blocks, row bands) is a performance choice
 * only: any plan accepts any N and computes the same outputs (Eq. 1).  Below
 * 16 images AUTO picks the data-driven direct kernel with a launch-time configuration for
 * batch_hint images (a compiled layer's code would be fetched cold by a few CTAs), from 16 up
 * the compiled-weights kernel (its 256-image configuration).  Errors: as skc_pack_csr_ex;
 * SKC_ERR_ARG if batch_hint < 1. */
skc_status skc_pack_csr_batch(const float *w_host, int K, int C, int R, int S, int H, int W,
                              int stride, int pad, int groups, int kernel, int batch_hint,
                              skc_plan **out);

/* Row f2 -- sparse fully connected layer as SpMDM: Y[M x B] = W[M x K] .
 * X[K x B] with W dense-pruned on the host (row-major [M][K]) and X, Y device row-major (the
 * batch is the fast axis -- SpMDM's dense operand).  This is exactly the 1x1 convolution of
 * one image with K channels of 1 x B pixels (the virtual dense matrix degenerates to X), so
 * the plan runs through the conv entry points: skc_plan_upload, then
 * skc_sparse_conv_forward(plan, X, Y, 1, stream) (X needs no padding; or _ex for bias+ReLU).
 * kernel: SKC_KERNEL_AUTO picks SKC_KERNEL_SPMDM when B % 4 == 0, else the direct kernel;
 * SKC_KERNEL_SPMDM with B % 4 != 0 is SKC_ERR_UNSUPPORTED.  SPMDM plans accept the fused
 * epilogue (bias, ReLU, out_pad, the next plan's layout).  Every output element is
 * accumulated by one thread in CSR order, so the SPMDM and direct kernels agree bit for bit.
 * The plan is specific to B.  Errors: as skc_pack_csr_ex. */
skc_status skc_pack_fc(const float *w_host, int M, int K, int B, int kernel, skc_plan **out);

skc_status skc_plan_info(const skc_plan *plan, skc_info *info);

/* Host views of the canonical CSR (valid until skc_plan_destroy): rowptr[K+1] int32,
 * colidx[nnz] int32, values[nnz] fp32. */
skc_status skc_plan_csr(const skc_plan *plan, const int32_t **rowptr, const int32_t **colidx,
                        const float **values);

/* Host view of the nnz-sorted channel order perm[K] (within-group, descending nnz, ties by
 * ascending k).  The kernels assign output channels to warps in this order. */
skc_status skc_plan_perm(const skc_plan *plan, const int32_t **perm);

/* Copy the plan's kernel-private arrays into a caller-owned device workspace of at least
 * skc_info.device_bytes bytes (16-byte aligned) on `stream`, and prepare the current device
 * for the plan's launches: kernel attributes; for JIT plans also the code (compiled now if
 * skc_plan_compile was not called; loaded as a cudaLibrary), occupancy figures, and -- at
 * the first JIT upload on a device -- the SM-topology probe (a few clustered probe kernels on
 * `stream`, using the workspace as scratch) whose GPC-major SM order goes into the
 * workspace.  SYNCHRONOUS: the one setup call that may block on `stream`; call it outside
 * stream capture.  The host arrays stay owned by the plan; the workspace must outlive every
 * launch using the plan, which must run on the device it was uploaded on (else forward
 * returns SKC_ERR_STATE).  Launch-scoped scheduling state lives in the workspace (see Thread
 * safety above).  Errors: SKC_ERR_ARG, SKC_ERR_ALIGN, SKC_ERR_UNSUPPORTED (JIT compile
 * failed), SKC_ERR_CUDA. */
skc_status skc_plan_upload(skc_plan *plan, void *d_workspace, size_t bytes, void *stream);

/* a2 -- padded-input layout (R1): d_in [N][C][H][W] ->
 * d_in_padded in the plan's layout (skc_info.layout): [N][C][Hp][Wp], or for
 * SKC_LAYOUT_PAIRS [ceil(N/2)][C][Hp][Wp][2]; zeros in the pad-wide border, interior copied
 * bit-exactly.  Both device pointers, caller-owned, must not overlap.  N = 0 is a no-op;
 * N < 0 is SKC_ERR_ARG. */
skc_status skc_pad_input(const skc_plan *plan, const float *d_in_nchw, float *d_in_padded,
                         int N, void *stream);

/* a3..a6 -- the sparse conv (PAPER.md:198-208 Fig. 2; :303-316).  d_in_padded as written by
 * skc_pad_input (or any buffer in the plan's layout, zero border required), d_out [N][K][Ho][Wo]
 * (fully overwritten, no accumulation into it).  Requires skc_plan_upload first
 * (else SKC_ERR_STATE).  Deterministic: each output element is accumulated by one thread in
 * a fixed order, so repeated calls are bitwise identical. */
skc_status skc_sparse_conv_forward(const skc_plan *plan, const float *d_in_padded,
                                   float *d_out, int N, void *stream);

/* Row f3 -- lowering for the comparison baseline "sparse convolution with lowering"
 * (PAPER.md:272-284; Fig. 3's "conv5 lowered", :413-414): d_lowered[n][(c*R + r)*S + s][y][x]
 * = in[n][c][y*stride + r - pad][x*stride + s - pad] (zero outside), i.e. the C*R*S x Ho*Wo
 * lowered matrix per image (R*S-fold replication of the input).  The geometry is the plan's.
 * Sparse conv with lowering = this + a 1x1 plan over the lowered tensor (weights reshaped
 * [K][C/g*R*S][1][1], same groups), whose CSR visits the nonzeros in the same (c, r, s)
 * order, so the two paths agree bit for bit.  Errors: SKC_ERR_ARG, SKC_ERR_OVERFLOW
 * (C*R*S*Ho*Wo >= 2^31). */
skc_status skc_im2col(const skc_plan *plan, const float *d_in_nchw, float *d_lowered, int N,
                      void *stream);

/* skc_im2col in a chosen layout of the lowered tensor: layout SKC_LAYOUT_NCHW as above, or
 * SKC_LAYOUT_PAIRS = the padded layout of a JIT (AUTO) 1x1 plan over it (pad 0):
 * d_lowered[p][(c*R + r)*S + s][y][x][j] = lowered image 2p+j ([ceil(N/2)][C*R*S][Ho][Wo][2],
 * zeros for a missing second image of an odd batch), so the compiled-weights kernel can run
 * the lowered SpMDM without a separate re-layout pass.  Errors: as skc_im2col, SKC_ERR_ARG for
 * another layout, SKC_ERR_ALIGN (PAIRS: pointers not 16-byte aligned). */
skc_status skc_im2col_ex(const skc_plan *plan, const float *d_in_nchw, float *d_lowered, int N,
                         int layout, void *stream);

/* Row f1 -- the same convolution with a fused epilogue (the layout
 * function makes writing into another layout legitimate):
 *     d_out[n][k][y + out_pad][x + out_pad] = act(conv(n, k, y, x) + bias[k])
 * d_bias: device [K] fp32 or NULL (no bias); relu: 0 (identity) or 1 (max(., 0));
 * d_out: [N][K][Ho + 2*out_pad][Wo + 2*out_pad] -- with out_pad equal to the next layer's pad
 * this IS the next layer's padded input, so no skc_pad_input pass is needed.  Only the
 * interior is written: the caller zero-fills the halo once (e.g. at allocation).
 * out_pad in [0, 64]; otherwise as skc_sparse_conv_forward. */
skc_status skc_sparse_conv_forward_ex(const skc_plan *plan, const float *d_in_padded,
                                      float *d_out, int N, const float *d_bias, int relu,
                                      int out_pad, void *stream);

/* Row f1 for chains: the same fused epilogue, written straight into the padded input buffer
 * of the NEXT layer's plan `next` (its pad and its layout, skc_info.layout), so the next
 * layer needs no skc_pad_input pass:
 *     d_next_in[n][k][y + pad'][x + pad'] (in next's layout) = act(conv(n, k, y, x) + bias[k])
 * Requires next's C == this K, next's H x W == this Ho x Wo (else SKC_ERR_GEOMETRY).  Only the
 * interior is written; the caller zero-fills the halo once.  Otherwise as
 * skc_sparse_conv_forward_ex. */
skc_status skc_sparse_conv_forward_into(const skc_plan *plan, const float *d_in_padded,
                                        const skc_plan *next, float *d_next_in, int N,
                                        const float *d_bias, int relu, void *stream);

/* End-to-end entry with HOST buffers (the host-buffer measurement): h_in [N][C][H][W] ->
 * h_out [N][K][Ho][Wo] (host memory; pinned for asynchronous overlap).  The batch is cut
 * into image chunks; the H2D copy of a chunk, pad + conv of the previous one (on `stream`)
 * and the D2H copy of the one before run concurrently on two internal copy streams.  The
 * call returns after enqueueing; `stream` completes after the last D2H copy.  It creates (and
 * releases) two internal non-blocking copy streams and a few events per call, so unlike the
 * device-buffer entry points it cannot be captured into a CUDA graph.  Caller-owned
 * device scratch for the whole batch: d_in [N][C][H][W], d_in_padded (in the plan's layout),
 * d_out.  Requires
 * skc_plan_upload.  Errors: as skc_pad_input / skc_sparse_conv_forward, SKC_ERR_CUDA for
 * stream/copy failures. */
skc_status skc_forward_host(const skc_plan *plan, const float *h_in, float *h_out, int N,
                            float *d_in, float *d_in_padded, float *d_out, void *stream);

/* Layout function f(c,y,x) of the padded input: test hook.
 * Returns -1 when (c,y,x) is outside [0,C) x [0,Hp) x [0,Wp). */
int64_t skc_layout_offset(const skc_plan *plan, int c, int y, int x);

/* JIT kernel only: generate, compile (PTX compiler library, one module per channel block,
 * in parallel host threads) and link (nvJitLink) the plan's code now, on the host -- no GPU
 * is needed.  Otherwise this happens in skc_plan_upload.  The linked cubin is cached on disk
 * under $SKC_JIT_CACHE (default $HOME/.cache/skc_jit), keyed by a hash of the generated
 * code; SKC_JIT_NOCACHE=1 disables the cache.  No-op for other kernels.
 * Errors: SKC_ERR_ARG (NULL), SKC_ERR_UNSUPPORTED (compile or link failed; message in
 * skc_last_error). */
skc_status skc_plan_compile(skc_plan *plan);

/* JIT kernel only: measure the launch-schedule variants of the plan's kernel on this device and
 * keep the fastest (first round of work items spread over the channel blocks or block-major;
 * work items numbered GPC-major or by cluster rank; clusters of 2 CTAs or none; lane table
 * dealt by shared-memory bank residue or contiguously; dry-run code prefetch by the first
 * CTAs or by every CTA -- DESIGN.md Sec. 7.4; skc_info.jit_sched reports the choice).  Times
 * each variant 5x on CALLER-OWNED scratch: d_in, a padded input of N images in the plan's
 * layout (any finite contents), d_out, an output of N images (overwritten), and optionally
 * d_flush, flush_bytes (NULL/0: no flush) -- a buffer larger than L2 that is written before
 * every timed launch so code and data start cold.  Synchronous on `stream`.  Every variant
 * computes bit-identical outputs, so tuning changes speed only.  Requires skc_plan_upload;
 * exclusive: no launch of this plan may run concurrently.  *best_ms (may be NULL) receives
 * the chosen variant's time (0 for non-JIT plans, for which this is a no-op).
 * Errors: SKC_ERR_ARG (NULL plan or scratch, N < 1), SKC_ERR_ALIGN, SKC_ERR_STATE (not
 * uploaded on this device), SKC_ERR_CUDA (a launch failed). */
skc_status skc_plan_tune(skc_plan *plan, int N, const float *d_in, float *d_out, void *d_flush,
                         size_t flush_bytes, void *stream, double *best_ms);

/* Static self-check of a plan (host only, no GPU): every kernel-private index the kernels
 * will dereference -- shared-memory windows and pixel slots against the stage and allocation
 * bounds, segment tables, op-stream structure (HDR before FMA ops, EXIT last) -- and that the
 * kernel streams decode back EXACTLY to the canonical CSR (each nonzero once, same weight
 * bits) and every output element is written exactly once.  SKC_OK or SKC_ERR_STATE with the
 * first violation in skc_last_error(). */
skc_status skc_plan_verify(const skc_plan *plan);

void skc_plan_destroy(skc_plan *plan);
const char *skc_last_error(void);

/* a7 -- roofline performance model, host fp64.
 *   C = 2*K*(C/g)*R*S*Ho*Wo*batch FLOP; S_A = 4*batch*(C*H*W + K*Ho*Wo) bytes;
 *   S_W = 4*K*(C/g)*R*S bytes (x batch unless amortised != 0).
 *   t_dense = C/F; t_sparse_compute = alpha*x*C/F; t_sparse_bw = (S_A + beta*x*S_W)/B;
 *   speedup = t_dense / max(t_sparse_compute, t_sparse_bw);
 *   x_hi = 1/alpha (sparse slower than dense above it);
 *   x_lo = S_A / (alpha*C*B/F - beta*S_W) (bandwidth crossover; +inf if denominator <= 0). */
typedef struct { double C, S_A, S_W; } skc_layer_cost;
typedef struct { double F, B, alpha, beta; } skc_platform;
typedef struct {
    double t_dense, t_sparse_compute, t_sparse_bw, t_sparse, speedup, effective_flops,
        actual_flops;
} skc_projection;
typedef struct { double x_lo, x_hi; int has_speedup_potential; } skc_window;

skc_status skc_model_layer_cost(int K, int C, int R, int S, int H, int W, int stride, int pad,
                                int groups, int64_t batch, int amortised, skc_layer_cost *out);
skc_status skc_model_project(const skc_layer_cost *cost, double x, const skc_platform *p,
                             skc_projection *out);
skc_status skc_model_window(const skc_layer_cost *cost, const skc_platform *p, skc_window *out);

/* Diagnostic: the GPC-major SM order the JIT kernel numbers its work items by (topo.cu;
 * DESIGN.md Sec. 7.4) for the current device: vid[smid] = position of SM smid when the SMs are
 * listed GPC by GPC, learned by launching thread-block clusters (which never span GPCs).
 * vid: host array of `cap` ints; *nsm receives the SM count.  Host only: returns the order the
 * probe found at the first skc_plan_upload of a JIT plan on this device.  Errors: SKC_ERR_ARG
 * (NULL, cap < SM count), SKC_ERR_STATE (no JIT plan uploaded on this device yet, or the
 * probe could not group the SMs). */
skc_status skc_sm_topology(int *vid, int cap, int *nsm);

/* Device micro-benchmarks that calibrate the B200 roofline -- the analogue of the paper's
 * measured SGEMM / STREAM "achievable" peaks: measured rates
 * rather than data-sheet numbers.  ffma: scalar FP32 FMA (16 independent chains per thread);
 * ffma2: packed fma.rn.f32x2 (FFMA2, the JIT kernel's instruction; 2 FMAs each); lds:
 * conflict-free 4-byte shared loads; lds64: conflict-free 8-byte shared loads (the JIT
 * kernel's window load).  `blocks` CTAs of 256 threads, `iters` loop trips; d_scratch: >= 4 MiB
 * device buffer (never read; defeats dead-code elimination).  *ms = device milliseconds of
 * one timed launch (after a warm-up launch), *flops / *bytes = the work it performed (FLOP =
 * 2 per FMA).  Synchronous on the legacy default stream.  Errors: SKC_ERR_ARG, SKC_ERR_CUDA. */
skc_status skc_bench_ffma(void *d_scratch, int blocks, int iters, double *ms, double *flops);
skc_status skc_bench_ffma2(void *d_scratch, int blocks, int iters, double *ms, double *flops);
skc_status skc_bench_lds(void *d_scratch, int blocks, int iters, double *ms, double *bytes);
skc_status skc_bench_lds64(void *d_scratch, int blocks, int iters, double *ms, double *bytes);

#ifdef __cplusplus
}
#endif
#endif /* SKC_H_ */
