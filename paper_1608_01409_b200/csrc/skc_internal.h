// skc_internal.h -- private interface between the host library (plan.cpp) and the CUDA
// kernels (pad.cu, sconv_direct.cu, sconv_regtile.cu).  Not part of the C-ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace skc {

constexpr int kMaxStages = 8;

// One kernel-private nonzero: the weight and its offset relative to the base of the
// shared-memory stage that holds its input channel (colidx = f(c,r,s),
// re-encoded against the staged slab instead of the whole padded tensor).
struct Nz {
    float w;
    int32_t off;
};

// Geometry of the staging pipeline shared by both conv kernels.
//  - A work item is (image n, output-row band, block of output channels of one group).
//  - Input channels of the group are staged CB at a time ("column blocking")
//    into a ring of NS shared-memory stages; each stage holds CB channels x BHin rows x Wp.
struct StageGeom {
    int N, C, K, Kg, Cg, Hp, Wp, Ho, Wo, stride;
    int BH;         // output rows per band
    int BHin;       // input rows staged per band = (BH-1)*stride + R
    int nbands;
    int CB;         // input channels per stage
    int nchunks;    // ceil(Cg / CB)
    int NS;         // stages in the ring
    int stage_floats;  // floats per stage (multiple of 4)
    int tail_floats;   // slack after the last stage: junk lane slots may read past a stage
    int bulk;       // 1: cp.async.bulk (TMA) staging; 0: LSU copy fallback
    int whole;      // 1: band covers all Hp rows -> one bulk copy per stage
};

struct DirectParams {
    StageGeom g;
    const float *in;       // padded input [N][C][Hp][Wp]
    float *out;            // [N][K][Ho][Wo]
    const Nz *nz;          // streams in perm order, chunk-major inside each row
    const int32_t *chunkptr;  // [K][nchunks+1] absolute indices into nz
    const int32_t *perm;   // perm position -> output channel
    int NW;                // compute warps per CTA
    int M;                 // channels per warp
    int cblocks;           // channel blocks per group = ceil(Kg / (NW*M))
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
    const int32_t *lanemap;  // [NG][32] (img << 24) | (y0 << 12) | x0, or -1
    int N, C, K, Cg, Kg, Hp, Wp, Ho, Wo, groups;
    int NI, CB, nchunks, NS;
    int img_stride;          // floats between image slots of a stage (multiple of 4)
    int slab_floats;         // NI * img_stride
    int stream_cap;          // uint2 entries per stage stream area (incl. slack)
    int stage_floats;        // slab_floats + 2 * stream_cap
    int NG, NT, nblocks;
};

struct RegtileShape {
    int R, S, TY, TX, M;
    int nwmax, minb;  // __launch_bounds__(nwmax*32, minb): register cap of the instance
};

// Launchers (defined in the .cu files).  Return cudaError_t of the launch.
cudaError_t launch_pad(const float *in, float *out, int64_t N, int C, int H, int W, int pad,
                       cudaStream_t st);
cudaError_t launch_direct(const DirectParams &p, int T, bool pitch, size_t smem,
                          cudaStream_t st);
bool direct_supported(int T, int M);
cudaError_t launch_regtile(const RegtileParams &p, const RegtileShape &sh, size_t smem,
                           cudaStream_t st);
// Instantiated register-tile shapes (count returned, shapes written to out[0..max)).
int regtile_shapes(RegtileShape *out, int max);
cudaError_t bench_ffma(void *scratch, int blocks, int iters, float *ms, double *flops);
cudaError_t bench_lds(void *scratch, int blocks, int iters, float *ms, double *bytes);

}  // namespace skc
