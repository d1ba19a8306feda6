// SM topology probe: which SMs share a GPC.  Thread-block clusters are always placed inside
// one GPC, so launching clusters of 16 / 8 / 4 CTAs (one CTA per SM, held resident) and
// joining the SMs of each cluster groups the SMs by GPC.  The JIT kernel uses the grouping
// to give the CTAs of one GPC neighbouring work items (the same channel block, whose code
// the GPC's shared instruction cache then holds for all of them); see jit.cpp.
#include "skc_internal.h"

#include <algorithm>
#include <mutex>
#include <numeric>
#include <vector>

namespace skc {
namespace {

__global__ void topo_probe_kernel(int *out, long long spin) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (threadIdx.x == 0) out[blockIdx.x] = int(smid);
    const long long t0 = clock64();
    while (clock64() - t0 < spin) {
    }
}

int find(std::vector<int> &par, int a) {
    while (par[size_t(a)] != a) a = par[size_t(a)] = par[size_t(par[size_t(a)])];
    return a;
}

}  // namespace

// vid[smid] = position of the SM in a GPC-major order (GPCs by lowest SM id, SMs ascending
// within a GPC); empty if the probe fails.  Computed once per device, synchronously on the
// caller's stream `st` with the caller's device scratch (skc_plan_upload passes a region of the
// plan workspace: libskc allocates no device memory).  Later calls return the cached order.
const std::vector<uint16_t> &sm_gpc_order(int dev, int *d, size_t scratch_ints, cudaStream_t st) {
    static std::mutex mu;
    static std::vector<std::vector<uint16_t>> cache(64);
    static std::vector<char> done(64, 0);
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 0 || dev >= 64) return cache[0];
    if (done[size_t(dev)] || !d) return cache[size_t(dev)];
    done[size_t(dev)] = 1;
    int nsm = 0;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || nsm < 1 ||
        nsm > 4096)
        return cache[size_t(dev)];
    std::vector<int> par(static_cast<size_t>(nsm));
    std::iota(par.begin(), par.end(), 0);
    const int smem = 160 * 1024;  // one CTA per SM
    bool ok = cudaFuncSetAttribute(topo_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   smem) == cudaSuccess;
    cudaFuncSetAttribute(topo_probe_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int linked = 0;
    for (int cs : {16, 8, 4, 2}) {
        if (!ok) break;
        cudaLaunchConfig_t lc{};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = unsigned(cs);
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        lc.blockDim = dim3(32);
        lc.dynamicSmemBytes = smem;
        lc.stream = st;
        lc.gridDim = dim3(unsigned(cs));
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, topo_probe_kernel, &lc) != cudaSuccess || ncl < 1) {
            cudaGetLastError();
            continue;
        }
        const int n = int(std::min<size_t>(size_t(ncl) * cs, scratch_ints));
        if (n < cs) continue;
        lc.gridDim = dim3(unsigned(n / cs * cs));
        std::vector<int> h(static_cast<size_t>(n));
        if (cudaLaunchKernelEx(&lc, topo_probe_kernel, d, 200000LL) != cudaSuccess ||
            cudaMemcpyAsync(h.data(), d, sizeof(int) * size_t(n), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
            cudaGetLastError();
            ok = false;
            break;
        }
        for (int c = 0; c + cs <= n; c += cs)
            for (int r = 1; r < cs; ++r) {
                const int a = h[size_t(c)], b = h[size_t(c + r)];
                if (a < 0 || a >= nsm || b < 0 || b >= nsm) continue;
                const int ra = find(par, a), rb = find(par, b);
                if (ra != rb) {
                    par[size_t(std::max(ra, rb))] = std::min(ra, rb);
                    ++linked;
                }
            }
    }
    if (!ok || linked == 0) return cache[size_t(dev)];
    // GPC-major order: groups by their lowest SM id (the root, since unions keep the minimum)
    std::vector<uint16_t> vid(static_cast<size_t>(nsm));
    int next = 0;
    for (int g = 0; g < nsm; ++g) {
        if (find(par, g) != g) continue;
        for (int s = g; s < nsm; ++s)
            if (find(par, s) == g) vid[size_t(s)] = uint16_t(next++);
    }
    cache[size_t(dev)] = vid;
    return cache[size_t(dev)];
}

bool sm_gpc_order_cached(int dev, std::vector<uint16_t> *out) {
    const std::vector<uint16_t> &v = sm_gpc_order(dev, nullptr, 0, nullptr);
    if (v.empty()) return false;
    *out = v;
    return true;
}

}  // namespace skc
