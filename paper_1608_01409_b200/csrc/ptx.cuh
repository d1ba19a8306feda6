// ptx.cuh -- thin inline-PTX wrappers for sm_100a: mbarrier, TMA bulk copy, fast division.
#pragma once
#include <cstdint>

namespace skc {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

// Make barrier initialisation visible to the async (TMA) proxy.
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "SKC_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra SKC_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// TMA bulk copy global -> shared (non-tensor), completion reported to `bar` as tx bytes.
// dst, src 16-byte aligned; bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// 4-byte asynchronous global -> shared copy (LDGSTS), completion tracked per thread.
__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src)
                 : "memory");
}

// Arrive on `bar` once all of this thread's prior cp.async copies have completed; the
// arrival is pre-counted in the barrier's initial count (.noinc).
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t *bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// Division by a runtime-constant divisor d (1 <= d < 2^31) for n < 2^31: q = (mulhi(n,m)+n)>>s.
struct FastDiv {
    uint32_t d, m, s;
};

inline FastDiv make_fastdiv(uint32_t d) {
    uint32_t s = 0;
    while (s < 32 && (1u << s) < d) ++s;
    const uint64_t one = 1;
    const uint64_t m = ((one << 32) * ((one << s) - d)) / d + 1;
    return FastDiv{d, static_cast<uint32_t>(m), s};
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv &f) {
    return (__umulhi(n, f.m) + n) >> f.s;
}

// Output element index of (image n, channel k, padded row yy, padded column xx) in the
// epilogue's output layout: olay 0 = [N][K][Hop][Wop]; olay 1 = image-pair interleaved
// [ceil(N/2)][K][Hop][Wop][2] (the padded input layout of a JIT plan, for chaining).
__device__ __forceinline__ int64_t out_index(int64_t n, int k, int yy, int xx, int K, int Hop,
                                             int Wop, int olay) {
    if (!olay) return ((n * K + k) * Hop + yy) * int64_t(Wop) + xx;
    return ((((n >> 1) * K + k) * Hop + yy) * int64_t(Wop) + xx) * 2 + (n & 1);
}

}  // namespace skc
