// common.cuh — shared helpers for the sm_100a kernels: error plumbing, combinatorial
// string addressing (colex rank == position in the reference's increasing-integer
// enumeration, determinants.hpp:41-59/88-92), and the FP64 tensor-core (DMMA) wrappers.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace sbg {

struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess)
        throw DeviceError(std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what + " at " + file + ":" +
                          std::to_string(line));
}
#define SBG_CUDA(x) ::sbg::cuda_check((x), #x, __FILE__, __LINE__)
#define SBG_LAUNCH_CHECK() ::sbg::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

constexpr int kMaxOrb = 32;   // FciProblem::resize bound (fcidump.hpp:36)
constexpr int kBinRows = 65;

__host__ __device__ inline uint64_t binom_host_calc(int n, int k) {
    if (k < 0 || k > n) return 0;
    if (k > n - k) k = n - k;
    uint64_t r = 1;
    for (int i = 1; i <= k; ++i) r = r * (uint64_t)(n - k + i) / (uint64_t)i;
    return r;
}

// Binomial table C(n,k) for n < 65, k < 34 in constant memory. Constant memory is per translation
// unit (no -rdc), so every .cu that uses it calls ensure_binomials() before its launches.
static __constant__ uint64_t c_binom[kBinRows][34];
static inline void ensure_binomials() {
    static int done[64] = {0};
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice", __FILE__, __LINE__);
    if (dev < 64 && done[dev]) return;
    uint64_t h[kBinRows][34];
    for (int n = 0; n < kBinRows; ++n)
        for (int k = 0; k < 34; ++k) h[n][k] = binom_host_calc(n, k);
    cuda_check(cudaMemcpyToSymbol(c_binom, h, sizeof(h)), "cudaMemcpyToSymbol", __FILE__, __LINE__);
    if (dev < 64) done[dev] = 1;
}

__device__ __forceinline__ uint64_t dbinom(int n, int k) { return (k < 0 || k > n) ? 0 : c_binom[n][k]; }

// colex rank of an occupation bitmask: sum_i C(c_i, i), c_1 < c_2 < ... the set bits.
__device__ __forceinline__ uint32_t string_rank(uint64_t s) {
    uint64_t r = 0;
    int i = 1;
    while (s) {
        const int c = __ffsll((long long)s) - 1;
        r += c_binom[c][i];
        ++i;
        s &= s - 1;
    }
    return (uint32_t)r;
}

// inverse of string_rank for k electrons in norb orbitals
__device__ __forceinline__ uint64_t string_unrank(uint64_t r, int k, int norb) {
    uint64_t s = 0;
    int c = norb - 1;
    for (int i = k; i >= 1; --i) {
        while (c_binom[c][i] > r) --c;
        s |= (uint64_t)1 << c;
        r -= c_binom[c][i];
        --c;
    }
    return s;
}

__device__ __forceinline__ int pop_below(uint64_t s, int orb) {
    return __popcll(s & (((uint64_t)1 << orb) - 1));
}

// packed symmetric pair index (p >= q): p(p+1)/2 + q
__host__ __device__ __forceinline__ int pair_sym(int p, int q) {
    return p >= q ? p * (p + 1) / 2 + q : q * (q + 1) / 2 + p;
}
// packed strict pair index (p < r): r(r-1)/2 + p
__host__ __device__ __forceinline__ int pair_strict(int p, int r) { return r * (r - 1) / 2 + p; }

// ---- FP64 tensor core (DMMA) wrappers; fragment layouts verified by sbg_selftest() ----
// m16n8k4: A 16x4 (row): a0=(g,t) a1=(g+8,t); B 4x8 (col): b0=(t,g); C 16x8: c0=(g,2t) c1=(g,2t+1) c2=(g+8,2t) c3=(g+8,2t+1)
__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a0), "d"(a1), "d"(b));
}
// m8n8k4: A 8x4: a0=(g,t); B 4x8: b0=(t,g); C 8x8: c0=(g,2t) c1=(g,2t+1)
__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- bulk copies (TMA engine, SASS UBLKCP) completing on an mbarrier ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// make the barrier initialisation visible to the async proxy (the bulk-copy engine)
__device__ __forceinline__ void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
// one arrival that also announces `bytes` of transactions the copies will complete
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// plain arrival (release at CTA scope): the arriving thread's earlier shared-memory accesses are
// ordered before the phase completion another thread observes with mbar_wait_parity
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// arrival that fires once every cp.async this thread has issued so far has landed (the barrier's
// count already includes it: .noinc) — the loader never blocks on its own copies
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// generic-proxy accesses to shared memory before this point are ordered before later async-proxy
// (bulk copy) writes by the same thread — the WAR hand-off when a consumed buffer is refilled
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// global -> shared bulk copy of `bytes` (multiple of 16, both addresses 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(smem_dst)),
                 "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// shared -> global bulk reduction gdst[i] += ssrc[i] (f64, `bytes` a multiple of 16, both
// 16-byte aligned), tracked per issuing thread in bulk async-groups (SASS UBLKRED)
__device__ __forceinline__ void bulk_reduce_add_f64(double* gdst, const double* ssrc, uint32_t bytes) {
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;\n" ::"l"(gdst),
                 "r"(smem_u32(ssrc)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
// this thread's bulk groups have finished READING their shared-memory sources
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
// ... and have completed (writes performed)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ void red_add_f64(double* p, double v) {
    asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;\n" ::"l"(p), "d"(v) : "memory");
}

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

}  // namespace sbg
