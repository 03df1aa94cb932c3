// spin.cu — <S^2> of a CI vector on the device (reference: fci/spin.hpp:17-51).
//   <S^2> = |S+ x|^2 / |x|^2 + S_z (S_z + 1),  S+ : (n_a, n_b) -> (n_a + 1, n_b - 1)
// The reference scatters w[a + p, b - p] += sign * x[a, b] over every source determinant; here every
// thread owns one target determinant (a2, b2) of the raised sector and gathers its sources
// x[a2 - p, b2 + p] for p in a2 \ b2, in the order the reference's scatter reaches that target
// (source alpha rank ascending = p descending), then accumulates w^2 — S+ x is never stored.
#include "common.cuh"
#include "kernels.cuh"

namespace sbg {

namespace {

constexpr int kSpinThreads = 256;

__global__ void __launch_bounds__(kSpinThreads) k_spin_raise(const double* x, int64_t ld, int na, int nb, int norb,
                                                             int64_t ja_lo, int64_t ja_hi, int64_t NB2,
                                                             double* partial) {
    __shared__ int s_ia[64], s_pb[64];
    __shared__ double red[kSpinThreads / 32];
    double acc = 0.0;
    for (int64_t ja = ja_lo + blockIdx.x; ja < ja_hi; ja += gridDim.x) {
        const uint64_t a2 = string_unrank((uint64_t)ja, na + 1, norb);
        __syncthreads();
        if (threadIdx.x < norb) {
            const int p = threadIdx.x;
            s_ia[p] = ((a2 >> p) & 1) ? (int)string_rank(a2 ^ ((uint64_t)1 << p)) : -1;
            s_pb[p] = pop_below(a2, p);
        }
        __syncthreads();
        for (int64_t jb = threadIdx.x; jb < NB2; jb += blockDim.x) {
            const uint64_t b2 = string_unrank((uint64_t)jb, nb - 1, norb);
            double w = 0.0;
            for (int p = norb - 1; p >= 0; --p) {
                const int ia = s_ia[p];
                if (ia < 0 || ((b2 >> p) & 1)) continue;
                const uint64_t b = b2 | ((uint64_t)1 << p);
                const int phase = na + pop_below(b2, p) + s_pb[p];
                const double c = x[(int64_t)ia * ld + string_rank(b)];
                w += (phase & 1) ? -c : c;
            }
            acc = fma(w, w, acc);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < kSpinThreads / 32; ++i) s += red[i];
        partial[blockIdx.x * kMaxRed] = s;
    }
}

}  // namespace

void launch_spin_raise(const double* x_full, int64_t ld, int na, int nb, int norb, int64_t ja_lo, int64_t ja_hi,
                       const ReduceWs& ws, cudaStream_t st) {
    ensure_binomials();
    if (norb > 64 || na + 1 > norb || nb < 1) throw InvalidArgument("spin_raise: sector has no S+ image");
    const int64_t NB2 = (int64_t)binom_host_calc(norb, nb - 1);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ws.grid, ja_hi - ja_lo));
    k_spin_raise<<<grid, kSpinThreads, 0, st>>>(x_full, ld, na, nb, norb, ja_lo, ja_hi, NB2, ws.partial);
    SBG_LAUNCH_CHECK();
    launch_reduce_finish(ws, grid, 1, st);
}

}  // namespace sbg
