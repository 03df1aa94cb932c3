// vec.cu — K7-K9: the SBCI update's length-n_det passes, each one fused trip through HBM with
// its dot products reduced on the fly (vector_ops.hpp:27-79, precond.hpp:30-111, sbci1.hpp:152-279).
// Element arithmetic uses explicit round-to-nearest products/sums (no FMA contraction), so every
// updated element is bit-identical to the reference's combine/axpy/scale for the same inputs;
// only the order of the dot-product sums differs (fixed-order tree: deterministic run to run).
#include <cfloat>
#include "common.cuh"
#include "kernels.cuh"

namespace sbg {

namespace {

constexpr int kThreads = 256;

template <int ND>
__device__ __forceinline__ void block_reduce_store(double (&acc)[ND], int ndot, double* partial) {
    __shared__ double red[kThreads / 32][kMaxDot];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
        if (d >= ndot) break;
        double v = acc[d];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[w][d] = v;
    }
    __syncthreads();
    if (threadIdx.x < ndot) {
        double s = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i][threadIdx.x];
        partial[blockIdx.x * kMaxDot + threadIdx.x] = s;
    }
}

__global__ void __launch_bounds__(kThreads) k_lincomb(const LinArgs a, double* partial) {
    double acc[kMaxDot];
#pragma unroll
    for (int d = 0; d < kMaxDot; ++d) acc[d] = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += stride) {
        double s[kMaxIn + kMaxOut];
#pragma unroll
        for (int k = 0; k < kMaxIn; ++k) s[k] = (k < a.nin) ? a.in[k][i] : 0.0;
#pragma unroll
        for (int j = 0; j < kMaxOut; ++j) {
            if (j >= a.nout) break;
            double v = 0.0;
            bool first = true;
#pragma unroll
            for (int k = 0; k < kMaxIn + kMaxOut; ++k) {
                if (k >= kMaxIn && k - kMaxIn >= j) break;
                const double c = a.coef[j][k];
                if (c != 0.0) {
                    const double term = __dmul_rn(c, s[k]);
                    v = first ? term : __dadd_rn(v, term);
                    first = false;
                }
            }
            s[kMaxIn + j] = v;
            if (a.out[j]) a.out[j][i] = v;
        }
#pragma unroll
        for (int d = 0; d < kMaxDot; ++d) {
            if (d >= a.ndot) break;
            acc[d] = fma(s[a.da[d]], s[a.db[d]], acc[d]);
        }
    }
    block_reduce_store<kMaxDot>(acc, a.ndot, partial);
}

__device__ __forceinline__ double precond_den(double d, double shift, double clamp) {
    const double den = __dsub_rn(d, shift);
    if (fabs(den) >= clamp) return den;
    return den < 0.0 ? -clamp : clamp;
}

// mode 0: overlaps o_c = xc_c . (zres / den)
// mode 1: z = zres/den - sum_c o_c xc_c ; dots xx, xz, zz [, xy, yy, yz]
__global__ void __launch_bounds__(kThreads) k_precond(const PrecArgs a, double* partial) {
    double acc[8];
#pragma unroll
    for (int d = 0; d < 8; ++d) acc[d] = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += stride) {
        double v = a.zres[i] / precond_den(a.D[i], a.shift, a.clamp);
        if (a.mode == 0) {
#pragma unroll
            for (int c = 0; c < 8; ++c)
                if (c < a.nxc) acc[c] = fma(a.xc[c][i], v, acc[c]);
        } else {
#pragma unroll
            for (int c = 0; c < 8; ++c)
                if (c < a.nxc) v = __dadd_rn(v, __dmul_rn(-a.o[c], a.xc[c][i]));
            a.z[i] = v;
            const double x = a.x[i];
            acc[0] = fma(x, x, acc[0]);
            acc[1] = fma(x, v, acc[1]);
            acc[2] = fma(v, v, acc[2]);
            if (a.y) {
                const double y = a.y[i];
                acc[3] = fma(x, y, acc[3]);
                acc[4] = fma(y, y, acc[4]);
                acc[5] = fma(y, v, acc[5]);
            }
        }
    }
    const int nd = a.mode == 0 ? a.nxc : (a.y ? 6 : 3);
    block_reduce_store<8>(acc, nd, partial);
}

// basis b = {Ax x, Bx x + By y, (Cx x + Cz z) + Cy y}, images likewise; dots d_ij = b_i . B_j
__global__ void __launch_bounds__(kThreads) k_subspace(const SubArgs a, double* partial) {
    double acc[9];
#pragma unroll
    for (int d = 0; d < 9; ++d) acc[d] = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += stride) {
        const double x = a.x[i], z = a.z[i], hx = a.hx[i], hz = a.hz[i];
        double b[3], B[3];
        b[0] = __dmul_rn(x, a.Ax);
        B[0] = __dmul_rn(hx, a.Ax);
        if (a.three) {
            const double y = a.y[i], hy = a.hy[i];
            b[1] = __dadd_rn(__dmul_rn(a.Bx, x), __dmul_rn(a.By, y));
            B[1] = __dadd_rn(__dmul_rn(a.Bx, hx), __dmul_rn(a.By, hy));
            b[2] = __dadd_rn(__dadd_rn(__dmul_rn(a.Cx, x), __dmul_rn(a.Cz, z)), __dmul_rn(a.Cy, y));
            B[2] = __dadd_rn(__dadd_rn(__dmul_rn(a.Cx, hx), __dmul_rn(a.Cz, hz)), __dmul_rn(a.Cy, hy));
#pragma unroll
            for (int p = 0; p < 3; ++p)
#pragma unroll
                for (int q = 0; q < 3; ++q) acc[p * 3 + q] = fma(b[p], B[q], acc[p * 3 + q]);
        } else {
            b[1] = __dadd_rn(__dmul_rn(a.Cx, x), __dmul_rn(a.Cz, z));
            B[1] = __dadd_rn(__dmul_rn(a.Cx, hx), __dmul_rn(a.Cz, hz));
#pragma unroll
            for (int p = 0; p < 2; ++p)
#pragma unroll
                for (int q = 0; q < 2; ++q) acc[p * 2 + q] = fma(b[p], B[q], acc[p * 2 + q]);
        }
    }
    block_reduce_store<9>(acc, a.three ? 9 : 4, partial);
}

__global__ void k_reduce_finish(const double* partial, int nblk, int ndot, double* result) {
    const int d = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (d >= ndot) return;
    double s = 0.0;
    for (int b = lane; b < nblk; b += 32) s += partial[b * kMaxDot + d];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) result[d] = s;
}

__device__ __forceinline__ bool lex_less(double v1, int64_t i1, double v2, int64_t i2) {
    return v1 < v2 || (v1 == v2 && i1 < i2);
}

__global__ void k_argmin_after(const double* D, int64_t nrows, int64_t ncols, int64_t ld, int64_t row_lo,
                               double prev_v, int64_t prev_i, double* part_v, int64_t* part_i) {
    double bv = DBL_MAX;
    int64_t bi = INT64_MAX;
    const int64_t n = nrows * ld, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += stride) {
        const int64_t r = k / ld, c = k % ld;
        if (c >= ncols) continue;
        const int64_t gi = (row_lo + r) * ncols + c;
        const double v = D[k];
        if (lex_less(prev_v, prev_i, v, gi) && lex_less(v, gi, bv, bi)) {
            bv = v;
            bi = gi;
        }
    }
    __shared__ double sv[kThreads];
    __shared__ int64_t si[kThreads];
    sv[threadIdx.x] = bv;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s && lex_less(sv[threadIdx.x + s], si[threadIdx.x + s], sv[threadIdx.x], si[threadIdx.x])) {
            sv[threadIdx.x] = sv[threadIdx.x + s];
            si[threadIdx.x] = si[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part_v[blockIdx.x] = sv[0];
        part_i[blockIdx.x] = si[0];
    }
}

// sum_i y_i^2 (D_i - shift)  (kinetic_scalar, sbci1.hpp:135-139)
__global__ void __launch_bounds__(kThreads) k_kinetic(const double* y, const double* D, double shift, int64_t n,
                                                      double* partial) {
    double acc[1] = {0.0};
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        acc[0] += __dmul_rn(__dmul_rn(y[i], y[i]), __dsub_rn(D[i], shift));
    block_reduce_store<1>(acc, 1, partial);
}

__global__ void k_fill(double* p, int64_t n, double v) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) p[i] = v;
}

__global__ void k_set(double* p, int64_t idx, double v) { p[idx] = v; }

}  // namespace

void launch_lincomb(const LinArgs& a, const ReduceWs& ws, cudaStream_t st) {
    k_lincomb<<<ws.grid, kThreads, 0, st>>>(a, ws.partial);
    SBG_LAUNCH_CHECK();
    if (a.ndot > 0) launch_reduce_finish(ws, a.ndot, st);
}

void launch_precond(const PrecArgs& a, const ReduceWs& ws, cudaStream_t st) {
    k_precond<<<ws.grid, kThreads, 0, st>>>(a, ws.partial);
    SBG_LAUNCH_CHECK();
    const int nd = a.mode == 0 ? a.nxc : (a.y ? 6 : 3);
    if (nd > 0) launch_reduce_finish(ws, nd, st);
}

void launch_subspace(const SubArgs& a, const ReduceWs& ws, cudaStream_t st) {
    k_subspace<<<ws.grid, kThreads, 0, st>>>(a, ws.partial);
    SBG_LAUNCH_CHECK();
    launch_reduce_finish(ws, a.three ? 9 : 4, st);
}

void launch_reduce_finish(const ReduceWs& ws, int ndot, cudaStream_t st) {
    k_reduce_finish<<<1, 32 * kMaxDot, 0, st>>>(ws.partial, ws.grid, ndot, ws.result);
    SBG_LAUNCH_CHECK();
}

void launch_argmin_after(const double* D, int64_t nrows, int64_t ncols, int64_t ld, int64_t row_lo, double prev_v,
                         int64_t prev_i, double* out_v, int64_t* out_i, double* part_v, int64_t* part_i, int grid,
                         cudaStream_t st) {
    (void)out_v;
    (void)out_i;
    k_argmin_after<<<grid, kThreads, 0, st>>>(D, nrows, ncols, ld, row_lo, prev_v, prev_i, part_v, part_i);
    SBG_LAUNCH_CHECK();
}

void launch_kinetic(const double* y, const double* D, double shift, int64_t n, const ReduceWs& ws, cudaStream_t st) {
    k_kinetic<<<ws.grid, kThreads, 0, st>>>(y, D, shift, n, ws.partial);
    SBG_LAUNCH_CHECK();
    launch_reduce_finish(ws, 1, st);
}

void launch_fill(double* p, int64_t n, double v, cudaStream_t st) {
    if (n <= 0) return;
    k_fill<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0, st>>>(p, n, v);
    SBG_LAUNCH_CHECK();
}

void launch_set_element(double* p, int64_t idx, double v, cudaStream_t st) {
    k_set<<<1, 1, 0, st>>>(p, idx, v);
    SBG_LAUNCH_CHECK();
}

}  // namespace sbg
