// vec.cu — K7-K9: the SBCI update's length-n_det passes, each one fused trip through HBM with
// its dot products reduced on the fly (vector_ops.hpp:27-79, precond.hpp:30-111, sbci1.hpp:152-279).
// Element arithmetic uses explicit round-to-nearest products/sums (no FMA contraction), so every
// updated element is bit-identical to the reference's combine/axpy/scale for the same inputs;
// only the order of the dot-product sums differs (fixed-order tree: deterministic run to run).
#include <cfloat>
#include <map>
#include <mutex>
#include "common.cuh"
#include "kernels.cuh"

namespace sbg {

namespace {

constexpr int kThreads = 256;
// resident blocks per SM the k_lincomb passes with <= 4 dots are compiled for (register cap
// 65536 / (256 * 3) = 85): more warps in flight to cover HBM latency (c4 commit pass, 11 vectors:
// 3.24 -> 2.90 ms under ncu)
#ifndef SBG_VEC_MINB
#define SBG_VEC_MINB 3
#endif

// Where a pass's dot products go: per-block partial sums, the final sums, and the ticket counter
// that elects the last block to finish them (so a pass is one launch, not pass + finish kernel).
struct RedOut {
    double* partial;  // [grid][kMaxRed]
    double* result;   // [kMaxRed]
    unsigned int* ticket;
    double* mirror;                // mapped host copy of result (nullptr: none)
    unsigned long long* flag;      // mapped host flag, set to seq once mirror is written
    unsigned long long seq;
};

// ndot: the dots this launch will finish (0: none — the zero-copy sequence is not advanced)
inline RedOut red_out(const ReduceWs& ws, int ndot) {
    RedOut r{ws.partial, ws.result, ws.ticket, nullptr, nullptr, 0};
    if (ws.zc && ndot > 0) {
        r.mirror = ws.zc->mirror;
        r.flag = ws.zc->flag;
        r.seq = ++ws.zc->seq;
        ws.zc->fresh = true;
    }
    return r;
}

template <int ND>
__device__ __forceinline__ void block_reduce_store(double (&acc)[ND], int ndot, const RedOut ro) {
    static_assert(ND <= kMaxRed, "reduction width");
    __shared__ double red[kThreads / 32][ND];
    __shared__ bool last;
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
        ro.partial[blockIdx.x * kMaxRed + threadIdx.x] = s;
    }
    if (ndot <= 0) return;
    // the last block to arrive sums every block's partials — in the fixed order of
    // k_reduce_finish (lane-strided, then a shuffle tree), so the results do not depend on which
    // block is last
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ro.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int nblk = gridDim.x, nw = blockDim.x >> 5;
    for (int d = w; d < ndot; d += nw) {
        double s = 0.0;
        for (int b = lane; b < nblk; b += 32) s += __ldcg(ro.partial + b * kMaxRed + d);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
            ro.result[d] = s;
            if (ro.mirror) ro.mirror[d] = s;
        }
    }
    if (ro.mirror) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence_system();  // the mirrored sums reach host memory before the flag does
            *reinterpret_cast<volatile unsigned long long*>(ro.flag) = ro.seq;
        }
    }
    if (threadIdx.x == 0) *ro.ticket = 0u;  // ready for the next pass on this stream
}

// One fused pass: up to NI inputs, NO outputs (each a linear combination of inputs and earlier
// outputs), ND dot products between any two slots. Two elements per thread per trip (16-byte
// loads/stores: n is even and every vector base is 16-byte aligned). Slots read by dots are staged
// in shared memory so the runtime slot indices never force the slot array into local memory.
template <int NI, int NO, int ND, bool DC = false>
__global__ void __launch_bounds__(kThreads, ND > 4 ? 2 : SBG_VEC_MINB) k_lincomb(const LinArgs a, const RedOut partial) {
    constexpr int NDS = ND > 0 ? ND : 1;
    __shared__ double stage[ND > 0 ? kMaxIn + kMaxOut : 1][kThreads];
    // DC: the coefficient table comes from device memory (written by launch_step_scalars)
    __shared__ double scoef[DC ? kMaxOut : 1][DC ? kMaxIn + kMaxOut : 1];
    if constexpr (DC) {
        for (int t = threadIdx.x; t < kMaxOut * (kMaxIn + kMaxOut); t += blockDim.x)
            scoef[t / (kMaxIn + kMaxOut)][t % (kMaxIn + kMaxOut)] = a.dcoef[t];
        __syncthreads();
    }
    double acc[NDS];
#pragma unroll
    for (int d = 0; d < NDS; ++d) acc[d] = 0.0;
    const int64_t n2 = a.n >> 1, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
        double2 in[NI];
#pragma unroll
        for (int k = 0; k < NI; ++k)
            if (k < a.nin) in[k] = reinterpret_cast<const double2*>(a.in[k])[i];
        const double2 kd = (ND > 0 && a.kdot >= 0) ? reinterpret_cast<const double2*>(a.kD)[i] : make_double2(0.0, 0.0);
        double2 outv[NO];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            double s[NI + NO];
#pragma unroll
            for (int k = 0; k < NI; ++k) s[k] = (k < a.nin) ? (h ? in[k].y : in[k].x) : 0.0;
#pragma unroll
            for (int j = 0; j < NO; ++j) {
                if (j >= a.nout) break;
                double v = 0.0;
                bool first = true;
#pragma unroll
                for (int k = 0; k < NI + j; ++k) {
                    const double c = DC ? scoef[j][k < NI ? k : kMaxIn + (k - NI)] : a.coef[j][k < NI ? k : kMaxIn + (k - NI)];
                    if (c != 0.0) {
                        const double term = __dmul_rn(c, s[k]);
                        v = first ? term : __dadd_rn(v, term);
                        first = false;
                    }
                }
                s[NI + j] = v;
                if (h) outv[j].y = v;
                else outv[j].x = v;
            }
            if constexpr (ND > 0) {
#pragma unroll
                for (int k = 0; k < NI + NO; ++k) {
                    const int sid = k < NI ? k : kMaxIn + (k - NI);
                    if ((a.dmask >> sid) & 1u) stage[sid][threadIdx.x] = s[k];
                }
#pragma unroll
                for (int d = 0; d < ND; ++d) {
                    if (d >= a.ndot) break;
                    if (d == a.kdot) {
                        const double yy = stage[a.da[d]][threadIdx.x];
                        acc[d] += __dmul_rn(__dmul_rn(yy, yy), __dsub_rn(h ? kd.y : kd.x, a.kshift));
                    } else {
                        acc[d] = fma(stage[a.da[d]][threadIdx.x], stage[a.db[d]][threadIdx.x], acc[d]);
                    }
                }
            }
        }
#pragma unroll
        for (int j = 0; j < NO; ++j)
            if (j < a.nout && a.out[j]) reinterpret_cast<double2*>(a.out[j])[i] = outv[j];
    }
    if constexpr (ND > 0) block_reduce_store<NDS>(acc, a.ndot, partial);
}

__device__ __forceinline__ double precond_den(double d, double shift, double clamp) {
    const double den = __dsub_rn(d, shift);
    if (fabs(den) >= clamp) return den;
    return den < 0.0 ? -clamp : clamp;
}

template <class T>
__device__ __forceinline__ double comp(const T& v, int h) {
    return h ? v.y : v.x;
}
__device__ __forceinline__ const double2* v2(const double* p) { return reinterpret_cast<const double2*>(p); }

// mode 0: overlaps o_c = xc_c . (zres / den)
// mode 1: z = zres/den - sum_c o_c xc_c ; dots xx, xz, zz [, xy, yy, yz]
constexpr int kPrecMaxC = 8;  // PrecArgs::xc capacity
// MAXC: compile-time bound on the deflated states (0 for the ground state: no x_c registers, more
// resident blocks per SM for this HBM stream)
template <int MAXC>
__global__ void __launch_bounds__(kThreads) k_precond(const PrecArgs a, const RedOut partial) {
    double acc[8];
#pragma unroll
    for (int d = 0; d < 8; ++d) acc[d] = 0.0;
    const int64_t n2 = a.n >> 1, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
        const double2 zr = v2(a.zres)[i], D = v2(a.D)[i];
        double2 xc[MAXC > 0 ? MAXC : 1];
#pragma unroll
        for (int c = 0; c < MAXC; ++c)
            if (c < a.nxc) xc[c] = v2(a.xc[c])[i];
        if (a.mode == 0) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const double v = comp(zr, h) / precond_den(comp(D, h), a.shift, a.clamp);
#pragma unroll
                for (int c = 0; c < MAXC; ++c)
                    if (c < a.nxc) acc[c] = fma(comp(xc[c], h), v, acc[c]);
            }
        } else {
            const double2 x2 = v2(a.x)[i];
            double2 y2 = make_double2(0.0, 0.0);
            if (a.y) y2 = v2(a.y)[i];
            double2 z2;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double v = comp(zr, h) / precond_den(comp(D, h), a.shift, a.clamp);
#pragma unroll
                for (int c = 0; c < MAXC; ++c)
                    if (c < a.nxc) v = __dadd_rn(v, __dmul_rn(-a.o[c], comp(xc[c], h)));
                if (h) z2.y = v;
                else z2.x = v;
                const double x = comp(x2, h);
                acc[0] = fma(x, x, acc[0]);
                acc[1] = fma(x, v, acc[1]);
                acc[2] = fma(v, v, acc[2]);
                if (a.y) {
                    const double y = comp(y2, h);
                    acc[3] = fma(x, y, acc[3]);
                    acc[4] = fma(y, y, acc[4]);
                    acc[5] = fma(y, v, acc[5]);
                }
            }
            reinterpret_cast<double2*>(a.z)[i] = z2;
        }
    }
    const int nd = a.mode == 0 ? a.nxc : (a.y ? 6 : 3);
    block_reduce_store<8>(acc, nd, partial);
}

// basis b = {Ax x, Bx x + By y, (Cx x + Cz z) + Cy y}, images likewise; dots d_ij = b_i . B_j
__global__ void __launch_bounds__(kThreads) k_subspace(const SubArgs a, const RedOut partial) {
    double acc[9];
#pragma unroll
    for (int d = 0; d < 9; ++d) acc[d] = 0.0;
    const int64_t n2 = a.n >> 1, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
        const double2 x2 = v2(a.x)[i], z2 = v2(a.z)[i], hx2 = v2(a.hx)[i], hz2 = v2(a.hz)[i];
        double2 y2 = make_double2(0.0, 0.0), hy2 = make_double2(0.0, 0.0);
        if (a.three) {
            y2 = v2(a.y)[i];
            hy2 = v2(a.hy)[i];
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const double x = comp(x2, h), z = comp(z2, h), hx = comp(hx2, h), hz = comp(hz2, h);
            double b[3], B[3];
            b[0] = __dmul_rn(x, a.Ax);
            B[0] = __dmul_rn(hx, a.Ax);
            if (a.three) {
                const double y = comp(y2, h), hy = comp(hy2, h);
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
    }
    block_reduce_store<9>(acc, a.three ? 9 : 4, partial);
}

__global__ void k_reduce_finish(const double* partial, int nblk, int ndot, double* result) {
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int d = threadIdx.x >> 5; d < ndot; d += nw) {
        double s = 0.0;
        for (int b = lane; b < nblk; b += 32) s += partial[b * kMaxRed + d];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) result[d] = s;
    }
}

// all dots v_i . v_j (i <= j) of up to 6 vectors in one pass
__global__ void __launch_bounds__(kThreads) k_gram(const PairSubArgs a, const RedOut partial) {
    double acc[21];
#pragma unroll
    for (int d = 0; d < 21; ++d) acc[d] = 0.0;
    const int64_t n2 = a.n >> 1, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
        double2 v[6];
#pragma unroll
        for (int k = 0; k < 6; ++k)
            if (k < a.m) v[k] = reinterpret_cast<const double2*>(a.v[k])[i];
        int d = 0;
#pragma unroll
        for (int p = 0; p < 6; ++p)
#pragma unroll
            for (int q = p; q < 6; ++q, ++d)
                if (q < a.m) acc[d] = fma(v[p].y, v[q].y, fma(v[p].x, v[q].x, acc[d]));
    }
    // compact the m(m+1)/2 used accumulators to the front (row-major upper triangle of size m)
    double out[21];
    int d = 0, o = 0;
#pragma unroll
    for (int p = 0; p < 6; ++p)
#pragma unroll
        for (int q = p; q < 6; ++q, ++d)
            if (q < a.m) out[o++] = acc[d];
#pragma unroll
    for (int k = 0; k < 21; ++k)
        if (k >= o) out[k] = 0.0;
    block_reduce_store<21>(out, a.m * (a.m + 1) / 2, partial);
}

// sbci2.hpp:144-176 per element: w_i = v_i * inv_n_i (scaled copy), basis b_c = sum_i P[i][c] w_i
// accumulated in input order from zero (apply_transform, ortho.hpp:220-230), images likewise;
// cross dots b_c . B_d for c, d < r
__global__ void __launch_bounds__(kThreads) k_pair_subspace(const PairSubArgs a, const RedOut partial) {
    double acc[36];
#pragma unroll
    for (int d = 0; d < 36; ++d) acc[d] = 0.0;
    const int64_t n2 = a.n >> 1, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
        double2 v[6], h[6];
#pragma unroll
        for (int k = 0; k < 6; ++k)
            if (k < a.m) {
                v[k] = reinterpret_cast<const double2*>(a.v[k])[i];
                h[k] = reinterpret_cast<const double2*>(a.h[k])[i];
            }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            double w[6], wh[6];
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                w[k] = k < a.m ? __dmul_rn(e ? v[k].y : v[k].x, a.inv_n[k]) : 0.0;
                wh[k] = k < a.m ? __dmul_rn(e ? h[k].y : h[k].x, a.inv_n[k]) : 0.0;
            }
            double b[6], B[6];
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                double s = 0.0, S = 0.0;
#pragma unroll
                for (int k = 0; k < 6; ++k)
                    if (k < a.m) {
                        s = __dadd_rn(s, __dmul_rn(a.P[k][c], w[k]));
                        S = __dadd_rn(S, __dmul_rn(a.P[k][c], wh[k]));
                    }
                b[c] = s;
                B[c] = S;
            }
#pragma unroll
            for (int c = 0; c < 6; ++c)
#pragma unroll
                for (int d2 = 0; d2 < 6; ++d2)
                    if (c < a.r && d2 < a.r) acc[c * 6 + d2] = fma(b[c], B[d2], acc[c * 6 + d2]);
        }
    }
    double out[36];
#pragma unroll
    for (int k = 0; k < 36; ++k) out[k] = 0.0;
#pragma unroll
    for (int c = 0; c < 6; ++c)
#pragma unroll
        for (int d2 = 0; d2 < 6; ++d2)
            if (c < a.r && d2 < a.r) out[c * a.r + d2] = acc[c * 6 + d2];
    block_reduce_store<36>(out, a.r * a.r, partial);
}

__global__ void __launch_bounds__(kThreads) k_ritz(const RitzArgs a, const RedOut partial) {
    double acc[kMaxRoots];
#pragma unroll
    for (int r = 0; r < kMaxRoots; ++r) acc[r] = 0.0;
    const int64_t n2 = a.n >> 1, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n2; e += stride) {
        double2 R[kMaxRoots], H[kMaxRoots];
#pragma unroll
        for (int r = 0; r < kMaxRoots; ++r) {
            if (r >= a.k) break;
            if (a.first) {
                R[r] = make_double2(0.0, 0.0);
                H[r] = make_double2(0.0, 0.0);
            } else {
                R[r] = reinterpret_cast<const double2*>(a.ritz[r])[e];
                H[r] = reinterpret_cast<const double2*>(a.ritz_im[r])[e];
            }
        }
        for (int i = 0; i < a.m; ++i) {
            const double2 b = reinterpret_cast<const double2*>(a.b[i])[e];
            const double2 h = reinterpret_cast<const double2*>(a.h[i])[e];
#pragma unroll
            for (int r = 0; r < kMaxRoots; ++r) {
                if (r >= a.k) break;
                const double c = a.coef[i][r];
                R[r].x = __dadd_rn(R[r].x, __dmul_rn(c, b.x));
                R[r].y = __dadd_rn(R[r].y, __dmul_rn(c, b.y));
                H[r].x = __dadd_rn(H[r].x, __dmul_rn(c, h.x));
                H[r].y = __dadd_rn(H[r].y, __dmul_rn(c, h.y));
            }
        }
#pragma unroll
        for (int r = 0; r < kMaxRoots; ++r) {
            if (r >= a.k) break;
            reinterpret_cast<double2*>(a.ritz[r])[e] = R[r];
            reinterpret_cast<double2*>(a.ritz_im[r])[e] = H[r];
            if (a.last) {
                const double t = -a.theta[r];
                double2 z;
                z.x = __dadd_rn(H[r].x, __dmul_rn(t, R[r].x));
                z.y = __dadd_rn(H[r].y, __dmul_rn(t, R[r].y));
                reinterpret_cast<double2*>(a.res[r])[e] = z;
                acc[r] = fma(z.y, z.y, fma(z.x, z.x, acc[r]));
            }
        }
    }
    block_reduce_store<kMaxRoots>(acc, a.last ? a.k : 0, partial);
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
                                                      const RedOut partial) {
    double acc[1] = {0.0};
    const int64_t n2 = n >> 1, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
        const double2 yv = v2(y)[i], Dv = v2(D)[i];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const double yy = comp(yv, h);
            acc[0] += __dmul_rn(__dmul_rn(yy, yy), __dsub_rn(comp(Dv, h), shift));
        }
    }
    block_reduce_store<1>(acc, 1, partial);
}

__global__ void k_fill(double* p, int64_t n, double v) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) p[i] = v;
}

__global__ void k_set(double* p, int64_t idx, double v) { p[idx] = v; }

// resident-block grid of one kernel, capped by the partial-sum capacity
int grid_of(const void* fn, const ReduceWs& ws) {
    static std::mutex mu;
    static std::map<const void*, int> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(fn);
    if (it == cache.end()) {
        int dev = 0, nsm = 0, nb = 0;
        SBG_CUDA(cudaGetDevice(&dev));
        SBG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        SBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kThreads, 0));
        it = cache.emplace(fn, std::max(1, nb) * nsm).first;
    }
    return std::min(it->second, ws.grid);
}

void check_aligned(const void* p) {
    if (reinterpret_cast<uintptr_t>(p) & 15u) throw InvalidArgument("vector pass: device vectors must be 16-byte aligned");
}

template <int NI, int NO, int ND>
void run_lincomb(const LinArgs& a, const ReduceWs& ws, cudaStream_t st) {
    if constexpr (NO == kMaxOut && ND > 0) {
        if (a.dcoef) {
            const void* fn = reinterpret_cast<const void*>(&k_lincomb<NI, NO, ND, true>);
            const int g = grid_of(fn, ws);
            k_lincomb<NI, NO, ND, true><<<g, kThreads, 0, st>>>(a, red_out(ws, a.ndot));
            SBG_LAUNCH_CHECK();
            return;
        }
    }
    if (a.dcoef) throw InvalidArgument("launch_lincomb: device coefficients need 6 outputs and dots");
    const void* fn = reinterpret_cast<const void*>(&k_lincomb<NI, NO, ND>);
    const int g = grid_of(fn, ws);
    k_lincomb<NI, NO, ND><<<g, kThreads, 0, st>>>(a, red_out(ws, a.ndot));
    SBG_LAUNCH_CHECK();
}

template <int NI, int NO>
void run_lincomb_nd(const LinArgs& a, const ReduceWs& ws, cudaStream_t st) {
    if (a.ndot == 0) run_lincomb<NI, NO, 0>(a, ws, st);
    else if (a.ndot <= 4) run_lincomb<NI, NO, 4>(a, ws, st);
    else run_lincomb<NI, NO, kMaxDot>(a, ws, st);
}
template <int NI>
void run_lincomb_no(const LinArgs& a, const ReduceWs& ws, cudaStream_t st) {
    if (a.nout <= 2) run_lincomb_nd<NI, 2>(a, ws, st);
    else run_lincomb_nd<NI, kMaxOut>(a, ws, st);
}

}  // namespace

void launch_lincomb(const LinArgs& args, const ReduceWs& ws, cudaStream_t st) {
    if (args.nin < 0 || args.nin > kMaxIn || args.nout < 0 || args.nout > kMaxOut || args.ndot < 0 ||
        args.ndot > kMaxDot || (args.n & 1))
        throw InvalidArgument("launch_lincomb: bad pass shape");
    LinArgs a = args;
    a.dmask = 0;
    for (int d = 0; d < a.ndot; ++d) a.dmask |= (1u << a.da[d]) | (1u << a.db[d]);
    for (int k = 0; k < a.nin; ++k) check_aligned(a.in[k]);
    for (int j = 0; j < a.nout; ++j) check_aligned(a.out[j]);
    if (a.kdot >= a.ndot || (a.kdot >= 0 && !a.kD)) throw InvalidArgument("launch_lincomb: bad weighted dot");
    if (a.kdot >= 0) check_aligned(a.kD);
    if (a.nin <= 3) run_lincomb_no<3>(a, ws, st);
    else if (a.nin <= 6) run_lincomb_no<6>(a, ws, st);
    else run_lincomb_no<kMaxIn>(a, ws, st);
}

void launch_precond(const PrecArgs& a, const ReduceWs& ws, cudaStream_t st) {
    if (a.n & 1) throw InvalidArgument("launch_precond: odd length");
    if (a.nxc < 0 || a.nxc > kPrecMaxC) throw InvalidArgument("launch_precond: bad deflation count");
    const void* fn = a.nxc == 0 ? reinterpret_cast<const void*>(&k_precond<0>)
                                : reinterpret_cast<const void*>(&k_precond<kPrecMaxC>);
    const int g = grid_of(fn, ws);
    const int nd = a.mode == 0 ? a.nxc : (a.y ? 6 : 3);
    if (a.nxc == 0) k_precond<0><<<g, kThreads, 0, st>>>(a, red_out(ws, nd));
    else k_precond<kPrecMaxC><<<g, kThreads, 0, st>>>(a, red_out(ws, nd));
    SBG_LAUNCH_CHECK();
}

void launch_subspace(const SubArgs& a, const ReduceWs& ws, cudaStream_t st) {
    if (a.n & 1) throw InvalidArgument("launch_subspace: odd length");
    const int g = grid_of(reinterpret_cast<const void*>(&k_subspace), ws);
    k_subspace<<<g, kThreads, 0, st>>>(a, red_out(ws, a.three ? 9 : 4));
    SBG_LAUNCH_CHECK();
}

void launch_reduce_finish(const ReduceWs& ws, int nblk, int ndot, cudaStream_t st) {
    if (ws.zc) ws.zc->fresh = false;  // result written without the host mirror
    if (ndot < 1 || ndot > kMaxRed) throw InvalidArgument("reduce: bad dot count");
    k_reduce_finish<<<1, 32 * std::min(ndot, 32), 0, st>>>(ws.partial, nblk, ndot, ws.result);
    SBG_LAUNCH_CHECK();
}

void launch_gram(const double* const* v, int m, int64_t n, const ReduceWs& ws, cudaStream_t st) {
    if (m < 1 || m > 6 || (n & 1)) throw InvalidArgument("launch_gram: 1..6 vectors of even length");
    PairSubArgs a{};
    a.n = n;
    a.m = m;
    for (int k = 0; k < m; ++k) {
        check_aligned(v[k]);
        a.v[k] = v[k];
    }
    const int g = grid_of(reinterpret_cast<const void*>(&k_gram), ws);
    k_gram<<<g, kThreads, 0, st>>>(a, red_out(ws, m * (m + 1) / 2));
    SBG_LAUNCH_CHECK();
}

void launch_ritz(const RitzArgs& a, const ReduceWs& ws, cudaStream_t st) {
    if (a.m < 1 || a.m > kRitzChunk || a.k < 1 || a.k > kMaxRoots || (a.n & 1))
        throw InvalidArgument("launch_ritz: bad shape");
    for (int i = 0; i < a.m; ++i) {
        check_aligned(a.b[i]);
        check_aligned(a.h[i]);
    }
    const int g = grid_of(reinterpret_cast<const void*>(&k_ritz), ws);
    k_ritz<<<g, kThreads, 0, st>>>(a, red_out(ws, a.last ? a.k : 0));
    SBG_LAUNCH_CHECK();
}

void launch_pair_subspace(const PairSubArgs& a, const ReduceWs& ws, cudaStream_t st) {
    if (a.m < 1 || a.m > 6 || a.r < 1 || a.r > a.m || (a.n & 1)) throw InvalidArgument("launch_pair_subspace: bad shape");
    for (int k = 0; k < a.m; ++k) {
        check_aligned(a.v[k]);
        check_aligned(a.h[k]);
    }
    const int g = grid_of(reinterpret_cast<const void*>(&k_pair_subspace), ws);
    k_pair_subspace<<<g, kThreads, 0, st>>>(a, red_out(ws, a.r * a.r));
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
    if (n & 1) throw InvalidArgument("launch_kinetic: odd length");
    const int g = grid_of(reinterpret_cast<const void*>(&k_kinetic), ws);
    k_kinetic<<<g, kThreads, 0, st>>>(y, D, shift, n, red_out(ws, 1));
    SBG_LAUNCH_CHECK();
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
