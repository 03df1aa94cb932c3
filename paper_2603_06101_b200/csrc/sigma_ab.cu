// sigma_ab.cu — K6: opposite-spin sigma term as gather -> FP64 tensor-core DGEMM -> scatter.
//
//   sigma_ab(Ia, Ib) = sum_{pq,rs} V'(pq,rs) <Ia|E^a_pq|Ja> <Ib|E^b_rs|Jb> c(Ja,Jb)
//   V'(pq,rs) = (pq|rs) + h_pq d_rs / n_beta + d_pq h_rs / n_alpha      (one-body folded in)
//
// is the reference's spin-summed contraction (fci/sigma.hpp:86-137) restricted to its alpha-beta
// cross terms plus both one-body terms; the same-spin two-body terms come from sigma_ss.cu.
// One CTA owns one alpha row Ia at a time (persistent over rows) and keeps sigma(Ia,:) in shared
// memory. Per 32-column tile of beta strings Jb:
//   gather  D[k][Jb] = c(J_k, Jb) for the K = 1 + n_a(norb-n_a) distinct alpha strings J_k linked
//           to Ia (k=0 is Ia itself carrying all occupation entries; sigma.hpp:33-35) — cp.async,
//           3-stage pipeline;
//   DGEMM   G[rs][Jb] = sum_k A[rs][k] D[k][Jb], A[rs][k] = sign_k V'(pair_k, rs), M = npair =
//           norb(norb+1)/2 packed symmetric pairs, A resident in registers for the whole row —
//           mma.sync m16n8k4 / m8n8k4 f64 (SASS DMMA.8x8x4);
//   scatter G[rs][Jb] -> sigma(Ia, E_rs Jb) with the beta link sign, fp64 shared-memory atomics.
// The row is then written once: y(Ia,:) = [y(Ia,:)] + sigma_row + e_core c(Ia,:).
#include <algorithm>
#include "common.cuh"
#include "kernels.cuh"

namespace sbg {

namespace {

constexpr int NT = 32;        // beta-string tile width (columns per tile)
constexpr int DSTRIDE = 36;   // smem row stride of a D tile (bank-conflict-free B fragments)
constexpr int STAGES = 3;

struct AbParams {
    const double* x;
    double* y;
    const double* Vp;
    const uint16_t* codes;
    int norb, na_el, npair, npad, mb16, extra, K, KP;
    int64_t NB, ld, row_lo, row_hi;
    double e_core;
    int accumulate;
};

template <int KS>
__global__ void __launch_bounds__(288, 1) k_sigma_ab(const AbParams p) {
    extern __shared__ __align__(16) double smem[];
    const int KP = KS * 4;
    double* srow = smem;                                  // [ld]
    double* Ds = smem + p.ld;                             // [STAGES][KP][DSTRIDE]
    int* sJ = reinterpret_cast<int*>(Ds + STAGES * KP * DSTRIDE);  // [KP]
    int* sPair = sJ + KP;                                 // [KP]  -1 = occupation row, -2 = padding
    double* sSign = reinterpret_cast<double*>(sPair + KP + (KP & 1));  // [KP]

    const int tid = threadIdx.x, nthr = blockDim.x;
    const int w = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int norb = p.norb, npair = p.npair;
    const int ntiles = (int)(p.ld / NT);
    const bool main_ok = w < p.mb16;
    const bool do_extra = p.extra && w < 4;

    for (int64_t ia = p.row_lo + blockIdx.x; ia < p.row_hi; ia += gridDim.x) {
        __syncthreads();  // previous row fully written out
        const uint64_t sa = string_unrank((uint64_t)ia, p.na_el, norb);
        // ---- K-list: k=0 the row itself (occupation entries), k>=1 singles (q occ asc, p virt asc)
        for (int k = tid; k < KP; k += nthr) {
            int J = (int)ia, pr = -2;
            double sg = 0.0;
            if (k == 0) {
                pr = -1;
                sg = 1.0;
            } else if (k < p.K) {
                const int nv = norb - p.na_el;
                const int qi = (k - 1) / nv, pi = (k - 1) % nv;
                uint64_t m = sa;
                for (int i = 0; i < qi; ++i) m &= m - 1;
                const int q = __ffsll((long long)m) - 1;
                uint64_t v = ~sa & (((uint64_t)1 << norb) - 1);
                for (int i = 0; i < pi; ++i) v &= v - 1;
                const int pp = __ffsll((long long)v) - 1;
                const uint64_t rem = sa ^ ((uint64_t)1 << q);
                J = (int)string_rank(rem | ((uint64_t)1 << pp));
                sg = ((pop_below(sa, q) + pop_below(rem, pp)) & 1) ? -1.0 : 1.0;
                pr = pair_sym(pp, q);
            }
            sJ[k] = J;
            sPair[k] = pr;
            sSign[k] = sg;
        }
        for (int64_t c = tid; c < p.ld; c += nthr) srow[c] = 0.0;
        __syncthreads();

        // ---- A fragments: rows rs of the packed pair space, columns k of the K-list
        auto aval = [&](int rs, int k) -> double {
            if (rs >= npair || k >= p.K) return 0.0;
            const int pr = sPair[k];
            if (pr == -1) {
                double s = 0.0;
                for (uint64_t m = sa; m; m &= m - 1) {
                    const int q = __ffsll((long long)m) - 1;
                    s += p.Vp[(size_t)pair_sym(q, q) * npair + rs];
                }
                return s;
            }
            return sSign[k] * p.Vp[(size_t)pr * npair + rs];
        };
        double a0[KS], a1[KS], ae[KS];
        const int r0 = 16 * w + g, re = 16 * p.mb16 + g;
#pragma unroll
        for (int j = 0; j < KS; ++j) {
            const int k = 4 * j + t;
            a0[j] = main_ok ? aval(r0, k) : 0.0;
            a1[j] = main_ok ? aval(r0 + 8, k) : 0.0;
            ae[j] = do_extra ? aval(re, k) : 0.0;
        }

        auto load_tile = [&](int stage, int jt) {
            double* dst = Ds + stage * KP * DSTRIDE;
            for (int c = tid; c < KP * (NT / 2); c += nthr) {
                const int k = c / (NT / 2), part = c % (NT / 2);
                cp_async16(dst + k * DSTRIDE + part * 2, p.x + (int64_t)sJ[k] * p.ld + (int64_t)jt * NT + part * 2);
            }
            cp_async_commit();
        };
#pragma unroll
        for (int s = 0; s < STAGES - 1; ++s) {
            if (s < ntiles) load_tile(s, s);
            else cp_async_commit();
        }

        for (int jt = 0; jt < ntiles; ++jt) {
            // scatter codes for this tile (independent of D; issued before the wait)
            uint16_t code[4][4], codee[2];
            const uint16_t* cbase = p.codes + ((int64_t)jt * NT) * p.npad;
#pragma unroll
            for (int nb = 0; nb < 4; ++nb)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int col = nb * 8 + 2 * t + (e & 1), row = r0 + (e >> 1) * 8;
                    code[nb][e] = main_ok ? cbase[(int64_t)col * p.npad + row] : (uint16_t)0xFFFF;
                }
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = w * 8 + 2 * t + e;
                codee[e] = do_extra ? cbase[(int64_t)col * p.npad + re] : (uint16_t)0xFFFF;
            }

            cp_async_wait<STAGES - 2>();
            __syncthreads();
            {
                const int pf = jt + STAGES - 1;
                if (pf < ntiles) load_tile(pf % STAGES, pf);
                else cp_async_commit();
            }
            const double* D = Ds + (jt % STAGES) * KP * DSTRIDE;
            double acc[4][4];
            double acce[2] = {0.0, 0.0};
#pragma unroll
            for (int nb = 0; nb < 4; ++nb)
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[nb][e] = 0.0;
#pragma unroll
            for (int j = 0; j < KS; ++j) {
                const double* Dk = D + (4 * j + t) * DSTRIDE + g;
                double b[4];
#pragma unroll
                for (int nb = 0; nb < 4; ++nb) b[nb] = Dk[nb * 8];
                if (main_ok) {
#pragma unroll
                    for (int nb = 0; nb < 4; ++nb) dmma_16x8x4(acc[nb], a0[j], a1[j], b[nb]);
                }
                if (do_extra) dmma_8x8x4(acce, ae[j], Dk[w * 8]);
            }
            // ---- scatter into the shared sigma row
#pragma unroll
            for (int nb = 0; nb < 4; ++nb)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint16_t cd = code[nb][e];
                    if (cd != 0xFFFF) atomicAdd(&srow[cd & 0x7FFF], (cd & 0x8000) ? -acc[nb][e] : acc[nb][e]);
                }
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const uint16_t cd = codee[e];
                if (cd != 0xFFFF) atomicAdd(&srow[cd & 0x7FFF], (cd & 0x8000) ? -acce[e] : acce[e]);
            }
        }
        cp_async_wait<0>();
        __syncthreads();
        // ---- write the row: y = [y] + sigma_ab + e_core * x
        const double* xr = p.x + ia * p.ld;
        double* yr = p.y + (ia - p.row_lo) * p.ld;
        for (int64_t c = tid; c < p.ld; c += nthr) {
            double v = 0.0;
            if (c < p.NB) {
                v = srow[c] + p.e_core * xr[c];
                if (p.accumulate) v += yr[c];
            }
            yr[c] = v;
        }
    }
}

template <int KS>
void launch_ks(const AbPlan& pl, const AbParams& prm, int grid, cudaStream_t st) {
    auto kern = k_sigma_ab<KS>;
    static thread_local int configured = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured != dev) {
        SBG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        configured = dev;
    }
    kern<<<grid, pl.threads, pl.smem, st>>>(prm);
    SBG_LAUNCH_CHECK();
}

}  // namespace

AbPlan plan_sigma_ab(int norb, int na_el, int nb_el, int64_t NA, int64_t NB, int64_t ld, int nsm) {
    (void)nsm;
    AbPlan pl{};
    pl.norb = norb;
    pl.na_el = na_el;
    pl.nb_el = nb_el;
    pl.NA = NA;
    pl.NB = NB;
    pl.ld = ld;
    pl.npair = norb * (norb + 1) / 2;
    pl.K = 1 + na_el * (norb - na_el);
    pl.KS = (pl.K + 3) / 4;
    const int full = pl.npair / 16, rem = pl.npair % 16;
    if (rem == 0) {
        pl.mb16 = full;
        pl.extra = 0;
    } else if (rem <= 8 && full >= 4) {
        pl.mb16 = full;  // the last 8 rows ride on m8n8k4 in warps 0..3 (balanced SMSP load)
        pl.extra = 1;
    } else {
        pl.mb16 = full + 1;
        pl.extra = 0;
    }
    pl.npad = pl.extra ? 16 * pl.mb16 + 8 : 16 * pl.mb16;
    pl.threads = 32 * std::max(pl.mb16, pl.extra ? 4 : 1);
    const int KP = pl.KS * 4;
    pl.smem = (size_t)ld * 8 + (size_t)STAGES * KP * DSTRIDE * 8 + (size_t)KP * 4 * 2 + 8 + (size_t)KP * 8;
    if (NB > 32767) throw InvalidArgument("sigma_ab: more than 32767 beta strings is not supported by this build");
    if (pl.smem > 227 * 1024) throw InvalidArgument("sigma_ab: beta row does not fit in shared memory");
    if (pl.KS > 24 || pl.threads > 288) throw InvalidArgument("sigma_ab: orbital space too large for this build");
    return pl;
}

void launch_sigma_ab(const AbPlan& pl, const double* x_full, double* y_local, const double* Vp, const uint16_t* codes,
                     int64_t row_lo, int64_t row_hi, double e_core, int accumulate, int grid, cudaStream_t st) {
    ensure_binomials();
    if (row_hi <= row_lo) return;
    AbParams prm{};
    prm.x = x_full;
    prm.y = y_local;
    prm.Vp = Vp;
    prm.codes = codes;
    prm.norb = pl.norb;
    prm.na_el = pl.na_el;
    prm.npair = pl.npair;
    prm.npad = pl.npad;
    prm.mb16 = pl.mb16;
    prm.extra = pl.extra;
    prm.K = pl.K;
    prm.KP = pl.KS * 4;
    prm.NB = pl.NB;
    prm.ld = pl.ld;
    prm.row_lo = row_lo;
    prm.row_hi = row_hi;
    prm.e_core = e_core;
    prm.accumulate = accumulate;
    grid = (int)std::min<int64_t>(grid, row_hi - row_lo);
    switch (pl.KS) {
#define SBG_KS(n) \
    case n: launch_ks<n>(pl, prm, grid, st); break;
        SBG_KS(1) SBG_KS(2) SBG_KS(3) SBG_KS(4) SBG_KS(5) SBG_KS(6) SBG_KS(7) SBG_KS(8) SBG_KS(9) SBG_KS(10)
        SBG_KS(11) SBG_KS(12) SBG_KS(13) SBG_KS(14) SBG_KS(15) SBG_KS(16) SBG_KS(17) SBG_KS(18) SBG_KS(19)
        SBG_KS(20) SBG_KS(21) SBG_KS(22) SBG_KS(23) SBG_KS(24)
#undef SBG_KS
        default: throw InvalidArgument("sigma_ab: unsupported K");
    }
}

}  // namespace sbg
