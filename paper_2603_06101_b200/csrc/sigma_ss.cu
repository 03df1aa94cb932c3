// sigma_ss.cu — K4/K5: same-spin two-body sigma terms through the (n-2)-electron intermediate,
// plus the tiled transposes that turn the beta-beta term into an alpha-alpha one, and the
// one-body kernel used only for sectors without an opposite-spin term.
//
// Normal-ordered same-spin two-body operator (the reference carries it inside its spin-summed
// h2e, fci/sigma.hpp:56-81 / 86-137):
//   1/2 sum (pq|rs) a+_p a+_r a_s a_q = sum_{p<r, q<s} W(pr,qs) a+_p a+_r a_s a_q,
//   W(pr,qs) = (pq|rs) - (ps|rq).
// Resolving through K = (n-2)-electron strings:
//   sigma(I,:) += sum_K phi(K;pr) W(pr,qs) phi(K;qs) c(J,:),  I = K+{p,r}, J = K+{q,s},
//   phi(K;q,s) = <K|a_s a_q|K+{q,s}> = (-1)^(pop_below(J,q) + pop_below(J-q,s)).
// Per K that is a dense (P x P) x (P x ncols) DGEMM with P = C(norb-n+2, 2) gathered rows and P
// scattered rows; the batch dimension (the other spin) is contiguous, so gathers are coalesced
// row reads and the scatter is a coalesced fp64 reduction (red.global.add.f64) into L2.
#include <algorithm>
#include <cstdlib>
#include "common.cuh"
#include "kernels.cuh"

namespace sbg {

namespace {

constexpr int NTS = 32;         // batch columns per tile (one warp-wide reduction segment)
constexpr int XSTRIDE = NTS + 4;
constexpr int YSTRIDE = NTS + 8;  // == 8 mod 16 doubles: conflict-free 16-byte accumulator stores
#ifndef SBG_SS_TPC
#define SBG_SS_TPC 128
#endif
#ifndef SBG_SS_MINB
#define SBG_SS_MINB 4
#endif
constexpr int kMaxTilesPerCta = SBG_SS_TPC;
#ifndef SBG_SS_STAGES
#define SBG_SS_STAGES 2
#endif
constexpr int SS_STAGES = SBG_SS_STAGES;  // X tiles in flight (3: P-row stages, the k padding rows alias the next buffer)
// bulk path, two stages: X tiles are announced on mbarriers by the threads' own cp.async completions
// and handed back per warp, instead of one block barrier per tile (the three warps of a CTA may then
// run up to a tile apart)
#ifndef SBG_SS_MBAR
#define SBG_SS_MBAR 1
#endif
constexpr bool SS_MBAR = SBG_SS_MBAR != 0;  // column tiles per CTA: amortizes the per-K setup (pair list, A)

struct SsParams {
    const double* x;
    double* y;  // column c of row I lives at y[I * ldy + c - ycol0] (a column window of the output)
    const double* Va;
    int norb, nel, P, npa;
    int64_t ldx, col_lo, col_hi;
    int tpc;  // column tiles per CTA
    int64_t ldy, ycol0;
    int bulk;        // full tiles reduced by bulk copies (TMA engine) instead of per-lane reds
    int64_t col_pad; // columns [col_hi, col_pad) are padding (x = 0 there, inside the y rows): a tile
                     // ending there still reduces whole (it adds exact zeros)
    // several vectors per launch (bulk path): the CTA's tile sequence runs over its column tiles of
    // vector 0, then of vector 1, ... so the per-K set-up is paid once
    int nvec;
    const double* xv[kMaxSigmaVec];
    double* yv[kMaxSigmaVec];
    int xrows;  // rows per X stage (KPP, or P with three stages)
    int mbar;   // bulk path: mbarrier-announced X tiles (long tile sequences) instead of a block barrier per tile
};

template <int KSS, bool MBAR>
// up to 4 MMA warps (P <= 64 pairs, KSS <= 16: the BASELINE sectors) with the register cap of 4
// resident CTAs; 5-6 warps (P <= 96) and 7-8 warps (P <= 128: few electrons in many orbitals) with
// looser caps
__global__ void __launch_bounds__(KSS > 24 ? 256 : (KSS > 16 ? 192 : 128), KSS > 24 ? 1 : (KSS > 16 ? 2 : SBG_SS_MINB))
    k_sigma_ss(const SsParams p) {
    constexpr int KPP = KSS * 4;
    extern __shared__ __align__(16) double smem[];
    uint64_t* mbF = reinterpret_cast<uint64_t*>(smem);  // [stages] X stage landed, [stages] X stage consumed
    uint64_t* mbE = mbF + SS_STAGES;
    double* Xs = smem + 8;                    // [stages][xrows][XSTRIDE]
    const int ysrows = max(KPP, 16 * (int)(blockDim.x >> 5));
    const int xstage = p.xrows * XSTRIDE;     // doubles per X stage
    double* Ys = Xs + SS_STAGES * xstage;     // [ysrows][YSTRIDE]
    int* sJ = reinterpret_cast<int*>(Ys + ysrows * YSTRIDE);
    int* sPi = sJ + KPP;
    double* sPhi = reinterpret_cast<double*>(sPi + KPP);
    int64_t* sRow = reinterpret_cast<int64_t*>(sPhi + KPP);  // row offsets sJ[i] * ldx
    int64_t* sRowY = sRow + KPP;                             // row offsets sJ[i] * ldy

    const int tid = threadIdx.x, nthr = blockDim.x;
    const int w = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int P = p.P, norb = p.norb;
    const uint64_t K = string_unrank(blockIdx.x, p.nel - 2, norb);
    const uint64_t full = ((uint64_t)1 << norb) - 1;

    // the barrier form is a kernel of its own (MBAR = false) and keeps its schedule; the mbarrier form
    // keeps the run-time test (the schedule ptxas finds with it is 2.5% faster at c4 than without)
    const bool use_mbar = MBAR && SS_MBAR && p.mbar;
    if (use_mbar && tid == 0) {
        for (int i = 0; i < SS_STAGES; ++i) {
            mbar_init(mbF + i, nthr);
            mbar_init(mbE + i, nthr >> 5);
        }
        mbar_init_fence();
    }
    for (int i = tid; i < KPP; i += nthr) {
        int J = -1, pi = 0;
        double phi = 0.0;
        if (i < P) {
            // i-th pair (q<s) of the empty orbitals of K, lexicographic in (s, q)
            const uint64_t vac = ~K & full;
            int cnt = 0, q = -1, s = -1;
            for (uint64_t ms = vac; ms && q < 0; ms &= ms - 1) {
                const int ss = __ffsll((long long)ms) - 1;
                for (uint64_t mq = vac & (((uint64_t)1 << ss) - 1); mq; mq &= mq - 1) {
                    if (cnt == i) {
                        q = __ffsll((long long)mq) - 1;
                        s = ss;
                        break;
                    }
                    ++cnt;
                }
            }
            const uint64_t Jm = K | ((uint64_t)1 << q) | ((uint64_t)1 << s);
            J = (int)string_rank(Jm);
            phi = ((pop_below(Jm, q) + pop_below(Jm ^ ((uint64_t)1 << q), s)) & 1) ? -1.0 : 1.0;
            pi = pair_strict(q, s);
        }
        sJ[i] = J;
        sPi[i] = pi;
        sPhi[i] = phi;
    }
    __syncthreads();
    if (sJ[0] < 0) return;  // no pairs (cannot happen for P >= 1)
    for (int i = tid; i < KPP; i += nthr) {
        if (i >= P) sJ[i] = sJ[0];  // padding rows read a valid row; their A entries are zero
        sRow[i] = (int64_t)sJ[i] * p.ldx;
        sRowY[i] = (int64_t)sJ[i] * p.ldy;
    }

    double a0[KSS], a1[KSS];
    const int i0 = 16 * w + g;
#pragma unroll
    for (int j = 0; j < KSS; ++j) {
        const int jj = 4 * j + t;
        a0[j] = (i0 < P && jj < P) ? sPhi[i0] * sPhi[jj] * p.Va[(size_t)sPi[i0] * p.npa + sPi[jj]] : 0.0;
        a1[j] = (i0 + 8 < P && jj < P) ? sPhi[i0 + 8] * sPhi[jj] * p.Va[(size_t)sPi[i0 + 8] * p.npa + sPi[jj]] : 0.0;
    }
    __syncthreads();

    // column tiles of this CTA, X tiles double-buffered with cp.async (tile tt+1 lands while the
    // DMMAs of tile tt run); Ys is a separate staging tile for the coalesced reductions. Tiles sit on
    // the NTS-aligned column grid (16-byte aligned cp.async for any window [col_lo, col_hi), e.g.
    // odd shard boundaries); columns outside the window are computed but never reduced.
    const int64_t c_begin = (p.col_lo / NTS + (int64_t)blockIdx.y * p.tpc) * NTS;
    const int64_t c_end = ((p.col_hi + NTS - 1) / NTS) * NTS;
    const int ntt = (int)std::min<int64_t>(p.tpc, (c_end - c_begin) / NTS);
    int ld_k = tid / (NTS / 2), ld_part2 = (tid % (NTS / 2)) * 2, ld_soff = ld_k * XSTRIDE + ld_part2;
    asm volatile("" : "+r"(ld_k), "+r"(ld_part2), "+r"(ld_soff));  // fixed per thread: not rebuilt per tile
    auto load = [&](int tcol, int vec, int stage) {  // column tile tcol of vector vec into X stage `stage`
        const int64_t c0 = c_begin + (int64_t)tcol * NTS;
        const double* xs = p.xv[vec] + c0;
        double* dst = Xs + stage * xstage;
        // a tile may overhang the padded row only when ldx is not a multiple of NTS: those columns
        // are never reduced
        const bool inside = c0 + NTS <= p.ldx;
        // chunk i of this thread: row ld_k + i * KSTEP, column pair ld_part2 (the block has a whole
        // number of 16-thread rows, so the column pair is the same for every chunk): one row-offset
        // load, one address add and one cp.async per chunk, unrolled
        constexpr int NTHR = 32 * ((KSS + 3) / 4), KSTEP = NTHR / (NTS / 2), NCH = (KPP + KSTEP - 1) / KSTEP;
        if (inside || c0 + ld_part2 < p.ldx) {
#pragma unroll
            for (int i = 0; i < NCH; ++i) {
                const int k = ld_k + i * KSTEP;
                if (k < p.xrows) cp_async16(dst + ld_soff + i * KSTEP * XSTRIDE, xs + sRow[k] + ld_part2);
            }
        }
    };
    if (SS_STAGES > 2) {  // aliased padding rows must hold finite numbers from the start
        for (int i = tid; i < SS_STAGES * xstage + ysrows * YSTRIDE; i += nthr) Xs[i] = 0.0;
        __syncthreads();
    }
    if (ntt > 0) load(0, 0, 0);
    cp_async_commit();
    if (p.bulk) {
        // One block barrier per tile. Each warp stages ITS OWN 16 rows of the tile in Ys and reduces
        // them into y itself — whole rows by bulk reductions issued from lanes 0-15 (one 256-byte
        // row segment each, executed by the TMA engine, not the LSU), edge tiles of a column window
        // by per-lane reds — so no barrier is needed between the DMMAs and the reductions. A lane
        // waits until the engine has read its previous row (wait_group.read) before the warp
        // overwrites it.
        const int64_t full_end = p.col_pad > p.col_hi ? p.col_pad : p.col_hi;
        const int nseq = ntt * p.nvec;
        // tile tt of the sequence is column tile tt % ntt of vector tt / ntt: running counters for the
        // tile being loaded (ld_*) and the tile being computed (cu_*) instead of divisions per tile
        int ld_t = 1 % ntt, ld_v = 1 / ntt, ld_s = 1 % SS_STAGES, cu_t = 0, cu_v = 0, cu_s = 0;
        auto load_next = [&]() {
            load(ld_t, ld_v, ld_s);
            if (++ld_t == ntt) {
                ld_t = 0;
                ++ld_v;
            }
            if (++ld_s == SS_STAGES) ld_s = 0;
        };
        uint32_t phF = 0, phE = 0;  // phase parity per X stage (landed / consumed)
        const int oX = t * XSTRIDE + g, oY = i0 * YSTRIDE + 2 * t;  // lane offsets into an X tile / the staging tile
        if (use_mbar) cp_async_mbar_arrive_noinc(mbF);  // tile 0's gathers, issued above
        if (SS_STAGES > 2) {  // tile 1 as well: the ring runs SS_STAGES - 1 tiles ahead
            if (1 < nseq) load_next();
            if (use_mbar) cp_async_mbar_arrive_noinc(mbF + 1);
            cp_async_commit();
        }
        for (int tt = 0; tt < nseq; ++tt) {
            const int64_t c0 = c_begin + (int64_t)cu_t * NTS;
            double* const yv = p.yv[cu_v];
            const int s = cu_s;
            const double* X = Xs + cu_s * xstage;
            if (++cu_t == ntt) {
                cu_t = 0;
                ++cu_v;
            }
            if (++cu_s == SS_STAGES) cu_s = 0;
            if (use_mbar) {
                if (tt + SS_STAGES - 1 < nseq) {
                    const int sn = ld_s;  // stage of tile tt + SS_STAGES - 1 = the stage tile tt - 1 used
                    if (tt >= 1) {  // every warp has consumed tile tt-1
                        mbar_wait_parity(mbE + sn, (phE >> sn) & 1u);
                        phE ^= 1u << sn;
                    }
                    load_next();
                    cp_async_mbar_arrive_noinc(mbF + sn);  // fires when this thread's chunks have landed
                }
                mbar_wait_parity(mbF + s, (phF >> s) & 1u);      // X(tt): every thread's chunks have landed
                phF ^= 1u << s;
            } else {
                cp_async_wait<SS_STAGES - 2>();
                __syncthreads();  // X(tt) visible; every warp is done with X(tt-1), whose buffer the next load refills
                if (tt + SS_STAGES - 1 < nseq) load_next();
                cp_async_commit();
            }
            double acc[NTS / 8][4];
#pragma unroll
            for (int nb = 0; nb < NTS / 8; ++nb)
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[nb][e] = 0.0;
            // B fragments double-buffered in registers: k-step j+1's loads are in flight while the
            // DMMAs of step j issue
            double bq[2][NTS / 8];
#pragma unroll
            for (int nb = 0; nb < NTS / 8; ++nb) bq[0][nb] = X[oX + nb * 8];
#pragma unroll
            for (int j = 0; j < KSS; ++j) {
                const int cur = j & 1;
                if (j + 1 < KSS) {
#pragma unroll
                    for (int nb = 0; nb < NTS / 8; ++nb) bq[cur ^ 1][nb] = X[oX + 4 * (j + 1) * XSTRIDE + nb * 8];
                }
#pragma unroll
                for (int nb = 0; nb < NTS / 8; ++nb) dmma_16x8x4(acc[nb], a0[j], a1[j], bq[cur][nb]);
            }
            if (use_mbar) {  // this warp is done with X(tt)
                __syncwarp();
                if (lane == 0) mbar_arrive(mbE + s);
            }
            if (lane < 16) bulk_wait_read_all();  // this lane's previous row segment has been read
            __syncwarp();
#pragma unroll
            for (int nb = 0; nb < NTS / 8; ++nb) {
                *reinterpret_cast<double2*>(Ys + oY + nb * 8) = make_double2(acc[nb][0], acc[nb][1]);
                *reinterpret_cast<double2*>(Ys + oY + 8 * YSTRIDE + nb * 8) = make_double2(acc[nb][2], acc[nb][3]);
            }
            const bool whole = c0 >= p.col_lo && c0 + NTS <= full_end;
            if (whole) {
                fence_proxy_async_smem();  // the staged row is visible to the bulk-copy engine
                __syncwarp();
                const int r = 16 * w + lane;
                if (lane < 16 && r < P) {
                    bulk_reduce_add_f64(yv + sRowY[r] + (c0 - p.ycol0), Ys + r * YSTRIDE, NTS * 8);
                    bulk_commit();
                }
            } else {
                __syncwarp();
                if (c0 + lane >= p.col_lo && c0 + lane < p.col_hi) {
                    double* ybase = yv + (c0 + lane - p.ycol0);
                    for (int r = 16 * w; r < 16 * w + 16 && r < P; ++r) red_add_f64(ybase + sRowY[r], Ys[r * YSTRIDE + lane]);
                }
            }
        }
        if (lane < 16) bulk_wait_all();  // every bulk reduction of this CTA has completed
        cp_async_wait<0>();
        return;
    }
    for (int tt = 0; tt < ntt; ++tt) {
        const int64_t c0 = c_begin + (int64_t)tt * NTS;
        if (tt + 1 < ntt) load(tt + 1, 0, (tt + 1) % SS_STAGES);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();  // X(tt) visible; the reductions of tile tt-1 finished reading Ys
        const double* X = Xs + (tt % SS_STAGES) * xstage;
        double acc[NTS / 8][4];
#pragma unroll
        for (int nb = 0; nb < NTS / 8; ++nb)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[nb][e] = 0.0;
#pragma unroll
        for (int j = 0; j < KSS; ++j) {
            const double* Xk = X + (4 * j + t) * XSTRIDE + g;
#pragma unroll
            for (int nb = 0; nb < NTS / 8; ++nb) dmma_16x8x4(acc[nb], a0[j], a1[j], Xk[nb * 8]);
        }
#pragma unroll
        for (int nb = 0; nb < NTS / 8; ++nb) {
            const int col = nb * 8 + 2 * t;
            *reinterpret_cast<double2*>(Ys + i0 * YSTRIDE + col) = make_double2(acc[nb][0], acc[nb][1]);
            *reinterpret_cast<double2*>(Ys + (i0 + 8) * YSTRIDE + col) = make_double2(acc[nb][2], acc[nb][3]);
        }
        __syncthreads();
        // one warp reduces one 32-column row segment per step: coalesced 256-byte reductions
        if (c0 + lane >= p.col_lo && c0 + lane < p.col_hi) {
            double* ybase = p.y + (c0 + lane - p.ycol0);
            const double* yl = Ys + lane;
            const int nw = nthr >> 5;
#pragma unroll 4
            for (int i = w; i < P; i += nw) red_add_f64(ybase + sRowY[i], yl[i * YSTRIDE]);
        }
    }
    cp_async_wait<0>();
}

template <int KSS, bool MBAR>
void launch_kss(const SsPlan& pl, const SsParams& prm, dim3 grid, cudaStream_t st) {
    auto kern = k_sigma_ss<KSS, MBAR>;
    static thread_local int configured = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured != dev) {  // the largest dynamic allocation any plan of this KSS may ask for
        SBG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        configured = dev;
    }
    kern<<<grid, pl.warps * 32, pl.smem, st>>>(prm);
    SBG_LAUNCH_CHECK();
}

// 32x32 tiled transpose of fp64 with a padded shared tile
__global__ void k_transpose(const double* __restrict__ src, int64_t R, int64_t C, int64_t lds, double* __restrict__ dst,
                            int64_t ldd, int64_t dst_rows, int64_t dst_cols, int accumulate) {
    __shared__ double tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;  // src rows / cols
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        tile[i][threadIdx.x] = (r < R && c < C) ? src[r * lds + c] : 0.0;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;  // dst row c, dst col r
        if (c < dst_rows && r < dst_cols) {
            double v = tile[threadIdx.x][i];
            if (accumulate) v += dst[c * ldd + r];
            dst[c * ldd + r] = v;
        }
    }
}

// sigma += h-part for sectors where one spin is empty (no alpha-beta kernel to fold it into):
// y(Ia,Ib) = [y] + e_core x + sum_{l in links_a(Ia)} s h_{p q} x(J,Ib) + sum_{m in links_b(Ib)} s h x(Ia,J)
__global__ void k_onebody(const double* x, double* y, const Excitation* la, int La, const Excitation* lb, int Lb,
                          const double* h1, int norb, int64_t NA, int64_t NB, int64_t ld, double e_core,
                          int accumulate) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= NA * ld) return;
    const int64_t ia = idx / ld, ib = idx % ld;
    double v = 0.0;
    if (ib < NB) {
        v = e_core * x[idx];
        for (int l = 0; l < La; ++l) {
            const Excitation e = la[ia * La + l];
            v += e.sign * h1[e.p * norb + e.q] * x[(int64_t)e.target * ld + ib];
        }
        for (int l = 0; l < Lb; ++l) {
            const Excitation e = lb[ib * Lb + l];
            v += e.sign * h1[e.p * norb + e.q] * x[ia * ld + e.target];
        }
        if (accumulate) v += y[idx];
    }
    y[idx] = v;
}

// Generic same-spin term for sectors with more than 96 pair rows per (n-2)-string: the one-spin
// two-body operator as a CSR matrix over strings (built on the host from the same normal-ordered
// pair form as k_sigma_ss), applied to the other spin's contiguous batch dimension:
//   y(I, c) += sum_J Wss(I, J) x(J, c) for columns c in [col_lo, col_hi).
// One warp per (output string, 32-column block), one lane per column.
__global__ void k_sigma_ss_csr(const double* __restrict__ x, double* __restrict__ y, const int64_t* __restrict__ rowptr,
                               const int* __restrict__ col, const double* __restrict__ val, int64_t nstr, int64_t ldx,
                               int64_t col_lo, int64_t col_hi, int64_t ldy, int64_t ycol0) {
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nblk = (col_hi - col_lo + 31) / 32;
    if (warp >= nstr * nblk) return;
    const int64_t I = warp / nblk, c = col_lo + (warp % nblk) * 32 + lane;
    if (c >= col_hi) return;
    double acc = 0.0;
    for (int64_t e = rowptr[I]; e < rowptr[I + 1]; ++e) acc = fma(val[e], x[(int64_t)col[e] * ldx + c], acc);
    y[I * ldy + c - ycol0] += acc;
}

}  // namespace

// host CSR of the one-spin two-body operator sum_{p<r,q<s} W(pr,qs) a+_p a+_r a_s a_q over the
// n-electron strings of norb orbitals (colex order), phases as in k_sigma_ss
void build_ss_csr(int norb, int nel, const double* Va, SsCsr& out) {
    const int npa = norb * (norb - 1) / 2;
    const int64_t nstr = (int64_t)binom_host_calc(norb, nel);
    auto rank = [&](uint64_t sb) {
        uint64_t r = 0;
        int i = 1;
        for (int o = 0; o < norb; ++o)
            if (sb >> o & 1) r += binom_host_calc(o, i++);
        return (int64_t)r;
    };
    auto popb = [](uint64_t sb, int o) { return __builtin_popcountll(sb & (((uint64_t)1 << o) - 1)); };
    auto phi = [&](uint64_t full, int q, int sq) {  // <K|a_s a_q|K+{q,s}>, q < s
        return ((popb(full, q) + popb(full ^ ((uint64_t)1 << q), sq)) & 1) ? -1.0 : 1.0;
    };
    std::vector<std::vector<std::pair<int, double>>> rows(nstr);
    // enumerate J in colex order: strings with nel bits (Gosper)
    if (nel >= 2 && nel <= norb) {
        uint64_t J = ((uint64_t)1 << nel) - 1;
        const uint64_t lim = (uint64_t)1 << norb;
        while (J < lim) {
            const int64_t jr = rank(J);
            for (int s = 0; s < norb; ++s) {
                if (!(J >> s & 1)) continue;
                for (int q = 0; q < s; ++q) {
                    if (!(J >> q & 1)) continue;
                    const uint64_t K = J & ~((uint64_t)1 << q) & ~((uint64_t)1 << s);
                    const double pj = phi(J, q, s);
                    const int qs = pair_strict(q, s);
                    for (int r = 0; r < norb; ++r) {
                        if (K >> r & 1) continue;
                        for (int p = 0; p < r; ++p) {
                            if (K >> p & 1) continue;
                            const uint64_t I = K | ((uint64_t)1 << p) | ((uint64_t)1 << r);
                            const double v = phi(I, p, r) * Va[(size_t)pair_strict(p, r) * npa + qs] * pj;
                            if (v != 0.0) rows[rank(I)].push_back({(int)jr, v});
                        }
                    }
                }
            }
            const uint64_t c = J & (~J + 1), rr = J + c;  // next string with the same popcount
            J = (((rr ^ J) >> 2) / c) | rr;
        }
    }
    out.nstr = nstr;
    out.rowptr.assign(nstr + 1, 0);
    out.col.clear();
    out.val.clear();
    for (int64_t i = 0; i < nstr; ++i) {
        auto& rw = rows[i];
        std::sort(rw.begin(), rw.end());
        for (size_t k = 0; k < rw.size();) {  // merge duplicate columns (diagonal / single excitations)
            size_t e = k;
            double v = 0.0;
            while (e < rw.size() && rw[e].first == rw[k].first) v += rw[e++].second;
            out.col.push_back(rw[k].first);
            out.val.push_back(v);
            k = e;
        }
        out.rowptr[i + 1] = (int64_t)out.col.size();
    }
}

void launch_sigma_ss_csr(const SsCsrDev& m, const double* x, double* y, int64_t ldx, int64_t col_lo, int64_t col_hi,
                         cudaStream_t st, int64_t ldy, int64_t ycol0) {
    if (ldy == 0) ldy = ldx;
    if (m.nstr == 0 || col_hi <= col_lo) return;
    const int64_t warps = m.nstr * ((col_hi - col_lo + 31) / 32);
    k_sigma_ss_csr<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(x, y, m.rowptr, m.col, m.val, m.nstr, ldx,
                                                                        col_lo, col_hi, ldy, ycol0);
    SBG_LAUNCH_CHECK();
}

SsPlan plan_sigma_ss(int norb, int nel) {
    SsPlan pl{};
    pl.norb = norb;
    pl.nel = nel;
    pl.npa = norb * (norb - 1) / 2;
    if (nel < 2) {
        pl.P = 0;
        pl.NK = 0;
        return pl;
    }
    const int nv = norb - nel + 2;
    pl.P = nv * (nv - 1) / 2;
    pl.NK = (int64_t)binom_host_calc(norb, nel - 2);
    pl.KSS = (pl.P + 3) / 4;
    pl.warps = (pl.P + 15) / 16;
    const int KPP = pl.KSS * 4;
    const int rows = std::max(KPP, 16 * pl.warps);
    pl.xrows = SS_STAGES > 2 ? pl.P : KPP;
    pl.smem = 64 + (size_t)(SS_STAGES * pl.xrows * XSTRIDE + rows * YSTRIDE) * 8 + (size_t)KPP * 8 * 5 + 16;
    // staged tiles reach y through TMA bulk reductions (cp.reduce.async.bulk .add.f64, one 256-byte
    // row segment per instruction); SBG_SS_BULK=0 keeps the per-lane red.global.add form
    const char* bulk_env = getenv("SBG_SS_BULK");
    pl.bulk = !(bulk_env && atoi(bulk_env) == 0);
    if (pl.KSS > 32 || pl.warps > 8) throw InvalidArgument("sigma_ss: orbital space too large for this build");
    return pl;
}

void launch_sigma_ss(const SsPlan& pl, const double* x, double* y, const double* Va, int64_t ldx, int64_t col_lo,
                     int64_t col_hi, cudaStream_t st, int64_t ldy, int64_t ycol0, int64_t col_pad) {
    launch_sigma_ss_multi(pl, &x, &y, 1, Va, ldx, col_lo, col_hi, st, ldy, ycol0, col_pad);
}

void launch_sigma_ss_multi(const SsPlan& pl, const double* const* xv, double* const* yvs, int nvec, const double* Va,
                           int64_t ldx, int64_t col_lo, int64_t col_hi, cudaStream_t st, int64_t ldy, int64_t ycol0,
                           int64_t col_pad) {
    const double* x = xv[0];
    double* y = yvs[0];
    if (ldy == 0) ldy = ldx;
    ensure_binomials();
    if (pl.P == 0 || pl.NK == 0 || col_hi <= col_lo) return;
    const int64_t ntiles = (col_hi + NTS - 1) / NTS - col_lo / NTS;  // aligned tile grid (see k_sigma_ss)
    // as many tiles per CTA as keep >= 8 CTAs per SM in flight
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    // long rows (c4: 403 tiles) do best with 128 tiles per CTA, shorter ones (c3: 108) with 32
    // (measured: c4 same-spin 33.4 -> 32.8 ms, c3 1.87 ms kept)
    int tpc = ntiles >= 256 ? kMaxTilesPerCta : std::min(kMaxTilesPerCta, 32);
    while (tpc > 4 && pl.NK * ((ntiles + tpc - 1) / tpc) < 8LL * nsm) tpc /= 2;
    if (const char* e = getenv("SBG_SS_TILES")) tpc = std::max(1, std::min(atoi(e), 4096));  // experiments
    // bulk reductions need 16-byte aligned row segments (any padded library buffer is 256-byte aligned)
    int bulk = pl.bulk && (ldy % 2 == 0) && (ycol0 % 2 == 0);
    for (int v = 0; v < nvec; ++v) bulk = bulk && ((uintptr_t)yvs[v] % 16 == 0);
    if (nvec < 1 || nvec > kMaxSigmaVec || (nvec > 1 && !bulk))
        throw InvalidArgument("sigma_ss: several vectors per launch need the bulk-reduction kernel");
    SsParams prm{x, y, Va, pl.norb, pl.nel, pl.P, pl.npa, ldx, col_lo, col_hi, tpc, ldy, ycol0, bulk, col_pad, nvec};
    prm.xrows = pl.xrows;
    // long rows (c4: 128 tiles per CTA) gain from the decoupled warps (32.3 -> 31.4 ms per sigma), short
    // tile sequences lose (c3: 1.67 -> 1.73 ms, c2: 0.116 -> 0.123 ms); SBG_SS_MBAR=0/1 forces either
    prm.mbar = ntiles >= 256;
    if (const char* e = getenv("SBG_SS_MBAR")) prm.mbar = atoi(e) != 0;
    for (int v = 0; v < nvec; ++v) {
        prm.xv[v] = xv[v];
        prm.yv[v] = yvs[v];
    }
    const int64_t gy = (ntiles + tpc - 1) / tpc;
    dim3 grid((unsigned)pl.NK, (unsigned)gy);
    switch (pl.KSS) {
#define SBG_KSS(n) \
    case n:                                              \
        if (prm.mbar) launch_kss<n, true>(pl, prm, grid, st); \
        else launch_kss<n, false>(pl, prm, grid, st);         \
        break;
        SBG_KSS(1) SBG_KSS(2) SBG_KSS(3) SBG_KSS(4) SBG_KSS(5) SBG_KSS(6) SBG_KSS(7) SBG_KSS(8) SBG_KSS(9)
        SBG_KSS(10) SBG_KSS(11) SBG_KSS(12) SBG_KSS(13) SBG_KSS(14) SBG_KSS(15) SBG_KSS(16) SBG_KSS(17)
        SBG_KSS(18) SBG_KSS(19) SBG_KSS(20) SBG_KSS(21) SBG_KSS(22) SBG_KSS(23) SBG_KSS(24) SBG_KSS(25)
        SBG_KSS(26) SBG_KSS(27) SBG_KSS(28) SBG_KSS(29) SBG_KSS(30) SBG_KSS(31) SBG_KSS(32)
#undef SBG_KSS
        default: throw InvalidArgument("sigma_ss: unsupported pair count");
    }
}

void launch_transpose(const double* src, int64_t R, int64_t C, int64_t lds, double* dst, int64_t ldd, int64_t dst_rows,
                      int64_t dst_cols, int accumulate, cudaStream_t st) {
    // grid over src tiles covering rows [0, max(R, dst_cols)): dst columns r in [R, dst_cols) (the
    // padding of a full-width destination) are written as zeros
    const int64_t rr = std::max(R, dst_cols), cc = std::max(C, dst_rows);
    dim3 grid((unsigned)((rr + 31) / 32), (unsigned)((cc + 31) / 32));
    k_transpose<<<grid, dim3(32, 8), 0, st>>>(src, R, C, lds, dst, ldd, dst_rows, dst_cols, accumulate);
    SBG_LAUNCH_CHECK();
}

void launch_onebody(const double* x, double* y, const Excitation* la, int La, const Excitation* lb, int Lb,
                    const double* h1, int norb, int64_t NA, int64_t NB, int64_t ld, double e_core, int accumulate,
                    cudaStream_t st) {
    const int64_t n = NA * ld;
    k_onebody<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, y, la, La, lb, Lb, h1, norb, NA, NB, ld, e_core,
                                                            accumulate);
    SBG_LAUNCH_CHECK();
}

}  // namespace sbg
