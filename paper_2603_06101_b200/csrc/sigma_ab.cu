// sigma_ab.cu — K6: opposite-spin sigma term as gather -> FP64 tensor-core DGEMM -> scatter.
//
//   sigma_ab(Ia, Ib) = sum_{pq,rs} V'(pq,rs) <Ia|E^a_pq|Ja> <Ib|E^b_rs|Jb> c(Ja,Jb)
//   V'(pq,rs) = (pq|rs) + h_pq d_rs / n_beta + d_pq h_rs / n_alpha      (one-body folded in)
//
// is the reference's spin-summed contraction (fci/sigma.hpp:86-137) restricted to its alpha-beta
// cross terms plus both one-body terms; the same-spin two-body terms come from sigma_ss.cu.
// One CTA owns one alpha row Ia at a time (persistent over rows) and keeps sigma(Ia,:) in shared
// memory. Per NT-column tile of beta strings Jb:
//   gather  D[k][Jb] = c(J_k, Jb) for the K = 1 + n_a(norb-n_a) distinct alpha strings J_k linked
//           to Ia (k=0 is Ia itself carrying all occupation entries; sigma.hpp:33-35);
//   DGEMM   G[rs][Jb] = sum_k A[rs][k] D[k][Jb], A[rs][k] = sign_k V'(pair_k, rs), M = npair =
//           norb(norb+1)/2 packed symmetric pairs, A resident in registers for the whole row —
//           mma.sync m16n8k4 / m8n8k4 f64 (SASS DMMA.8x8x4);
//   scatter sigma(Ia, Ib) += sum over the tile's (rs, Jb) with E_rs Jb = Ib of sign * G[rs][Jb],
//           through per-tile target-sorted segment lists precomputed once (build_ab_scatter):
//           every target of a tile is reduced by one thread in a fixed order — no atomics,
//           bit-reproducible sums.
// Warp specialisation: warps 0..7 only issue DMMAs (A in registers) and stage G; warps 8..11
// gather D tiles and scatter lists with cp.async (3 stages) and run the scatter. The two groups
// hand tiles over with named barriers (bar.arrive / bar.sync), so the FP64 tensor pipe never waits
// for the scatter. The row is written once: y(Ia,:) = [y(Ia,:)] + sigma_row + e_core c(Ia,:).
#include <algorithm>
#include <cstdlib>
#include <vector>
#include "common.cuh"
#include "kernels.cuh"

namespace sbg {

namespace {

constexpr int MMA_WARPS = 8, HELPER_WARPS = 4;
constexpr int THREADS = 32 * (MMA_WARPS + HELPER_WARPS);
constexpr int MMA_THREADS = 32 * MMA_WARPS, HELPER_THREADS = 32 * HELPER_WARPS;
constexpr int SD = 3;         // D tile / scatter-list stages
constexpr int SG = 2;         // staged G tiles
// named barriers (0 is __syncthreads)
constexpr int BAR_DFULL = 1;  // + stage (SD of them)
constexpr int BAR_GFULL = 4;  // + G buffer
constexpr int BAR_GEMPTY = 6; // + G buffer
constexpr int BAR_MMA = 8;    // DMMA warps only
constexpr int BAR_HELPER = 9; // load / scatter warps only

template <int NT> struct Tile {
    static constexpr int NBT = NT / 8;         // n8 blocks per tile
    static constexpr int DSTRIDE = NT + 4;     // D row stride: bank-conflict-free B fragments (== 4 mod 16)
    static constexpr int GSTRIDE = NT + 1;     // staged G row stride
};

__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }

struct AbParams {
    const double* x;
    double* y;
    const double* Vp;
    const uint32_t* tgt;        // per tile: (target << 16) | segment end, concatenated
    const uint16_t* ent;        // per tile: (G offset) | (negative << 15), target-sorted
    const uint32_t* tile_tgt;   // [ntiles+1] offsets into tgt (16-byte aligned segments)
    const uint32_t* tile_ent;   // [ntiles+1] offsets into ent
    int norb, na_el, npair, mb16, extra, K, KP, grows, maxT, maxE;
    int64_t NB, ld, row_lo, row_hi;
    double e_core;
    int accumulate;
    int dbg;  // profiling experiments only (SBG_AB_DEBUG): 1 = skip scatter, 4 = scatter without FP64 adds
};

template <int KS, int NT>
__global__ void __launch_bounds__(THREADS, 1) k_sigma_ab(const AbParams p) {
    constexpr int NBT = Tile<NT>::NBT, DSTRIDE = Tile<NT>::DSTRIDE, GSTRIDE = Tile<NT>::GSTRIDE;
    constexpr int KP = KS * 4;
    constexpr int KH = (KS + 1) / 2;  // k-steps of the first half (extra rows are split in k)
    extern __shared__ __align__(16) double smem[];
    const int ntiles = (int)(p.ld / NT);
    double* srow = smem;                                             // [ld]
    double* Ds = srow + p.ld;                                        // [SD][KP][DSTRIDE]
    double* sAe = Ds + SD * KP * DSTRIDE;                            // [KP][8] A of the extra m8 rows
    double* Gs = sAe + KP * 8;                                       // [SG][grows][GSTRIDE]
    uint32_t* Lt = reinterpret_cast<uint32_t*>(Gs + SG * p.grows * GSTRIDE);  // [SD][maxT]
    uint16_t* Le = reinterpret_cast<uint16_t*>(Lt + SD * p.maxT);             // [SD][maxE]
    uint32_t* sTT = reinterpret_cast<uint32_t*>(Le + SD * p.maxE);            // [ntiles+1]
    uint32_t* sTE = sTT + ntiles + 1;                                         // [ntiles+1]
    int* sJ = reinterpret_cast<int*>(sTE + ntiles + 1);                       // [KP]
    int* sPair = sJ + KP;                                 // [KP]  -1 = occupation row, -2 = padding
    double* sSign = reinterpret_cast<double*>(sPair + KP);  // [KP] (8-byte aligned: KP % 4 == 0)

    const int tid = threadIdx.x;
    const int w = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int norb = p.norb, npair = p.npair;
    const bool is_mma = w < MMA_WARPS;
    const bool main_ok = w < p.mb16;
    // extra m8 rows (npair % 16 <= 8): warps 0..2*NBT-1, n8 block (w % NBT), k half (w / NBT)
    const bool do_extra = p.extra && w < 2 * NBT;
    const int ex_nb = w % NBT, ex_half = w / NBT;
    const int r0 = 16 * w + g, re = 16 * p.mb16;

    for (int i = tid; i <= ntiles; i += THREADS) {
        sTT[i] = p.tile_tgt[i];
        sTE[i] = p.tile_ent[i];
    }

    for (int64_t ia = p.row_lo + blockIdx.x; ia < p.row_hi; ia += gridDim.x) {
        __syncthreads();  // previous row fully written out
        const uint64_t sa = string_unrank((uint64_t)ia, p.na_el, norb);
        // ---- K-list: k=0 the row itself (occupation entries), k>=1 singles (q occ asc, p virt asc)
        for (int k = tid; k < KP; k += THREADS) {
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
        for (int64_t c = tid; c < p.ld; c += THREADS) srow[c] = 0.0;
        __syncthreads();

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

        if (is_mma) {
            // =============================== DMMA warps ===============================
            double a0[KS], a1[KS];
#pragma unroll
            for (int j = 0; j < KS; ++j) {
                const int k = 4 * j + t;
                a0[j] = main_ok ? aval(r0, k) : 0.0;
                a1[j] = main_ok ? aval(r0 + 8, k) : 0.0;
            }
            if (p.extra)
                for (int i = tid; i < KP * 8; i += MMA_THREADS) sAe[i] = aval(re + (i & 7), i >> 3);
            nbar_sync(BAR_MMA, MMA_THREADS);  // sAe complete among the DMMA warps

            for (int it = 0; it < ntiles; ++it) {
                const int sd = it % SD, sg = it & 1;
                nbar_sync(BAR_DFULL + sd, THREADS);
                const double* D = Ds + sd * KP * DSTRIDE;
                double acc[NBT][4];
                double ace[2] = {0.0, 0.0};
#pragma unroll
                for (int nb = 0; nb < NBT; ++nb)
#pragma unroll
                    for (int e = 0; e < 4; ++e) acc[nb][e] = 0.0;
                if (main_ok) {
                    double b[2][NBT];
#pragma unroll
                    for (int nb = 0; nb < NBT; ++nb) b[0][nb] = D[t * DSTRIDE + g + nb * 8];
#pragma unroll
                    for (int j = 0; j < KS; ++j) {
                        const int cur = j & 1;
                        if (j + 1 < KS) {
#pragma unroll
                            for (int nb = 0; nb < NBT; ++nb) b[cur ^ 1][nb] = D[(4 * (j + 1) + t) * DSTRIDE + g + nb * 8];
                        }
#pragma unroll
                        for (int nb = 0; nb < NBT; ++nb) dmma_16x8x4(acc[nb], a0[j], a1[j], b[cur][nb]);
                    }
                }
                if (do_extra) {
                    const int j0 = ex_half ? KH : 0, j1 = ex_half ? KS : KH;
                    for (int j = j0; j < j1; ++j) {
                        const double ae = sAe[(4 * j + t) * 8 + g];
                        const double be = D[(4 * j + t) * DSTRIDE + g + ex_nb * 8];
                        dmma_8x8x4(ace, ae, be);
                    }
                }
                if (it >= SG) nbar_sync(BAR_GEMPTY + sg, THREADS);  // scatter of tile it-2 done
                double* G = Gs + sg * p.grows * GSTRIDE;
                if (main_ok) {
#pragma unroll
                    for (int nb = 0; nb < NBT; ++nb) {
                        const int col = nb * 8 + 2 * t;
                        G[r0 * GSTRIDE + col] = acc[nb][0];
                        G[r0 * GSTRIDE + col + 1] = acc[nb][1];
                        G[(r0 + 8) * GSTRIDE + col] = acc[nb][2];
                        G[(r0 + 8) * GSTRIDE + col + 1] = acc[nb][3];
                    }
                }
                if (do_extra) {  // the two k halves land in rows re.. and re+8.. (summed by the scatter lists)
                    const int row = re + 8 * ex_half + g;
                    G[row * GSTRIDE + ex_nb * 8 + 2 * t] = ace[0];
                    G[row * GSTRIDE + ex_nb * 8 + 2 * t + 1] = ace[1];
                }
                nbar_arrive(BAR_GFULL + sg, THREADS);
            }
        } else {
            // ============================ load / scatter warps =========================
            const int ht = tid - MMA_THREADS;
            auto load_tile = [&](int jt) {
                const int s = jt % SD;
                double* dst = Ds + s * KP * DSTRIDE;
                for (int c = ht; c < KP * (NT / 2); c += HELPER_THREADS) {
                    const int k = c / (NT / 2), part = c % (NT / 2);
                    cp_async16(dst + k * DSTRIDE + part * 2, p.x + (int64_t)sJ[k] * p.ld + (int64_t)jt * NT + part * 2);
                }
                const uint32_t t0 = sTT[jt], nt4 = (sTT[jt + 1] - t0 + 3) / 4;
                const uint32_t e0 = sTE[jt], ne8 = (sTE[jt + 1] - e0 + 7) / 8;
                for (uint32_t c = ht; c < nt4; c += HELPER_THREADS) cp_async16(Lt + s * p.maxT + 4 * c, p.tgt + t0 + 4 * c);
                for (uint32_t c = ht; c < ne8; c += HELPER_THREADS) cp_async16(Le + s * p.maxE + 8 * c, p.ent + e0 + 8 * c);
            };
            auto scatter = [&](int jt) {
                const double* G = Gs + (jt & 1) * p.grows * GSTRIDE;
                const uint32_t* lt = Lt + (jt % SD) * p.maxT;
                const uint16_t* le = Le + (jt % SD) * p.maxE;
                const uint32_t nt = sTT[jt + 1] - sTT[jt];
                for (uint32_t i = ht; i < nt; i += HELPER_THREADS) {
                    const uint32_t tg = lt[i];
                    const uint32_t beg = (i == 0) ? 0u : (lt[i - 1] & 0xFFFFu);
                    const uint32_t end = tg & 0xFFFFu;
                    // the zero padding that ends a tile's segment is an empty segment: skip it,
                    // or its +0 read-modify-write of srow[0] would race with the real target 0
                    if (end <= beg) continue;
                    // signs are applied by flipping the sign bit (integer pipe): the FP64 pipe,
                    // shared with the DMMA warps, only sees the (entries - 1) + 1 real additions
                    auto signed_g = [&](uint32_t e) {
                        const uint16_t en = le[e];
                        const long long bits = __double_as_longlong(G[en & 0x7FFF]);
                        return __longlong_as_double(bits ^ ((long long)(en & 0x8000) << 48));
                    };
                    if (p.dbg & 4) {  // profiling experiment: same memory traffic, no FP64 adds
                        long long v = __double_as_longlong(signed_g(beg));
                        for (uint32_t e = beg + 1; e < end; ++e) v ^= __double_as_longlong(signed_g(e));
                        srow[tg >> 16] = __longlong_as_double(v);
                        continue;
                    }
                    double v = signed_g(beg);
                    for (uint32_t e = beg + 1; e < end; ++e) v += signed_g(e);
                    srow[tg >> 16] += v;
                }
            };
            // cp.async groups: g0..g2 = tiles 0..2, then iteration i commits g(3+i) holding tile i+2
            // (empty at i = 0), so tile k >= 3 lives in g(k+1) and waiting until <= 1 group is
            // pending at iteration it always covers tile it.
#pragma unroll 1
            for (int s = 0; s < SD; ++s) {
                if (s < ntiles) load_tile(s);
                cp_async_commit();
            }
            for (int it = 0; it < ntiles; ++it) {
                cp_async_wait<1>();                // tile it (and its lists) landed (see group numbering below)
                nbar_arrive(BAR_DFULL + it % SD, THREADS);
                if (it >= 1) {
                    const int jt = it - 1;
                    nbar_sync(BAR_GFULL + (jt & 1), THREADS);   // G(jt) staged (and D(jt) consumed)
                    if (!(p.dbg & 1)) scatter(jt);
                    if (jt + SG < ntiles) nbar_arrive(BAR_GEMPTY + (jt & 1), THREADS);
                    // D stage and list stage of tile jt are free once every helper finished the
                    // scatter of jt: prefetch tile jt + SD into them
                    nbar_sync(BAR_HELPER, HELPER_THREADS);
                    if (jt + SD < ntiles) load_tile(jt + SD);
                }
                cp_async_commit();
            }
            if (ntiles >= 1) {
                const int jt = ntiles - 1;
                nbar_sync(BAR_GFULL + (jt & 1), THREADS);
                scatter(jt);
            }
            cp_async_wait<0>();
        }
        __syncthreads();
        // ---- write the row: y = [y] + sigma_ab + e_core * x
        const double* xr = p.x + ia * p.ld;
        double* yr = p.y + (ia - p.row_lo) * p.ld;
        for (int64_t c = tid; c < p.ld; c += THREADS) {
            double v = 0.0;
            if (c < p.NB) {
                v = srow[c] + p.e_core * xr[c];
                if (p.accumulate) v += yr[c];
            }
            yr[c] = v;
        }
    }
}

template <int KS, int NT>
void launch_ks(const AbPlan& pl, const AbParams& prm, int grid, cudaStream_t st) {
    auto kern = k_sigma_ab<KS, NT>;
    static int configured[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !configured[dev]) {
        SBG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        configured[dev] = 1;
    }
    kern<<<grid, THREADS, pl.smem, st>>>(prm);
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
    const int KP = pl.KS * 4;
    const int full = pl.npair / 16, rem = pl.npair % 16;
    auto configure = [&](int nt) {
        const int nbt = nt / 8;
        if (rem == 0) {
            pl.mb16 = full;
            pl.extra = 0;
        } else if (rem <= 8 && full >= 2 * nbt) {
            pl.mb16 = full;  // the last 8 rows: m8n8k4 on warps 0..2*nbt-1 (n8 block x k half)
            pl.extra = 1;
        } else {
            pl.mb16 = full + 1;
            pl.extra = 0;
        }
        pl.npad = pl.extra ? 16 * pl.mb16 + 8 : 16 * pl.mb16;
        pl.threads = THREADS;
        pl.nt = nt;
        const int grows = pl.npad + (pl.extra ? 8 : 0);  // + the second k half of the extra rows
        // scatter-list buffers: bounded by the tile's valid (rs, column) entries (+ extra-row halves)
        pl.maxT = 4 * ((nt * (1 + nb_el * (norb - nb_el)) + 3) / 4);
        pl.maxE = 8 * ((nt * (nb_el + nb_el * (norb - nb_el) + (pl.extra ? 8 : 0)) + 7) / 8);
        const int64_t ntiles = ld / nt;
        pl.smem = (size_t)ld * 8 + (size_t)SD * KP * (nt + 4) * 8 + (size_t)KP * 8 * 8 +
                  (size_t)SG * grows * (nt + 1) * 8 + (size_t)SD * (pl.maxT * 4 + pl.maxE * 2) +
                  (size_t)(ntiles + 1) * 8 + (size_t)KP * 16 + 16;
    };
    configure(32);
    if (pl.smem > 227 * 1024) configure(16);
    if (NB > 32767) throw InvalidArgument("sigma_ab: more than 32767 beta strings is not supported by this build");
    if ((size_t)(pl.npad + 8) * (pl.nt + 1) >= 32768) throw InvalidArgument("sigma_ab: pair space too large for this build");
    if (pl.smem > 227 * 1024) throw InvalidArgument("sigma_ab: beta row does not fit in shared memory");
    if (pl.KS > 24 || pl.mb16 > MMA_WARPS) throw InvalidArgument("sigma_ab: orbital space too large for this build");
    return pl;
}

// Per-tile target-sorted scatter lists from the (rs, Jb) -> (Ib, sign) codes ([ld][npad] u16,
// 0xFFFF = none). Sort key: target, then (rs, column) — a fixed summation order per target. The
// extra m8 rows are produced as two k halves (rows rs and rs+8 of the staged tile): both enter
// the segment of the target.
void build_ab_scatter(const AbPlan& pl, const std::vector<uint16_t>& codes, std::vector<uint32_t>& tgt,
                      std::vector<uint16_t>& ent, std::vector<uint32_t>& tile_tgt, std::vector<uint32_t>& tile_ent) {
    const int NT = pl.nt, GSTRIDE = pl.nt + 1;
    const int64_t ntiles = pl.ld / NT;
    const int re = 16 * pl.mb16;
    tgt.clear();
    ent.clear();
    tile_tgt.assign(ntiles + 1, 0);
    tile_ent.assign(ntiles + 1, 0);
    std::vector<std::pair<uint32_t, uint16_t>> items;
    for (int64_t jt = 0; jt < ntiles; ++jt) {
        items.clear();
        for (int rs = 0; rs < pl.npad; ++rs)
            for (int c = 0; c < NT; ++c) {
                const uint16_t code = codes[(size_t)(jt * NT + c) * pl.npad + rs];
                if (code == 0xFFFF) continue;
                items.push_back({(uint32_t)(code & 0x7FFF), (uint16_t)((rs * GSTRIDE + c) | (code & 0x8000))});
                if (pl.extra && rs >= re)
                    items.push_back({(uint32_t)(code & 0x7FFF), (uint16_t)(((rs + 8) * GSTRIDE + c) | (code & 0x8000))});
            }
        std::stable_sort(items.begin(), items.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        while (tgt.size() % 4) tgt.push_back(0);  // 16-byte aligned tile segments (cp.async)
        while (ent.size() % 8) ent.push_back(0);
        tile_tgt[jt] = (uint32_t)tgt.size();
        tile_ent[jt] = (uint32_t)ent.size();
        for (size_t i = 0; i < items.size(); ++i) {
            ent.push_back(items[i].second);
            if (i + 1 == items.size() || items[i + 1].first != items[i].first) {
                if (i + 1 > 0xFFFF) throw InvalidArgument("sigma_ab: tile segment overflow");
                tgt.push_back((items[i].first << 16) | (uint32_t)(i + 1));
            }
        }
        if ((int64_t)(tgt.size() - tile_tgt[jt]) > pl.maxT || (int64_t)(ent.size() - tile_ent[jt]) > pl.maxE)
            throw InvalidArgument("sigma_ab: tile scatter list exceeds its buffer");
    }
    while (tgt.size() % 4) tgt.push_back(0);
    while (ent.size() % 8) ent.push_back(0);
    tile_tgt[ntiles] = (uint32_t)tgt.size();
    tile_ent[ntiles] = (uint32_t)ent.size();
}

void launch_sigma_ab(const AbPlan& pl, const AbScatter& sc, const double* x_full, double* y_local, const double* Vp,
                     int64_t row_lo, int64_t row_hi, double e_core, int accumulate, int grid, cudaStream_t st) {
    ensure_binomials();
    if (row_hi <= row_lo) return;
    AbParams prm{};
    prm.x = x_full;
    prm.y = y_local;
    prm.Vp = Vp;
    prm.tgt = sc.tgt;
    prm.ent = sc.ent;
    prm.tile_tgt = sc.tile_tgt;
    prm.tile_ent = sc.tile_ent;
    prm.norb = pl.norb;
    prm.na_el = pl.na_el;
    prm.npair = pl.npair;
    prm.mb16 = pl.mb16;
    prm.extra = pl.extra;
    prm.K = pl.K;
    prm.KP = pl.KS * 4;
    prm.grows = pl.npad + (pl.extra ? 8 : 0);
    prm.maxT = pl.maxT;
    prm.maxE = pl.maxE;
    prm.NB = pl.NB;
    prm.ld = pl.ld;
    prm.row_lo = row_lo;
    prm.row_hi = row_hi;
    prm.e_core = e_core;
    prm.accumulate = accumulate;
    prm.dbg = getenv("SBG_AB_DEBUG") ? atoi(getenv("SBG_AB_DEBUG")) : 0;
    grid = (int)std::min<int64_t>(grid, row_hi - row_lo);
    switch (pl.KS) {
#define SBG_KS(n) \
    case n: if (pl.nt == 32) launch_ks<n, 32>(pl, prm, grid, st); else launch_ks<n, 16>(pl, prm, grid, st); break;
        SBG_KS(1) SBG_KS(2) SBG_KS(3) SBG_KS(4) SBG_KS(5) SBG_KS(6) SBG_KS(7) SBG_KS(8) SBG_KS(9) SBG_KS(10)
        SBG_KS(11) SBG_KS(12) SBG_KS(13) SBG_KS(14) SBG_KS(15) SBG_KS(16) SBG_KS(17) SBG_KS(18) SBG_KS(19)
        SBG_KS(20) SBG_KS(21) SBG_KS(22) SBG_KS(23) SBG_KS(24)
#undef SBG_KS
        default: throw InvalidArgument("sigma_ab: unsupported K");
    }
}

}  // namespace sbg
