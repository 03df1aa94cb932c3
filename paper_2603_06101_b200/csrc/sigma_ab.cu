// sigma_ab.cu — K6: opposite-spin sigma term as gather -> FP64 tensor-core DGEMM -> scatter.
//
//   sigma_ab(Ia, Ib) = sum_{pq,rs} V'(pq,rs) <Ia|E^a_pq|Ja> <Ib|E^b_rs|Jb> c(Ja,Jb)
//   V'(pq,rs) = (pq|rs) + h_pq d_rs / n_beta + d_pq h_rs / n_alpha      (one-body folded in)
//
// is the reference's spin-summed contraction (fci/sigma.hpp:86-137) restricted to its alpha-beta
// cross terms plus both one-body terms; the same-spin two-body terms come from sigma_ss.cu.
//
// A thread-block CLUSTER OF TWO CTAs (two SMs) owns one alpha row Ia at a time (persistent over
// rows). The sigma row is split between the pair's shared memories: CTA h owns targets
// [h*ld/2, (h+1)*ld/2). Columns (beta strings Jb) are processed as pair-tiles of 2*NT: CTA h
// computes the NT-column sub-tile h of each pair-tile:
//   gather  D[k][Jb] = c(J_k, Jb) for the K = 1 + n_a(norb-n_a) distinct alpha strings J_k linked
//           to Ia (k=0 is Ia itself carrying all occupation entries; sigma.hpp:33-35) — cp.async;
//   DGEMM   G[rs][Jb] = sum_k A[rs][k] D[k][Jb], A[rs][k] = sign_k V'(pair_k, rs), M = npair =
//           norb(norb+1)/2 packed symmetric pairs, A resident in registers for the whole row —
//           mma.sync m16n8k4 / m8n8k4 f64 (SASS DMMA.8x8x4); G staged in shared memory;
//   scatter CTA h reduces every target of its half from BOTH sub-tiles' G (the partner's through
//           distributed shared memory) with per-(pair-tile, half) target-sorted segment lists
//           precomputed once (build_ab_scatter): one thread per target, fixed order — no atomics,
//           bit-reproducible sums.
// Splitting the row across the pair frees the shared memory for 32-column sub-tiles with
// double-buffered D, G and lists; one cluster barrier per pair-tile, and the scatter of pair-tile
// i-1 overlaps the DMMAs of pair-tile i (warps w and w+4, which share an SM sub-partition, run the
// two phases in opposite order). Each CTA finally writes its half of y(Ia,:) = [y] + sigma + e_core c.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <vector>
#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace sbg {

namespace {

template <int NT> struct Tile {
    static constexpr int NBT = NT / 8;         // n8 blocks per sub-tile
    static constexpr int DSTRIDE = NT + 4;     // D row stride: bank-conflict-free B fragments (== 4 mod 16)
    static constexpr int GSTRIDE = NT + 1;     // staged G row stride
};
constexpr int STAGES = 2;  // D sub-tiles, G sub-tiles and scatter lists are double buffered
constexpr int THREADS = 256;

struct AbParams {
    const double* x;
    double* y;
    const double* Vp;
    const uint32_t* tgt;        // per (pair-tile, half): (local target << 16) | segment end
    const uint16_t* ent;        // G offset | (partner's G) << 14 | (negative) << 15
    const uint32_t* seg_tgt;    // [2*npt+1] offsets into tgt (16-byte aligned segments)
    const uint32_t* seg_ent;    // [2*npt+1] offsets into ent
    int norb, na_el, npair, mb16, extra, K, grows, maxT, maxE;
    int64_t NB, ld, row_lo, row_hi;
    double e_core;
    int accumulate;
};

template <int KS, int NT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1) k_sigma_ab(const AbParams p) {
    constexpr int NBT = Tile<NT>::NBT, DSTRIDE = Tile<NT>::DSTRIDE, GSTRIDE = Tile<NT>::GSTRIDE;
    constexpr int KP = KS * 4;
    extern __shared__ __align__(16) double smem[];
    cg::cluster_group cluster = cg::this_cluster();
    const int h = (int)cluster.block_rank();
    const int64_t half = p.ld / 2;
    const int npt = (int)(p.ld / (2 * NT));
    double* srow = smem;                                             // [half]  targets of this CTA
    double* Ds = srow + half;                                        // [STAGES][KP][DSTRIDE]
    double* sAe = Ds + STAGES * KP * DSTRIDE;                        // [KP][8] A of the extra m8 rows
    double* Gs = sAe + KP * 8;                                       // [STAGES][grows][GSTRIDE]
    uint32_t* Lt = reinterpret_cast<uint32_t*>(Gs + STAGES * p.grows * GSTRIDE);  // [STAGES][maxT]
    uint16_t* Le = reinterpret_cast<uint16_t*>(Lt + STAGES * p.maxT);             // [STAGES][maxE]
    uint32_t* sST = reinterpret_cast<uint32_t*>(Le + STAGES * p.maxE);            // [2*npt+1]
    uint32_t* sSE = sST + 2 * npt + 1;                                            // [2*npt+1]
    int* sJ = reinterpret_cast<int*>(sSE + 2 * npt + 1);                          // [KP]
    int* sPair = sJ + KP;                                 // [KP]  -1 = occupation row, -2 = padding
    double* sSign = reinterpret_cast<double*>(sPair + KP);  // [KP] (offset 16*npt + 8 + 8*KP: 8-byte aligned)
    const double* Gpartner = cluster.map_shared_rank(Gs, h ^ 1);

    const int tid = threadIdx.x;
    const int w = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int norb = p.norb, npair = p.npair;
    const bool main_ok = w < p.mb16;
    const bool do_extra = p.extra && w < NBT;  // extra m8 rows: one n8 block per warp
    const int r0 = 16 * w + g, re = 16 * p.mb16;

    for (int i = tid; i <= 2 * npt; i += THREADS) {
        sST[i] = p.seg_tgt[i];
        sSE[i] = p.seg_ent[i];
    }

    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    for (int64_t ia = p.row_lo + cid; ia < p.row_hi; ia += ncl) {
        cluster.sync();  // previous row written out by both CTAs; partner done reading my G
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
        for (int64_t c = tid; c < half; c += THREADS) srow[c] = 0.0;
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
        double a0[KS], a1[KS];
#pragma unroll
        for (int j = 0; j < KS; ++j) {
            const int k = 4 * j + t;
            a0[j] = main_ok ? aval(r0, k) : 0.0;
            a1[j] = main_ok ? aval(r0 + 8, k) : 0.0;
        }
        if (p.extra)
            for (int i = tid; i < KP * 8; i += THREADS) sAe[i] = aval(re + (i & 7), i >> 3);

        auto load_d = [&](int pt) {  // this CTA's sub-tile of pair-tile pt
            double* dst = Ds + (pt & 1) * KP * DSTRIDE;
            const int64_t c0 = (int64_t)pt * 2 * NT + (int64_t)h * NT;
            for (int c = tid; c < KP * (NT / 2); c += THREADS) {
                const int k = c / (NT / 2), part = c % (NT / 2);
                cp_async16(dst + k * DSTRIDE + part * 2, p.x + (int64_t)sJ[k] * p.ld + c0 + part * 2);
            }
        };
        auto load_lists = [&](int pt) {  // this CTA's half of pair-tile pt (16-byte aligned segments)
            const int sg = 2 * pt + h, st = pt & 1;
            const uint32_t t0 = sST[sg], nt4 = (sST[sg + 1] - t0 + 3) / 4;
            const uint32_t e0 = sSE[sg], ne8 = (sSE[sg + 1] - e0 + 7) / 8;
            for (uint32_t c = tid; c < nt4; c += THREADS) cp_async16(Lt + st * p.maxT + 4 * c, p.tgt + t0 + 4 * c);
            for (uint32_t c = tid; c < ne8; c += THREADS) cp_async16(Le + st * p.maxE + 8 * c, p.ent + e0 + 8 * c);
        };
        load_d(0);
        cp_async_commit();

        for (int it = 0; it <= npt; ++it) {
            cp_async_wait<0>();
            cluster.sync();  // D(it) local; both G(it-1) staged; both CTAs done with scatter(it-2)
            if (it + 1 < npt) load_d(it + 1);
            if (it < npt) load_lists(it);
            cp_async_commit();
            auto do_mma = [&]() {
                if (it >= npt || !main_ok) return;
                const double* D = Ds + (it & 1) * KP * DSTRIDE;
                double* G = Gs + (it & 1) * p.grows * GSTRIDE;
                double acc[NBT][4];
                double ace0[2] = {0.0, 0.0}, ace1[2] = {0.0, 0.0};
#pragma unroll
                for (int nb = 0; nb < NBT; ++nb)
#pragma unroll
                    for (int e = 0; e < 4; ++e) acc[nb][e] = 0.0;
                // B fragments double-buffered in registers: loads of k-step j+1 in flight while the
                // DMMAs of step j issue
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
                    if (do_extra) {
                        const double ae = sAe[(4 * j + t) * 8 + g];
                        const double be = D[(4 * j + t) * DSTRIDE + g + w * 8];
                        if (cur) dmma_8x8x4(ace1, ae, be);
                        else dmma_8x8x4(ace0, ae, be);
                    }
                }
#pragma unroll
                for (int nb = 0; nb < NBT; ++nb) {
                    const int col = nb * 8 + 2 * t;
                    G[r0 * GSTRIDE + col] = acc[nb][0];
                    G[r0 * GSTRIDE + col + 1] = acc[nb][1];
                    G[(r0 + 8) * GSTRIDE + col] = acc[nb][2];
                    G[(r0 + 8) * GSTRIDE + col + 1] = acc[nb][3];
                }
                if (do_extra) {
                    G[(re + g) * GSTRIDE + w * 8 + 2 * t] = ace0[0] + ace1[0];
                    G[(re + g) * GSTRIDE + w * 8 + 2 * t + 1] = ace0[1] + ace1[1];
                }
            };
            auto do_scatter = [&]() {  // targets of my half from both sub-tiles of pair-tile it-1
                if (it < 1) return;
                const int pt = it - 1, sg = 2 * pt + h;
                const double* Gl = Gs + (pt & 1) * p.grows * GSTRIDE;
                const double* Gr = Gpartner + (pt & 1) * p.grows * GSTRIDE;
                const uint32_t* lt = Lt + (pt & 1) * p.maxT;
                const uint16_t* le = Le + (pt & 1) * p.maxE;
                const uint32_t nt = sST[sg + 1] - sST[sg];
                for (uint32_t i = tid; i < nt; i += THREADS) {
                    const uint32_t tg = lt[i];
                    const uint32_t beg = (i == 0) ? 0u : (lt[i - 1] & 0xFFFFu);
                    const uint32_t end = tg & 0xFFFFu;
                    // the zero padding that ends a segment is an empty segment: skip it, or its +0
                    // read-modify-write of srow[0] would race with the real target 0
                    if (end <= beg) continue;
                    // signs flip the sign bit (integer pipe): the FP64 pipe, shared with the other
                    // warps' DMMAs, only sees the (entries - 1) + 1 real additions
                    auto signed_g = [&](uint32_t e) {
                        const uint16_t en = le[e];
                        const double* G = (en & 0x4000) ? Gr : Gl;
                        const long long bits = __double_as_longlong(G[en & 0x3FFF]);
                        return __longlong_as_double(bits ^ ((long long)(en & 0x8000) << 48));
                    };
                    double v = signed_g(beg);
                    for (uint32_t e = beg + 1; e < end; ++e) v += signed_g(e);
                    srow[tg >> 16] += v;
                }
            };
            if (((w >> 2) & 1) == 0) {
                do_mma();
                do_scatter();
            } else {
                do_scatter();
                do_mma();
            }
        }
        __syncthreads();
        // ---- write my half of the row: y = [y] + sigma_ab + e_core * x
        const double* xr = p.x + ia * p.ld;
        double* yr = p.y + (ia - p.row_lo) * p.ld;
        const int64_t c0 = (int64_t)h * half;
        for (int64_t c = tid; c < half; c += THREADS) {
            const int64_t col = c0 + c;
            double v = 0.0;
            if (col < p.NB) {
                v = srow[c] + p.e_core * xr[col];
                if (p.accumulate) v += yr[col];
            }
            yr[col] = v;
        }
    }
    cluster.sync();  // keep this CTA's shared memory alive until the partner's last remote reads
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

int ab_ld_multiple() { return 64; }  // pair-tiles of 2 x 32 columns

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
    const int nt = 32, nbt = nt / 8;
    if (ld % (2 * nt)) throw InvalidArgument("sigma_ab: row length must be a multiple of 64");
    if (rem == 0) {
        pl.mb16 = full;
        pl.extra = 0;
    } else if (rem <= 8 && full >= nbt) {
        pl.mb16 = full;  // the last 8 rows ride on m8n8k4 in warps 0..nbt-1
        pl.extra = 1;
    } else {
        pl.mb16 = full + 1;
        pl.extra = 0;
    }
    pl.npad = pl.extra ? 16 * pl.mb16 + 8 : 16 * pl.mb16;
    pl.threads = THREADS;
    pl.nt = nt;
    pl.maxT = pl.maxE = 0;  // set by finalize_sigma_ab once the lists are built
    if (NB > 65535) throw InvalidArgument("sigma_ab: more than 65535 beta strings is not supported by this build");
    if ((size_t)pl.npad * (nt + 1) >= 16384) throw InvalidArgument("sigma_ab: pair space too large for this build");
    if (pl.KS > 24 || pl.mb16 > 8) throw InvalidArgument("sigma_ab: orbital space too large for this build");
    return pl;
}

void finalize_sigma_ab(AbPlan& pl, int maxT, int maxE) {
    pl.maxT = 4 * ((maxT + 3) / 4);
    pl.maxE = 8 * ((maxE + 7) / 8);
    const int KP = pl.KS * 4, nt = pl.nt;
    const int64_t npt = pl.ld / (2 * nt);
    pl.smem = (size_t)(pl.ld / 2) * 8 + (size_t)STAGES * KP * (nt + 4) * 8 + (size_t)KP * 8 * 8 +
              (size_t)STAGES * pl.npad * (nt + 1) * 8 + (size_t)STAGES * (pl.maxT * 4 + pl.maxE * 2) +
              (size_t)(2 * npt + 1) * 8 + 8 + (size_t)KP * 16 + 16;
    if (pl.smem > 227 * 1024) throw InvalidArgument("sigma_ab: half row does not fit in shared memory");
}

// Per-(pair-tile, half) target-sorted scatter lists from the (rs, Jb) -> (Ib, sign) codes
// ([ld][npad] u16, 0xFFFF = none). Sort key: target, then (sub-tile, rs, column) — a fixed
// summation order per target. Entries: G offset (14 bits) | sub-tile owned by the partner CTA
// (bit 14, relative to the half's owner) | negative sign (bit 15).
void build_ab_scatter(const AbPlan& pl, const std::vector<uint16_t>& codes, std::vector<uint32_t>& tgt,
                      std::vector<uint16_t>& ent, std::vector<uint32_t>& seg_tgt, std::vector<uint32_t>& seg_ent,
                      int* maxT, int* maxE) {
    const int NT = pl.nt, GSTRIDE = pl.nt + 1;
    const int64_t npt = pl.ld / (2 * NT), half = pl.ld / 2;
    tgt.clear();
    ent.clear();
    seg_tgt.assign(2 * npt + 1, 0);
    seg_ent.assign(2 * npt + 1, 0);
    *maxT = *maxE = 0;
    std::vector<std::pair<uint32_t, uint16_t>> items[2];
    for (int64_t pt = 0; pt < npt; ++pt) {
        items[0].clear();
        items[1].clear();
        for (int sub = 0; sub < 2; ++sub)
            for (int rs = 0; rs < pl.npad; ++rs)
                for (int c = 0; c < NT; ++c) {
                    const uint16_t code = codes[(size_t)(pt * 2 * NT + sub * NT + c) * pl.npad + rs];
                    if (code == 0xFFFF) continue;
                    const uint32_t target = code & 0x7FFF;
                    const int owner = target >= (uint32_t)half ? 1 : 0;
                    const uint16_t e = (uint16_t)((rs * GSTRIDE + c) | (sub != owner ? 0x4000 : 0) | (code & 0x8000));
                    items[owner].push_back({target - (uint32_t)(owner * half), e});
                }
        for (int hh = 0; hh < 2; ++hh) {
            auto& it = items[hh];
            std::stable_sort(it.begin(), it.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
            while (tgt.size() % 4) tgt.push_back(0);  // 16-byte aligned segments (cp.async)
            while (ent.size() % 8) ent.push_back(0);
            seg_tgt[2 * pt + hh] = (uint32_t)tgt.size();
            seg_ent[2 * pt + hh] = (uint32_t)ent.size();
            for (size_t i = 0; i < it.size(); ++i) {
                ent.push_back(it[i].second);
                if (i + 1 == it.size() || it[i + 1].first != it[i].first) {
                    if (i + 1 > 0xFFFF) throw InvalidArgument("sigma_ab: tile segment overflow");
                    tgt.push_back((it[i].first << 16) | (uint32_t)(i + 1));
                }
            }
            *maxT = std::max<int>(*maxT, (int)(tgt.size() - seg_tgt[2 * pt + hh]) + 4);
            *maxE = std::max<int>(*maxE, (int)(ent.size() - seg_ent[2 * pt + hh]) + 8);
        }
    }
    while (tgt.size() % 4) tgt.push_back(0);
    while (ent.size() % 8) ent.push_back(0);
    seg_tgt[2 * npt] = (uint32_t)tgt.size();
    seg_ent[2 * npt] = (uint32_t)ent.size();
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
    prm.seg_tgt = sc.tile_tgt;
    prm.seg_ent = sc.tile_ent;
    prm.norb = pl.norb;
    prm.na_el = pl.na_el;
    prm.npair = pl.npair;
    prm.mb16 = pl.mb16;
    prm.extra = pl.extra;
    prm.K = pl.K;
    prm.grows = pl.npad;
    prm.maxT = pl.maxT;
    prm.maxE = pl.maxE;
    prm.NB = pl.NB;
    prm.ld = pl.ld;
    prm.row_lo = row_lo;
    prm.row_hi = row_hi;
    prm.e_core = e_core;
    prm.accumulate = accumulate;
    // clusters of two CTAs, one per SM pair, persistent over the rows
    grid = 2 * (int)std::min<int64_t>(std::max(1, grid / 2), row_hi - row_lo);
    switch (pl.KS) {
#define SBG_KS(n) \
    case n: launch_ks<n, 32>(pl, prm, grid, st); break;
        SBG_KS(1) SBG_KS(2) SBG_KS(3) SBG_KS(4) SBG_KS(5) SBG_KS(6) SBG_KS(7) SBG_KS(8) SBG_KS(9) SBG_KS(10)
        SBG_KS(11) SBG_KS(12) SBG_KS(13) SBG_KS(14) SBG_KS(15) SBG_KS(16) SBG_KS(17) SBG_KS(18) SBG_KS(19)
        SBG_KS(20) SBG_KS(21) SBG_KS(22) SBG_KS(23) SBG_KS(24)
#undef SBG_KS
        default: throw InvalidArgument("sigma_ab: unsupported K");
    }
}

}  // namespace sbg
