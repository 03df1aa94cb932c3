// sigma_ab.cu — K6: opposite-spin sigma term as gather -> FP64 tensor-core DGEMM -> scatter.
//
//   sigma_ab(Ia, Ib) = sum_{pq,rs} V'(pq,rs) <Ia|E^a_pq|Ja> <Ib|E^b_rs|Jb> c(Ja,Jb)
//   V'(pq,rs) = (pq|rs) + h_pq d_rs / n_beta + d_pq h_rs / n_alpha      (one-body folded in)
//
// is the reference's spin-summed contraction (fci/sigma.hpp:86-137) restricted to its alpha-beta
// cross terms plus both one-body terms; the same-spin two-body terms come from sigma_ss.cu.
// One CTA owns one alpha row Ia at a time (persistent over rows). Per 32-column tile of beta
// strings Jb:
//   gather  D[k][Jb] = c(J_k, Jb) for the K = 1 + n_a(norb-n_a) distinct alpha strings J_k linked
//           to Ia (k=0 is Ia itself carrying all occupation entries; sigma.hpp:33-35) — cp.async,
//           double-buffered;
//   DGEMM   G[rs][Jb] = sum_k A[rs][k] D[k][Jb], A[rs][k] = sign_k V'(pair_k, rs), M = npair =
//           norb(norb+1)/2 packed symmetric pairs, A resident in registers for the whole row —
//           mma.sync m16n8k4 / m8n8k4 f64 (SASS DMMA.8x8x4); G staged once in shared memory;
//   scatter sigma(Ia, Ib) += sign * G[rs][Jb] over the tile's (rs, Jb) with E_rs Jb = Ib; the
//           (rs,Jb) -> Ib map depends only on the tile and is precomputed once per operator.
// Default kernel (k_sigma_ab_ws): warp-specialized (8 DMMA warps, 8 gather/scatter warps) and the
// scatter is one red.global.add.f64 per entry into y from a target-sorted list (build_ab_red_list);
// e_core c(Ia,:) is added the same way. SBG_AB_RED=0 selects the deterministic form: sigma(Ia,:)
// in shared memory, every target of a tile summed by one thread in a fixed order from a segment
// list (build_ab_scatter), the row written once — bit-reproducible sums (k_sigma_ab, or the
// warp-specialized kernel with SBG_AB_WS=1).
#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <vector>
#include "common.cuh"
#include "kernels.cuh"

namespace sbg {

namespace {

// NT: beta-string tile width (16 or 32 columns); chosen per sector by shared-memory budget.
template <int NT> struct Tile {
    static constexpr int NBT = NT / 8;         // n8 blocks per tile
    static constexpr int DSTRIDE = NT + 4;     // D row stride: bank-conflict-free B fragments (== 4 mod 16)
    // staged G row stride: == 8 mod 16 doubles, so the MMA warps' 16-byte accumulator stores are
    // bank-conflict free (a quarter warp covers 8 distinct 16-byte bank groups)
    static constexpr int GSTRIDE = NT + 8;
};
constexpr int STAGES = 2;     // D tiles, G tiles and scatter lists are double buffered

struct AbParams {
    const double* x;
    double* y;
    const double* Vp;
    const uint32_t* tgt;        // per tile: (target << 16) | segment end, concatenated
    const uint16_t* ent;        // per tile: (G offset) | (negative << 15), target-sorted
    const uint32_t* tile_tgt;   // [ntiles+1] offsets into tgt
    const uint32_t* tile_ent;   // [ntiles+1] offsets into ent
    int norb, na_el, npair, mb16, extra, K, KP, grows, maxT, maxE;
    int64_t NB, ld, row_lo, row_hi;
    double e_core;
    int accumulate;
    int dbg;  // profiling experiments only: 1 = skip scatter, 2 = skip MMA, 4 = skip gathers (ws kernel)
    int red;  // k_sigma_ab_ws: 1 = scatter by red.global.add into y (no sigma row in shared memory)
    const uint32_t* ent32;      // red mode, per tile: [npos][target << 16 | G byte offset ...] (build_ab_red_list)
    const uint32_t* tile_ent32; // [ntiles+1] offsets into ent32 (multiples of 4)
    int m0;                     // first pair row of this pass (pair-row blocks when npair > 136)
    int add_ecore;              // this pass adds e_core * x
    int tma;                    // k_sigma_ab_ws red mode: D rows and reduction lists by bulk copies
    // several vectors in one launch (tma path): tile T of a row is tile T % ntiles of vector
    // T / ntiles, so the per-row set-up (K-list, A fragments, pipeline fill) is paid once per row
    int nvec;
    const double* xv[kMaxSigmaVec];
    double* yv[kMaxSigmaVec];
    // decoupled hand-offs (tma path): number of D stages (2 or 3), 0 = named-barrier hand-offs.
    // D(it) is announced on an mbarrier by the loaders' own cp.async completions and the G buffer is
    // handed back on an mbarrier the MMA warps only look at AFTER their DMMAs, so neither a slow
    // scatter nor a late gather stops the tensor pipe unless it is a whole tile late
    int dc;
};

// Software pipeline per alpha row, one __syncthreads per tile: iteration `it` prefetches D(it+1)
// and the scatter lists of tile it, runs the DMMAs of tile it into G[it&1], and scatters tile it-1
// from G[(it-1)&1] — so warps that finish their MMAs scatter while the others still feed the
// FP64 tensor pipe.
template <int KS, int NT>
__global__ void __launch_bounds__(256, 1) k_sigma_ab(const AbParams p) {
    constexpr int NBT = Tile<NT>::NBT, DSTRIDE = Tile<NT>::DSTRIDE, GSTRIDE = Tile<NT>::GSTRIDE;
    extern __shared__ __align__(16) double smem[];
    const int KP = KS * 4;
    const int ntiles = (int)(p.ld / NT);
    double* srow = smem;                                             // [ld]
    double* Ds = srow + p.ld;                                        // [STAGES][KP][DSTRIDE]
    double* sAe = Ds + STAGES * KP * DSTRIDE;                        // [KP][8] A of the extra m8 rows
    double* Gs = sAe + KP * 8;                                       // [STAGES][grows][GSTRIDE]
    uint32_t* Lt = reinterpret_cast<uint32_t*>(Gs + STAGES * p.grows * GSTRIDE);  // [STAGES][maxT]
    uint16_t* Le = reinterpret_cast<uint16_t*>(Lt + STAGES * p.maxT);             // [STAGES][maxE]
    uint32_t* sTT = reinterpret_cast<uint32_t*>(Le + STAGES * p.maxE);            // [ntiles+1]
    uint32_t* sTE = sTT + ntiles + 1;                                             // [ntiles+1]
    int* sJ = reinterpret_cast<int*>(sTE + ntiles + 1);                           // [KP]
    int* sPair = sJ + KP;                                 // [KP]  -1 = occupation row, -2 = padding
    double* sSign = reinterpret_cast<double*>(sPair + KP);  // [KP] (8-byte aligned: KP % 4 == 0)

    const int tid = threadIdx.x, nthr = blockDim.x;
    const int w = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int norb = p.norb, npair = p.npair;
    const bool main_ok = w < p.mb16;
    const bool do_extra = p.extra && w < NBT;  // extra m8 rows: one n8 block per warp

    for (int i = tid; i <= ntiles; i += nthr) {
        sTT[i] = p.tile_tgt[i];
        sTE[i] = p.tile_ent[i];
    }

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
        double a0[KS], a1[KS];
        const int r0 = 16 * w + g, re = 16 * p.mb16;
#pragma unroll
        for (int j = 0; j < KS; ++j) {
            const int k = 4 * j + t;
            a0[j] = main_ok ? aval(r0, k) : 0.0;
            a1[j] = main_ok ? aval(r0 + 8, k) : 0.0;
        }
        if (p.extra)
            for (int i = tid; i < KP * 8; i += nthr) sAe[i] = aval(re + (i & 7), i >> 3);

        auto load_d = [&](int stage, int jt) {
            double* dst = Ds + stage * KP * DSTRIDE;
            for (int c = tid; c < KP * (NT / 2); c += nthr) {
                const int k = c / (NT / 2), part = c % (NT / 2);
                cp_async16(dst + k * DSTRIDE + part * 2, p.x + (int64_t)sJ[k] * p.ld + (int64_t)jt * NT + part * 2);
            }
        };
        auto load_lists = [&](int stage, int jt) {  // 16-byte aligned, padded segments
            const uint32_t t0 = sTT[jt], nt4 = (sTT[jt + 1] - t0 + 3) / 4;
            const uint32_t e0 = sTE[jt], ne8 = (sTE[jt + 1] - e0 + 7) / 8;
            for (uint32_t c = tid; c < nt4; c += nthr) cp_async16(Lt + stage * p.maxT + 4 * c, p.tgt + t0 + 4 * c);
            for (uint32_t c = tid; c < ne8; c += nthr) cp_async16(Le + stage * p.maxE + 8 * c, p.ent + e0 + 8 * c);
        };
        load_d(0, 0);
        cp_async_commit();

        for (int it = 0; it <= ntiles; ++it) {
            cp_async_wait<0>();
            __syncthreads();
            if (it + 1 < ntiles) load_d((it + 1) & 1, it + 1);
            if (it < ntiles) load_lists(it & 1, it);
            cp_async_commit();
            // warps w and w+4 share an SM sub-partition: one issues its DMMAs while the other
            // scatters, so the FP64 tensor pipe is not idle during the scatter phase
            auto do_mma = [&]() {
            if (it < ntiles) {
                    const double* D = Ds + (it & 1) * KP * DSTRIDE;
                    double* G = Gs + (it & 1) * p.grows * GSTRIDE;
                    double acc[NBT][4];
                    double ace0[2] = {0.0, 0.0}, ace1[2] = {0.0, 0.0};
    #pragma unroll
                    for (int nb = 0; nb < NBT; ++nb)
    #pragma unroll
                        for (int e = 0; e < 4; ++e) acc[nb][e] = 0.0;
                    if (main_ok) {
                        // B fragments double-buffered in registers: loads of k-step j+1 are in flight
                        // while the DMMAs of step j issue
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
                    }
                }
            };
            auto do_scatter = [&]() {
            if (it >= 1) {  // segmented scatter of tile it-1: one thread per distinct target
                    const int jt = it - 1;
                    const double* G = Gs + (jt & 1) * p.grows * GSTRIDE;
                    const uint32_t* lt = Lt + (jt & 1) * p.maxT;
                    const uint16_t* le = Le + (jt & 1) * p.maxE;
                    const uint32_t nt = sTT[jt + 1] - sTT[jt];
                    for (uint32_t i = tid; i < nt; i += nthr) {
                        const uint32_t tg = lt[i];
                        const uint32_t beg = (i == 0) ? 0u : (lt[i - 1] & 0xFFFFu);
                        const uint32_t end = tg & 0xFFFFu;
                        // the 16-byte padding that ends a tile's segment (zeros) is an empty
                        // segment: skip it, or its +0 read-modify-write of srow[0] would race
                        // with the real update of target 0 by another thread
                        if (end <= beg) continue;
                        // signs flip the sign bit (integer pipe): the FP64 pipe, shared with the
                        // other warps' DMMAs, only sees the (entries - 1) + 1 real additions
                        auto signed_g = [&](uint32_t e) {
                            const uint16_t en = le[e];
                            const long long bits = __double_as_longlong(G[en & 0x7FFF]);
                            return __longlong_as_double(bits ^ ((long long)(en & 0x8000) << 48));
                        };
                        double v = signed_g(beg);
                        for (uint32_t e = beg + 1; e < end; ++e) v += signed_g(e);
                        srow[tg >> 16] += v;
                    }
                }
            };
            if (((w >> 2) & 1) == 0) {
                if (!(p.dbg & 2)) do_mma();
                if (!(p.dbg & 1)) do_scatter();
            } else {
                if (!(p.dbg & 1)) do_scatter();
                if (!(p.dbg & 2)) do_mma();
            }
        }
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

// ---------------------------------------------------------------------------------------------
// Warp-specialized variant: 16 warps. Warps 0-7 (two warpgroups, 2 per SM sub-partition) only run
// the DMMA GEMM; warps 8-15 load (cp.async) and scatter. setmaxnreg moves registers to the MMA
// warpgroups (A fragments stay resident), named barriers hand tiles over:
//   DREADY[b]  loaders -> MMA   D(it) has landed in stage b
//   FULL[b]    MMA -> scatter   G(it) is staged in buffer b
//   EMPTY[b]   scatter -> MMA   G buffer b may be overwritten (tile it+2)
// so tile it's scatter overlaps tile it+1's DMMAs on other warps of the same sub-partition.
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
constexpr int kWsThreads = 512, kWsHalf = 256;
#ifndef SBG_XS_WAITG
#define SBG_XS_WAITG 4   // uniform stream: k-steps between the G hand-back wait and the end of the tile
#endif
#ifndef SBG_TALL_WAITG
#define SBG_TALL_WAITG 3   // TALL kernel, warps 0-3 (c3: 4.57 / 4.54 / 4.50 / 4.54 / 4.58 ms for 1 / 2 / 3 / 4 / 6)
#endif
// The SBG_AB_DEBUG timing experiments (skip the scatter / the DMMAs / the gathers / every hand-off)
// are compiled into k_sigma_ab_ws only with -DSBG_AB_DEBUG_SWITCHES (tools/ab_variant.sh): every
// instruction in the DMMA warps' tile loop costs tensor-pipe time.
#ifdef SBG_AB_DEBUG_SWITCHES
#define SBG_DBG(bit) (p.dbg & (bit))
#else
#define SBG_DBG(bit) (false)
#endif
// register split between the MMA and the loader/scatter warpgroups (sum 256: 256 threads each)
#ifndef SBG_WS_MREG
#define SBG_WS_MREG 200
#endif
#define SBG_WS_SREG (256 - SBG_WS_MREG)
#define SBG_STR2(x) #x
#define SBG_STR(x) SBG_STR2(x)
#ifndef SBG_WSU
#define SBG_WSU 2
#endif
constexpr int WSU = SBG_WSU;
#ifndef SBG_RED_UNROLL
#define SBG_RED_UNROLL 4
#endif
constexpr int RED_UNROLL = SBG_RED_UNROLL;  // scatter entries per thread in flight
constexpr int BAR_DREADY = 1, BAR_FULL = 3, BAR_EMPTY = 5, BAR_SINT = 7, BAR_MINT = 8, BAR_KLIST = 9;

// XS (NT = 32, reduction mode, not TALL): the uniform MMA instruction stream. Every DMMA warp runs
// the same code with no per-k-step branch or select chain:
//  * n8 blocks are interleaved over the tile's columns (local block L of the pair P = L >> 1 holds
//    columns 16 P' + 2 n + (L & 1), n = 0..7), so a lane's B fragments for two blocks are adjacent:
//    two conflict-free LDS.128 per k-step instead of four LDS.64, and a lane's accumulators cover
//    four adjacent columns per pair (16-byte stores; G row stride NT + 2 keeps them conflict free);
//  * XS == 2 (8 m16 blocks + 8 extra rows, the 16-orbital sectors): the extra rows' m8n8k4 DMMAs
//    are split over ALL eight warps — warp w takes n8 block w & 3 on half of the k range (warps
//    4-7 walk the k-steps rotated by half, so "the first KH iterations" means the upper half for
//    them) and stages its partial sums in its own G rows (re + g, re + 8 + g); the reduction list
//    carries both partials. 136 DMMA.8x8x4 per tile on every warp instead of 144 / 128.
template <int KS, int NT, bool K0E, bool TALL, int XS>
__global__ void __launch_bounds__(kWsThreads, 1) k_sigma_ab_ws(const AbParams p) {
    static_assert(XS == 0 || (NT == 32 && !TALL), "uniform stream: 32-column tiles, no TALL");
    constexpr int NBT = Tile<NT>::NBT, DSTRIDE = Tile<NT>::DSTRIDE, GSTRIDE = XS ? NT + 2 : Tile<NT>::GSTRIDE;
    extern __shared__ __align__(16) double smem[];
    // D rows: k = 0 is the row Ia itself (all occupation entries, sigma.hpp:33-35), k = 1..K-1 its
    // single excitations. K0E (when (K-1) % 4 == 0): the DMMAs cover k = 1 .. 4*KS and k = 0 is a
    // rank-1 term added in the epilogue (G += A(:,0) c(Ia,:)), so the K - 1 = n(norb-n) links need
    // no padded k-step (c4: 16 instead of 17); otherwise the DMMAs cover k = 0 .. 4*KS-1.
    constexpr int K0 = K0E ? 1 : 0;
    const int KP = K0 + KS * 4;
    const int ntiles = (int)(p.ld / NT);
    const int ntot = ntiles * p.nvec;  // tiles per alpha row over all vectors
    // mbarriers: [0..2] D stage s landed, [3..4] list stage b landed, [5..6] G buffer b scattered
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
    uint64_t* const mbD = mbar;
    uint64_t* const mbL = mbar + 3;
    uint64_t* const mbE = mbar + 5;
    const int nds = p.dc ? p.dc : STAGES;    // D stages
    double* srow = smem + 8;                 // [ld], absent in red mode
    double* Ds = srow + (p.red ? 0 : p.ld);
    double* sAe = Ds + nds * KP * DSTRIDE;
    double* Gs = sAe + KP * 8;
    uint32_t* Lt = reinterpret_cast<uint32_t*>(Gs + STAGES * p.grows * GSTRIDE);
    uint16_t* Le = reinterpret_cast<uint16_t*>(Lt + STAGES * p.maxT);   // red mode: u32 entries
    uint32_t* sTT = reinterpret_cast<uint32_t*>(Le + STAGES * p.maxE);
    uint32_t* sTE = sTT + ntiles + 1;
    // K-list of an alpha row, double buffered (the loaders build row r+1's while row r runs):
    // sJ = linked alpha string, sOff = its pair's row of V' (pair * npair), sSign = +-1 (0 for k = 0
    // and padding), sOcc = the occupation column A(:, 0) of this pass's pair rows
    int* sJ = reinterpret_cast<int*>(sTE + ntiles + 1);        // [2][KP]
    int* sOff = sJ + 2 * KP;                                   // [2][KP]
    double* sSign = reinterpret_cast<double*>(sOff + 2 * KP);  // [2][KP]
    double* sOcc = sSign + 2 * KP;                             // [2][grows]

    const int tid = threadIdx.x;
    const int w = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int norb = p.norb, npair = p.npair;
    // the two roles never rejoin, so ptxas can give each its own register budget
    if (w < 8) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 " SBG_STR(SBG_WS_MREG) ";\n");
        // TALL (5-7 m16 blocks, no extra rows; c2, c3): warps 0-3 own m16 blocks 0-3 with every n8
        // block, warps 4-7 own blocks 4 .. mb16-1 for one n8 block each (w - 4), so every SM
        // sub-partition gets mb16 units of DMMA work instead of 2x4 on some and 4 on others
        const bool tall = TALL && w >= 4;
        const int mbh = TALL ? p.mb16 - 4 : 0;
        const bool main_ok = TALL ? w < 4 : w < p.mb16;
        const bool do_extra = p.extra && w < NBT;
        uint32_t phDm = 0, phEm = 0;  // decoupled hand-offs: phase parity per D stage / G buffer
        // tile it of a row: wait for D (stage returned), and the hand-back of G buffer b
        auto wait_d = [&](int it, int& sd) -> const double* {
            const int b = it & 1;
            if SBG_DBG(16) return Ds + b * KP * DSTRIDE;  // timing experiment: no hand-offs at all
            if (p.dc) {
                mbar_wait_parity(mbD + sd, (phDm >> sd) & 1u);
                phDm ^= 1u << sd;
                const double* D = Ds + sd * KP * DSTRIDE;
                sd = (sd + 1 == p.dc) ? 0 : sd + 1;
                return D;
            }
            bar_sync(BAR_DREADY + b, kWsThreads);
            if (it >= 2) bar_sync(BAR_EMPTY + b, kWsThreads);
            return Ds + b * KP * DSTRIDE;
        };
        auto wait_g = [&](int it) {  // decoupled: just before the accumulators are staged
            const int b = it & 1;
            if SBG_DBG(16) return;
            if (p.dc && it >= 2) {
                mbar_wait_parity(mbE + b, (phEm >> b) & 1u);
                phEm ^= 1u << b;
            }
        };
        auto drain_g = [&](int ntot) {  // row end: the last two tiles have been scattered
            if SBG_DBG(16) return;
            for (int it = ntot - 2 < 0 ? 0 : ntot - 2; it < ntot; ++it) {
                const int b = it & 1;
                if (p.dc) {
                    mbar_wait_parity(mbE + b, (phEm >> b) & 1u);
                    phEm ^= 1u << b;
                } else {
                    bar_sync(BAR_EMPTY + b, kWsThreads);
                }
            }
        };
        int kb = 0;  // K-list buffer of this row
        for (int64_t ia = p.row_lo + blockIdx.x; ia < p.row_hi; ia += gridDim.x, kb ^= p.tma ? 1 : 0) {
            bar_sync(0, kWsThreads);           // row start (bulk-copy path: this row's K-list was built during the previous row)
            if (!p.tma) bar_sync(BAR_KLIST, kWsThreads);   // K-list of row ia ready (built by the loader warps)
            const int* sOffB = sOff + kb * KP;
            const double* sSignB = sSign + kb * KP;
            const double* sOccB = sOcc + kb * p.grows;
            // A(rs, k) = sign_k V'(pair_k, rs), branch free so that a warp's loads of V' go out together
            // (one L2 round trip per row instead of one per element)
            auto aocc = [&](int rs) -> double { return sOccB[rs]; };
            auto aval = [&](int rs, int k) -> double {
                const int rr = rs + p.m0;  // pair-row block of this pass
                const double v = p.Vp[(size_t)sOffB[k] + (rr < npair ? rr : 0)];
                double a = (rr < npair) ? sSignB[k] * v : 0.0;
                if (!K0E) a = (k == 0) ? sOccB[rs] : a;
                return a;
            };
            if constexpr (TALL) {
                if (tall) {
                    constexpr int MH = 3;  // up to 3 m16 blocks per tall warp (mb16 <= 7)
                    const int nbh = w - 4;  // this warp's n8 block
                    double ah0[MH][KS], ah1[MH][KS], ak0[MH], ak1[MH];
#pragma unroll
                    for (int mb = 0; mb < MH; ++mb) {
                        const int rh = 16 * (4 + mb) + g;
                        const bool ok = mb < mbh && nbh < NBT;
#pragma unroll
                        for (int j = 0; j < KS; ++j) {
                            ah0[mb][j] = ok ? aval(rh, K0 + 4 * j + t) : 0.0;
                            ah1[mb][j] = ok ? aval(rh + 8, K0 + 4 * j + t) : 0.0;
                        }
                        ak0[mb] = (K0E && ok) ? aocc(rh) : 0.0;
                        ak1[mb] = (K0E && ok) ? aocc(rh + 8) : 0.0;
                    }
                    bar_sync(BAR_MINT, kWsHalf);
                    int sd = 0;
                    // lane-dependent offsets pinned in registers (not rebuilt from the thread index per tile)
                    int oB = (K0 + t) * DSTRIDE + g + nbh * 8, oGt = (16 * 4 + g) * GSTRIDE + nbh * 8 + 2 * t;
                    asm volatile("" : "+r"(oB), "+r"(oGt));
                    for (int it = 0; it < ntot; ++it) {
                        const int b = it & 1;
                        const double* D = wait_d(it, sd);
                        if (!SBG_DBG(2) && nbh < NBT) {
                            double* G = Gs + b * p.grows * GSTRIDE;
                            const double* D1 = D + oB;  // row K0 + t, this warp's n8 block
                            double acc[MH][4];
#pragma unroll
                            for (int mb = 0; mb < MH; ++mb)
#pragma unroll
                                for (int e = 0; e < 4; ++e) acc[mb][e] = 0.0;
                            double bq[2];
                            bq[0] = D1[0];
#pragma unroll
                            for (int j = 0; j < KS; ++j) {
                                const int cur = j & 1;
                                if (j == KS - 1) wait_g(it);
                                if (j + 1 < KS) bq[cur ^ 1] = D1[4 * (j + 1) * DSTRIDE];
#pragma unroll
                                for (int mb = 0; mb < MH; ++mb)
                                    if (mb < mbh) dmma_16x8x4(acc[mb], ah0[mb][j], ah1[mb][j], bq[cur]);
                            }
                            const int col = nbh * 8 + 2 * t;
                            const double2 cv = K0E ? *reinterpret_cast<const double2*>(D + col) : make_double2(0.0, 0.0);
#pragma unroll
                            for (int mb = 0; mb < MH; ++mb) {
                                if (mb >= mbh) break;
                                double* gr = G + oGt + 16 * mb * GSTRIDE;
                                if constexpr (K0E) {  // (without it no FP64 add may reach the pipe the DMMAs use)
                                    acc[mb][0] = fma(ak0[mb], cv.x, acc[mb][0]);
                                    acc[mb][1] = fma(ak0[mb], cv.y, acc[mb][1]);
                                    acc[mb][2] = fma(ak1[mb], cv.x, acc[mb][2]);
                                    acc[mb][3] = fma(ak1[mb], cv.y, acc[mb][3]);
                                }
                                *reinterpret_cast<double2*>(gr) = make_double2(acc[mb][0], acc[mb][1]);
                                *reinterpret_cast<double2*>(gr + 8 * GSTRIDE) = make_double2(acc[mb][2], acc[mb][3]);
                            }
                        } else {
                            wait_g(it);
                        }
                        if (!SBG_DBG(16)) bar_arrive(BAR_FULL + b, kWsThreads);
                    }
                    drain_g(ntot);
                    continue;  // next row
                }
                // warps 0-3 of the TALL kernel: m16 block w with every n8 block, the blocks interleaved
                // over the tile's columns as in the uniform stream (two LDS.128 per k-step, no per-k-step
                // branch)
                static_assert(NT == 32, "TALL: 32-column tiles");
                const int r0 = 16 * w + g;
                double a0[KS], a1[KS];
#pragma unroll
                for (int j = 0; j < KS; ++j) {
                    a0[j] = aval(r0, K0 + 4 * j + t);
                    a1[j] = aval(r0 + 8, K0 + 4 * j + t);
                }
                const double a00 = K0E ? aocc(r0) : 0.0, a01 = K0E ? aocc(r0 + 8) : 0.0;
                bar_sync(BAR_MINT, kWsHalf);
                int oB = (K0 + t) * DSTRIDE + 2 * g, oG = r0 * GSTRIDE + 4 * t;
                asm volatile("" : "+r"(oB), "+r"(oG));
                int sd = 0;
                for (int it = 0; it < ntot; ++it) {
                    const int b = it & 1;
                    const double* D = wait_d(it, sd);
                    if (!SBG_DBG(2)) {
                        double* G = Gs + b * p.grows * GSTRIDE;
                        const double* pB = D + oB;
                        double acc[4][4];
#pragma unroll
                        for (int nb = 0; nb < 4; ++nb)
#pragma unroll
                            for (int e = 0; e < 4; ++e) acc[nb][e] = 0.0;
                        double2 q[2][2];
                        q[0][0] = *reinterpret_cast<const double2*>(pB);
                        q[0][1] = *reinterpret_cast<const double2*>(pB + 16);
#pragma unroll
                        for (int j = 0; j < KS; ++j) {
                            const int cur = j & 1;
                            if (j == (KS > SBG_TALL_WAITG ? KS - SBG_TALL_WAITG : 0)) wait_g(it);
                            if (j + 1 < KS) {
                                q[cur ^ 1][0] = *reinterpret_cast<const double2*>(pB + 4 * (j + 1) * DSTRIDE);
                                q[cur ^ 1][1] = *reinterpret_cast<const double2*>(pB + 4 * (j + 1) * DSTRIDE + 16);
                            }
                            dmma_16x8x4(acc[0], a0[j], a1[j], q[cur][0].x);
                            dmma_16x8x4(acc[1], a0[j], a1[j], q[cur][0].y);
                            dmma_16x8x4(acc[2], a0[j], a1[j], q[cur][1].x);
                            dmma_16x8x4(acc[3], a0[j], a1[j], q[cur][1].y);
                        }
                        // column of acc[L][e] = 16 (L >> 1) + 4 t + 2 (e & 1) + (L & 1), rows g (e < 2), g + 8
                        if constexpr (K0E) {
                            const double2 va0 = *reinterpret_cast<const double2*>(D + 4 * t), va1 = *reinterpret_cast<const double2*>(D + 4 * t + 2);
                            const double2 vb0 = *reinterpret_cast<const double2*>(D + 16 + 4 * t), vb1 = *reinterpret_cast<const double2*>(D + 18 + 4 * t);
                            acc[0][0] = fma(a00, va0.x, acc[0][0]); acc[1][0] = fma(a00, va0.y, acc[1][0]);
                            acc[0][1] = fma(a00, va1.x, acc[0][1]); acc[1][1] = fma(a00, va1.y, acc[1][1]);
                            acc[0][2] = fma(a01, va0.x, acc[0][2]); acc[1][2] = fma(a01, va0.y, acc[1][2]);
                            acc[0][3] = fma(a01, va1.x, acc[0][3]); acc[1][3] = fma(a01, va1.y, acc[1][3]);
                            acc[2][0] = fma(a00, vb0.x, acc[2][0]); acc[3][0] = fma(a00, vb0.y, acc[3][0]);
                            acc[2][1] = fma(a00, vb1.x, acc[2][1]); acc[3][1] = fma(a00, vb1.y, acc[3][1]);
                            acc[2][2] = fma(a01, vb0.x, acc[2][2]); acc[3][2] = fma(a01, vb0.y, acc[3][2]);
                            acc[2][3] = fma(a01, vb1.x, acc[2][3]); acc[3][3] = fma(a01, vb1.y, acc[3][3]);
                        }
                        double* g0 = G + oG;
                        double* g1 = g0 + 8 * GSTRIDE;
                        *reinterpret_cast<double2*>(g0) = make_double2(acc[0][0], acc[1][0]);
                        *reinterpret_cast<double2*>(g0 + 2) = make_double2(acc[0][1], acc[1][1]);
                        *reinterpret_cast<double2*>(g1) = make_double2(acc[0][2], acc[1][2]);
                        *reinterpret_cast<double2*>(g1 + 2) = make_double2(acc[0][3], acc[1][3]);
                        *reinterpret_cast<double2*>(g0 + 16) = make_double2(acc[2][0], acc[3][0]);
                        *reinterpret_cast<double2*>(g0 + 18) = make_double2(acc[2][1], acc[3][1]);
                        *reinterpret_cast<double2*>(g1 + 16) = make_double2(acc[2][2], acc[3][2]);
                        *reinterpret_cast<double2*>(g1 + 18) = make_double2(acc[2][3], acc[3][3]);
                    } else {
                        wait_g(it);
                    }
                    if (!SBG_DBG(16)) bar_arrive(BAR_FULL + b, kWsThreads);
                }
                drain_g(ntot);
                continue;  // next row
            }
            if constexpr (XS > 0) {
                constexpr int KH = (KS + 1) / 2;          // iterations carrying an extra-row DMMA
                const int koff = (XS == 2 && w >= 4) ? KS - KH : 0;  // k-step of iteration 0
                const int xb = w & 3;                     // extra rows: this warp's n8 block
                const bool xodd = xb & 1;
                const int c01 = XS == 2 ? 16 * (xb >> 1) : 0, c23 = 16 - c01;  // columns of local blocks 0,1 / 2,3
                const int r0 = 16 * w + g, re = 16 * p.mb16;
                double a0[KS], a1[KS], aer[XS == 2 ? KH : 1];
#pragma unroll
                for (int i = 0; i < KS; ++i) {
                    int kk = i + koff;
                    if (kk >= KS) kk -= KS;
                    const int k = K0 + 4 * kk + t;
                    a0[i] = aval(main_ok ? r0 : 0, k);  // rows of idle warps (mb16 < 8) are never staged
                    a1[i] = aval(main_ok ? r0 + 8 : 0, k);
                }
                if constexpr (XS == 2) {
#pragma unroll
                    for (int i = 0; i < KH; ++i) {
                        const int kk = i + koff;  // odd KS: the middle k-step belongs to warps 0-3
                        aer[i] = (w >= 4 && kk < KH) ? 0.0 : aval(re + g, K0 + 4 * kk + t);
                    }
                } else {
                    aer[0] = 0.0;
                }
                const double a00 = (K0E && main_ok) ? aocc(r0) : 0.0, a01 = (K0E && main_ok) ? aocc(r0 + 8) : 0.0;
                const double ae0 = (XS == 2 && K0E && w < 4) ? aocc(re + g) : 0.0;
                // lane-dependent byte offsets, fixed for the kernel: pinned in registers (the opaque asm
                // stops the compiler from rebuilding them from the thread index in every tile)
                int oB01 = ((K0 + 4 * koff + t) * DSTRIDE + 2 * g + c01) * 8;  // B fragments, blocks 0,1, iterations < KH
                int oB23 = oB01 + (c23 - c01) * 8;                             // ... blocks 2,3
                int oHi = koff ? -4 * KS * DSTRIDE * 8 : 0;                    // ... iterations >= KH (rotated k order)
                int oG01 = (r0 * GSTRIDE + 4 * t + c01) * 8;                   // staged accumulators, row g of the block
                int oG23 = oG01 + (c23 - c01) * 8;
                int oX = ((re + (w >= 4 ? 8 : 0) + g) * GSTRIDE + c01 + 4 * t + (xodd ? 1 : 0)) * 8;  // extra partials
                int oC01 = (c01 + 4 * t) * 8, oC23 = (c23 + 4 * t) * 8;        // the row's own tile (k = 0 term)
                asm volatile("" : "+r"(oB01), "+r"(oB23), "+r"(oHi), "+r"(oG01), "+r"(oG23), "+r"(oX), "+r"(oC01), "+r"(oC23));
                // the tile loop, compiled once per parity of the extra block (a sub-partition's two DMMA
                // warps share it): picking the odd or even block's B fragment costs no select
                auto tile_loop = [&](auto xodd_c) {
                    [[maybe_unused]] constexpr bool XODD = decltype(xodd_c)::value;
                    int sd = 0;
                    for (int it = 0; it < ntot; ++it) {
                        const int b = it & 1;
                        const char* D = reinterpret_cast<const char*>(wait_d(it, sd));
                        if (!SBG_DBG(2) && (main_ok || XS == 2)) {
                            char* G = reinterpret_cast<char*>(Gs + b * p.grows * GSTRIDE);
                            const char* pLo01 = D + oB01;
                            const char* pLo23 = D + oB23;
                            const char* pHi01 = pLo01 + oHi;
                            const char* pHi23 = pLo23 + oHi;
                            double acc[4][4];
                            [[maybe_unused]] double acx[2] = {0.0, 0.0};
#pragma unroll
                            for (int nb = 0; nb < 4; ++nb)
#pragma unroll
                                for (int e = 0; e < 4; ++e) acc[nb][e] = 0.0;
                            double2 q[2][2];  // B fragments of local blocks (0,1) and (2,3), one k-step ahead
                            q[0][0] = *reinterpret_cast<const double2*>(pLo01);
                            q[0][1] = *reinterpret_cast<const double2*>(pLo23);
#pragma unroll
                            for (int i = 0; i < KS; ++i) {
                                const int cur = i & 1;
                                // G buffer b is needed after the last k-step; the wait sits WG k-steps earlier: its
                                // position steers the schedule ptxas builds around it (c4, KS = 17: 92.2 / 92.4 /
                                // 91.2 / 90.4 / 91.3 / 91.0 / 91.5 ms for 1 / 2 / 3 / 4 / 5 / 6 / 8 k-steps)
                                constexpr int WG = KS > SBG_XS_WAITG ? KS - SBG_XS_WAITG : 0;
                                if (i == WG) wait_g(it);
                                if (i + 1 < KS) {
                                    constexpr int STEP = 4 * DSTRIDE * 8;
                                    q[cur ^ 1][0] = *reinterpret_cast<const double2*>(((i + 1 < KH) ? pLo01 : pHi01) + (i + 1) * STEP);
                                    q[cur ^ 1][1] = *reinterpret_cast<const double2*>(((i + 1 < KH) ? pLo23 : pHi23) + (i + 1) * STEP);
                                }
#ifdef SBG_XS_EXTRA_FIRST
                                if constexpr (XS == 2) {
                                    if (i < KH) dmma_8x8x4(acx, aer[i], XODD ? q[cur][0].y : q[cur][0].x);
                                }
#endif
                                dmma_16x8x4(acc[0], a0[i], a1[i], q[cur][0].x);
                                dmma_16x8x4(acc[1], a0[i], a1[i], q[cur][0].y);
                                dmma_16x8x4(acc[2], a0[i], a1[i], q[cur][1].x);
                                dmma_16x8x4(acc[3], a0[i], a1[i], q[cur][1].y);
#ifndef SBG_XS_EXTRA_FIRST
                                if constexpr (XS == 2) {
                                    if (i < KH) dmma_8x8x4(acx, aer[i], XODD ? q[cur][0].y : q[cur][0].x);
                                }
#endif
                            }
                            // epilogue: column of acc[L][e] = (L < 2 ? c01 : c23) + 4 t + 2 (e & 1) + (L & 1),
                            // rows g (e < 2) and g + 8; the k = 0 rank-1 term (K0E) first
                            if constexpr (K0E) {
                                const double2 va0 = *reinterpret_cast<const double2*>(D + oC01), va1 = *reinterpret_cast<const double2*>(D + oC01 + 16);
                                const double2 vb0 = *reinterpret_cast<const double2*>(D + oC23), vb1 = *reinterpret_cast<const double2*>(D + oC23 + 16);
                                acc[0][0] = fma(a00, va0.x, acc[0][0]); acc[1][0] = fma(a00, va0.y, acc[1][0]);
                                acc[0][1] = fma(a00, va1.x, acc[0][1]); acc[1][1] = fma(a00, va1.y, acc[1][1]);
                                acc[0][2] = fma(a01, va0.x, acc[0][2]); acc[1][2] = fma(a01, va0.y, acc[1][2]);
                                acc[0][3] = fma(a01, va1.x, acc[0][3]); acc[1][3] = fma(a01, va1.y, acc[1][3]);
                                acc[2][0] = fma(a00, vb0.x, acc[2][0]); acc[3][0] = fma(a00, vb0.y, acc[3][0]);
                                acc[2][1] = fma(a00, vb1.x, acc[2][1]); acc[3][1] = fma(a00, vb1.y, acc[3][1]);
                                acc[2][2] = fma(a01, vb0.x, acc[2][2]); acc[3][2] = fma(a01, vb0.y, acc[3][2]);
                                acc[2][3] = fma(a01, vb1.x, acc[2][3]); acc[3][3] = fma(a01, vb1.y, acc[3][3]);
                                if constexpr (XS == 2) {  // warps 0-3 carry the extra rows' k = 0 term
                                    acx[0] = fma(ae0, XODD ? va0.y : va0.x, acx[0]);
                                    acx[1] = fma(ae0, XODD ? va1.y : va1.x, acx[1]);
                                }
                            }
                            if (main_ok) {
                                constexpr int ROW8 = 8 * GSTRIDE * 8;
                                *reinterpret_cast<double2*>(G + oG01) = make_double2(acc[0][0], acc[1][0]);
                                *reinterpret_cast<double2*>(G + oG01 + 16) = make_double2(acc[0][1], acc[1][1]);
                                *reinterpret_cast<double2*>(G + oG01 + ROW8) = make_double2(acc[0][2], acc[1][2]);
                                *reinterpret_cast<double2*>(G + oG01 + ROW8 + 16) = make_double2(acc[0][3], acc[1][3]);
                                *reinterpret_cast<double2*>(G + oG23) = make_double2(acc[2][0], acc[3][0]);
                                *reinterpret_cast<double2*>(G + oG23 + 16) = make_double2(acc[2][1], acc[3][1]);
                                *reinterpret_cast<double2*>(G + oG23 + ROW8) = make_double2(acc[2][2], acc[3][2]);
                                *reinterpret_cast<double2*>(G + oG23 + ROW8 + 16) = make_double2(acc[2][3], acc[3][3]);
                            }
                            if constexpr (XS == 2) {
                                *reinterpret_cast<double*>(G + oX) = acx[0];
                                *reinterpret_cast<double*>(G + oX + 16) = acx[1];
                            }
                        } else {
                            wait_g(it);
                        }
                        if (!SBG_DBG(16)) bar_arrive(BAR_FULL + b, kWsThreads);
                    }
                };
                if (XS == 2 && xodd) tile_loop(std::true_type{});
                else tile_loop(std::false_type{});
                drain_g(ntot);
                continue;  // next row
            }
            double a0[KS], a1[KS];
            const int r0 = 16 * w + g, re = 16 * p.mb16;
#pragma unroll
            for (int j = 0; j < KS; ++j) {
                const int k = K0 + 4 * j + t;
                a0[j] = main_ok ? aval(r0, k) : 0.0;
                a1[j] = main_ok ? aval(r0 + 8, k) : 0.0;
            }
            const double a00 = (K0E && main_ok) ? aocc(r0) : 0.0, a01 = (K0E && main_ok) ? aocc(r0 + 8) : 0.0;
            if (p.extra)
                for (int i = tid; i < KP * 8; i += kWsHalf)
                    sAe[i] = (K0E && (i >> 3) == 0) ? aocc(re + (i & 7)) : aval(re + (i & 7), i >> 3);
            bar_sync(BAR_MINT, kWsHalf);
            // the extra m8 rows' A fragments stay in registers too (warps w < NBT)
            double aer[KS];
#pragma unroll
            for (int j = 0; j < KS; ++j) aer[j] = do_extra ? sAe[(K0 + 4 * j + t) * 8 + g] : 0.0;
            const double ae0 = (K0E && do_extra) ? sAe[g] : 0.0;
            int sd = 0;
            // lane-dependent offsets pinned in registers (not rebuilt from the thread index per tile)
            int oBm = (K0 + t) * DSTRIDE + g, oGm = r0 * GSTRIDE + 2 * t;
            asm volatile("" : "+r"(oBm), "+r"(oGm));
            for (int it = 0; it < ntot; ++it) {
                const int b = it & 1;
                const double* D = wait_d(it, sd);
                if (!SBG_DBG(2) && main_ok) {
                    double* G = Gs + b * p.grows * GSTRIDE;
                    double acc[NBT][4];
                    double ace0[2] = {0.0, 0.0}, ace1[2] = {0.0, 0.0};
#pragma unroll
                    for (int nb = 0; nb < NBT; ++nb)
#pragma unroll
                        for (int e = 0; e < 4; ++e) acc[nb][e] = 0.0;
                    const double* D1 = D + oBm;  // row K0 + t, column g: B fragments of the DMMA k range
#ifndef SBG_BF_DEPTH
#define SBG_BF_DEPTH 2
#endif
                    constexpr int BFD = SBG_BF_DEPTH;  // B-fragment register ring (loads BFD-1 k-steps ahead)
                    double bf[BFD][NBT];
#pragma unroll
                    for (int jj = 0; jj < BFD - 1; ++jj)
                        if (jj < KS) {
#pragma unroll
                            for (int nb = 0; nb < NBT; ++nb) bf[jj][nb] = D1[4 * jj * DSTRIDE + nb * 8];
                        }
#pragma unroll
                    for (int j = 0; j < KS; ++j) {
                        const int cur = j % BFD;
                        // decoupled: G buffer b is needed from here on (before the last k-step, so the
                        // staging stores still interleave with the tail of the DMMA chains)
                        if (j == KS - 1) wait_g(it);
                        if (j + BFD - 1 < KS) {
#pragma unroll
                            for (int nb = 0; nb < NBT; ++nb)
                                bf[(j + BFD - 1) % BFD][nb] = D1[4 * (j + BFD - 1) * DSTRIDE + nb * 8];
                        }
#pragma unroll
                        for (int nb = 0; nb < NBT; ++nb) dmma_16x8x4(acc[nb], a0[j], a1[j], bf[cur][nb]);
                        if (do_extra) {
                            // warp w's extra n8 block is column block w: its B fragment is bf[cur][w]
                            double be = bf[cur][0];
#pragma unroll
                            for (int nb = 1; nb < NBT; ++nb)
                                if (w == nb) be = bf[cur][nb];
                            if (cur) dmma_8x8x4(ace1, aer[j], be);
                            else dmma_8x8x4(ace0, aer[j], be);
                        }
                    }
                    // epilogue: the k = 0 rank-1 term (K0E; a00 = a01 = ae0 = 0 otherwise), then
                    // 16-byte stores of the tile (decoupled: once the scatter has handed buffer b back)
                    if constexpr (K0E) {
#pragma unroll
                        for (int nb = 0; nb < NBT; ++nb) {
                            const double2 cv = *reinterpret_cast<const double2*>(D + nb * 8 + 2 * t);
                            acc[nb][0] = fma(a00, cv.x, acc[nb][0]);
                            acc[nb][1] = fma(a00, cv.y, acc[nb][1]);
                            acc[nb][2] = fma(a01, cv.x, acc[nb][2]);
                            acc[nb][3] = fma(a01, cv.y, acc[nb][3]);
                        }
                    }
                    double2 ge = make_double2(0.0, 0.0);
                    if (do_extra) {
                        ge = make_double2(ace0[0] + ace1[0], ace0[1] + ace1[1]);
                        if constexpr (K0E) {
                            const double2 cv = *reinterpret_cast<const double2*>(D + w * 8 + 2 * t);
                            ge = make_double2(fma(ae0, cv.x, ge.x), fma(ae0, cv.y, ge.y));
                        }
                    }
#pragma unroll
                    for (int nb = 0; nb < NBT; ++nb) {
                        double* gr = G + oGm + nb * 8;
                        *reinterpret_cast<double2*>(gr) = make_double2(acc[nb][0], acc[nb][1]);
                        *reinterpret_cast<double2*>(gr + 8 * GSTRIDE) = make_double2(acc[nb][2], acc[nb][3]);
                    }
                    if (do_extra) *reinterpret_cast<double2*>(G + (re + g) * GSTRIDE + w * 8 + 2 * t) = ge;
                } else {
                    wait_g(it);
                }
                if (!SBG_DBG(16)) bar_arrive(BAR_FULL + b, kWsThreads);
            }
            drain_g(ntot);
        }
    } else {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 " SBG_STR(SBG_WS_SREG) ";\n");
        const int stid = tid - kWsHalf;
        for (int i = stid; i <= ntiles; i += kWsHalf) {
            sTT[i] = p.red ? 0u : p.tile_tgt[i];
            sTE[i] = p.red ? p.tile_ent32[i] : p.tile_ent[i];
        }
        // K-list of alpha row ia into buffer kb: k = 0 the row itself (occupation column, carried by
        // sOcc), k >= 1 its single excitations (q occupied ascending, p virtual ascending)
        auto build_klist = [&](int64_t ia, int kb) {
            const uint64_t sa = string_unrank((uint64_t)ia, p.na_el, norb);
            for (int k = stid; k < KP; k += kWsHalf) {
                int J = (int)ia, off = 0;
                double sg = 0.0;
                if (k >= 1 && k < p.K) {
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
                    off = pair_sym(pp, q) * npair;
                }
                sJ[kb * KP + k] = J;
                sOff[kb * KP + k] = off;
                sSign[kb * KP + k] = sg;
            }
            for (int rs = stid; rs < p.grows; rs += kWsHalf) {  // A(rs, 0) = sum over occupied q of V'(qq, rs)
                double sum = 0.0;
                if (rs + p.m0 < npair)
                    for (uint64_t m = sa; m; m &= m - 1) {
                        const int q = __ffsll((long long)m) - 1;
                        sum += p.Vp[(size_t)pair_sym(q, q) * npair + rs + p.m0];
                    }
                sOcc[kb * p.grows + rs] = sum;
            }
        };
        // One reduction per list entry. Tile blob (build_ab_red_list): [npos][entries], the first npos
        // entries add +G, the rest add -G (the sign is loop invariant: no per-entry sign arithmetic);
        // entry = target column << 16 | byte offset into the G tile; the 16-byte padding at the end
        // points at a G padding column that holds 0.0, so it needs no test either.
        auto scatter_tile = [&](const double* G, const uint32_t* blob, uint32_t nwords, double* yrow) {
            if (nwords == 0) return;
            const uint32_t npos = blob[0], n = nwords - 1;
            const uint32_t* l32 = blob + 1;
            const char* Gb = reinterpret_cast<const char*>(G);
#pragma unroll RED_UNROLL
            for (uint32_t i = stid; i < npos; i += kWsHalf) {
                const uint32_t en = l32[i];
                red_add_f64(yrow + (en >> 16), *reinterpret_cast<const double*>(Gb + (en & 0xFFFFu)));
            }
#pragma unroll RED_UNROLL
            for (uint32_t i = npos + stid; i < n; i += kWsHalf) {
                const uint32_t en = l32[i];
                const double v = *reinterpret_cast<const double*>(Gb + (en & 0xFFFFu));
                red_add_f64(yrow + (en >> 16), __hiloint2double(__double2hiint(v) ^ 0x80000000, __double2loint(v)));
            }
        };
        if (p.red)  // the G padding columns the lists' padding entries read (never written by the MMA warps)
            for (int i = stid; i < STAGES * p.grows; i += kWsHalf) Gs[i * GSTRIDE + NT] = 0.0;
        if (p.tma) {
            if (stid == 0) {
                // D stages: one deferred arrival per loader thread (its cp.async completions); lists:
                // tx-counted bulk copy; G hand-back: one arrival per loader warp
                for (int i = 0; i < 3; ++i) mbar_init(mbD + i, kWsHalf);
                for (int i = 0; i < 2; ++i) mbar_init(mbL + i, 1);
                for (int i = 0; i < 2; ++i) mbar_init(mbE + i, kWsHalf / 32);
                mbar_init_fence();
            }
            // Decoupled pipeline (reduction mode): all loader threads gather the D rows with cp.async
            // and announce them on mbD through their own completions; warp 8 brings the tile's
            // reduction list with one bulk copy (TMA engine) onto mbL; the DMMA warps hand G back
            // through mbE. This loop only meets the DMMA warps at FULL (G(it) staged, D stage free).
            uint32_t phL = 0;
            const bool prod = (stid >> 5) == 0;
            const int plane = stid & 31;
            // this thread's 16-byte chunks of a D tile (row k, column pair `part`): shared offsets are
            // fixed, global offsets (16-byte units, from the K-list) change per row — a tile's gathers
            // cost one add and one cp.async per chunk
            constexpr int NCH = 5;  // >= ceil(KP * (NT / 2) / 256), KP <= 69
            uint32_t soff[NCH], goff[NCH];
#pragma unroll
            for (int i = 0; i < NCH; ++i) {
                const int c = stid + i * kWsHalf;
                soff[i] = c < KP * (NT / 2) ? (uint32_t)((c / (NT / 2)) * DSTRIDE + (c % (NT / 2)) * 2) : 0xFFFFFFFFu;
            }
            // the K-list of a row is built one row ahead (double buffered): the row-start barrier
            // publishes it, so neither the MMA warps' A fragments nor the first gathers wait for it
            int kb = 0;
            if (p.row_lo + blockIdx.x < p.row_hi) build_klist(p.row_lo + blockIdx.x, 0);
            for (int64_t ia = p.row_lo + blockIdx.x; ia < p.row_hi; ia += gridDim.x, kb ^= 1) {
                bar_sync(0, kWsThreads);  // row start: K-list kb published; everyone is done with buffer kb ^ 1
                const int* sJ_row = sJ + kb * KP;
                if SBG_DBG(16) {  // timing experiment: the MMA warps free-run
                    if (ia + gridDim.x < p.row_hi) build_klist(ia + gridDim.x, kb ^ 1);
                    continue;
                }
#pragma unroll
                for (int i = 0; i < NCH; ++i) {
                    const int c = stid + i * kWsHalf;
                    if (soff[i] != 0xFFFFFFFFu)
                        goff[i] = (uint32_t)(((int64_t)sJ_row[c / (NT / 2)] * p.ld) >> 1) + (uint32_t)(c % (NT / 2));
                }
                // tiles are gathered / listed in sequence order: running (tile, vector) counters
                int g_t = 0, g_v = 0, l_t = 0;
                auto gather_next = [&](int stage) {
                    if (!SBG_DBG(4)) {
                        const double* xs = p.xv[g_v] + (int64_t)g_t * NT;
                        double* dst = Ds + stage * KP * DSTRIDE;
#pragma unroll
                        for (int i = 0; i < NCH; ++i)
                            if (soff[i] != 0xFFFFFFFFu) cp_async16(dst + soff[i], xs + ((int64_t)goff[i] << 1));
                        if (++g_t == ntiles) {
                            g_t = 0;
                            ++g_v;
                        }
                    }
                    cp_async_mbar_arrive_noinc(mbD + stage);  // fires when this thread's chunks have landed
                };
                auto list_next = [&](int stage) {  // producer warp
                    if (plane == 0) {
                        const uint32_t e0 = sTE[l_t], bytes = (sTE[l_t + 1] - e0) * 4;
                        fence_proxy_async_smem();
                        mbar_arrive_expect_tx(mbL + stage, bytes);
                        if (bytes) bulk_g2s(Le + stage * p.maxE, p.ent32 + e0, bytes, mbL + stage);
                    }
                    if (++l_t == ntiles) l_t = 0;
                };
                for (int jt = 0; jt < p.dc && jt < ntot; ++jt) gather_next(jt);
                for (int jt = 0; jt < 2 && jt < ntot; ++jt)
                    if (prod) list_next(jt);
                if (ia + gridDim.x < p.row_hi) build_klist(ia + gridDim.x, kb ^ 1);  // next row's K-list
                int sd = 0, s_t = 0, s_v = 0;  // D stage, tile and vector of the tile being scattered
                double* yrow = p.yv[0] + (ia - p.row_lo) * p.ld;
                for (int it = 0; it < ntot; ++it) {
                    const int b = it & 1;
                    bar_sync(BAR_FULL + b, kWsThreads);   // G(it) staged; D stage sd free
                    if (it + p.dc < ntot) gather_next(sd);
                    sd = (sd + 1 == p.dc) ? 0 : sd + 1;
                    mbar_wait_parity(mbL + b, (phL >> b) & 1u);  // lists(it) landed
                    phL ^= 1u << b;
                    if (!SBG_DBG(1))
                        scatter_tile(Gs + b * p.grows * GSTRIDE, reinterpret_cast<const uint32_t*>(Le + b * p.maxE),
                                     sTE[s_t + 1] - sTE[s_t], yrow);
                    if (++s_t == ntiles) {
                        s_t = 0;
                        if (++s_v < p.nvec) yrow = p.yv[s_v] + (ia - p.row_lo) * p.ld;
                    }
                    __syncwarp();
                    if (plane == 0) mbar_arrive(mbE + b);  // this warp is done with G(it)
                    bar_sync(BAR_SINT, kWsHalf);           // lists stage b read by every loader
                    if (it + 2 < ntot && prod) list_next(b);
                }
                if (p.e_core != 0.0 && p.add_ecore)  // e_core * x, reduced like the tiles
                    for (int v = 0; v < p.nvec; ++v) {
                        const double* xr = p.xv[v] + ia * p.ld;
                        double* yr = p.yv[v] + (ia - p.row_lo) * p.ld;
                        for (int64_t c = stid; c < p.NB; c += kWsHalf) red_add_f64(yr + c, p.e_core * xr[c]);
                    }
            }
            return;
        }
        for (int64_t ia = p.row_lo + blockIdx.x; ia < p.row_hi; ia += gridDim.x) {
            bar_sync(0, kWsThreads);  // row start: the MMA warps are done with the previous K-list
            build_klist(ia, 0);
            if (!p.red)
                for (int64_t c = stid; c < p.ld; c += kWsHalf) srow[c] = 0.0;
            bar_sync(BAR_SINT, kWsHalf);       // sJ visible to every loader
            bar_arrive(BAR_KLIST, kWsThreads);
            auto load_d = [&](int stage, int jt) {
                if SBG_DBG(4) return;  // experiment: no gathers
                double* dst = Ds + stage * KP * DSTRIDE;
                for (int c = stid; c < KP * (NT / 2); c += kWsHalf) {
                    const int k = c / (NT / 2), part = c % (NT / 2);
                    cp_async16(dst + k * DSTRIDE + part * 2, p.x + (int64_t)sJ[k] * p.ld + (int64_t)jt * NT + part * 2);
                }
            };
            auto load_lists = [&](int stage, int jt) {
                if (p.red) {
                    const uint32_t e0 = sTE[jt], ne4 = (sTE[jt + 1] - e0) / 4;
                    uint32_t* dst = reinterpret_cast<uint32_t*>(Le + stage * p.maxE);
                    for (uint32_t c = stid; c < ne4; c += kWsHalf) cp_async16(dst + 4 * c, p.ent32 + e0 + 4 * c);
                    return;
                }
                const uint32_t t0 = sTT[jt], nt4 = (sTT[jt + 1] - t0 + 3) / 4;
                const uint32_t e0 = sTE[jt], ne8 = (sTE[jt + 1] - e0 + 7) / 8;
                for (uint32_t c = stid; c < nt4; c += kWsHalf) cp_async16(Lt + stage * p.maxT + 4 * c, p.tgt + t0 + 4 * c);
                for (uint32_t c = stid; c < ne8; c += kWsHalf) cp_async16(Le + stage * p.maxE + 8 * c, p.ent + e0 + 8 * c);
            };
            double* yrow = p.y + (ia - p.row_lo) * p.ld;
            // prologue: tiles 0 and 1
            for (int jt = 0; jt < 2 && jt < ntiles; ++jt) {
                load_d(jt, jt);
                load_lists(jt, jt);
            }
            cp_async_commit();
            cp_async_wait<0>();
            bar_sync(BAR_SINT, kWsHalf);
            for (int jt = 0; jt < 2 && jt < ntiles; ++jt) bar_arrive(BAR_DREADY + jt, kWsThreads);
            // steady state: tile it's scatter runs while the MMA warps work on tile it+1; D(it+2)
            // streams in meanwhile and is released to them as soon as the scatter is done
            for (int it = 0; it < ntiles; ++it) {
                const int b = it & 1;
                bar_sync(BAR_FULL + b, kWsThreads);   // G(it) staged; D stage b free
                if (it + 2 < ntiles) load_d(b, it + 2);
                cp_async_commit();
                if (p.red && !SBG_DBG(1)) {  // one reduction into y per (rs, column) entry
                    scatter_tile(Gs + b * p.grows * GSTRIDE, reinterpret_cast<const uint32_t*>(Le + b * p.maxE),
                                 sTE[it + 1] - sTE[it], yrow);
                } else if (!SBG_DBG(1)) {
                    const double* G = Gs + b * p.grows * GSTRIDE;
                    const uint32_t* lt = Lt + b * p.maxT;
                    const uint16_t* le = Le + b * p.maxE;
                    const uint32_t nt = sTT[it + 1] - sTT[it];
                    auto signed_g = [&](uint32_t e) {
                        const uint16_t en = le[e];
                        const long long bits = __double_as_longlong(G[en & 0x7FFF]);
                        return __longlong_as_double(bits ^ ((long long)(en & 0x8000) << 48));
                    };
                    // WSU targets per thread in flight (independent smem chains)
                    for (uint32_t i0 = stid; i0 < nt; i0 += WSU * kWsHalf) {
                        uint32_t tg[WSU], beg[WSU], end[WSU];
                        double v[WSU];
#pragma unroll
                        for (int u = 0; u < WSU; ++u) {
                            const uint32_t i = i0 + u * kWsHalf;
                            tg[u] = i < nt ? lt[i] : 0u;
                            beg[u] = (i == 0 || i >= nt) ? 0u : (lt[i - 1] & 0xFFFFu);
                            end[u] = tg[u] & 0xFFFFu;
                        }
#pragma unroll
                        for (int u = 0; u < WSU; ++u) v[u] = end[u] > beg[u] ? signed_g(beg[u]) : 0.0;
#pragma unroll
                        for (int u = 0; u < WSU; ++u)
                            for (uint32_t e = beg[u] + 1; e < end[u]; ++e) v[u] += signed_g(e);
#pragma unroll
                        for (int u = 0; u < WSU; ++u)  // padding segments (end <= beg) write nothing
                            if (end[u] > beg[u]) srow[tg[u] >> 16] += v[u];
                    }
                }
                bar_arrive(BAR_EMPTY + b, kWsThreads);
                cp_async_wait<0>();                    // D(it+2) (and lists(it+1)) landed
                bar_sync(BAR_SINT, kWsHalf);           // ... for every loader; lists stage b free
                if (it + 2 < ntiles) {
                    bar_arrive(BAR_DREADY + b, kWsThreads);
                    load_lists(b, it + 2);
                }
                cp_async_commit();
            }
            cp_async_wait<0>();
            const double* xr = p.x + ia * p.ld;
            if (p.red) {  // y already accumulates the reductions; add e_core * x the same way
                if (p.e_core != 0.0 && p.add_ecore)
                    for (int64_t c = stid; c < p.NB; c += kWsHalf) red_add_f64(yrow + c, p.e_core * xr[c]);
                continue;
            }
            // ---- write the row: y = [y] + sigma_ab + e_core * x (srow complete after the barrier)
            double* yr = yrow;
            for (int64_t c = stid; c < p.ld; c += kWsHalf) {
                double v = 0.0;
                if (c < p.NB) {
                    v = srow[c] + p.e_core * xr[c];
                    if (p.accumulate) v += yr[c];
                }
                yr[c] = v;
            }
        }
    }
}

template <int KS, int NT, bool K0E, bool TALL = false, int XS = 0>
void launch_ks(const AbPlan& pl, const AbParams& prm, int grid, cudaStream_t st) {
    auto kern = pl.ws ? k_sigma_ab_ws<KS, NT, K0E, TALL, XS> : k_sigma_ab<KS, NT>;
    static int configured[2][64] = {{0}};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !configured[pl.ws][dev]) {
        SBG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        configured[pl.ws][dev] = 1;
    }
    kern<<<grid, pl.threads, pl.smem, st>>>(prm);
    SBG_LAUNCH_CHECK();
}

// Generic opposite-spin term for sectors outside the tensor-core kernel's limits (more than 136
// pair rows, more than 68 alpha links, more than 32767 beta strings): the gather form straight from
// the reference's link tables (sigma.hpp:27-50),
//   y(Ia, Ib) += sum_{l in links(Ia)} sum_{m in links(Ib)} s_l s_m V'(pair_l, pair_m) x(J_l, J_m)
//                + e_core x(Ia, Ib).
// One warp per (row, 32-column block), one lane per column; plain FP64 FMAs.
__global__ void k_sigma_ab_direct(const double* __restrict__ x, double* __restrict__ y, const double* __restrict__ Vp,
                                  int npair, const Excitation* __restrict__ la, int La, const Excitation* __restrict__ lb,
                                  int Lb, int64_t row_lo, int64_t nrows, int64_t NB, int64_t ld, double e_core) {
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nblk = (NB + 31) / 32;
    if (warp >= nrows * nblk) return;
    const int64_t r = warp / nblk, Ib = (warp % nblk) * 32 + lane;
    const int64_t Ia = row_lo + r;
    if (Ib >= NB) return;
    double acc = 0.0;
    const Excitation* lbi = lb + Ib * Lb;
    for (int l = 0; l < La; ++l) {
        const Excitation e = la[Ia * La + l];
        const double* vrow = Vp + (size_t)pair_sym(e.p, e.q) * npair;
        const double* xr = x + (int64_t)e.target * ld;
        double part = 0.0;
        for (int m = 0; m < Lb; ++m) {
            const Excitation f = lbi[m];
            part = fma(f.sign * vrow[pair_sym(f.p, f.q)], xr[f.target], part);
        }
        acc = fma(e.sign, part, acc);
    }
    y[r * ld + Ib] += acc + e_core * x[Ia * ld + Ib];
}

}  // namespace

void launch_sigma_ab_direct(const double* x_full, double* y_local, const double* Vp, int npair, const Excitation* la,
                            int La, const Excitation* lb, int Lb, int64_t row_lo, int64_t row_hi, int64_t NB, int64_t ld,
                            double e_core, cudaStream_t st) {
    const int64_t nrows = row_hi - row_lo;
    if (nrows <= 0) return;
    const int64_t warps = nrows * ((NB + 31) / 32);
    k_sigma_ab_direct<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(x_full, y_local, Vp, npair, la, La, lb, Lb,
                                                                           row_lo, nrows, NB, ld, e_core);
    SBG_LAUNCH_CHECK();
}

namespace {
// k0e_allowed: the occupation column k = 0 may leave the DGEMM (rank-1 epilogue term, K0E)
AbPlan plan_sigma_ab_impl(int norb, int na_el, int nb_el, int64_t NA, int64_t NB, int64_t ld, bool k0e_allowed) {
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
    // more pair rows than eight MMA warps + one m8 block hold (norb > 16): passes over blocks of
    // 128 pair rows (warp-specialized reduction kernel only)
    const int red_default = !(getenv("SBG_AB_RED") && atoi(getenv("SBG_AB_RED")) == 0);
    pl.npass = 1;
    int mrows = pl.npair;
    if (pl.npair > 136 && red_default) {
        pl.npass = (pl.npair + 127) / 128;
        mrows = 128;
    }
    const int full = mrows / 16, rem = mrows % 16;
    // default: k_sigma_ab_ws with reductions into y (SBG_AB_RED=0 selects the shared-memory sigma
    // row with the target-sorted segment scatter, SBG_AB_WS then picks its warp-specialized form)
    const char* red_env = getenv("SBG_AB_RED");
    pl.red = red_env ? (atoi(red_env) != 0) : 1;
    const char* ws_env = getenv("SBG_AB_WS");
    pl.ws = (ws_env ? (atoi(ws_env) != 0) : 0) || pl.red;
    // k_sigma_ab_ws with K0E (the K - 1 links fill whole k-steps): KS = (K - 1) / 4 DMMA k-steps,
    // k = 0 an epilogue rank-1 term, D tiles of 1 + 4 KS rows; otherwise KS = ceil(K / 4), 4 KS rows
    pl.k0e = pl.ws && pl.K > 1 && (pl.K - 1) % 4 == 0 && k0e_allowed;
    if (pl.k0e) pl.KS = (pl.K - 1) / 4;
    const int KP = pl.k0e ? 1 + 4 * pl.KS : 4 * pl.KS;
    auto configure = [&](int nt) {
        const int nbt = nt / 8;
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
        pl.code_ld = pl.npass > 1 ? pl.npass * 128 : pl.npad;  // rows of the scatter-code table
        pl.threads = 32 * pl.mb16;
        pl.nt = nt;
        // scatter-list buffers: bounded by the tile's valid (rs, column) entries
        pl.maxT = 4 * ((nt * (1 + nb_el * (norb - nb_el)) + 3) / 4);
        pl.maxE = 8 * ((nt * (nb_el + nb_el * (norb - nb_el)) + 7) / 8);
        if (pl.red) {  // one u32 per entry (maxE counts u16 slots), no target lists, no sigma row
            pl.maxT = 0;
            pl.maxE = 2 * 4 * ((nt * (nb_el + nb_el * (norb - nb_el)) + 1 + 3) / 4);  // + the npos header
        }
        const int64_t ntiles = ld / nt;
        pl.smem = 64 + (size_t)(pl.red ? 0 : ld) * 8 + (size_t)STAGES * KP * (nt + 4) * 8 + (size_t)KP * 8 * 8 +
                  (size_t)STAGES * pl.npad * (nt + 8) * 8 + (size_t)STAGES * (pl.maxT * 4 + pl.maxE * 2) +
                  (size_t)(ntiles + 1) * 8 + (size_t)KP * 32 + (size_t)(pl.npad + 8) * 16 + 16;
    };
    const char* nt_env = getenv("SBG_AB_NT");
    const int nt_force = nt_env ? atoi(nt_env) : 0;
    if (nt_force == 16 || nt_force == 32) configure(nt_force);
    else {
        configure(32);
        if (pl.smem > 227 * 1024) configure(16);
    }
    if (NB > 32767) throw InvalidArgument("sigma_ab: more than 32767 beta strings is not supported by this build");
    if ((size_t)pl.npad * (pl.nt + 8) >= 32768) throw InvalidArgument("sigma_ab: pair space too large for this build");
    if (pl.smem > 227 * 1024) throw InvalidArgument("sigma_ab: beta row does not fit in shared memory");
    if (pl.KS > 17 || pl.threads > 256) throw InvalidArgument("sigma_ab: orbital space too large for this build");
    // warp-specialized kernel (k_sigma_ab_ws): 8 MMA warps + 8 load/scatter warps; 5-7 m16 blocks
    // without extra rows use the balanced TALL warp assignment (SBG_AB_TALL=0 disables it)
    const char* tall_env = getenv("SBG_AB_TALL");
    pl.tall = pl.ws && pl.nt == 32 && !pl.extra && pl.mb16 >= 5 && pl.mb16 <= 7 && pl.KS <= 13 &&
              !(tall_env && atoi(tall_env) == 0);
    if (pl.ws) pl.threads = kWsThreads;
    // bulk copies (TMA engine) for the gathers and lists of the reduction kernel; SBG_AB_TMA=0 keeps
    // the 256-thread cp.async gathers
    // 1 = reduction lists by bulk copy (D rows by cp.async), 2 = D rows too (one 256-byte bulk copy
    // per linked row: measured slower at c4, 107.7 vs 100.7 ms — the 2-stage ring does not hide its
    // latency), 0 = cp.async for both
    const char* tma_env = getenv("SBG_AB_TMA");
    const char* dc_env0 = getenv("SBG_AB_DC");
    pl.tma = (pl.ws && pl.red) ? ((tma_env ? atoi(tma_env) != 0 : 1) && !(dc_env0 && atoi(dc_env0) == 0)) : 0;
    // 16-byte-unit row offsets of the hoisted gathers are 32-bit: vectors up to 64 GB
    if ((double)NA * (double)ld >= 8.0e9) pl.tma = 0;
    // decoupled hand-offs (mbarrier D announcements, G handed back after the DMMAs) with a third D
    // stage when it fits; SBG_AB_DC=0 keeps the named-barrier hand-offs, =2 two D stages
    // uniform MMA instruction stream (see k_sigma_ab_ws): 1 = no extra rows, 2 = extra rows split
    // over all eight warps (needs all eight m16 blocks in use); SBG_AB_XS=0 keeps the older stream
    const char* xs_env = getenv("SBG_AB_XS");
    pl.xs = 0;
    if (pl.tma && pl.nt == 32 && !pl.tall && !(xs_env && atoi(xs_env) == 0)) {
        // split extra rows: 8 m16 blocks + 8 rows = 16 orbitals; built for the k-step counts of
        // K = 1 + n (16 - n), 1 <= n <= 15 (a full alpha shell, K = 1, keeps the older stream)
        const int ks = (pl.K + 3) / 4;  // the uniform stream keeps k = 0 in the DGEMM (plan_sigma_ab)
        const bool ks2 = ks == 4 || ks == 8 || ks == 10 || ks == 13 || ks == 14 || ks == 16 || ks == 17;
        if (!pl.extra) pl.xs = 1;
        else if (pl.mb16 == 8 && ks2) pl.xs = 2;
    }
    pl.gstride = pl.xs ? pl.nt + 2 : pl.nt + 8;
    pl.grows = pl.npad + (pl.xs == 2 ? 8 : 0);
    if (pl.xs) {  // G tiles: grows x gstride instead of npad x (nt + 8); lists: both partials of the extra rows
        pl.smem -= (size_t)STAGES * pl.npad * (pl.nt + 8) * 8;
        pl.smem += (size_t)STAGES * pl.grows * pl.gstride * 8;
        if (pl.xs == 2) {
            pl.smem += (size_t)STAGES * 2 * (pl.nt * 8) * 2;
            pl.maxE += 2 * pl.nt * 8;
        }
    }
    const char* dc_env = getenv("SBG_AB_DC");
    pl.dc = pl.tma ? (dc_env ? atoi(dc_env) : 3) : 0;
    if (pl.tma && pl.dc != 2 && pl.dc != 3) pl.dc = 3;
    const size_t dstage = (size_t)KP * (pl.nt + 4) * 8;
    if (pl.dc == 3 && pl.smem + dstage > 227 * 1024) pl.dc = 2;
    if (pl.dc == 3) pl.smem += dstage;
    return pl;
}
}  // namespace

AbPlan plan_sigma_ab(int norb, int na_el, int nb_el, int64_t NA, int64_t NB, int64_t ld, int nsm) {
    (void)nsm;
    // K0E (k = 0 as an epilogue rank-1 term, one k-step fewer when K - 1 is a multiple of 4) pays in
    // the TALL kernel (c2: 0.301 vs 0.335 ms) but not in the uniform stream, whose DMMA warps then
    // push 16 DFMAs per tile through the FP64 pipe they share with the other warp's DMMAs (c4: 93.9
    // ms with it, 92.2 ms with a 17th k-step instead). SBG_AB_K0E=0 turns it off everywhere.
    const char* env = getenv("SBG_AB_K0E");
    const bool allow = !(env && atoi(env) == 0);
    AbPlan pl = plan_sigma_ab_impl(norb, na_el, nb_el, NA, NB, ld, allow);
    if (pl.k0e && pl.xs) {  // the uniform stream is only built without the epilogue form
        const AbPlan alt = plan_sigma_ab_impl(norb, na_el, nb_el, NA, NB, ld, false);
        if (alt.xs) return alt;
        // the extra k-step changed the plan (it no longer takes the uniform stream): fall back to the
        // older stream with the epilogue form
        pl.xs = 0;
        const int gold = pl.gstride, rold = pl.grows;
        pl.gstride = pl.nt + 8;
        pl.grows = pl.npad;
        pl.smem += (size_t)STAGES * ((size_t)pl.grows * pl.gstride - (size_t)rold * gold) * 8;
        if (pl.smem > 227 * 1024 && pl.dc == 3) {
            pl.dc = 2;
            pl.smem -= (size_t)(pl.k0e ? 1 + 4 * pl.KS : 4 * pl.KS) * (pl.nt + 4) * 8;
        }
        if (pl.smem > 227 * 1024) throw InvalidArgument("sigma_ab: beta row does not fit in shared memory");
    }
    return pl;
}

// Per-tile target-sorted scatter lists from the (rs, Jb) -> (Ib, sign) codes ([ld][npad] u16,
// 0xFFFF = none). Sort key: target, then (rs, column) — a fixed summation order per target.
void build_ab_scatter(const AbPlan& pl, const std::vector<uint16_t>& codes, std::vector<uint32_t>& tgt,
                      std::vector<uint16_t>& ent, std::vector<uint32_t>& tile_tgt, std::vector<uint32_t>& tile_ent) {
    const int NT = pl.nt, GSTRIDE = pl.nt + 8;  // Tile<NT>::GSTRIDE
    const int64_t ntiles = pl.ld / NT;
    tgt.clear();
    ent.clear();
    tile_tgt.assign(ntiles + 1, 0);
    tile_ent.assign(ntiles + 1, 0);
    std::vector<std::pair<uint32_t, uint16_t>> items;
    for (int64_t jt = 0; jt < ntiles; ++jt) {
        items.clear();
        for (int rs = 0; rs < pl.npad; ++rs)
            for (int c = 0; c < NT; ++c) {
                const uint16_t code = codes[(size_t)(jt * NT + c) * pl.code_ld + rs];
                if (code == 0xFFFF) continue;
                items.push_back({(uint32_t)(code & 0x7FFF), (uint16_t)((rs * GSTRIDE + c) | (code & 0x8000))});
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
    }
    while (tgt.size() % 4) tgt.push_back(0);
    while (ent.size() % 8) ent.push_back(0);
    tile_tgt[ntiles] = (uint32_t)tgt.size();
    tile_ent[ntiles] = (uint32_t)ent.size();
}

// red mode: per tile every (rs, column) entry as target << 16 | negative << 15 | G offset, in G
// order, padded to 4 entries
void build_ab_red_list(const AbPlan& pl, const std::vector<uint16_t>& codes, std::vector<uint32_t>& ent,
                       std::vector<uint32_t>& tile_ent, int m0) {
    const int NT = pl.nt, GSTRIDE = pl.gstride ? pl.gstride : pl.nt + 8;  // the kernel's G row stride
    const int64_t ntiles = pl.ld / NT;
    ent.clear();
    tile_ent.assign(ntiles + 1, 0);
    std::vector<std::pair<uint32_t, uint32_t>> items;
    for (int64_t jt = 0; jt < ntiles; ++jt) {
        items.clear();
        for (int rs = 0; rs < pl.npad; ++rs)
            for (int c = 0; c < NT; ++c) {
                if (rs + m0 >= pl.npair) continue;
                const uint16_t code = codes[(size_t)(jt * NT + c) * pl.code_ld + rs + m0];
                if (code == 0xFFFF) continue;
                items.push_back({(uint32_t)(code & 0x7FFF), (uint32_t)((rs * GSTRIDE + c) | (code & 0x8000))});
                // xs == 2: the extra rows' second partial sum (warps 4-7) sits eight G rows further
                if (pl.xs == 2 && rs >= 16 * pl.mb16)
                    items.push_back({(uint32_t)(code & 0x7FFF), (uint32_t)(((rs + 8) * GSTRIDE + c) | (code & 0x8000))});
            }
        tile_ent[jt] = (uint32_t)ent.size();
        // Tile blob: [npos][positive entries][negative entries][padding to 16 bytes]; entry = target
        // column << 16 | byte offset into the staged G tile. Each sign group is kept in G order
        // (rs-major): a warp's shared-memory reads of G are then near-contiguous; target-sorting them
        // instead (a warp reducing into neighbouring y elements) measured slightly slower, and one
        // reduction per distinct target (a thread summing a target's entries first) much slower
        // (146 vs 98 ms at c4: divergent dependent chains). Padding entries read the G padding
        // column (0.0) and add it to column 0.
        uint32_t npos = 0;
        for (auto& it : items) npos += (it.second & 0x8000u) ? 0u : 1u;
        ent.push_back(npos);
        for (int neg = 0; neg < 2; ++neg)
            for (auto& it : items) {
                if (((it.second & 0x8000u) != 0) != (neg != 0)) continue;
                const uint32_t byte_off = (it.second & 0x7FFFu) * 8u;
                if (byte_off > 0xFFFFu) throw InvalidArgument("sigma_ab: staged tile too large for 16-bit list offsets");
                ent.push_back((it.first << 16) | byte_off);
            }
        while (ent.size() % 4) ent.push_back((uint32_t)(NT * 8));
        if ((int64_t)(ent.size() - tile_ent[jt]) * 2 > pl.maxE) throw InvalidArgument("sigma_ab: red list overflow");
    }
    tile_ent[ntiles] = (uint32_t)ent.size();
}

void launch_sigma_ab(const AbPlan& pl, const AbScatter& sc, const double* x_full, double* y_local, const double* Vp,
                     int64_t row_lo, int64_t row_hi, double e_core, int accumulate, int grid, cudaStream_t st, int pass) {
    launch_sigma_ab_multi(pl, sc, &x_full, &y_local, 1, Vp, row_lo, row_hi, e_core, accumulate, grid, st, pass);
}

void launch_sigma_ab_multi(const AbPlan& pl, const AbScatter& sc, const double* const* x_full, double* const* y_local,
                           int nvec, const double* Vp, int64_t row_lo, int64_t row_hi, double e_core, int accumulate,
                           int grid, cudaStream_t st, int pass) {
    ensure_binomials();
    if (row_hi <= row_lo) return;
    if (nvec < 1 || nvec > kMaxSigmaVec || (nvec > 1 && !pl.tma))
        throw InvalidArgument("sigma_ab: several vectors per launch need the bulk-copy reduction kernel");
    AbParams prm{};
    prm.x = x_full[0];
    prm.y = y_local[0];
    prm.nvec = nvec;
    for (int v = 0; v < nvec; ++v) {
        prm.xv[v] = x_full[v];
        prm.yv[v] = y_local[v];
    }
    prm.Vp = Vp;
    prm.tgt = sc.tgt;
    prm.ent = sc.ent;
    prm.tile_tgt = sc.tile_tgt;
    prm.tile_ent = sc.tile_ent;
    prm.red = pl.red;
    prm.ent32 = sc.ent32;
    prm.tile_ent32 = sc.tile_ent32;
    prm.m0 = pass * 128;
    prm.tma = pl.tma;
    prm.dc = pl.dc;
    prm.add_ecore = pass == 0;
    if (pass > 0 && !(pl.red && pl.ws)) throw InvalidArgument("sigma_ab: pair-row passes need the reduction kernel");
    if (pl.red && !accumulate) throw InvalidArgument("sigma_ab: reduction mode needs an initialised y");
    prm.norb = pl.norb;
    prm.na_el = pl.na_el;
    prm.npair = pl.npair;
    prm.mb16 = pl.mb16;
    prm.extra = pl.extra;
    prm.K = pl.K;
    prm.KP = pl.k0e ? 1 + 4 * pl.KS : 4 * pl.KS;
    prm.grows = pl.grows ? pl.grows : pl.npad;
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
#define SBG_KS(n)                                                                                   \
    case n:                                                                                         \
        if (pl.nt == 32 && pl.tall) {                                                               \
            if constexpr (n <= 13) {                                                                \
                if (pl.k0e) launch_ks<n, 32, true, true>(pl, prm, grid, st);                        \
                else launch_ks<n, 32, false, true>(pl, prm, grid, st);                              \
            }                                                                                       \
        } else if (pl.nt == 32 && pl.xs == 2) { /* the uniform stream keeps k = 0 in the DGEMM */  \
            /* 8 m16 blocks + 8 extra rows = 16 orbitals: K = 1 + n (16 - n), these k-step counts */  \
            if constexpr (n == 4 || n == 8 || n == 10 || n == 13 || n == 14 || n == 16 || n == 17)    \
                launch_ks<n, 32, false, false, 2>(pl, prm, grid, st);                               \
            else throw InvalidArgument("sigma_ab: no split-extra-rows kernel for this K");          \
        } else if (pl.nt == 32 && pl.xs == 1) {                                                     \
            launch_ks<n, 32, false, false, 1>(pl, prm, grid, st);                                   \
        } else if (pl.nt == 32) {                                                                   \
            if (pl.k0e) launch_ks<n, 32, true>(pl, prm, grid, st);                                  \
            else launch_ks<n, 32, false>(pl, prm, grid, st);                                        \
        } else {                                                                                    \
            if (pl.k0e) launch_ks<n, 16, true>(pl, prm, grid, st);                                  \
            else launch_ks<n, 16, false>(pl, prm, grid, st);                                        \
        }                                                                                           \
        break;
#ifdef SBG_KS_ONLY  // developer builds: one k-step count (c4: 16) compiles in seconds
        SBG_KS(SBG_KS_ONLY)
#else
        SBG_KS(1) SBG_KS(2) SBG_KS(3) SBG_KS(4) SBG_KS(5) SBG_KS(6) SBG_KS(7) SBG_KS(8) SBG_KS(9) SBG_KS(10)
        SBG_KS(11) SBG_KS(12) SBG_KS(13) SBG_KS(14) SBG_KS(15) SBG_KS(16) SBG_KS(17)
#endif
#undef SBG_KS
        default: throw InvalidArgument("sigma_ab: unsupported K");
    }
}

}  // namespace sbg
