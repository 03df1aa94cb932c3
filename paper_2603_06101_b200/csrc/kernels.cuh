// kernels.cuh — launch interfaces of the sm_100a kernels (host-callable).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <vector>

namespace sbg {

// byte-compatible with sbg_excitation / sbci::fci::Excitation (fci/sigma.hpp:19-23)
struct Excitation {
    uint16_t p, q;
    uint32_t target;
    double sign;
};
static_assert(sizeof(Excitation) == 16, "Excitation layout");

// ---- tables.cu ----
void launch_strings(uint64_t* out, int64_t n, int nel, int norb, cudaStream_t st);
void launch_links(const uint64_t* strings, int64_t n, int norb, int row_len, Excitation* out, cudaStream_t st);
void launch_string_energy(const uint64_t* strings, int64_t n, int norb, const double* h1, const double* eri,
                          double* out, cudaStream_t st);
void launch_diag(const uint64_t* sa, const uint64_t* sb, const double* ea, const double* eb, int64_t row_lo,
                 int64_t nrows, int64_t nb, int64_t ld, int norb, const double* eri, double e_core, double* out,
                 cudaStream_t st);
void launch_scatter_codes(const uint64_t* sb, int64_t nb, int64_t ld, int norb, int npair, int npad, uint16_t* out,
                          cudaStream_t st);

constexpr int kMaxSigmaVec = 4;  // vectors per multi-vector sigma launch

// ---- sigma_ab.cu: opposite-spin term (+ folded one-body, + e_core), K6 ----
struct AbPlan {
    int norb, na_el, nb_el, npair, npad, mb16, extra, K, KS, threads, maxT, maxE, nt, ws, red;
    int k0e;  // ws kernel: occupation column k = 0 as an epilogue rank-1 term (K - 1 divisible by 4)
    int tall; // ws kernel: balanced warp assignment for 5-7 m16 blocks (warps 4-7 span the rest)
    int npass = 1;    // pair-row blocks of 128 rows (npair > 136); 1 = one pass over all rows
    int tma = 0;      // ws red kernel: D rows and reduction lists by bulk copies (UBLKCP) on mbarriers
    int dc = 0;       // ws red kernel: decoupled (mbarrier) hand-offs with this many D stages (0 = off)
    int xs = 0;       // ws red kernel: uniform MMA instruction stream (1 = no extra rows, 2 = split extra rows)
    int gstride = 0;  // staged G tile: row stride in doubles (nt + 8, or nt + 2 with xs) ...
    int grows = 0;    // ... and rows (npad, + 8 with xs == 2: both partial sums of the extra rows)
    int code_ld = 0;  // rows per beta string of the scatter-code table (npad, or npass * 128)
    int64_t NA, NB, ld;
    size_t smem;
};
struct AbScatter {  // device pointers of the per-tile segment lists (build_ab_scatter)
    const uint32_t* tgt;
    const uint16_t* ent;
    const uint32_t* tile_tgt;
    const uint32_t* tile_ent;
    const uint32_t* ent32;       // red mode (build_ab_red_list)
    const uint32_t* tile_ent32;
};
AbPlan plan_sigma_ab(int norb, int na_el, int nb_el, int64_t NA, int64_t NB, int64_t ld, int nsm);
void build_ab_scatter(const AbPlan& pl, const std::vector<uint16_t>& codes, std::vector<uint32_t>& tgt,
                      std::vector<uint16_t>& ent, std::vector<uint32_t>& tile_tgt, std::vector<uint32_t>& tile_ent);
void build_ab_red_list(const AbPlan& pl, const std::vector<uint16_t>& codes, std::vector<uint32_t>& ent,
                       std::vector<uint32_t>& tile_ent, int m0 = 0);
void launch_sigma_ab(const AbPlan& pl, const AbScatter& sc, const double* x_full, double* y_local, const double* Vp,
                     int64_t row_lo, int64_t row_hi, double e_core, int accumulate, int grid, cudaStream_t st,
                     int pass = 0);
// the same for nvec <= kMaxSigmaVec vectors in one launch (bulk-copy reduction kernel, pl.tma)
void launch_sigma_ab_multi(const AbPlan& pl, const AbScatter& sc, const double* const* x_full, double* const* y_local,
                           int nvec, const double* Vp, int64_t row_lo, int64_t row_hi, double e_core, int accumulate,
                           int grid, cudaStream_t st, int pass = 0);
// generic fallback outside plan_sigma_ab's limits: y(local rows) += sigma_ab + e_core x from the link tables
void launch_sigma_ab_direct(const double* x_full, double* y_local, const double* Vp, int npair, const Excitation* la,
                            int La, const Excitation* lb, int Lb, int64_t row_lo, int64_t row_hi, int64_t NB, int64_t ld,
                            double e_core, cudaStream_t st);

// ---- sigma_ss.cu: same-spin term via the (n-2)-electron intermediate, K4/K5 ----
struct SsPlan {
    int norb, nel, P, KSS, warps, npa;
    int64_t NK;
    size_t smem;
    int bulk = 1;  // staged tiles reduced into y by TMA bulk reductions (UBLKRED)
    int xrows = 0; // rows per staged X tile
};
SsPlan plan_sigma_ss(int norb, int nel);
// generic fallback outside plan_sigma_ss's limits: the one-spin two-body operator as CSR
struct SsCsr {
    int64_t nstr = 0;
    std::vector<int64_t> rowptr;
    std::vector<int> col;
    std::vector<double> val;
};
struct SsCsrDev {
    int64_t nstr = 0;
    const int64_t* rowptr = nullptr;
    const int* col = nullptr;
    const double* val = nullptr;
};
void build_ss_csr(int norb, int nel, const double* Va, SsCsr& out);
// y may be a column window of the output: column c of row I at y[I * ldy + c - ycol0] (ldy 0 = ldx)
void launch_sigma_ss_csr(const SsCsrDev& m, const double* x, double* y, int64_t ldx, int64_t col_lo, int64_t col_hi,
                         cudaStream_t st, int64_t ldy = 0, int64_t ycol0 = 0);
// col_pad > col_hi: columns [col_hi, col_pad) are zero padding of x inside y's rows (whole tiles may
// reduce across them)
void launch_sigma_ss(const SsPlan& pl, const double* x, double* y, const double* Va, int64_t ldx, int64_t col_lo,
                     int64_t col_hi, cudaStream_t st, int64_t ldy = 0, int64_t ycol0 = 0, int64_t col_pad = 0);
// nvec <= kMaxSigmaVec vectors (same layout each) in one launch (bulk-reduction kernel)
void launch_sigma_ss_multi(const SsPlan& pl, const double* const* x, double* const* y, int nvec, const double* Va,
                           int64_t ldx, int64_t col_lo, int64_t col_hi, cudaStream_t st, int64_t ldy = 0,
                           int64_t ycol0 = 0, int64_t col_pad = 0);
// dst[c][r] = src[r][c] (+ dst if accumulate), for r < R, c < C; dst columns r in [R, dst_cols) zeroed,
// columns >= dst_cols untouched (a column window of a wider destination).
void launch_transpose(const double* src, int64_t R, int64_t C, int64_t lds, double* dst, int64_t ldd, int64_t dst_rows,
                      int64_t dst_cols, int accumulate, cudaStream_t st);
// one-body + e_core sigma for sectors without an opposite-spin term (n_alpha == 0 or n_beta == 0)
void launch_onebody(const double* x, double* y, const Excitation* la, int La, const Excitation* lb, int Lb,
                    const double* h1, int norb, int64_t NA, int64_t NB, int64_t ld, double e_core, int accumulate,
                    cudaStream_t st);

// ---- vec.cu: fused HBM passes of the SBCI update (K7-K9) ----
constexpr int kMaxIn = 10, kMaxOut = 6, kMaxDot = 16;
constexpr int kMaxRed = 64;  // dot products per reduction workspace (pair subspace: 36 cross dots)
struct LinArgs {
    int64_t n;  // doubles per vector (padded local length, even)
    int nin, nout, ndot;
    const double* in[kMaxIn];
    double* out[kMaxOut];
    // out[j] = sum_s coef[j][s] * slot[s], slots 0..9 = inputs, 10..15 = outputs already computed (j' < j);
    // out[j] may be null (value only used by later outputs / dots)
    double coef[kMaxOut][kMaxIn + kMaxOut];
    unsigned char da[kMaxDot], db[kMaxDot];  // dot slots
    unsigned int dmask;                       // slots read by the dots (set by launch_lincomb)
    // optional weighted dot: dot index kdot accumulates s[da]^2 (kD_i - kshift) instead of
    // s[da] s[db] (the trace's kinetic scalar y^T (D - E0) y, sbci1.hpp:135-139), kdot < 0: none
    int kdot;
    const double* kD;
    double kshift;
    // coefficients read from device memory ([kMaxOut][kMaxIn + kMaxOut], written by an earlier kernel
    // of the same stream) instead of coef: the SBCI1 commit pass after launch_step_scalars
    const double* dcoef;
};
// ---- step_scalars.cu: the SBCI1 step's 2x2/3x3 algebra on one device thread ----
struct StepScalarArgs {
    double Ax, Bx, By, Cx, Cy, Cz;  // Gram-Schmidt triangle (ortho.hpp:45-76)
    int three;                      // 3-vector {x, y, z} form
};
// dots: the subspace pass's m x m cross dots; coef: the commit pass's coefficient table; out[0..8]:
// restart flag, k, b, c, E', second Ritz value, its x/y/z coefficients
void launch_step_scalars(const double* dots, const StepScalarArgs& a, double* coef, double* out, cudaStream_t st);
struct ReduceWs {
    double* partial;  // [grid][kMaxRed]
    double* result;   // [kMaxRed] device
    double* host;     // pinned [kMaxRed]
    int grid;         // capacity of partial in blocks; each pass launches min(grid, resident blocks)
    unsigned int* ticket;  // device counter electing the block that finishes a pass's sums (0 between passes)
    // single GPU: the finishing block also writes the sums into mapped host memory and then bumps a
    // sequence flag there, so the host reads a pass's dots by polling host memory instead of a copy
    // plus a stream synchronisation (Context::finish_dots; small sectors are latency bound)
    struct ZeroCopy {
        double* mirror;                 // mapped pinned [kMaxRed] (UVA: valid on host and device)
        unsigned long long* flag;       // mapped pinned: seq of the last finished pass
        unsigned long long seq = 0;     // host: seq handed to the latest pass with dots
        bool fresh = false;             // host: the latest writer of the dot buffer was such a pass
    };
    ZeroCopy* zc = nullptr;
};
// returns nothing; results land in ws.result (device). Caller copies to host after collectives.
void launch_lincomb(const LinArgs& a, const ReduceWs& ws, cudaStream_t st);
// z = zres / den(D - shift) - sum_c o_c xc_c ; with dots per LinArgs-like slot spec on (zres=0, D=1, x=2, y=3, z_out=8)
struct PrecArgs {
    int64_t n;
    const double* zres;
    const double* D;
    double shift, clamp;
    int nxc;
    const double* xc[8];
    double o[8];     // overlaps to subtract (used when mode == 1)
    int mode;        // 0: only compute overlaps xc_c . (zres/den) ; 1: write z and compute dots
    double* z;
    const double* x;
    const double* y;  // may be null
};
void launch_precond(const PrecArgs& a, const ReduceWs& ws, cudaStream_t st);
// subspace matrix of the materialized basis (sbci1.hpp:193-219): returns V00,V01,V11 (two) or
// V00,V01,V02,V11,V12,V22 (three)
struct SubArgs {
    int64_t n;
    const double *x, *y, *z, *hx, *hy, *hz;
    double Ax, Bx, By, Cx, Cy, Cz;
    int three;
};
void launch_subspace(const SubArgs& a, const ReduceWs& ws, cudaStream_t st);
// generic deterministic dot/norm reductions finish: partials -> result
void launch_reduce_finish(const ReduceWs& ws, int nblk, int ndot, cudaStream_t st);
// Gram matrix of up to 6 vectors: dots v_i . v_j for i <= j, row-major upper triangle
void launch_gram(const double* const* v, int m, int64_t n, const ReduceWs& ws, cudaStream_t st);
// SBCI2 subspace matrix over the materialized orthonormal basis (sbci2.hpp:144-176): w_i = v_i/|v_i|
// (inv_n[i] = 0 drops v_i), b_c = sum_i P[i][c] w_i, B_c likewise from the images; returns the r x r
// cross dots b_c . B_d (row-major)
struct PairSubArgs {
    int64_t n;
    int m, r;
    const double* v[6];
    const double* h[6];
    double inv_n[6];
    double P[6][6];
};
void launch_pair_subspace(const PairSubArgs& a, const ReduceWs& ws, cudaStream_t st);
// Davidson Ritz vectors (davidson.hpp:96-105, 109-111) over one chunk of <= kRitzChunk basis vectors:
// ritz_k (+)= sum_i coef[i][k] b_i and ritz_im_k likewise from the images, accumulated in basis order
// (first: from zero); on the last chunk also res_k = ritz_im_k - theta_k ritz_k and |res_k|^2
constexpr int kRitzChunk = 16, kMaxRoots = 9;
struct RitzArgs {
    int64_t n;
    int m, k, first, last;
    const double* b[kRitzChunk];
    const double* h[kRitzChunk];
    double coef[kRitzChunk][kMaxRoots];
    double theta[kMaxRoots];
    double* ritz[kMaxRoots];
    double* ritz_im[kMaxRoots];
    double* res[kMaxRoots];
};
void launch_ritz(const RitzArgs& a, const ReduceWs& ws, cudaStream_t st);
// argmin with index tie-break over a padded matrix (valid cols < ncols), excluding (value,index) <= prev
void launch_argmin_after(const double* D, int64_t nrows, int64_t ncols, int64_t ld, int64_t row_lo, double prev_v,
                         int64_t prev_i, double* out_v, int64_t* out_i, double* part_v, int64_t* part_i, int grid,
                         cudaStream_t st);
void launch_kinetic(const double* y, const double* D, double shift, int64_t n, const ReduceWs& ws, cudaStream_t st);
void launch_fill(double* p, int64_t n, double v, cudaStream_t st);
void launch_set_element(double* p, int64_t idx, double v, cudaStream_t st);

// ---- spin.cu ----
// |S+ x|^2 over raised-sector alpha strings [ja_lo, ja_hi) (fci/spin.hpp:17-51); x_full is the whole
// padded vector; the result lands in ws.result[0]
void launch_spin_raise(const double* x_full, int64_t ld, int na, int nb, int norb, int64_t ja_lo, int64_t ja_hi,
                       const ReduceWs& ws, cudaStream_t st);

// ---- selftest.cu ----
int run_mma_selftest();
int run_nccl_selftest();

}  // namespace sbg
