// tables.cu — K1 string addressing, K2 single-excitation tables, K3 exact diagonal, and the
// beta-side scatter codes of the alpha-beta sigma kernel. Integer work is bit-exact with the
// reference by construction; the diagonal follows the reference's summation order with every
// product/sum rounded separately (no FMA contraction; this file is also built with --fmad=false).
#include "common.cuh"
#include "kernels.cuh"

namespace sbg {


// K1: strings in increasing-integer order (determinants.hpp:41-59) by colex unranking.
__global__ void k_strings(uint64_t* out, int64_t n, int nel, int norb) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = string_unrank((uint64_t)i, nel, norb);
}

// K2: link table rows in the reference order (sigma.hpp:27-50): for q ascending over occupied
// orbitals, the occupation entry (q,q,self,+1), then p ascending over empty orbitals of str-q
// (p != q) with sign (-1)^(popcount_below(str,q) + popcount_below(str-q,p)).
__global__ void k_links(const uint64_t* strings, int64_t n, int norb, int row_len, Excitation* out) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= n) return;
    const uint64_t str = strings[s];
    Excitation* row = out + s * row_len;
    int o = 0;
    for (int q = 0; q < norb; ++q) {
        if (!((str >> q) & 1)) continue;
        row[o++] = Excitation{(uint16_t)q, (uint16_t)q, (uint32_t)s, 1.0};
        const uint64_t rem = str ^ ((uint64_t)1 << q);
        const int sq = pop_below(str, q);
        for (int p = 0; p < norb; ++p) {
            if (((rem >> p) & 1) || p == q) continue;
            const int sp = pop_below(rem, p);
            row[o++] = Excitation{(uint16_t)p, (uint16_t)q, string_rank(rem | ((uint64_t)1 << p)),
                                  ((sq + sp) & 1) ? -1.0 : 1.0};
        }
    }
}

// Same-spin part of the diagonal for one string (fci_operator.hpp:29-35), rounded step by step.
__global__ void k_string_energy(const uint64_t* strings, int64_t n, int norb, const double* h1, const double* eri,
                                double* out) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= n) return;
    const uint64_t str = strings[s];
    int occ[kMaxOrb];
    int no = 0;
    for (int p = 0; p < norb; ++p)
        if ((str >> p) & 1) occ[no++] = p;
    double e = 0.0;
    for (int a = 0; a < no; ++a) e = __dadd_rn(e, h1[occ[a] * norb + occ[a]]);
    const size_t n2 = (size_t)norb * norb;
    for (int a = 0; a < no; ++a)
        for (int b = 0; b < no; ++b) {
            const int i = occ[a], j = occ[b];
            const double iijj = eri[(size_t)(i * norb + i) * n2 + j * norb + j];
            const double ijji = eri[(size_t)(i * norb + j) * n2 + j * norb + i];
            e = __dadd_rn(e, __dmul_rn(0.5, __dsub_rn(iijj, ijji)));
        }
    out[s] = e;
}

// K3: D[ia,ib] = ((e_core + e_a) + e_b) + cross, cross summed i over occ(a), j over occ(b)
// in ascending order (fci_operator.hpp:49-55). Output in the padded local layout.
__global__ void k_diag(const uint64_t* sa, const uint64_t* sb, const double* ea, const double* eb, int64_t row_lo,
                       int64_t nrows, int64_t nb, int64_t ld, int norb, const double* eri, double e_core,
                       double* out) {
    __shared__ double J[kMaxOrb * kMaxOrb];
    const size_t n2 = (size_t)norb * norb;
    for (int t = threadIdx.x; t < norb * norb; t += blockDim.x) {
        const int i = t / norb, j = t % norb;
        J[t] = eri[(size_t)(i * norb + i) * n2 + j * norb + j];
    }
    __syncthreads();
    const int64_t r = blockIdx.y;
    if (r >= nrows) return;
    const int64_t ia = row_lo + r;
    const uint64_t a = sa[ia];
    int oa[kMaxOrb];
    int na = 0;
    for (int p = 0; p < norb; ++p)
        if ((a >> p) & 1) oa[na++] = p;
    const double base = __dadd_rn(e_core, ea[ia]);
    for (int64_t ib = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ib < ld; ib += (int64_t)gridDim.x * blockDim.x) {
        double d = 0.0;
        if (ib < nb) {
            const uint64_t b = sb[ib];
            double cross = 0.0;
            for (int x = 0; x < na; ++x) {
                const double* Jr = J + oa[x] * norb;
                for (uint64_t bb = b; bb; bb &= bb - 1) cross = __dadd_rn(cross, Jr[__ffsll((long long)bb) - 1]);
            }
            d = __dadd_rn(__dadd_rn(base, eb[ib]), cross);
        }
        out[r * ld + ib] = d;
    }
}

// Beta-side scatter codes of the alpha-beta kernel: for column string Jb and packed pair
// rs=(r>=s): the one determinant E_rs|Jb> or E_sr|Jb> reaches (if any) and its sign.
// code = target | (sign<0) << 15, 0xFFFF = no contribution. Layout [ld][npad].
__global__ void k_scatter_codes(const uint64_t* sb, int64_t nb, int64_t ld, int norb, int npair, int npad,
                                uint16_t* out) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= ld * npad) return;
    const int64_t jb = idx / npad;
    const int rs = (int)(idx % npad);
    uint16_t code = 0xFFFF;
    if (jb < nb && rs < npair) {
        int r = 0;
        while ((r + 1) * (r + 2) / 2 <= rs) ++r;
        const int s = rs - r * (r + 1) / 2;
        const uint64_t str = sb[jb];
        const bool orr = (str >> r) & 1, os = (str >> s) & 1;
        if (r == s) {
            if (orr) code = (uint16_t)jb;
        } else if (orr != os) {
            const int o = orr ? r : s, v = orr ? s : r;
            const uint64_t rem = str ^ ((uint64_t)1 << o);
            const int par = pop_below(str, o) + pop_below(rem, v);
            code = (uint16_t)(string_rank(rem | ((uint64_t)1 << v)) | ((par & 1) << 15));
        }
    }
    out[idx] = code;
}

void launch_strings(uint64_t* out, int64_t n, int nel, int norb, cudaStream_t st) {
    ensure_binomials();
    k_strings<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(out, n, nel, norb);
    SBG_LAUNCH_CHECK();
}
void launch_links(const uint64_t* strings, int64_t n, int norb, int row_len, Excitation* out, cudaStream_t st) {
    ensure_binomials();
    k_links<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(strings, n, norb, row_len, out);
    SBG_LAUNCH_CHECK();
}
void launch_string_energy(const uint64_t* strings, int64_t n, int norb, const double* h1, const double* eri,
                          double* out, cudaStream_t st) {
    ensure_binomials();
    k_string_energy<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(strings, n, norb, h1, eri, out);
    SBG_LAUNCH_CHECK();
}
void launch_diag(const uint64_t* sa, const uint64_t* sb, const double* ea, const double* eb, int64_t row_lo,
                 int64_t nrows, int64_t nb, int64_t ld, int norb, const double* eri, double e_core, double* out,
                 cudaStream_t st) {
    if (nrows == 0) return;
    dim3 grid((unsigned)std::min<int64_t>((ld + 255) / 256, 64), (unsigned)nrows);
    k_diag<<<grid, 256, 0, st>>>(sa, sb, ea, eb, row_lo, nrows, nb, ld, norb, eri, e_core, out);
    SBG_LAUNCH_CHECK();
}
void launch_scatter_codes(const uint64_t* sb, int64_t nb, int64_t ld, int norb, int npair, int npad, uint16_t* out,
                          cudaStream_t st) {
    ensure_binomials();
    const int64_t n = ld * npad;
    k_scatter_codes<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(sb, nb, ld, norb, npair, npad, out);
    SBG_LAUNCH_CHECK();
}

}  // namespace sbg
