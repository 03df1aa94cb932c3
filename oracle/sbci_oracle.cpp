// oracle/sbci_oracle.cpp — TEST INFRASTRUCTURE ONLY. This is the CPU restatement of the
// reference's hot-path arithmetic (arXiv 2603.06101 reference, /root/reference/proj). It is
// the checker for the CUDA product path: only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load it. It is never linked into libsbg.so.
//
// Pinning: every function here is checked against the compiled reference itself
// (oracle/_ref/libsbci_ref.so, built from /root/reference by oracle/Makefile) and against the
// reference's checked-in fixtures (tests/golden/h4_2e.fcidump, h6_4e.fcidump) by
// tests/test_oracle_pins.py. The exact blocked sigma is pinned BIT-EXACTLY against
// sbci::fci::contract_sigma.
//
// Restated routines (reference file:line each follows):
//   or_strings            determinants.hpp:41-59   (Gosper enumeration, increasing integers)
//   or_links              sigma.hpp:27-50          (link table order and signs)
//   or_absorb_h1          sigma.hpp:56-81
//   or_diag               fci_operator.hpp:16-57   (same summation order, no FMA)
//   or_sigma_blocked      sigma.hpp:86-137         (contract_sigma, processed in alpha-row blocks;
//                                                   exact=1 reproduces the reference's accumulation
//                                                   order bit for bit)
//   or_sc_element / or_dense_h / or_sigma_rows
//                         tests/support/dense_oracle.hpp:101-189 (textbook Slater-Condon rules)
//   or_synthetic          BASELINE.json integral generator (not in the reference; pinned here)
#include <algorithm>
#include <bit>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

using u64 = std::uint64_t;

u64 binom(int n, int k) {
    if (k < 0 || k > n) return 0;
    k = std::min(k, n - k);
    unsigned __int128 r = 1;
    for (int i = 1; i <= k; ++i) r = r * (unsigned)(n - k + i) / (unsigned)i;
    return (u64)r;
}

// Gosper's hack, strictly increasing (determinants.hpp:41-59).
std::vector<u64> strings_of(int norb, int k) {
    std::vector<u64> out;
    if (k == 0) { out.push_back(0); return out; }
    const u64 limit = (norb == 63) ? (~u64{0} >> 1) : (u64{1} << norb);
    u64 v = (u64{1} << k) - 1;
    while (v < limit) {
        out.push_back(v);
        const u64 c = v & (~v + 1);
        const u64 r = v + c;
        if (c == 0) break;
        v = (((r ^ v) >> 2) / c) | r;
    }
    return out;
}

int pop_below(u64 s, int orb) { return std::popcount(s & ((u64{1} << orb) - 1)); }

size_t index_of(const std::vector<u64>& strs, u64 s) {
    auto it = std::lower_bound(strs.begin(), strs.end(), s);
    if (it == strs.end() || *it != s) throw std::logic_error("string not in enumeration");
    return (size_t)(it - strs.begin());
}

struct Link { int p, q; uint32_t target; double sign; };

// sigma.hpp:27-50: per string, q ascending over occupied: (q,q,self,+1) then p ascending
// over orbitals empty after removing q (p != q).
std::vector<std::vector<Link>> links_of(const std::vector<u64>& strs, int norb) {
    std::vector<std::vector<Link>> L(strs.size());
    for (size_t s = 0; s < strs.size(); ++s) {
        const u64 str = strs[s];
        for (int q = 0; q < norb; ++q) {
            if (!((str >> q) & 1)) continue;
            L[s].push_back({q, q, (uint32_t)s, 1.0});
            const u64 rem = str ^ (u64{1} << q);
            const int sq = pop_below(str, q);
            for (int p = 0; p < norb; ++p) {
                if (((rem >> p) & 1) || p == q) continue;
                const int sp = pop_below(rem, p);
                L[s].push_back({p, q, (uint32_t)index_of(strs, rem | (u64{1} << p)), ((sq + sp) % 2 == 0) ? 1.0 : -1.0});
            }
        }
    }
    return L;
}

struct Prob {
    int norb, nelec, ms2;
    double e_core;
    const double* h1;
    const double* eri;
    int na() const { return (nelec + ms2) / 2; }
    int nb() const { return (nelec - ms2) / 2; }
    double h(int i, int j) const { return h1[i * norb + j]; }
    double g(int i, int j, int k, int l) const { return eri[(((size_t)i * norb + j) * norb + k) * norb + l]; }
};

// sigma.hpp:56-81
std::vector<double> absorb(const Prob& P, int nsec) {
    const int no = P.norb;
    const size_t no2 = (size_t)no * no;
    std::vector<double> h2e(P.eri, P.eri + no2 * no2);
    std::vector<double> f(no2);
    for (int p = 0; p < no; ++p)
        for (int q = 0; q < no; ++q) {
            double corr = 0.0;
            for (int r = 0; r < no; ++r) corr += P.g(p, r, r, q);
            f[p * no + q] = (P.h(p, q) - 0.5 * corr) / (double)nsec;
        }
    for (int k = 0; k < no; ++k)
        for (int p = 0; p < no; ++p)
            for (int q = 0; q < no; ++q) {
                h2e[((size_t)(k * no + k)) * no2 + p * no + q] += f[p * no + q];
                h2e[((size_t)(p * no + q)) * no2 + k * no + k] += f[p * no + q];
            }
    for (double& v : h2e) v *= 0.5;
    return h2e;
}

std::vector<int> occ_of(u64 s, int norb) {
    std::vector<int> o;
    for (int p = 0; p < norb; ++p) if ((s >> p) & 1) o.push_back(p);
    return o;
}

// ---- Slater-Condon rules (dense_oracle.hpp:101-189), restated ----
double phase_between(u64 str, int hole, int part) {
    const int lo = std::min(hole, part) + 1, hi = std::max(hole, part);
    int c = 0;
    for (int p = lo; p < hi; ++p) c += (str >> p) & 1;
    return (c % 2 == 0) ? 1.0 : -1.0;
}

double sc_element(const Prob& P, u64 a1, u64 b1, u64 a2, u64 b2) {
    const int no = P.norb;
    const int da = std::popcount(a1 ^ a2) / 2, db = std::popcount(b1 ^ b2) / 2;
    if (da + db > 2) return 0.0;
    const auto oa = occ_of(a1, no), ob = occ_of(b1, no);
    if (da == 0 && db == 0) {
        double e = P.e_core;
        for (int i : oa) e += P.h(i, i);
        for (int i : ob) e += P.h(i, i);
        for (int i : oa) for (int j : oa) e += 0.5 * (P.g(i, i, j, j) - P.g(i, j, j, i));
        for (int i : ob) for (int j : ob) e += 0.5 * (P.g(i, i, j, j) - P.g(i, j, j, i));
        for (int i : oa) for (int j : ob) e += P.g(i, i, j, j);
        return e;
    }
    auto single = [&](u64 s1, u64 s2, const std::vector<int>& other) {
        const int i = std::countr_zero(s1 & ~s2), j = std::countr_zero(s2 & ~s1);
        double e = P.h(i, j);
        for (int k : occ_of(s1 & s2, no)) e += P.g(i, j, k, k) - P.g(i, k, k, j);
        for (int k : other) e += P.g(i, j, k, k);
        return phase_between(s1, i, j) * e;
    };
    if (da == 1 && db == 0) return single(a1, a2, ob);
    if (da == 0 && db == 1) return single(b1, b2, oa);
    if (da == 1 && db == 1) {
        const int ia = std::countr_zero(a1 & ~a2), pa = std::countr_zero(a2 & ~a1);
        const int ib = std::countr_zero(b1 & ~b2), pb = std::countr_zero(b2 & ~b1);
        return phase_between(a1, ia, pa) * phase_between(b1, ib, pb) * P.g(ia, pa, ib, pb);
    }
    auto dbl = [&](u64 s1, u64 s2) {
        const auto h = occ_of(s1 & ~s2, no), p = occ_of(s2 & ~s1, no);
        const u64 mid = (s1 ^ (u64{1} << h[0])) | (u64{1} << p[0]);
        const double ph = phase_between(s1, h[0], p[0]) * phase_between(mid, h[1], p[1]);
        return ph * (P.g(h[0], p[0], h[1], p[1]) - P.g(h[0], p[1], h[1], p[0]));
    };
    return da == 2 ? dbl(a1, a2) : dbl(b1, b2);
}

// colex rank == position in the increasing-integer enumeration
struct Ranker {
    int norb;
    std::vector<u64> C;  // C[n*(norb+1)+k]
    explicit Ranker(int no) : norb(no), C((size_t)(no + 1) * (no + 2), 0) {
        for (int n = 0; n <= no; ++n) for (int k = 0; k <= no + 1; ++k) C[n * (no + 2) + k] = binom(n, k);
    }
    u64 rank(u64 s) const {
        u64 r = 0; int i = 1;
        while (s) { int c = std::countr_zero(s); r += C[c * (norb + 2) + i]; ++i; s &= s - 1; }
        return r;
    }
};

// splitmix-free pinned normal sampler for the BASELINE generator
struct Normal {
    std::mt19937_64 eng;
    explicit Normal(u64 seed) : eng(seed) {}
    double uni() { return (double)(eng() >> 11) * 0x1.0p-53; }
    double operator()() {
        const double u1 = uni(), u2 = uni();
        return std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(6.283185307179586476925286766559 * u2);
    }
};

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try { f(); return 0; }
    catch (const std::invalid_argument& e) { g_err = e.what(); return 1; }
    catch (const std::exception& e) { g_err = e.what(); return 4; }
}

}  // namespace

extern "C" {

const char* or_last_error() { return g_err.c_str(); }
uint64_t or_binomial(int n, int k) { return binom(n, k); }

int or_strings(int norb, int k, uint64_t* out) {
    return guarded([&] { auto s = strings_of(norb, k); std::memcpy(out, s.data(), s.size() * 8); });
}

int or_links(int norb, int k, uint16_t* p, uint16_t* q, uint32_t* t, double* sign) {
    return guarded([&] {
        auto L = links_of(strings_of(norb, k), norb);
        size_t o = 0;
        for (auto& row : L) for (auto& e : row) { p[o] = (uint16_t)e.p; q[o] = (uint16_t)e.q; t[o] = e.target; sign[o] = e.sign; ++o; }
    });
}

int or_absorb_h1(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri, double* out) {
    return guarded([&] {
        Prob P{norb, nelec, ms2, e_core, h1, eri};
        auto v = absorb(P, P.na() + P.nb());
        std::memcpy(out, v.data(), v.size() * 8);
    });
}

// fci_operator.hpp:16-57; compiled with -ffp-contract=off so every product/sum rounds as in the reference.
int or_diag(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri, double* out) {
    return guarded([&] {
        Prob P{norb, nelec, ms2, e_core, h1, eri};
        auto sa = strings_of(norb, P.na()), sb = strings_of(norb, P.nb());
        auto senergy = [&](const std::vector<int>& o) {
            double e = 0.0;
            for (int i : o) e += P.h(i, i);
            for (int i : o) for (int j : o) e += 0.5 * (P.g(i, i, j, j) - P.g(i, j, j, i));
            return e;
        };
        std::vector<std::vector<int>> oa(sa.size()), ob(sb.size());
        std::vector<double> ea(sa.size()), eb(sb.size());
        for (size_t i = 0; i < sa.size(); ++i) { oa[i] = occ_of(sa[i], norb); ea[i] = senergy(oa[i]); }
        for (size_t i = 0; i < sb.size(); ++i) { ob[i] = occ_of(sb[i], norb); eb[i] = senergy(ob[i]); }
        for (size_t a = 0; a < sa.size(); ++a)
            for (size_t b = 0; b < sb.size(); ++b) {
                double cross = 0.0;
                for (int i : oa[a]) for (int j : ob[b]) cross += P.g(i, i, j, j);
                out[a * sb.size() + b] = P.e_core + ea[a] + eb[b] + cross;
            }
    });
}

// Tables of one sector for the blocked restatement (built once, reused by every call).
struct Blocked {
    Prob P;
    std::vector<u64> sa, sb;
    std::vector<std::vector<Link>> La, Lb;
    std::vector<double> h2e;
    // reverse alpha links: for intermediate row K, the (source ia, link) pairs targeting K, in the
    // reference's scatter order (ia ascending, link order)
    std::vector<std::vector<std::pair<uint32_t, int>>> rev;
    size_t na = 0, nb = 0, ndet = 0, no2 = 0;
    explicit Blocked(const Prob& p) : P(p) {
        sa = strings_of(P.norb, P.na());
        sb = strings_of(P.norb, P.nb());
        La = links_of(sa, P.norb);
        Lb = links_of(sb, P.norb);
        na = sa.size();
        nb = sb.size();
        ndet = na * nb;
        no2 = (size_t)P.norb * P.norb;
        h2e = absorb(P, P.na() + P.nb());
        rev.resize(na);
        for (size_t ia = 0; ia < na; ++ia)
            for (size_t l = 0; l < La[ia].size(); ++l) rev[La[ia][l].target].push_back({(uint32_t)ia, (int)l});
    }
    // contract_sigma (sigma.hpp:86-137) on intermediate alpha rows [row_lo, row_hi) in blocks of
    // block_rows, accumulating into y (not cleared here). exact=1 runs the blocks twice (alpha scatter
    // of every block, then beta scatter of every block): the reference's accumulation order exactly.
    void run(const double* x, double* y, size_t B, int exact, size_t row_lo, size_t row_hi, std::vector<double>& t1,
             std::vector<double>& g1) const {
        const int norb = P.norb;
        B = std::max<size_t>(1, B);
        const int passes = exact ? 2 : 1;
        for (int pass = 0; pass < passes; ++pass) {
            for (size_t k0 = row_lo; k0 < row_hi; k0 += B) {
                const size_t k1 = std::min(row_hi, k0 + B), nk = k1 - k0, bd = nk * nb;
                t1.assign(no2 * bd, 0.0);
                // phase A restricted to targets in [k0,k1): t1[pq][K,ib] += sign*x[ia,ib]
                for (size_t K = k0; K < k1; ++K)
                    for (auto [ia, l] : rev[K]) {
                        const auto& e = La[ia][l];
                        double* dst = t1.data() + (size_t)(e.p * norb + e.q) * bd + (K - k0) * nb;
                        const double* src = x + ia * nb;
                        for (size_t ib = 0; ib < nb; ++ib) dst[ib] += e.sign * src[ib];
                    }
                // phase B: t1[pq][K,target] += sign*x[K,ib]
                for (size_t ib = 0; ib < nb; ++ib)
                    for (const auto& e : Lb[ib]) {
                        double* dst = t1.data() + (size_t)(e.p * norb + e.q) * bd;
                        for (size_t K = k0; K < k1; ++K) dst[(K - k0) * nb + e.target] += e.sign * x[K * nb + ib];
                    }
                // phase C: g1 = h2e . t1 (axpy order, zero coefficients skipped)
                g1.assign(no2 * bd, 0.0);
                for (size_t pq = 0; pq < no2; ++pq) {
                    double* out = g1.data() + pq * bd;
                    const double* hrow = h2e.data() + pq * no2;
                    for (size_t rs = 0; rs < no2; ++rs) {
                        const double c = hrow[rs];
                        if (c == 0.0) continue;
                        const double* src = t1.data() + rs * bd;
                        for (size_t d = 0; d < bd; ++d) out[d] += c * src[d];
                    }
                }
                if (!exact || pass == 0) {  // phase D: alpha scatter
                    for (size_t K = k0; K < k1; ++K)
                        for (const auto& e : La[K]) {
                            const double* src = g1.data() + (size_t)(e.p * norb + e.q) * bd + (K - k0) * nb;
                            double* dst = y + (size_t)e.target * nb;
                            for (size_t ib = 0; ib < nb; ++ib) dst[ib] += e.sign * src[ib];
                        }
                }
                if (!exact || pass == 1) {  // phase E: beta scatter
                    for (size_t ib = 0; ib < nb; ++ib)
                        for (const auto& e : Lb[ib]) {
                            const double* src = g1.data() + (size_t)(e.p * norb + e.q) * bd;
                            for (size_t K = k0; K < k1; ++K) y[K * nb + e.target] += e.sign * src[(K - k0) * nb + ib];
                        }
                }
            }
        }
    }
};

// contract_sigma processed in blocks of `block_rows` alpha rows of the t1/g1 intermediate, so the
// 2*norb^2*n_det workspace shrinks to 2*norb^2*block_rows*nb. row_lo/row_hi restrict which
// intermediate alpha rows are processed; pass 0 / n_alpha_strings for the full sigma (then
// e_core * x is added last, as sigma.hpp:135 does).
int or_sigma_blocked(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri,
                     const double* x, double* y, int block_rows, int exact, int64_t row_lo, int64_t row_hi) {
    return guarded([&] {
        Blocked T(Prob{norb, nelec, ms2, e_core, h1, eri});
        std::fill(y, y + T.ndet, 0.0);
        std::vector<double> t1, g1;
        T.run(x, y, (size_t)block_rows, exact, (size_t)row_lo, (size_t)row_hi, t1, g1);
        if (row_lo == 0 && (size_t)row_hi == T.na)
            for (size_t i = 0; i < T.ndet; ++i) y[i] += e_core * x[i];
    });
}

// Complete sigma rows of selected alpha strings, in contract_sigma's exact accumulation order
// (sigma.hpp:86-137): only intermediate rows K that scatter into a selected row are formed — the
// row itself (its occupation entries and the phase-E beta scatter) and its single excitations (the
// link table is symmetric: K -> Ia iff Ia -> K). Phase D contributions reach y[Ia] in ascending K
// and link order and phase E (K = Ia) comes after all of them, exactly as in the full reference
// sweep, so each returned row is bit-identical to the reference's sigma row (the same restatement
// that is pinned bit-for-bit by tests/test_oracle_pins.py). Size-independent: a (16e,16o) row needs
// ~65 intermediate rows. Phase C (the h2e . t1 product) runs on `nthreads` threads over pq.
// out: n_rows x n_beta_strings, row-major.
int or_sigma_alpha_rows(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri,
                        const double* x, const int64_t* rows, int64_t n_rows, int block_rows, int nthreads,
                        double* out) {
    return guarded([&] {
        Prob P{norb, nelec, ms2, e_core, h1, eri};
        auto sa = strings_of(norb, P.na()), sb = strings_of(norb, P.nb());
        const auto La = links_of(sa, norb), Lb = links_of(sb, norb);
        const size_t na = sa.size(), nb = sb.size();
        const size_t no2 = (size_t)norb * norb;
        const auto h2e = absorb(P, P.na() + P.nb());
        std::vector<int64_t> slot(na, -1);  // alpha row -> output row
        for (int64_t r = 0; r < n_rows; ++r) {
            if (rows[r] < 0 || (size_t)rows[r] >= na) throw std::invalid_argument("alpha row out of range");
            slot[rows[r]] = r;
        }
        std::vector<uint32_t> ks;
        for (int64_t r = 0; r < n_rows; ++r)
            for (const auto& e : La[rows[r]]) ks.push_back(e.target);
        std::sort(ks.begin(), ks.end());
        ks.erase(std::unique(ks.begin(), ks.end()), ks.end());
        std::vector<std::vector<std::pair<uint32_t, int>>> rev(na);
        {
            std::vector<char> need(na, 0);
            for (auto K : ks) need[K] = 1;
            for (size_t ia = 0; ia < na; ++ia)
                for (size_t l = 0; l < La[ia].size(); ++l)
                    if (need[La[ia][l].target]) rev[La[ia][l].target].push_back({(uint32_t)ia, (int)l});
        }
        std::fill(out, out + (size_t)n_rows * nb, 0.0);
        std::vector<std::vector<double>> g_self(n_rows);  // g1[pq][Ia, :] for phase E
        const size_t B = (size_t)std::max(1, block_rows);
        const int nt = std::max(1, nthreads);
        std::vector<double> t1, g1;
        for (size_t b0 = 0; b0 < ks.size(); b0 += B) {
            const size_t nk = std::min(B, ks.size() - b0), bd = nk * nb;
            t1.assign(no2 * bd, 0.0);
            for (size_t i = 0; i < nk; ++i) {  // phase A
                const uint32_t K = ks[b0 + i];
                for (auto [ia, l] : rev[K]) {
                    const auto& e = La[ia][l];
                    double* dst = t1.data() + (size_t)(e.p * norb + e.q) * bd + i * nb;
                    const double* src = x + (size_t)ia * nb;
                    for (size_t ib = 0; ib < nb; ++ib) dst[ib] += e.sign * src[ib];
                }
            }
            for (size_t ib = 0; ib < nb; ++ib)  // phase B
                for (const auto& e : Lb[ib]) {
                    double* dst = t1.data() + (size_t)(e.p * norb + e.q) * bd;
                    for (size_t i = 0; i < nk; ++i) dst[i * nb + e.target] += e.sign * x[(size_t)ks[b0 + i] * nb + ib];
                }
            g1.assign(no2 * bd, 0.0);  // phase C, pq rows split over threads
            {
                std::vector<std::thread> th;
                for (int t = 0; t < nt; ++t)
                    th.emplace_back([&, t] {
                        for (size_t pq = t; pq < no2; pq += nt) {
                            double* o = g1.data() + pq * bd;
                            const double* hrow = h2e.data() + pq * no2;
                            for (size_t rs = 0; rs < no2; ++rs) {
                                const double c = hrow[rs];
                                if (c == 0.0) continue;
                                const double* src = t1.data() + rs * bd;
                                for (size_t d = 0; d < bd; ++d) o[d] += c * src[d];
                            }
                        }
                    });
                for (auto& t : th) t.join();
            }
            for (size_t i = 0; i < nk; ++i) {  // phase D into the selected rows only
                const uint32_t K = ks[b0 + i];
                for (const auto& e : La[K]) {
                    const int64_t r = slot[e.target];
                    if (r < 0) continue;
                    const double* src = g1.data() + (size_t)(e.p * norb + e.q) * bd + i * nb;
                    double* dst = out + (size_t)r * nb;
                    for (size_t ib = 0; ib < nb; ++ib) dst[ib] += e.sign * src[ib];
                }
                if (slot[K] >= 0) {  // keep g1[.][K, :] for its phase E
                    auto& gs = g_self[slot[K]];
                    gs.resize(no2 * nb);
                    for (size_t pq = 0; pq < no2; ++pq)
                        std::memcpy(gs.data() + pq * nb, g1.data() + pq * bd + i * nb, nb * 8);
                }
            }
        }
        for (int64_t r = 0; r < n_rows; ++r) {  // phase E, then e_core * x (sigma.hpp:133-136)
            const auto& gs = g_self[r];
            double* dst = out + (size_t)r * nb;
            for (size_t ib = 0; ib < nb; ++ib)
                for (const auto& e : Lb[ib]) dst[e.target] += e.sign * gs[(size_t)(e.p * norb + e.q) * nb + ib];
            const double* xr = x + (size_t)rows[r] * nb;
            for (size_t ib = 0; ib < nb; ++ib) dst[ib] += P.e_core * xr[ib];
        }
    });
}

// CPU-baseline timing context (bench.py cpu_baseline / --impl reference): the sector tables and
// one full-length output vector per worker thread are built ONCE here, outside any timed region.
struct SampleBench {
    Blocked T;
    std::vector<std::vector<double>> y;   // per-thread private sigma accumulators (n_det each)
    std::vector<std::vector<double>> t1, g1;
    SampleBench(const Prob& p, int nthreads) : T(p), y(nthreads), t1(nthreads), g1(nthreads) {
        for (auto& v : y) v.assign(T.ndet, 0.0);
    }
};

void* or_bench_create(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri, int nthreads) {
    try {
        return new SampleBench(Prob{norb, nelec, ms2, e_core, h1, eri}, std::max(1, nthreads));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void or_bench_destroy(void* b) { delete static_cast<SampleBench*>(b); }

// Timed bounded sample of the single-pass blocked restatement: each worker thread processes
// `rows_per_thread` intermediate alpha rows (disjoint ranges starting at `row0`, wrapping) into its
// private y. *seconds = wall time from the release of the workers to the last join (steady clock).
int or_bench_run(void* handle, const double* x, int nthreads, int64_t rows_per_thread, int block_rows, int64_t row0,
                 double* seconds) {
    return guarded([&] {
        auto* b = static_cast<SampleBench*>(handle);
        if (!b || nthreads < 1 || nthreads > (int)b->y.size()) throw std::invalid_argument("or_bench_run: bad thread count");
        const int64_t na = (int64_t)b->T.na;
        std::vector<std::thread> th;
        std::vector<int> rc(nthreads, 0);
        const auto t0 = std::chrono::steady_clock::now();
        for (int t = 0; t < nthreads; ++t)
            th.emplace_back([&, t] {
                try {
                    const int64_t lo = (row0 + t * rows_per_thread) % na;
                    const int64_t hi = std::min<int64_t>(na, lo + rows_per_thread);
                    b->T.run(x, b->y[t].data(), (size_t)block_rows, 0, (size_t)lo, (size_t)hi, b->t1[t], b->g1[t]);
                } catch (...) {
                    rc[t] = 1;
                }
            });
        for (auto& t : th) t.join();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (int r : rc)
            if (r) throw std::runtime_error("sample worker failed");
    });
}

double or_sc_element(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri,
                     uint64_t a1, uint64_t b1, uint64_t a2, uint64_t b2) {
    Prob P{norb, nelec, ms2, e_core, h1, eri};
    return sc_element(P, a1, b1, a2, b2);
}

// Dense H element by element (dense_oracle.hpp:269-285), row-major n_det x n_det.
int or_dense_h(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri, double* out) {
    return guarded([&] {
        Prob P{norb, nelec, ms2, e_core, h1, eri};
        auto sa = strings_of(norb, P.na()), sb = strings_of(norb, P.nb());
        const size_t nb = sb.size(), n = sa.size() * nb;
        for (size_t r = 0; r < n; ++r)
            for (size_t c = 0; c < n; ++c)
                out[r * n + c] = sc_element(P, sa[r / nb], sb[r % nb], sa[c / nb], sb[c % nb]);
    });
}

// sigma(I) = sum_J H_IJ x_J for selected determinants I, enumerating only the J within two
// excitations of I (Slater-Condon). Size-independent: usable at (16e,16o).
int or_sigma_rows(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri,
                  const double* x, const int64_t* rows, int64_t nrows, double* out) {
    return guarded([&] {
        Prob P{norb, nelec, ms2, e_core, h1, eri};
        const int na_e = P.na(), nb_e = P.nb();
        auto sa = strings_of(norb, na_e), sb = strings_of(norb, nb_e);
        const size_t nb = sb.size();
        Ranker R(norb);
        const u64 full = (norb == 64) ? ~u64{0} : ((u64{1} << norb) - 1);
        auto singles = [&](u64 s, std::vector<u64>& v) {
            v.clear();
            for (u64 o = s; o; o &= o - 1)
                for (u64 e = full & ~s; e; e &= e - 1) v.push_back((s & ~(o & -o)) | (e & -e));
        };
        auto doubles = [&](u64 s, std::vector<u64>& v) {
            v.clear();
            for (u64 o1 = s; o1; o1 &= o1 - 1)
                for (u64 o2 = o1 & (o1 - 1); o2; o2 &= o2 - 1)
                    for (u64 e1 = full & ~s; e1; e1 &= e1 - 1)
                        for (u64 e2 = e1 & (e1 - 1); e2; e2 &= e2 - 1)
                            v.push_back((s & ~(o1 & -o1) & ~(o2 & -o2)) | (e1 & -e1) | (e2 & -e2));
        };
        std::vector<u64> sa1, sb1, sa2, sb2;
        for (int64_t r = 0; r < nrows; ++r) {
            const u64 a = sa[rows[r] / nb], b = sb[rows[r] % nb];
            singles(a, sa1); singles(b, sb1); doubles(a, sa2); doubles(b, sb2);
            auto X = [&](u64 ja, u64 jb) { return x[R.rank(ja) * nb + R.rank(jb)]; };
            double s = sc_element(P, a, b, a, b) * X(a, b);
            for (u64 j : sa1) s += sc_element(P, a, b, j, b) * X(j, b);
            for (u64 j : sb1) s += sc_element(P, a, b, a, j) * X(a, j);
            for (u64 j : sa2) s += sc_element(P, a, b, j, b) * X(j, b);
            for (u64 j : sb2) s += sc_element(P, a, b, a, j) * X(a, j);
            for (u64 ja : sa1) for (u64 jb : sb1) s += sc_element(P, a, b, ja, jb) * X(ja, jb);
            out[r] = s;
        }
    });
}

// BASELINE.json synthetic integrals (pinned here; the product's generator in
// paper_2603_06101_b200/csrc/synthetic.cpp must match this bit for bit):
//   rng = std::mt19937_64(seed); normal = Box-Muller (cos branch) on two 53-bit uniforms.
//   draw order: h upper triangle row-major (p <= q): h_pq = [p==q](-1 + 2p/norb) + 0.05 N,
//   then for k = 0..norb-1 the upper triangle of L^k row-major: L_pp = 0.5 + 0.1 N,
//   L_pq = offdiag_scale * N. (pq|rs) = sum_k L^k_pq L^k_rs (k ascending).
int or_synthetic(int norb, uint64_t seed, double offdiag_scale, double* h1, double* eri) {
    return guarded([&] {
        Normal N(seed);
        for (int p = 0; p < norb; ++p)
            for (int q = p; q < norb; ++q) {
                const double base = (p == q) ? (-1.0 + 2.0 * p / norb) : 0.0;
                const double v = base + 0.05 * N();
                h1[p * norb + q] = v;
                h1[q * norb + p] = v;
            }
        const size_t no2 = (size_t)norb * norb;
        std::vector<double> L((size_t)norb * no2);
        for (int k = 0; k < norb; ++k)
            for (int p = 0; p < norb; ++p)
                for (int q = p; q < norb; ++q) {
                    const double v = (p == q) ? 0.5 + 0.1 * N() : offdiag_scale * N();
                    L[k * no2 + p * norb + q] = v;
                    L[k * no2 + q * norb + p] = v;
                }
        for (size_t pq = 0; pq < no2; ++pq)
            for (size_t rs = 0; rs < no2; ++rs) {
                double s = 0.0;
                for (int k = 0; k < norb; ++k) s += L[k * no2 + pq] * L[k * no2 + rs];
                eri[pq * no2 + rs] = s;
            }
    });
}

}  // extern "C"
