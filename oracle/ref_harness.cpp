// oracle/ref_harness.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// Compiles the UNMODIFIED reference library (header-only C++20, read in place from
// /root/reference/proj/include) into oracle/_ref/libsbci_ref.so and exposes a tiny
// extern "C" surface so the pytest suite and bench.py's CPU arm can drive the
// reference's own code path:
//   * strings / link tables   -> sbci::fci::enumerate_strings, build_link_table (determinants.hpp:41-59, sigma.hpp:27-50)
//   * diagonal                -> sbci::fci::hamiltonian_diagonal (fci_operator.hpp:16-57)
//   * sigma                   -> sbci::fci::FciOperator::apply -> contract_sigma (operator.hpp:25-31, sigma.hpp:86-137)
//   * solvers                 -> solve_n_states_sbci1 / _sbci2 / davidson_solve (sbci1.hpp:526, sbci2.hpp:527, davidson.hpp:231)
//   * FCIDUMP                 -> parse_fcidump_file (fcidump.hpp:171)
//   * <S^2>                   -> spin_squared (spin.hpp:17-51)
// Built by oracle/Makefile with the reference's own Release flags (-O3, no -march) plus
// -ffp-contract=off so the diagonal stays bit-identical on any host ISA (SURVEY §7 hazard 4d).
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>

#include "sbci/sbci.hpp"
#include "sbci/fci/fci_operator.hpp"
#include "sbci/fci/fcidump.hpp"
#include "sbci/fci/spin.hpp"

using namespace sbci;
using namespace sbci::fci;

namespace {
thread_local std::string g_err;

FciProblem make_problem(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri) {
    FciProblem p(norb);
    p.nelec = nelec;
    p.ms2 = ms2;
    p.e_core = e_core;
    std::memcpy(p.h1.data(), h1, sizeof(double) * norb * norb);
    std::memcpy(p.eri.data(), eri, sizeof(double) * (size_t)norb * norb * norb * norb);
    return p;
}

SolverConfig make_cfg(const double* d, const long* i) {
    // d = {eps0, r0, b_th, eps1, x_th1, x_th2, r1, lindep, clamp_delta}; i = {max_cycle, t_max, hx_refresh}
    SolverConfig c;
    if (d) {
        c.eps0 = d[0]; c.r0 = d[1]; c.b_th = d[2]; c.eps1 = d[3]; c.x_th1 = d[4]; c.x_th2 = d[5];
        c.r1 = d[6]; c.lindep = d[7]; c.clamp_delta = d[8];
    }
    if (i) {
        c.max_cycle = (int)i[0]; c.t_max = i[1]; c.hx_refresh_restarts = (int)i[2];
    }
    return c;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const NonConvergenceError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int64_t ref_num_strings(int norb, int k) { return (int64_t)binomial(norb, k); }

int ref_strings(int norb, int k, uint64_t* out) {
    return guarded([&] {
        auto s = enumerate_strings(norb, k);
        std::memcpy(out, s.data(), s.size() * sizeof(uint64_t));
    });
}

// Flattened link table: row-major [nstr][L] of {p, q, target, sign}.
int ref_links(int norb, int k, uint16_t* p, uint16_t* q, uint32_t* target, double* sign, int64_t* row_len) {
    return guarded([&] {
        auto s = enumerate_strings(norb, k);
        LinkTable lt = build_link_table(s, norb);
        size_t o = 0;
        for (size_t r = 0; r < lt.size(); ++r) {
            row_len[r] = (int64_t)lt[r].size();
            for (const auto& e : lt[r]) {
                p[o] = e.p; q[o] = e.q; target[o] = e.target; sign[o] = e.sign;
                ++o;
            }
        }
    });
}

int ref_diag(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri, double* out) {
    return guarded([&] {
        FciProblem p = make_problem(norb, nelec, ms2, e_core, h1, eri);
        DeterminantBasis b = enumerate_basis(norb, p.n_alpha(), p.n_beta());
        Vector d = hamiltonian_diagonal(p, b);
        std::memcpy(out, d.data(), d.size() * sizeof(double));
    });
}

int ref_sigma(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri,
              const double* x, double* y, int nvec) {
    return guarded([&] {
        FciProblem p = make_problem(norb, nelec, ms2, e_core, h1, eri);
        auto op = as_operator(p, ms2, ~uint64_t{0});
        const size_t n = op->dim();
        for (int v = 0; v < nvec; ++v) {
            Vector xv(x + v * n, x + (v + 1) * n);
            Vector yv = op->apply(xv);
            std::memcpy(y + v * n, yv.data(), n * sizeof(double));
        }
    });
}

// method: 1 = sbci1, 2 = sbci2, 3 = davidson.  Outputs sorted by energy (as the drivers return).
int ref_solve(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri, int method,
              int nroots, const double* cfgd, const long* cfgi, double* energies, int* iterations,
              int* restarts, double* residuals, uint64_t* matvecs, double* vectors, double* s_squared,
              double* wall_s, const char* trace_csv) {
    return guarded([&] {
        FciProblem p = make_problem(norb, nelec, ms2, e_core, h1, eri);
        auto op = as_operator(p, ms2, ~uint64_t{0});
        SolverConfig cfg = make_cfg(cfgd, cfgi);
        std::unique_ptr<CsvTraceSink> sink;
        if (trace_csv && trace_csv[0]) sink = std::make_unique<CsvTraceSink>(std::string(trace_csv));
        MultiStateResult r;
        if (method == 1) r = solve_n_states_sbci1(*op, nroots, cfg, sink.get());
        else if (method == 2) r = solve_n_states_sbci2(*op, nroots, cfg, sink.get());
        else {
            DavidsonResult d = davidson_solve(*op, nroots, cfg, sink.get());
            r.pairs = d.pairs;
            r.summary = d.summary;
        }
        const size_t n = op->dim();
        for (int k = 0; k < nroots; ++k) {
            energies[k] = r.pairs[k].energy;
            if (iterations) iterations[k] = r.pairs[k].iterations;
            if (restarts) restarts[k] = r.pairs[k].restarts;
            if (residuals) residuals[k] = r.pairs[k].final_residual;
            if (vectors) std::memcpy(vectors + k * n, r.pairs[k].vector.data(), n * sizeof(double));
            if (s_squared) s_squared[k] = spin_squared(op->basis(), r.pairs[k].vector);
        }
        if (matvecs) *matvecs = r.summary.matvecs;
        if (wall_s) *wall_s = r.summary.wall_time_s;
    });
}

int ref_parse_fcidump(const char* path, int* norb, int* nelec, int* ms2, double* e_core, double* h1,
                      double* eri, int cap_norb) {
    return guarded([&] {
        FciProblem p = parse_fcidump_file(path);
        *norb = p.norb; *nelec = p.nelec; *ms2 = p.ms2; *e_core = p.e_core;
        if (h1 && eri) {
            if (p.norb > cap_norb) throw std::invalid_argument("capacity");
            std::memcpy(h1, p.h1.data(), p.h1.size() * sizeof(double));
            std::memcpy(eri, p.eri.data(), p.eri.size() * sizeof(double));
        }
    });
}

int ref_spin_squared(int norb, int n_alpha, int n_beta, const double* x, double* out) {
    return guarded([&] {
        DeterminantBasis b = enumerate_basis(norb, n_alpha, n_beta);
        Vector v(x, x + b.n_det());
        *out = spin_squared(b, v);
    });
}

}  // extern "C"
