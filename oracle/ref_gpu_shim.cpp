// oracle/ref_gpu_shim.cpp — TEST INFRASTRUCTURE: the drop-in demonstration of INTEGRATION.md.
//
// Compiles the reference's headers (unmodified, from /root/reference/proj/include) together with
// the product's C++ drop-in header include/sbg.hpp, and exercises it through ctypes entry points:
//   * the reference's own solver drivers (sbci1.hpp, sbci2.hpp, davidson.hpp) on
//     sbci::gpu::CudaFciOperator (replaces FciOperator, fci_operator.hpp:60-86);
//   * the device-resident drivers sbci::gpu::solve_n_states_sbci1/_sbci2/davidson_solve with the
//     reference signature and error mapping (SBG_ENONCONV -> sbci::NonConvergenceError);
//   * the operator's threading contract: T threads x N applies through SymmetricOperator::apply
//     (operator.hpp:14-18, 47; the reference's test_operator.cpp:49-64 pattern);
//   * the plain-vector warm start sbci::gpu::solve_state_sbci1 against the reference's own
//     solve_state_sbci1 (sbci1.hpp:477-486) on the same operator.
// Built by oracle/Makefile into oracle/_ref/libsbci_ref_gpu.so.
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "sbg.hpp"

namespace {

thread_local std::string g_err;

sbci::fci::FciProblem make_problem(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri) {
    sbci::fci::FciProblem p(norb);
    p.nelec = nelec;
    p.ms2 = ms2;
    p.e_core = e_core;
    p.h1.assign(h1, h1 + (size_t)norb * norb);
    p.eri.assign(eri, eri + (size_t)norb * norb * norb * norb);
    return p;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const sbci::NonConvergenceError& e) {
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

void fill(const sbci::MultiStateResult& r, int nroots, double* energies, int* iterations, uint64_t* matvecs) {
    for (int k = 0; k < nroots; ++k) {
        energies[k] = r.pairs[k].energy;
        if (iterations) iterations[k] = r.pairs[k].iterations;
    }
    if (matvecs) *matvecs = r.summary.matvecs;
}

}  // namespace

extern "C" {

const char* refgpu_last_error() { return g_err.c_str(); }

// The reference's solver (method 1 = solve_n_states_sbci1, 2 = solve_n_states_sbci2,
// 3 = davidson_solve) on the GPU operator, default SolverConfig.
int refgpu_solve(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri, int method,
                 int nroots, double* energies, int* iterations, uint64_t* matvecs) {
    return guarded([&] {
        sbci::gpu::CudaFciOperator op(make_problem(norb, nelec, ms2, e_core, h1, eri), ~std::uint64_t{0});
        sbci::SolverConfig cfg;
        sbci::MultiStateResult r;
        if (method == 1) r = sbci::solve_n_states_sbci1(op, nroots, cfg);
        else if (method == 2) r = sbci::solve_n_states_sbci2(op, nroots, cfg);
        else {
            auto d = sbci::davidson_solve(op, nroots, cfg);
            r.pairs = d.pairs;
            r.summary = d.summary;
        }
        fill(r, nroots, energies, iterations, matvecs);
    });
}

// The product's device-resident drivers through include/sbg.hpp (t_max < 0 keeps the default).
int refgpu_device_solve(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri, int method,
                        int nroots, long t_max, double* energies, int* iterations, uint64_t* matvecs, int* failed_state) {
    return guarded([&] {
        auto op = sbci::gpu::as_operator(make_problem(norb, nelec, ms2, e_core, h1, eri), ms2, ~std::uint64_t{0});
        sbci::SolverConfig cfg;
        if (t_max >= 0) cfg.t_max = t_max;
        sbci::MemoryTraceSink sink;
        try {
            sbci::MultiStateResult r = method == 1   ? sbci::gpu::solve_n_states_sbci1(*op, nroots, cfg, &sink)
                                       : method == 2 ? sbci::gpu::solve_n_states_sbci2(*op, nroots, cfg, &sink)
                                                     : sbci::gpu::davidson_solve(*op, nroots, cfg, &sink);
            fill(r, nroots, energies, iterations, matvecs);
            if (sink.records().empty()) throw std::runtime_error("no trace records reached the TraceSink");
            if (r.pairs.size() != (size_t)nroots || r.pairs[0].vector.size() != op->dim())
                throw std::runtime_error("result shape");
        } catch (const sbci::NonConvergenceError& e) {
            if (failed_state) *failed_state = e.state;
            throw;
        }
    });
}

// T threads x N applies of one CudaFciOperator through the reference's SymmetricOperator::apply;
// every result must equal the single-threaded sigma (to L2-reduction rounding) and the reference's
// atomic counter must read T * N. Returns the number of bad results (or -1 on a wrong count).
int refgpu_concurrent_applies(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri,
                              int nthreads, int napply, int* bad_out) {
    return guarded([&] {
        sbci::gpu::CudaFciOperator op(make_problem(norb, nelec, ms2, e_core, h1, eri), ~std::uint64_t{0});
        const size_t n = op.dim();
        std::vector<sbci::Vector> xs(nthreads, sbci::Vector(n)), refs(nthreads);
        for (int t = 0; t < nthreads; ++t)
            for (size_t i = 0; i < n; ++i) xs[t][i] = std::sin(0.37 * (double)i + 1.3 * t);
        double scale = 0.0;
        for (int t = 0; t < nthreads; ++t) {
            refs[t] = op.apply(xs[t]);
            for (double v : refs[t]) scale = std::max(scale, std::abs(v));
        }
        op.reset_apply_count();
        std::vector<int> bad(nthreads, 0);
        std::vector<std::thread> th;
        for (int t = 0; t < nthreads; ++t)
            th.emplace_back([&, t] {
                for (int k = 0; k < napply; ++k) {
                    const sbci::Vector y = op.apply(xs[t]);
                    double err = 0.0;
                    for (size_t i = 0; i < n; ++i) err = std::max(err, std::abs(y[i] - refs[t][i]));
                    if (!(err <= 1e-13 * scale)) ++bad[t];
                }
            });
        for (auto& t : th) t.join();
        int total = 0;
        for (int b : bad) total += b;
        if (op.apply_count() != (std::uint64_t)nthreads * napply) total = -1;
        *bad_out = total;
    });
}

// Warm start: the reference's solve_state_sbci1 (host driver on the GPU operator) and the device
// sbci::gpu::solve_state_sbci1 from the same plain vector, shift and deflation set. out[0..3] =
// reference energy, device energy, reference iterations, device iterations; out[4] = the device
// run's |<x_ref|x_dev>|.
int refgpu_warm_start(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri, int with_defl,
                      double* out) {
    return guarded([&] {
        sbci::gpu::CudaFciOperator op(make_problem(norb, nelec, ms2, e_core, h1, eri), ~std::uint64_t{0});
        sbci::SolverConfig cfg;
        const auto guesses = sbci::init_guess_from_diagonal(op, 2, cfg.lindep);
        sbci::DeflationSet defl;
        int alpha = 0;
        double shift = guesses[0].energy;
        if (with_defl) {  // deflate the reference-converged ground state, then warm-start state 1
            sbci::GroundShiftPreconditioner pre0(op.diagonal(), guesses[0].energy, cfg.clamp_delta);
            auto g = sbci::solve_state_sbci1(op, pre0, defl, guesses[0].x, guesses[0].energy, cfg);
            defl.add_with_image(g.pair.vector, g.converged_image, g.pair.energy);
            shift = g.pair.energy;
            alpha = 1;
        }
        const sbci::Vector& x0 = guesses[with_defl ? 1 : 0].x;
        const double e0 = guesses[with_defl ? 1 : 0].energy;
        sbci::GroundShiftPreconditioner pr(op.diagonal(), shift, cfg.clamp_delta);
        auto r = sbci::solve_state_sbci1(op, pr, defl, x0, e0, cfg, alpha);
        sbci::GroundShiftPreconditioner pd(op.diagonal(), shift, cfg.clamp_delta);
        auto d = sbci::gpu::solve_state_sbci1(op, pd, defl, x0, e0, cfg, alpha);
        double ov = 0.0;
        for (size_t i = 0; i < op.dim(); ++i) ov += r.pair.vector[i] * d.pair.vector[i];
        out[0] = r.pair.energy;
        out[1] = d.pair.energy;
        out[2] = r.pair.iterations;
        out[3] = d.pair.iterations;
        out[4] = std::abs(ov);
        out[5] = pr.shift;
        out[6] = pd.shift;
    });
}

}  // extern "C"
