/*
 * sbg.hpp — header-only C++ drop-in of the B200 path for the reference library.
 *
 * A maintainer adds this header (and links libsbg.so) to the reference build; it needs the
 * reference's own headers on the include path (`-I proj/include`), because the types it returns ARE
 * the reference's: sbci::SymmetricOperator, sbci::MultiStateResult, sbci::SolverConfig,
 * sbci::TraceSink, sbci::NonConvergenceError, sbci::fci::FciProblem. Everything crosses into the GPU
 * library through the C ABI of sbg.h only (plain pointers, error codes).
 *
 *   sbci::gpu::CudaFciOperator       drop-in for sbci::fci::FciOperator (fci_operator.hpp:60-86):
 *                                    dim(), apply() (the reference's own non-virtual apply, with its
 *                                    dimension check and atomic counter), diagonal() — usable by every
 *                                    reference driver unchanged; apply() is safe from several threads
 *                                    (libsbg serialises the context, operator.hpp:14-18).
 *   sbci::gpu::as_operator           fci_operator.hpp:103-120 (same guard, same messages).
 *   sbci::gpu::solve_n_states_sbci1  sbci1.hpp:526 with the whole solve device-resident (vectors in
 *   sbci::gpu::solve_n_states_sbci2  HBM, fused update passes); the reference signature, results in the
 *   sbci::gpu::davidson_solve        reference's types, errors mapped back: SBG_EINVAL ->
 *                                    std::invalid_argument, SBG_ENONCONV -> sbci::NonConvergenceError
 *                                    {state, best_energy, best_residual}, anything else ->
 *                                    std::runtime_error.
 *   sbci::gpu::solve_state_sbci1     the plain-vector warm start (sbci1.hpp:477-486).
 */
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "sbci/sbci.hpp"
#include "sbg.h"

namespace sbci::gpu {

namespace detail {

[[noreturn]] inline void throw_code(int rc, const sbg_stats* st = nullptr) {
    const std::string msg = sbg_last_error();
    if (rc == SBG_EINVAL) throw std::invalid_argument(msg);
    if (rc == SBG_ENONCONV && st) throw sbci::NonConvergenceError(st->failed_state, st->best_energy, st->best_residual);
    throw std::runtime_error(msg);
}

inline void check(int rc, const sbg_stats* st = nullptr) {
    if (rc != SBG_OK) throw_code(rc, st);
}

inline sbg_config to_c(const sbci::SolverConfig& c) {
    sbg_config o = sbg_config_default();
    o.eps0 = c.eps0;
    o.r0 = c.r0;
    o.b_th = c.b_th;
    o.eps1 = c.eps1;
    o.x_th1 = c.x_th1;
    o.x_th2 = c.x_th2;
    o.r1 = c.r1;
    o.max_cycle = c.max_cycle;
    o.hx_refresh_restarts = c.hx_refresh_restarts;
    o.t_max = c.t_max;
    o.lindep = c.lindep;
    o.clamp_delta = c.clamp_delta;
    return o;
}

// sbg_trace_record -> sbci::TraceRecord (trace.hpp:22-44)
inline void forward_trace(const sbg_trace_record* r, void* user) {
    auto* sink = static_cast<sbci::TraceSink*>(user);
    static const char* methods[] = {"", "sbci1", "sbci2", "davidson"};
    static const char* reasons[] = {"stall_small_b", "norm_out_of_range", "residual_blowup", "max_cycle"};
    sbci::TraceRecord t;
    t.method = (r->method >= 1 && r->method <= 3) ? methods[r->method] : "";
    t.state = r->state;
    t.pair_partner = r->pair_partner;
    t.t = r->t;
    t.energy = r->energy;
    t.dE = r->dE;
    t.res_norm = r->res_norm;
    t.x_norm = r->x_norm;
    t.kinetic = r->kinetic;
    t.matvecs = r->matvecs;
    if (r->restart_reason >= 0 && r->restart_reason < 4) t.restart_reason = reasons[r->restart_reason];
    t.b = r->b;
    t.c = r->c;
    t.b_ab = r->b_ab;
    t.b_ba = r->b_ba;
    t.b_bb = r->b_bb;
    t.c_ab = r->c_ab;
    t.c_ba = r->c_ba;
    t.c_bb = r->c_bb;
    t.a_ab = r->a_ab;
    t.a_ba = r->a_ba;
    t.energy_partner = r->energy_partner;
    t.x_norm_partner = r->x_norm_partner;
    t.res_norm_partner = r->res_norm_partner;
    sink->record(t);
}

}  // namespace detail

/// The determinant CI Hamiltonian of one (nelec, ms2) sector on a B200 (replaces
/// sbci::fci::FciOperator). The diagonal is the exact, bit-identical hamiltonian_diagonal.
class CudaFciOperator final : public sbci::SymmetricOperator {
public:
    CudaFciOperator(const sbci::fci::FciProblem& prob, std::uint64_t max_determinants = sbci::fci::kDefaultDeterminantGuard,
                    int device = 0)
        : SymmetricOperator(0) {
        if (prob.h1.size() != static_cast<std::size_t>(prob.norb) * prob.norb ||
            prob.eri.size() != static_cast<std::size_t>(prob.norb) * prob.norb * prob.norb * prob.norb)
            throw std::invalid_argument("CudaFciOperator: integral arrays do not match norb");
        sbg_ctx* c = nullptr;
        detail::check(sbg_create(prob.norb, prob.nelec, prob.ms2, prob.e_core, prob.h1.data(), prob.eri.data(), device,
                                 max_determinants, &c));
        ctx_.reset(c);
        dim_ = static_cast<std::size_t>(sbg_dim(c));
        diag_.assign(dim_, 0.0);
        detail::check(sbg_diagonal(c, diag_.data()));
    }

    sbg_ctx* handle() const { return ctx_.get(); }
    std::uint64_t device_sigma_count() const { return sbg_apply_count(ctx_.get()); }

    /// <S^2> of a CI vector (fci/spin.hpp:17-51), on the device.
    double spin_squared(const sbci::Vector& x) const {
        if (x.size() != dim_) throw std::invalid_argument("spin_squared: vector length mismatch");
        double s = 0.0;
        detail::check(sbg_spin_squared(ctx_.get(), x.data(), &s));
        return s;
    }

private:
    struct Del {
        void operator()(sbg_ctx* c) const { sbg_destroy(c); }
    };
    void apply_impl(const sbci::Vector& x, sbci::Vector& y) const override {
        detail::check(sbg_sigma(ctx_.get(), x.data(), y.data(), 1));
    }
    std::unique_ptr<sbg_ctx, Del> ctx_;
};

/// fci_operator.hpp:103-120: sector from (nelec, ms2_override), the determinant guard (overridable).
inline std::shared_ptr<CudaFciOperator> as_operator(const sbci::fci::FciProblem& prob, int ms2_override,
                                                    std::uint64_t max_determinants = sbci::fci::kDefaultDeterminantGuard,
                                                    int device = 0) {
    sbci::fci::FciProblem p = prob;
    p.ms2 = ms2_override;
    if ((p.nelec + p.ms2) % 2 != 0) throw std::invalid_argument("as_operator: MS2 parity mismatch");
    return std::make_shared<CudaFciOperator>(p, max_determinants, device);
}

namespace detail {

inline sbci::MultiStateResult solve(const CudaFciOperator& op, int method, int n, const sbci::SolverConfig& cfg,
                                    sbci::TraceSink* sink, int max_space = 0) {
    cfg.validate();
    const sbg_config c = to_c(cfg);
    std::vector<double> e(static_cast<std::size_t>(std::max(n, 0)));
    std::vector<double> v(static_cast<std::size_t>(std::max(n, 0)) * op.dim());
    sbg_stats st{};
    const int rc = method == 3 ? sbg_solve_davidson(op.handle(), n, max_space, &c, e.data(), v.data(), &st,
                                                    sink ? &forward_trace : nullptr, sink)
                               : sbg_solve(op.handle(), method, n, &c, e.data(), v.data(), &st,
                                           sink ? &forward_trace : nullptr, sink);
    check(rc, &st);
    sbci::MultiStateResult out;
    out.summary.method = method == 1 ? "sbci1" : method == 2 ? "sbci2" : "davidson";
    for (int k = 0; k < n; ++k) {
        sbci::ConvergedEigenpair p;
        p.state = k;
        p.energy = e[static_cast<std::size_t>(k)];
        p.vector.assign(v.begin() + static_cast<std::ptrdiff_t>(k * op.dim()),
                        v.begin() + static_cast<std::ptrdiff_t>((k + 1) * op.dim()));
        p.iterations = st.iterations[k];
        p.restarts = st.restarts[k];
        p.final_residual = st.final_residual[k];
        sbci::StateSummary ss;
        ss.state = k;
        ss.energy = p.energy;
        ss.iterations = p.iterations;
        ss.restarts = p.restarts;
        ss.final_residual = p.final_residual;
        ss.s_squared = st.s_squared[k];
        out.summary.states.push_back(ss);
        out.pairs.push_back(std::move(p));
    }
    out.summary.total_iterations = st.total_iterations;
    out.summary.total_restarts = st.total_restarts;
    out.summary.matvecs = st.matvecs;
    out.summary.hx_refreshes = st.hx_refreshes;
    out.summary.peak_vectors = st.peak_vectors;
    out.summary.wall_time_s = st.wall_time_s;
    // summary.matvecs is the device solve's sigma count (op.device_sigma_count() advances by the
    // same); op.apply_count() keeps counting host-side apply() calls only
    return out;
}

}  // namespace detail

/// sbci1.hpp:526 on device-resident vectors.
inline sbci::MultiStateResult solve_n_states_sbci1(const CudaFciOperator& op, int n, const sbci::SolverConfig& cfg,
                                                   sbci::TraceSink* sink = nullptr) {
    if (n < 1) throw std::invalid_argument("solve_n_states_sbci1: n must be >= 1");
    return detail::solve(op, 1, n, cfg, sink);
}

/// sbci2.hpp:527 on device-resident vectors.
inline sbci::MultiStateResult solve_n_states_sbci2(const CudaFciOperator& op, int n, const sbci::SolverConfig& cfg,
                                                   sbci::TraceSink* sink = nullptr) {
    if (n < 1) throw std::invalid_argument("solve_n_states_sbci2: n must be >= 1");
    return detail::solve(op, 2, n, cfg, sink);
}

/// davidson.hpp:228-244 (block Davidson cross-check); max_space 0 = 12 * nroots.
inline sbci::MultiStateResult davidson_solve(const CudaFciOperator& op, int nroots, const sbci::SolverConfig& cfg,
                                             sbci::TraceSink* sink = nullptr, int max_space = 0) {
    return detail::solve(op, 3, nroots, cfg, sink, max_space);
}

/// Plain-vector warm start, sbci1.hpp:477-486: one state from x0 with the caller's energy label E0,
/// preconditioner shift pre.shift (and clamp), deflated against defl's stored vectors. The stored
/// images of defl are private to the reference's DeflationSet, so the device rebuilds H x_c with one
/// sigma each (exact by linearity; not counted as applications). Returns the reference's
/// Sbci1Result with pair, converged_image and hx_refreshes filled (next_seed stays empty).
inline sbci::Sbci1Result solve_state_sbci1(const CudaFciOperator& op, sbci::GroundShiftPreconditioner& pre,
                                           const sbci::DeflationSet& defl, const sbci::Vector& x0, double E0,
                                           const sbci::SolverConfig& cfg, int alpha = 0, sbci::TraceSink* sink = nullptr) {
    cfg.validate();
    if (x0.size() != op.dim()) throw std::invalid_argument("SymmetricOperator::apply: dimension mismatch");
    sbci::SolverConfig c2 = cfg;
    c2.clamp_delta = pre.clamp_delta;
    const sbg_config c = detail::to_c(c2);
    const std::size_t nd = defl.size();
    std::vector<double> dx(nd * op.dim()), de(nd);
    for (std::size_t i = 0; i < nd; ++i) {
        std::copy(defl.vector(i).begin(), defl.vector(i).end(), dx.begin() + static_cast<std::ptrdiff_t>(i * op.dim()));
        de[i] = defl.energy(i);
    }
    double energy = 0.0, shift_out = pre.shift;
    sbci::Sbci1Result r;
    r.pair.vector.assign(op.dim(), 0.0);
    r.converged_image.assign(op.dim(), 0.0);
    sbg_stats st{};
    detail::check(sbg_solve_state_sbci1(op.handle(), x0.data(), E0, &shift_out, alpha, static_cast<int>(nd),
                                        nd ? dx.data() : nullptr, nullptr, nd ? de.data() : nullptr, &c, &energy,
                                        r.pair.vector.data(), r.converged_image.data(), &st,
                                        sink ? &detail::forward_trace : nullptr, sink),
                  &st);
    if (alpha == 0) pre.update_shift(shift_out);   // track_ground_shift (sbci1.hpp:381, 416)
    r.pair.state = alpha;
    r.pair.energy = energy;
    r.pair.iterations = st.iterations[0];
    r.pair.restarts = st.restarts[0];
    r.pair.final_residual = st.final_residual[0];
    r.hx_refreshes = st.hx_refreshes;
    return r;
}

}  // namespace sbci::gpu
