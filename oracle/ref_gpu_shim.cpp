// oracle/ref_gpu_shim.cpp — TEST INFRASTRUCTURE: the drop-in demonstration of INTEGRATION.md.
//
// The reference's own solver drivers (sbci1.hpp, sbci2.hpp, davidson.hpp — compiled unmodified
// from /root/reference/proj/include) run on the B200 sigma through the C ABI of libsbg.so: the
// only new code is a SymmetricOperator subclass whose apply_impl calls sbg_sigma and whose
// diagonal comes from sbg_diagonal (operator.hpp:19-48; replaces FciOperator,
// fci_operator.hpp:60-86). Built by oracle/Makefile into oracle/_ref/libsbci_ref_gpu.so.
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "sbci/sbci.hpp"
#include "sbg.h"

namespace {

thread_local std::string g_err;

class CudaFciOperator final : public sbci::SymmetricOperator {
public:
    CudaFciOperator(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri,
                    std::uint64_t max_det)
        : SymmetricOperator(0) {
        if (int rc = sbg_create(norb, nelec, ms2, e_core, h1, eri, /*device=*/0, max_det, &ctx_); rc != SBG_OK)
            throw_code(rc);
        dim_ = static_cast<std::size_t>(sbg_dim(ctx_));
        diag_.assign(dim_, 0.0);
        if (int rc = sbg_diagonal(ctx_, diag_.data()); rc != SBG_OK) throw_code(rc);
    }
    ~CudaFciOperator() override { sbg_destroy(ctx_); }

private:
    [[noreturn]] static void throw_code(int rc) {
        const std::string msg = sbg_last_error();
        if (rc == SBG_EINVAL) throw std::invalid_argument(msg);
        throw std::runtime_error(msg);
    }
    void apply_impl(const sbci::Vector& x, sbci::Vector& y) const override {
        if (int rc = sbg_sigma(ctx_, x.data(), y.data(), 1); rc != SBG_OK) throw_code(rc);
    }
    sbg_ctx* ctx_ = nullptr;
};

}  // namespace

extern "C" {

const char* refgpu_last_error() { return g_err.c_str(); }

// The reference's solver (method 1 = solve_n_states_sbci1, 2 = solve_n_states_sbci2,
// 3 = davidson_solve) on the GPU operator, default SolverConfig.
int refgpu_solve(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri, int method,
                 int nroots, double* energies, int* iterations, uint64_t* matvecs) {
    try {
        CudaFciOperator op(norb, nelec, ms2, e_core, h1, eri, ~std::uint64_t{0});
        sbci::SolverConfig cfg;
        sbci::MultiStateResult r;
        if (method == 1) r = sbci::solve_n_states_sbci1(op, nroots, cfg);
        else if (method == 2) r = sbci::solve_n_states_sbci2(op, nroots, cfg);
        else {
            auto d = sbci::davidson_solve(op, nroots, cfg);
            r.pairs = d.pairs;
            r.summary = d.summary;
        }
        for (int k = 0; k < nroots; ++k) {
            energies[k] = r.pairs[k].energy;
            if (iterations) iterations[k] = r.pairs[k].iterations;
        }
        if (matvecs) *matvecs = r.summary.matvecs;
        return 0;
    } catch (const sbci::NonConvergenceError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

}  // extern "C"
