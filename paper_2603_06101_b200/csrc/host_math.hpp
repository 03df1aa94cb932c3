// host_math.hpp — the solver's host-scalar pieces, restated from the reference so the branch
// decisions of the device-resident solver match it exactly:
//   SolverConfig / RestartReason / StepOutcome / NonConvergenceError   (config.hpp:10-100)
//   SmallMatrix + cyclic Jacobi eigensolver                             (small_eig.hpp:13-106)
//   Gram-Schmidt coefficients from six inner products                   (ortho.hpp:31-76)
#pragma once

#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

namespace sbg {

struct SolverConfig {
    double eps0 = 1e-10, r0 = 1e-5, b_th = 1e-2, eps1 = 1e-7, x_th1 = 0.1, x_th2 = 1.2, r1 = 1.0;
    int max_cycle = 0;
    long t_max = 10000;
    double lindep = 1e-14, clamp_delta = 1e-10;
    int hx_refresh_restarts = 5;

    int effective_max_cycle(int method_default) const { return max_cycle > 0 ? max_cycle : method_default; }
    void validate() const {
        auto positive = [](double v, const char* name) {
            if (!(v > 0.0)) throw std::invalid_argument(std::string("SolverConfig: ") + name + " must be > 0");
        };
        positive(eps0, "eps0");
        positive(r0, "r0");
        positive(b_th, "b_th");
        positive(eps1, "eps1");
        positive(x_th1, "x_th1");
        positive(x_th2, "x_th2");
        positive(r1, "r1");
        positive(lindep, "lindep");
        positive(clamp_delta, "clamp_delta");
        if (!(x_th1 < 1.0 && 1.0 < x_th2)) throw std::invalid_argument("SolverConfig: need x_th1 < 1 < x_th2");
        if (max_cycle != 0 && max_cycle < 2) throw std::invalid_argument("SolverConfig: max_cycle must be >= 2");
        if (t_max < 1) throw std::invalid_argument("SolverConfig: t_max must be >= 1");
    }
};

enum class RestartReason { StallSmallB = 0, NormOutOfRange = 1, ResidualBlowup = 2, MaxCycle = 3 };

struct StepOutcome {
    enum class Kind { Continue, Converged, Restart } kind = Kind::Continue;
    RestartReason reason = RestartReason::StallSmallB;
    static StepOutcome cont() { return {Kind::Continue, RestartReason::StallSmallB}; }
    static StepOutcome converged() { return {Kind::Converged, RestartReason::StallSmallB}; }
    static StepOutcome restart(RestartReason r) { return {Kind::Restart, r}; }
};

struct NonConvergenceError : std::runtime_error {
    int state;
    double best_energy, best_residual;
    NonConvergenceError(int s, double e, double r)
        : std::runtime_error("state " + std::to_string(s) + " did not converge (best E = " + std::to_string(e) +
                             ", |z'| = " + std::to_string(r) + ")"),
          state(s), best_energy(e), best_residual(r) {}
};

struct SmallMatrix {
    int n = 0;
    std::vector<double> a;
    SmallMatrix() = default;
    explicit SmallMatrix(int d) : n(d), a((size_t)d * d, 0.0) {}
    double& operator()(int i, int j) { return a[(size_t)i * n + j]; }
    double operator()(int i, int j) const { return a[(size_t)i * n + j]; }
};

struct SmallEigResult {
    std::vector<double> eigenvalues;
    SmallMatrix eigenvectors;
};

// Cyclic Jacobi with the reference's rotation formula, sweep order, stopping rule and the stable
// ascending sort (small_eig.hpp:46-106).
inline SmallEigResult jacobi_symmetric_eig(SmallMatrix m) {
    const int n = m.n;
    SmallEigResult out;
    out.eigenvectors = SmallMatrix(n);
    for (int i = 0; i < n; ++i) out.eigenvectors(i, i) = 1.0;
    if (n == 0) return out;
    if (n == 1) {
        out.eigenvalues = {m(0, 0)};
        return out;
    }
    double fro = 0.0;
    for (double v : m.a) fro += v * v;
    const double stop = 1e-30 * std::max(fro, 1e-300);
    auto offdiag = [&]() {
        double s = 0.0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                if (i != j) s += m(i, j) * m(i, j);
        return s;
    };
    SmallMatrix& v = out.eigenvectors;
    for (int sweep = 0; sweep < 100 && offdiag() > stop; ++sweep)
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                const double apq = m(p, q);
                if (apq == 0.0) continue;
                const double tau = (m(q, q) - m(p, p)) / (2.0 * apq);
                const double t = (tau >= 0.0) ? 1.0 / (tau + std::sqrt(1.0 + tau * tau))
                                              : 1.0 / (tau - std::sqrt(1.0 + tau * tau));
                const double c = 1.0 / std::sqrt(1.0 + t * t), s = t * c;
                for (int k = 0; k < n; ++k) {
                    const double a = m(k, p), b = m(k, q);
                    m(k, p) = c * a - s * b;
                    m(k, q) = s * a + c * b;
                }
                for (int k = 0; k < n; ++k) {
                    const double a = m(p, k), b = m(q, k);
                    m(p, k) = c * a - s * b;
                    m(q, k) = s * a + c * b;
                }
                for (int k = 0; k < n; ++k) {
                    const double a = v(k, p), b = v(k, q);
                    v(k, p) = c * a - s * b;
                    v(k, q) = s * a + c * b;
                }
            }
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::vector<double> diag(n);
    for (int i = 0; i < n; ++i) diag[i] = m(i, i);
    std::stable_sort(order.begin(), order.end(), [&](int i, int j) { return diag[i] < diag[j]; });
    out.eigenvalues.resize(n);
    SmallMatrix sorted(n);
    for (int k = 0; k < n; ++k) {
        out.eigenvalues[k] = diag[order[k]];
        for (int i = 0; i < n; ++i) sorted(i, k) = v(i, order[k]);
    }
    out.eigenvectors = std::move(sorted);
    return out;
}

struct GramSchmidtCoeffs {
    double A_x = 0.0, B_x = 0.0, B_y = 0.0, C_x = 0.0, C_y = 0.0, C_z = 0.0;
    bool has_y = false, y_degenerate = false, z_degenerate = false, x_degenerate = false;
};

// ortho.hpp:45-76
inline GramSchmidtCoeffs gram_schmidt_from_dots(double nxx, double nxy, double nyy, double nxz, double nyz,
                                                double nzz, bool has_y, double lindep) {
    GramSchmidtCoeffs g;
    g.has_y = has_y;
    if (!(nxx > 0.0)) {
        g.x_degenerate = true;
        return g;
    }
    g.A_x = 1.0 / std::sqrt(nxx);
    double proj = 0.0;
    if (has_y) {
        const double yres = nyy - nxy * nxy / nxx;
        if (!(nyy > 0.0) || yres <= lindep * lindep * nyy) {
            g.y_degenerate = true;
            return g;
        }
        g.B_y = 1.0 / std::sqrt(yres);
        g.B_x = -(nxy / nxx) * g.B_y;
        proj = g.B_x * nxz + g.B_y * nyz;
    }
    const double zres = nzz - nxz * nxz / nxx - proj * proj;
    if (!(nzz > 0.0) || zres <= lindep * lindep * nzz) {
        g.z_degenerate = true;
        return g;
    }
    g.C_z = 1.0 / std::sqrt(zres);
    g.C_y = -proj * g.B_y * g.C_z;
    g.C_x = -(nxz / nxx + proj * g.B_x) * g.C_z;
    return g;
}

// Canonical orthogonalization P = U s^{-1/2} from a precomputed overlap matrix (ortho.hpp:155-184):
// Jacobi on s, keep modes with eigenvalue >= cutoff in descending order, coeff(i, c) = U(i, m)/sqrt(l_m).
// Throws std::runtime_error when every mode is discarded, as the reference does.
struct OrthoTransform {
    int n_inputs = 0, rank = 0;
    std::vector<double> p;  // [n_inputs][rank]
    double coeff(int i, int c) const { return p[(size_t)i * rank + c]; }
    double& coeff(int i, int c) { return p[(size_t)i * rank + c]; }
};

inline OrthoTransform canonical_orthogonalize_overlap(const SmallMatrix& s, double cutoff = 1e-14) {
    const int k = s.n;
    if (k < 1) throw std::invalid_argument("canonical_orthogonalize: need at least one vector");
    const SmallEigResult eig = jacobi_symmetric_eig(s);
    OrthoTransform t;
    t.n_inputs = k;
    std::vector<int> kept;
    for (int m = k - 1; m >= 0; --m)
        if (eig.eigenvalues[m] >= cutoff) kept.push_back(m);
    if (kept.empty()) throw std::runtime_error("canonical_orthogonalize: all overlap modes below cutoff");
    t.rank = (int)kept.size();
    t.p.assign((size_t)k * t.rank, 0.0);
    for (int c = 0; c < t.rank; ++c) {
        const int m = kept[c];
        const double inv_sqrt = 1.0 / std::sqrt(eig.eigenvalues[m]);
        for (int i = 0; i < k; ++i) t.coeff(i, c) = eig.eigenvectors(i, m) * inv_sqrt;
    }
    return t;
}

}  // namespace sbg
