// davidson.cu — block Davidson on device-resident vectors (reference: davidson.hpp:19-244): the
// cross-method check of the SBCI energies, with the same (D - E0)^-1 preconditioner.
// Host logic (Rayleigh-Ritz, convergence, collapse, expansion acceptance) follows the reference;
// the vector work is fused:
//   cross dots     b_i . h_j for the new basis rows/columns only (the reference recomputes the whole
//                  m x m projection every pass; cached values are the same dots)
//   ritz           all Ritz vectors, their images and residuals in one streaming pass per 16 basis
//                  vectors (k_ritz), accumulated in basis order like the reference's axpy chain
//   expansion      preconditioned residual, two classical Gram-Schmidt sweeps against the basis
//                  (block dots + one fused subtraction per 9 basis vectors; the reference runs the
//                  two sweeps vector by vector), normalisation, one sigma
#include "solver_detail.hpp"

namespace sbg {
namespace detail {

namespace {

struct DavidsonConfig {  // davidson.hpp:19-38
    int nroots = 1, max_space = 0;
    double eps0 = 1e-10, r0 = 1e-5, lindep = 1e-14;
    long max_iter = 400;
    int effective_max_space() const { return std::max(max_space > 0 ? max_space : 12 * nroots, 2 * nroots); }
    void validate() const {
        if (nroots < 1) throw std::invalid_argument("DavidsonConfig: nroots must be >= 1");
        if (!(eps0 > 0.0) || !(r0 > 0.0) || !(lindep > 0.0))
            throw std::invalid_argument("DavidsonConfig: tolerances must be > 0");
        if (max_space != 0 && max_space < 2 * nroots)
            throw std::invalid_argument("DavidsonConfig: max_space must be >= 2*nroots");
    }
};

// dots a . v_j for a list of vectors, kMaxIn - 1 per fused pass
std::vector<double> dots_against(Context& c, const DBuf& a, const std::vector<const DBuf*>& vs) {
    std::vector<double> out;
    for (size_t j0 = 0; j0 < vs.size(); j0 += kMaxIn - 1) {
        Lin L;
        const int sa = L.in(a.p);
        for (size_t j = j0; j < std::min(vs.size(), j0 + kMaxIn - 1); ++j) L.dot(sa, L.in(vs[j]->p));
        const auto r = L.run(c);
        out.insert(out.end(), r.begin(), r.end());
    }
    return out;
}

// t -= sum_j o_j v_j (kMaxIn - 1 basis vectors per fused pass)
void subtract_combination(Context& c, DBuf& t, const std::vector<const DBuf*>& vs, const std::vector<double>& o) {
    for (size_t j0 = 0; j0 < vs.size(); j0 += kMaxIn - 1) {
        Lin L;
        LinArgs& A = L.a;
        const int st = L.in(t.p);
        const int j = A.nout++;
        A.out[j] = t.p;
        A.coef[j][st] = 1.0;
        for (size_t i = j0; i < std::min(vs.size(), j0 + kMaxIn - 1); ++i) A.coef[j][L.in(vs[i]->p)] = -o[i];
        L.run(c);
    }
}

class Davidson {
public:
    Davidson(Context& c, const DavidsonConfig& d) : c_(c), o_(c), d_(d) {}

    // X(i, j) = b_i . h_j for every pair not yet known
    void update_cross() {
        const int m = (int)basis_.size();
        const int known = (int)X_.size();
        X_.resize(m);
        for (auto& row : X_) row.resize(m, 0.0);
        for (int n = known; n < m; ++n) {
            // new row n: b_n . h_j for j <= n ; new column n: b_j . h_n for j < n
            std::vector<const DBuf*> hs, bs;
            for (int j = 0; j <= n; ++j) hs.push_back(&images_[j]);
            for (int j = 0; j < n; ++j) bs.push_back(&basis_[j]);
            const auto row = dots_against(c_, basis_[n], hs);
            const auto col = dots_against(c_, images_[n], bs);
            for (int j = 0; j <= n; ++j) X_[n][j] = row[j];
            for (int j = 0; j < n; ++j) X_[j][n] = col[j];
        }
    }

    // Ritz vectors, images, residuals and residual norms for the lowest k roots
    std::vector<double> ritz(const SmallEigResult& eig, int k, const std::vector<double>& theta) {
        const int m = (int)basis_.size();
        while ((int)ritz_.size() < k) {
            ritz_.push_back(c_.vec());
            ritz_im_.push_back(c_.vec());
            res_.push_back(c_.vec());
        }
        std::vector<double> norms2;
        for (int i0 = 0; i0 < m; i0 += kRitzChunk) {
            RitzArgs a{};
            a.n = c_.padded_len();
            a.m = std::min(kRitzChunk, m - i0);
            a.k = k;
            a.first = i0 == 0;
            a.last = i0 + kRitzChunk >= m;
            for (int i = 0; i < a.m; ++i) {
                a.b[i] = basis_[i0 + i].p;
                a.h[i] = images_[i0 + i].p;
                for (int r = 0; r < k; ++r) a.coef[i][r] = eig.eigenvectors(i0 + i, r);
            }
            for (int r = 0; r < k; ++r) {
                a.theta[r] = theta[r];
                a.ritz[r] = ritz_[r].p;
                a.ritz_im[r] = ritz_im_[r].p;
                a.res[r] = res_[r].p;
            }
            launch_ritz(a, c_.rws, c_.st);
            c_.launches += 1;
            if (a.last) {
                const double* h = c_.finish_dots(k);
                norms2.assign(h, h + k);
            }
        }
        return norms2;
    }

    Context& c_;
    Ops o_;
    DavidsonConfig d_;
    std::vector<DBuf> basis_, images_, ritz_, ritz_im_, res_;
    std::vector<std::vector<double>> X_;
};

}  // namespace
}  // namespace detail

using namespace detail;

// davidson_solve(op, nroots, cfg) (davidson.hpp:53-244)
MultiStateResult davidson_solve(Context& c, int nroots, const SolverConfig& cfg,
                                const std::function<void(const TraceRec&)>& trace, int max_space_opt) {
    DavidsonConfig dcfg;
    dcfg.nroots = nroots;
    dcfg.max_space = max_space_opt;
    dcfg.eps0 = cfg.eps0;
    dcfg.r0 = cfg.r0;
    dcfg.lindep = cfg.lindep;
    dcfg.validate();
    if (nroots > kMaxRoots) throw std::invalid_argument("davidson_solve: at most 9 roots");
    if ((int64_t)nroots > c.ndet) throw std::invalid_argument("davidson_solve: nroots exceeds dimension");
    const int max_space = dcfg.effective_max_space();
    const auto t0 = std::chrono::steady_clock::now();
    const uint64_t applies_before = c.applies().load();

    Davidson dv(c, dcfg);
    Ops& o = dv.o_;
    // the starting shift is min(D); it is replaced by the first Ritz value before any use
    const auto lo = o.lowest_diagonal(1);
    Precond pre{&c.diagonal(), o.read(c.diagonal(), lo[0]), cfg.clamp_delta};
    if (!(pre.clamp > 0.0)) throw std::invalid_argument("clamp_delta must be positive");

    std::vector<Seed> guesses = init_guess(c, o, nroots);
    std::vector<double> prev_theta(nroots);
    for (int k = 0; k < nroots; ++k) {
        prev_theta[k] = guesses[k].energy;
        dv.basis_.push_back(std::move(guesses[k].x));
        dv.images_.push_back(std::move(guesses[k].hx));
    }
    std::vector<double> theta(nroots, 0.0), res_norms(nroots, std::numeric_limits<double>::infinity());
    std::vector<char> converged(nroots, 0);
    int peak_space = (int)dv.basis_.size();
    DBuf t = c.vec();

    for (long iter = 0; iter < dcfg.max_iter; ++iter) {
        const int m = (int)dv.basis_.size();
        dv.update_cross();
        SmallMatrix proj(m);
        for (int i = 0; i < m; ++i)
            for (int j = i; j < m; ++j) proj(i, j) = proj(j, i) = 0.5 * (dv.X_[i][j] + dv.X_[j][i]);
        const SmallEigResult eig = jacobi_symmetric_eig(proj);
        for (int k = 0; k < nroots; ++k) theta[k] = eig.eigenvalues[k];
        const auto n2 = dv.ritz(eig, nroots, theta);

        bool all_done = true;
        for (int k = 0; k < nroots; ++k) {
            res_norms[k] = std::sqrt(n2[k]);
            const double dE = std::abs(theta[k] - prev_theta[k]);
            converged[k] = dE < dcfg.eps0 && res_norms[k] < dcfg.r0;
            if (!converged[k]) all_done = false;
            if (trace) {
                TraceRec rec;
                rec.method = 3;
                rec.state = k;
                rec.t = (int)iter;
                rec.energy = theta[k];
                rec.dE = dE;
                rec.res_norm = res_norms[k];
                rec.x_norm = 1.0;
                rec.matvecs = c.applies().load();
                trace(rec);
            }
        }
        pre.update_shift(theta[0]);
        prev_theta = theta;

        if (all_done) {
            MultiStateResult out;
            for (int k = 0; k < nroots; ++k) {
                StateResult p;
                p.state = k;
                p.energy = theta[k];
                const double nm = o.norm(dv.ritz_[k]);
                p.vector = std::move(dv.ritz_[k]);
                if (nm > 0.0) o.scale(p.vector, 1.0 / nm);
                p.iterations = (int)iter + 1;
                p.final_residual = res_norms[k];
                out.pairs.push_back(std::move(p));
            }
            out.total_iterations = iter + 1;
            out.matvecs = c.applies().load() - applies_before;
            out.peak_vectors = 2 * peak_space + nroots;
            SBG_CUDA(cudaStreamSynchronize(c.st));
            out.wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            return out;
        }

        int pending = 0;
        for (int k = 0; k < nroots; ++k)
            if (!converged[k]) ++pending;
        if (m + pending > max_space) {  // collapse to the current Ritz vectors (davidson.hpp:156-176)
            std::vector<DBuf> nb, ni;
            for (int k = 0; k < nroots; ++k) {
                DBuf v = o.clone(dv.ritz_[k]);
                DBuf w = o.clone(dv.ritz_im_[k]);
                for (const auto& b : nb) {
                    const double ov = o.dot(b, v);
                    if (ov != 0.0) {
                        Lin L;
                        const int sv = L.in(v.p), sb = L.in(b.p);
                        L.out(v.p, {{sv, 1.0}, {sb, -ov}});
                        L.run(c);
                    }
                }
                const double nm = o.norm(v);
                if (nm < dcfg.lindep) continue;
                o.scale2(v, w, 1.0 / nm);
                nb.push_back(std::move(v));
                ni.push_back(std::move(w));
            }
            dv.basis_ = std::move(nb);
            dv.images_ = std::move(ni);
            dv.X_.clear();
        }

        int added = 0;
        for (int k = 0; k < nroots; ++k) {  // expansion (davidson.hpp:178-193)
            if (converged[k]) continue;
            PrecArgs pa{};
            pa.n = c.padded_len();
            pa.zres = dv.res_[k].p;
            pa.D = pre.D->p;
            pa.shift = pre.shift;
            pa.clamp = pre.clamp;
            pa.mode = 1;
            pa.z = t.p;
            pa.x = dv.res_[k].p;
            launch_precond(pa, c.rws, c.st);
            c.launches += 1;
            const double before = std::sqrt(c.finish_dots(3)[2]);
            if (before == 0.0) continue;
            std::vector<const DBuf*> bs;
            for (const auto& b : dv.basis_) bs.push_back(&b);
            for (int pass = 0; pass < 2; ++pass) subtract_combination(c, t, bs, dots_against(c, t, bs));
            const double nm = o.norm(t);
            if (nm < std::sqrt(dcfg.lindep) * before) continue;  // direction already represented
            o.scale(t, 1.0 / nm);
            // the image is built after the loop, with the other new directions (orthogonalising the
            // next correction needs the basis, not the images): one multi-vector sigma per block
            dv.basis_.push_back(std::move(t));
            t = c.vec();
            ++added;
        }
        if (added > 0) {  // images of the expansion block (davidson.hpp:184-194), in basis order
            std::vector<const DBuf*> xs;
            std::vector<DBuf*> ys;
            const size_t first = dv.basis_.size() - (size_t)added;
            for (int k = 0; k < added; ++k) dv.images_.push_back(c.vec());
            for (int k = 0; k < added; ++k) {
                xs.push_back(&dv.basis_[first + k]);
                ys.push_back(&dv.images_[first + k]);
            }
            o.apply_multi(xs, ys);
        }
        peak_space = std::max(peak_space, (int)dv.basis_.size());
        if (added == 0 && !all_done) {
            bool residual_ok = true;
            for (int k = 0; k < nroots; ++k)
                if (res_norms[k] >= dcfg.r0) residual_ok = false;
            if (!residual_ok) break;
            for (int k = 0; k < nroots; ++k) converged[k] = 1;
            prev_theta = theta;
        }
    }
    throw NonConvergenceError(-1, theta.empty() ? 0.0 : theta[0], *std::max_element(res_norms.begin(), res_norms.end()));
}

}  // namespace sbg
