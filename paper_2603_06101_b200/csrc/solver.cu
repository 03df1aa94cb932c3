// solver.cu — the SBCI1 driver on device-resident vectors (reference: sbci1.hpp:45-579,
// precond.hpp:19-111). Structure and scalar logic follow the reference line by line; the vector
// work is issued as fused passes (vec.cu) whose dot products are the only data that crosses to
// the host each step.
#include "solver_detail.hpp"

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <optional>

namespace sbg {

namespace detail {

// ------------------------------------------------------------------ state
struct State {  // Sbci1State (sbci1.hpp:95-105)
    int alpha = 0, t = 0;
    DBuf x, hx, y, hy, zres;
    double energy = 0.0;
    double b_prev = 1.0, c_prev = 0.0, k_prev = 1.0;
    int restart_count = 0;
    long total_iterations = 0;
};

struct StepData {
    StepOutcome outcome;
    double dE = 0.0, dz = 0.0;
    bool have_ritz = false;
    double sx = 0, sy = 0, sz = 0, b = 0, c = 0, ritz_e = 0;
    bool three = false;
    bool committed = false;
    double x_norm = 0.0;  // |x| after the step (valid when committed)
    bool have_kinetic = false;  // kinetic scalar of the committed y' (traced solves, fused in the commit pass)
    double kinetic = 0.0;
};

std::optional<RestartReason> check_restart(int alpha, double b, double dE, double x_norm, double dz, int t,
                                           const SolverConfig& cfg, int max_cycle) {  // sbci1.hpp:109-117
    if (alpha > 0 && std::abs(b) < cfg.b_th && dE < cfg.eps1) return RestartReason::StallSmallB;
    if (x_norm < cfg.x_th1 || x_norm > cfg.x_th2) return RestartReason::NormOutOfRange;
    if (dz > cfg.r1 && t > 0) return RestartReason::ResidualBlowup;
    if (t + 1 >= max_cycle) return RestartReason::MaxCycle;
    return std::nullopt;
}

static std::vector<double> h_ovl(Context& c, int n) {
    const double* h = c.finish_dots(n);
    return std::vector<double>(h, h + n);
}

// precondition() up to the dots: z is enqueued, its dots are posted (Context::post_dots); returns
// their count. The caller collects them with Context::wait_dots.
int precondition_post(Context& c, const DBuf& zres, const Precond& pre, const Deflation& defl, DBuf& z,
                      const DBuf& x, const DBuf* y) {
    PrecArgs pa{};
    pa.n = c.padded_len();
    pa.zres = zres.p;
    pa.D = pre.D->p;
    pa.shift = pre.shift;
    pa.clamp = pre.clamp;
    pa.nxc = (int)defl.size();
    if (pa.nxc > kMaxDeflated) throw std::invalid_argument("precondition: at most 8 deflated states (9 roots)");
    for (size_t i = 0; i < defl.size(); ++i) pa.xc[i] = defl.m[i].x.p;
    if (pa.nxc > 0) {  // overlaps x_c . (D - E0)^-1 zres first, then the deflated z in one pass
        pa.mode = 0;
        launch_precond(pa, c.rws, c.st);
        c.launches += 1;
        const auto o = defl.sequential(std::vector<double>(h_ovl(c, pa.nxc)));
        for (int i = 0; i < pa.nxc; ++i) pa.o[i] = o[i];
    }
    pa.mode = 1;
    pa.z = z.p;
    pa.x = x.p;
    pa.y = y ? y->p : nullptr;
    launch_precond(pa, c.rws, c.st);
    c.launches += 1;
    const int nd = y ? 6 : 3;
    c.post_dots(nd);
    return nd;
}

std::vector<double> precondition(Context& c, const DBuf& zres, const Precond& pre, const Deflation& defl, DBuf& z,
                                 const DBuf& x, const DBuf* y) {
    const int nd = precondition_post(c, zres, pre, defl, z, x, y);
    const double* h = c.wait_dots();
    return std::vector<double>(h, h + nd);  // xx, xz, zz [, xy, yy, yz]
}

class Driver {
public:
    Driver(Context& c, const SolverConfig& cfg, const std::function<void(const TraceRec&)>& trace)
        : c_(c), o_(c), cfg_(cfg), trace_(trace), z_(c.vec()), hz_(c.vec()) {}

    std::vector<double> make_z(const State& st, const Precond& pre, const Deflation& defl, bool with_y) {
        return precondition(c_, st.zres, pre, defl, z_, st.x, with_y ? &st.y : nullptr);
    }

    // sbci1_step_impl (sbci1.hpp:147-323)
    StepData step(State& st, const Precond& pre, Deflation& defl, int max_cycle) {
        StepData out;
        bool use_three = st.t >= 1;
        auto tp = Clk::now();
        // H z is enqueued right behind z, before the host reads z's dots: the Gram-Schmidt scalars
        // are formed while the sigma kernels run. The branches that end the step before the
        // reference applies the operator (sbci1.hpp:153-184) take that application back from the
        // counter, so matvec counts stay the reference's.
        const int nd = precondition_post(c_, st.zres, pre, defl, z_, st.x, use_three ? &st.y : nullptr);
        if (speculate_) o_.apply(z_, hz_);
        const double* hd = c_.wait_dots();
        const std::vector<double> d(hd, hd + nd);
        g_ph[0] += ms_since(tp);
        struct Unapply {  // the speculative sigma is not an application of the reference's step
            Context& c;
            bool on;
            ~Unapply() {
                if (on) c.applies().fetch_sub(1, std::memory_order_relaxed);
            }
        } unapply{c_, speculate_};
        const double nxx = d[0], nxz = d[1], nzz = d[2];
        if (std::sqrt(nzz) < cfg_.lindep * std::sqrt(nxx)) {
            const double xhx = o_.dot(st.x, st.hx);
            if (nxx == 0.0) throw std::invalid_argument("rayleigh_quotient: zero vector");
            st.energy = xhx / nxx;
            out.outcome = StepOutcome::converged();
            out.dE = 0.0;
            out.dz = o_.norm(st.zres);
            out.x_norm = std::sqrt(nxx);
            return out;
        }
        GramSchmidtCoeffs gs;
        if (use_three) {
            gs = gram_schmidt_from_dots(nxx, d[3], d[4], nxz, d[5], nzz, true, cfg_.lindep);
            if (gs.y_degenerate) use_three = false;
            else if (gs.z_degenerate) {
                out.outcome = StepOutcome::restart(RestartReason::StallSmallB);
                return out;
            }
        }
        if (!use_three) {
            gs = gram_schmidt_from_dots(nxx, 0.0, 0.0, nxz, 0.0, nzz, false, cfg_.lindep);
            if (gs.z_degenerate) {
                out.outcome = StepOutcome::restart(RestartReason::StallSmallB);
                return out;
            }
        }
        unapply.on = false;  // the step applies the operator here (sbci1.hpp:186)
        tp = Clk::now();
        if (!speculate_) o_.apply(z_, hz_);
        g_ph[1] += ms_since(tp);
        tp = Clk::now();

        SubArgs sa{};
        sa.n = c_.padded_len();
        sa.x = st.x.p;
        sa.y = st.y.p;
        sa.z = z_.p;
        sa.hx = st.hx.p;
        sa.hy = st.hy.p;
        sa.hz = hz_.p;
        sa.Ax = gs.A_x;
        sa.Bx = gs.B_x;
        sa.By = gs.B_y;
        sa.Cx = gs.C_x;
        sa.Cy = gs.C_y;
        sa.Cz = gs.C_z;
        sa.three = use_three;
        launch_subspace(sa, c_.rws, c_.st);
        c_.launches += 1;
        const int m = use_three ? 3 : 2;
        double e_new = 0.0, k = 0.0, b = 0.0, c = 0.0;
        double zz2, xx2;
        std::vector<double> ovl;
        if (device_scalars_ && spares()) {
            // The subspace matrix, its Jacobi eigenpairs, k, b, c and the commit coefficients are
            // formed on one device thread (step_scalars.cu, the host's arithmetic bit for bit) and
            // the commit pass reads its coefficients from device memory: no host round trip between
            // the subspace pass and the commit pass. The scalars come back with the commit's dots.
            StepScalarArgs sca{gs.A_x, gs.B_x, gs.B_y, gs.C_x, gs.C_y, gs.C_z, use_three ? 1 : 0};
            c_.allreduce_inplace_device(c_.rws.result, m * m);  // world > 1: every rank's partial dots
            launch_step_scalars(c_.rws.result, sca, dcoef_.p, dscal_.p, c_.st);
            c_.launches += 1;
            SBG_CUDA(cudaMemcpyAsync(hscal_, dscal_.p, 9 * sizeof(double), cudaMemcpyDeviceToHost, c_.st));
            Lin L;
            const int sx = L.in(st.x.p), sy = L.in(st.y.p), sz = L.in(z_.p), shx = L.in(st.hx.p),
                      shy = L.in(st.hy.p), shz = L.in(hz_.p);
            std::vector<int> sxc;
            const bool fused_ovl = L.fits((int)defl.size());
            if (fused_ovl)
                for (auto& mm : defl.m) sxc.push_back(L.in(mm.x.p));
            // the same pass shape as below; the coefficients themselves come from dcoef_
            const int yn = use_three ? L.out(sp_y_.p, {{sy, 1.0}, {sz, 1.0}}) : L.out(sp_y_.p, {{sz, 1.0}});
            const int hyn = use_three ? L.out(sp_hy_.p, {{shy, 1.0}, {shz, 1.0}}) : L.out(sp_hy_.p, {{shz, 1.0}});
            const int xn = L.out(sp_x_.p, {{sx, 1.0}, {yn, 1.0}});
            const int hxn = L.out(sp_hx_.p, {{shx, 1.0}, {hyn, 1.0}});
            const int zn = L.out(sp_z_.p, {{hxn, 1.0}, {xn, 1.0}});
            L.a.dcoef = dcoef_.p;
            L.dot(zn, zn);
            L.dot(xn, xn);
            L.dot(yn, yn);
            for (int s2 : sxc) L.dot(s2, zn);
            if (trace_) L.kinetic(yn, pre.D->p, pre.shift);
            const auto r = L.run(c_);  // synchronises: hscal_ is valid too
            g_ph[2] += ms_since(tp);
            tp = Clk::now();
            if (hscal_[0] != 0.0) {  // |k_den| or |b_den| < 1e-14 (sbci1.hpp:230-246): restart, no commit
                out.outcome = StepOutcome::restart(RestartReason::StallSmallB);
                return out;
            }
            k = hscal_[1];
            b = hscal_[2];
            c = hscal_[3];
            e_new = hscal_[4];
            out.ritz_e = hscal_[5];
            out.sx = hscal_[6];
            out.sy = hscal_[7];
            out.sz = hscal_[8];
            zz2 = r[0];
            xx2 = r[1];
            if (std::sqrt(nxx) + std::abs(b) * std::sqrt(r[2]) > 1e6 * std::max(std::sqrt(xx2), 1e-300)) {
                out.outcome = StepOutcome::restart(RestartReason::StallSmallB);
                return out;
            }
            if (trace_) {
                out.have_kinetic = true;
                out.kinetic = r.back();
            }
            std::swap(st.y, sp_y_);
            std::swap(st.hy, sp_hy_);
            std::swap(st.x, sp_x_);
            std::swap(st.hx, sp_hx_);
            std::swap(st.zres, sp_z_);
            ovl.assign(r.begin() + 3, r.begin() + 3 + sxc.size());
            if (!fused_ovl) ovl = deflation_overlaps(c_, defl, st.zres);
            ovl = defl.sequential(std::move(ovl));
        } else {
            const double* h = c_.finish_dots(m * m);
            SmallMatrix v(m);
            for (int i = 0; i < m; ++i)
                for (int j = i; j < m; ++j) v(i, j) = v(j, i) = 0.5 * (h[i * m + j] + h[j * m + i]);
            g_ph[2] += ms_since(tp);
            tp = Clk::now();
            const SmallEigResult eig = jacobi_symmetric_eig(v);
            g_ph[3] += ms_since(tp);
            tp = Clk::now();

            const double vx = eig.eigenvectors(0, 0), vy = use_three ? eig.eigenvectors(1, 0) : 0.0,
                         vz = eig.eigenvectors(m - 1, 0);
            const double wx = eig.eigenvectors(0, 1), wy = use_three ? eig.eigenvectors(1, 1) : 0.0,
                         wz = eig.eigenvectors(m - 1, 1);
            e_new = eig.eigenvalues[0];
            const double k_den = vx * gs.A_x + vy * gs.B_x + vz * gs.C_x;
            if (std::abs(k_den) < 1e-14) {
                out.outcome = StepOutcome::restart(RestartReason::StallSmallB);
                return out;
            }
            k = 1.0 / k_den;
            if (use_three) {
                const double b_den = vy * gs.B_y + vz * gs.C_y;
                if (std::abs(b_den) < 1e-14) {
                    out.outcome = StepOutcome::restart(RestartReason::StallSmallB);
                    return out;
                }
                b = k * b_den;
                c = -vz * gs.C_z / b_den;
            } else {
                b = 1.0;
                c = -k * vz * gs.C_z;
            }
            // guard + commit in one pass (sbci1.hpp:259-267): y' = y - c z, Hy' = Hy - c Hz,
            // x' = x + b y', Hx' = Hx + b Hy', z' = (1/k) Hx' - (E'/k) x' are written into spare
            // buffers with |z'|^2, |x'|^2, |y'|^2 and the deflation overlaps x_c . z'; the cancellation
            // guard is then evaluated from those norms and the spares are swapped in only if it passes
            // (a rejected step leaves the state untouched, as in the reference)
            // second-lowest Ritz vector coefficients (sbci1.hpp:287-311)
            out.sx = wx * gs.A_x + wy * gs.B_x + wz * gs.C_x;
            out.sy = wy * gs.B_y + wz * gs.C_y;
            out.sz = wz * gs.C_z;
            out.ritz_e = eig.eigenvalues[1];
            if (!spares()) {
                // two-pass form when the five spares do not fit in HBM (or SBG_GUARD_TWO_PASS=1): the
                // candidate norms first (read-only pass, the same per-element arithmetic and reduction
                // tree, so the same values), then — only if the guard passes — the commit in place
                Lin L;
                const int sx = L.in(st.x.p), sy = L.in(st.y.p), sz = L.in(z_.p), shx = L.in(st.hx.p),
                          shy = L.in(st.hy.p), shz = L.in(hz_.p);
                std::vector<int> sxc;
                const bool fused_ovl = L.fits((int)defl.size());
                if (fused_ovl)
                    for (auto& mm : defl.m) sxc.push_back(L.in(mm.x.p));
                const int yn = use_three ? L.out(nullptr, {{sy, 1.0}, {sz, -c}}) : L.out(nullptr, {{sz, -c}});
                const int hyn = use_three ? L.out(nullptr, {{shy, 1.0}, {shz, -c}}) : L.out(nullptr, {{shz, -c}});
                const int xn = L.out(nullptr, {{sx, 1.0}, {yn, b}});
                const int hxn = L.out(nullptr, {{shx, 1.0}, {hyn, b}});
                const int zn = L.out(nullptr, {{hxn, 1.0 / k}, {xn, -e_new / k}});
                L.dot(zn, zn);
                L.dot(xn, xn);
                L.dot(yn, yn);
                for (int s : sxc) L.dot(s, zn);
                if (trace_) L.kinetic(yn, pre.D->p, pre.shift);
                const auto r = L.run(c_);
                zz2 = r[0];
                xx2 = r[1];
                if (std::sqrt(nxx) + std::abs(b) * std::sqrt(r[2]) > 1e6 * std::max(std::sqrt(xx2), 1e-300)) {
                    out.outcome = StepOutcome::restart(RestartReason::StallSmallB);
                    return out;
                }
                if (trace_) {
                    out.have_kinetic = true;
                    out.kinetic = r.back();
                }
                Lin W;
                const int wx = W.in(st.x.p), wy = W.in(st.y.p), wz = W.in(z_.p), whx = W.in(st.hx.p), why = W.in(st.hy.p),
                          whz = W.in(hz_.p);
                const int y2 = use_three ? W.out(st.y.p, {{wy, 1.0}, {wz, -c}}) : W.out(st.y.p, {{wz, -c}});
                const int hy2 = use_three ? W.out(st.hy.p, {{why, 1.0}, {whz, -c}}) : W.out(st.hy.p, {{whz, -c}});
                const int x2 = W.out(st.x.p, {{wx, 1.0}, {y2, b}});
                const int hx2 = W.out(st.hx.p, {{whx, 1.0}, {hy2, b}});
                W.out(st.zres.p, {{hx2, 1.0 / k}, {x2, -e_new / k}});
                W.run(c_);
                ovl.assign(r.begin() + 3, r.begin() + 3 + sxc.size());
                if (!fused_ovl) ovl = deflation_overlaps(c_, defl, st.zres);
                ovl = defl.sequential(std::move(ovl));
            } else {
                Lin L;
                const int sx = L.in(st.x.p), sy = L.in(st.y.p), sz = L.in(z_.p), shx = L.in(st.hx.p),
                          shy = L.in(st.hy.p), shz = L.in(hz_.p);
                std::vector<int> sxc;
                const bool fused_ovl = L.fits((int)defl.size());
                if (fused_ovl)
                    for (auto& mm : defl.m) sxc.push_back(L.in(mm.x.p));
                const int yn = use_three ? L.out(sp_y_.p, {{sy, 1.0}, {sz, -c}}) : L.out(sp_y_.p, {{sz, -c}});
                const int hyn = use_three ? L.out(sp_hy_.p, {{shy, 1.0}, {shz, -c}}) : L.out(sp_hy_.p, {{shz, -c}});
                const int xn = L.out(sp_x_.p, {{sx, 1.0}, {yn, b}});
                const int hxn = L.out(sp_hx_.p, {{shx, 1.0}, {hyn, b}});
                const int zn = L.out(sp_z_.p, {{hxn, 1.0 / k}, {xn, -e_new / k}});
                L.dot(zn, zn);
                L.dot(xn, xn);
                L.dot(yn, yn);
                for (int s : sxc) L.dot(s, zn);
                if (trace_) L.kinetic(yn, pre.D->p, pre.shift);  // folded here instead of a pass of its own
                const auto r = L.run(c_);
                zz2 = r[0];
                xx2 = r[1];
                if (std::sqrt(nxx) + std::abs(b) * std::sqrt(r[2]) > 1e6 * std::max(std::sqrt(xx2), 1e-300)) {
                    out.outcome = StepOutcome::restart(RestartReason::StallSmallB);
                    return out;
                }
                if (trace_) {
                    out.have_kinetic = true;
                    out.kinetic = r.back();
                }
                std::swap(st.y, sp_y_);
                std::swap(st.hy, sp_hy_);
                std::swap(st.x, sp_x_);
                std::swap(st.hx, sp_hx_);
                std::swap(st.zres, sp_z_);
                ovl.assign(r.begin() + 3, r.begin() + 3 + sxc.size());
                if (!fused_ovl) ovl = deflation_overlaps(c_, defl, st.zres);
                ovl = defl.sequential(std::move(ovl));
            }
        }
        g_ph[4] += ms_since(tp);
        out.committed = true;
        out.dE = std::abs(e_new - st.energy);
        out.dz = std::sqrt(zz2);
        out.x_norm = std::sqrt(xx2);
        double dz_defl = out.dz;
        if (!defl.empty()) {  // |(1 - sum x_c x_c^T) z'| (sbci1.hpp:274-279)
            Lin L;
            const int sz = L.in(st.zres.p);
            std::vector<std::pair<int, double>> terms{{sz, 1.0}};
            std::vector<int> sxc;
            for (size_t i = 0; i < defl.size(); ++i) sxc.push_back(L.in(defl.m[i].x.p));
            LinArgs& A = L.a;
            const int j = A.nout++;
            A.out[j] = nullptr;
            A.coef[j][sz] = 1.0;
            for (size_t i = 0; i < sxc.size(); ++i) A.coef[j][sxc[i]] = -ovl[i];
            L.dot(kMaxIn + j, kMaxIn + j);
            dz_defl = std::sqrt(L.run(c_)[0]);
        }
        st.energy = e_new;
        st.b_prev = b;
        st.c_prev = c;
        st.k_prev = k;
        // second-lowest Ritz vector (coefficients set above); materialized only on convergence
        out.have_ritz = true;
        out.b = b;
        out.c = c;
        out.three = use_three;

        if (out.dE < cfg_.eps0 && std::min(out.dz, dz_defl) < cfg_.r0) {
            out.outcome = StepOutcome::converged();
            return out;
        }
        if (auto reason = check_restart(st.alpha, b, out.dE, out.x_norm, out.dz, st.t, cfg_, max_cycle)) {
            out.outcome = StepOutcome::restart(*reason);
            return out;
        }
        out.outcome = StepOutcome::cont();
        return out;
    }

    // the converged step's second Ritz vector (sbci1.hpp:287-311), rebuilt from x_{t+1}, y_{t+1},
    // z, Hz: x_t = x - b y, y_t = y + c z, s = sx x_t + sy y_t + sz z (same summation order)
    Seed second_ritz(const State& st, const StepData& s) {
        Seed r;
        r.x = c_.vec();
        r.hx = c_.vec();
        for (int pass = 0; pass < 2; ++pass) {
            Lin L;
            const int sx = L.in(pass ? st.hx.p : st.x.p), sy = L.in(pass ? st.hy.p : st.y.p),
                      sz = L.in(pass ? hz_.p : z_.p);
            const int xt = L.out(nullptr, {{sx, 1.0}, {sy, -s.b}});
            const int yt = L.out(nullptr, {{sy, 1.0}, {sz, s.c}});
            const int zc = L.out(nullptr, {{sz, 1.0}});
            if (s.three) L.out(pass ? r.hx.p : r.x.p, {{xt, s.sx}, {yt, s.sy}, {zc, s.sz}});
            else L.out(pass ? r.hx.p : r.x.p, {{xt, s.sx}, {zc, s.sz}});
            L.run(c_);
        }
        r.energy = s.ritz_e;
        return r;
    }

    StepData last_;
    Context& c_;
    Ops o_;
    SolverConfig cfg_;
    const std::function<void(const TraceRec&)>& trace_;
    DBuf z_, hz_;
    DBuf sp_y_, sp_hy_, sp_x_, sp_hx_, sp_z_;  // candidate state of the merged guard + commit pass
    bool two_pass_ = std::getenv("SBG_GUARD_TWO_PASS") && std::atoi(std::getenv("SBG_GUARD_TWO_PASS")) != 0;
    bool speculate_ = !(std::getenv("SBG_SPECULATE") && std::atoi(std::getenv("SBG_SPECULATE")) == 0);
    // step scalars on the device (SBG_DEVICE_SCALARS=0: on the host, with a round trip per step)
    bool device_scalars_ = !(std::getenv("SBG_DEVICE_SCALARS") && std::atoi(std::getenv("SBG_DEVICE_SCALARS")) == 0);
    DBuf dcoef_{(int64_t)kMaxOut * (kMaxIn + kMaxOut)}, dscal_{16};
    struct PinnedScalars {
        double* p = nullptr;
        PinnedScalars() { SBG_CUDA(cudaMallocHost(&p, 16 * sizeof(double))); }
        ~PinnedScalars() { cudaFreeHost(p); }
    } pinned_;
    double* hscal_ = pinned_.p;

    // the merged guard + commit pass needs five spare vectors; without room for them the step
    // falls back to the two-pass form for the rest of the solve (large sectors)
    bool spares() {
        if (two_pass_) return false;
        if (!sp_y_.empty()) return true;
        try {
            sp_y_ = c_.vec();
            sp_hy_ = c_.vec();
            sp_x_ = c_.vec();
            sp_hx_ = c_.vec();
            sp_z_ = c_.vec();
            return true;
        } catch (const DeviceError&) {
            cudaGetLastError();  // the failed cudaMalloc leaves no sticky error
            for (DBuf* b : {&sp_y_, &sp_hy_, &sp_x_, &sp_hx_, &sp_z_}) *b = DBuf();
            two_pass_ = true;
            return false;
        }
    }
};


// solve_state_sbci1 (sbci1.hpp:357-473)
Sbci1Result solve_state(Driver& dr, Precond& pre, Deflation& defl, Seed seed, int alpha, bool track) {
    Context& c = dr.c_;
    Ops& o = dr.o_;
    const SolverConfig& cfg = dr.cfg_;
    cfg.validate();
    const int max_cycle = cfg.effective_max_cycle(kSbci1DefaultMaxCycle);
    defl.project_out_pair(o, seed.x, seed.hx);
    const double seed_norm = o.norm(seed.x);
    if (seed_norm < cfg.lindep) throw std::invalid_argument("solve_state_sbci1: seed collapsed under deflation");
    o.scale2(seed.x, seed.hx, 1.0 / seed_norm);

    State st;
    st.alpha = alpha;
    st.x = std::move(seed.x);
    st.hx = std::move(seed.hx);
    st.y = c.vec();
    st.hy = c.vec();
    st.zres = c.vec();
    st.energy = o.dot(st.x, st.hx);
    o.combine(st.zres, 1.0, st.hx, -st.energy, st.x);

    Sbci1Result result;
    if (track) pre.update_shift(st.energy);
    {
        const auto d = dr.make_z(st, pre, defl, false);
        if (std::sqrt(d[2]) < cfg.lindep) {
            result.pair.state = alpha;
            result.pair.energy = st.energy;
            result.pair.final_residual = o.norm(st.zres);
            result.pair.vector = std::move(st.x);
            result.converged_image = std::move(st.hx);
            return result;
        }
    }
    while (st.total_iterations < cfg.t_max) {
        StepData step = dr.step(st, pre, defl, max_cycle);
        ++st.total_iterations;
        auto tq = Clk::now();
        if (dr.trace_) {
            TraceRec rec;
            rec.state = alpha;
            rec.t = st.t;
            rec.energy = st.energy;
            rec.dE = step.dE;
            rec.res_norm = step.dz;
            rec.x_norm = step.committed ? step.x_norm : o.norm(st.x);
            if (step.have_kinetic) {
                rec.kinetic = step.kinetic;
            } else {  // no commit this step: y is unchanged, one pass of its own
                launch_kinetic(st.y.p, pre.D->p, pre.shift, c.padded_len(), c.rws, c.st);
                c.launches += 1;
                rec.kinetic = c.finish_dots(1)[0];
            }
            rec.matvecs = c.applies().load();
            rec.b = st.b_prev;
            rec.c = st.c_prev;
            rec.restart_reason = step.outcome.kind == StepOutcome::Kind::Restart ? (int)step.outcome.reason : -1;
            dr.trace_(rec);
        }
        g_ph[5] += ms_since(tq);
        tq = Clk::now();
        if (track) pre.update_shift(st.energy);
        switch (step.outcome.kind) {
            case StepOutcome::Kind::Converged: {
                StateResult pair;
                pair.state = alpha;
                const double xx = o.dot(st.x, st.x);
                if (xx == 0.0) throw std::invalid_argument("rayleigh_quotient: zero vector");
                pair.energy = o.dot(st.x, st.hx) / xx;
                const double nm = std::sqrt(xx);
                if (step.have_ritz) result.next_seed = dr.second_ritz(st, step);
                pair.vector = std::move(st.x);
                if (nm > 0.0) o.scale(pair.vector, 1.0 / nm);
                for (auto& mm : defl.m)
                    if (std::abs(o.dot(mm.x, pair.vector)) > 1e-9)
                        throw NonConvergenceError(alpha, pair.energy, step.dz);
                pair.iterations = (int)st.total_iterations;
                pair.restarts = st.restart_count;
                pair.final_residual = step.dz;
                result.pair = std::move(pair);
                o.scale(st.hx, nm > 0.0 ? 1.0 / nm : 1.0);
                result.converged_image = std::move(st.hx);
                return result;
            }
            case StepOutcome::Kind::Restart: {
                double nm = o.norm(st.x);
                if (nm < cfg.lindep) throw NonConvergenceError(alpha, st.energy, step.dz);
                o.scale2(st.x, st.hx, 1.0 / nm);
                if (!defl.empty()) {
                    defl.project_out_pair(o, st.x, st.hx);
                    nm = o.norm(st.x);
                    if (nm < cfg.lindep) throw NonConvergenceError(alpha, st.energy, step.dz);
                    o.scale2(st.x, st.hx, 1.0 / nm);
                    st.energy = o.dot(st.x, st.hx);
                }
                o.zero(st.y);
                o.zero(st.hy);
                ++st.restart_count;
                if (cfg.hx_refresh_restarts > 0 && st.restart_count % cfg.hx_refresh_restarts == 0) {
                    o.apply(st.x, st.hx);
                    ++result.hx_refreshes;
                }
                o.combine(st.zres, 1.0, st.hx, -st.energy, st.x);
                st.t = 0;
                g_ph[6] += ms_since(tq);
                break;
            }
            case StepOutcome::Kind::Continue:
                ++st.t;
                break;
        }
    }
    throw NonConvergenceError(alpha, st.energy, o.norm(st.zres));
}

Sbci1Result solve_state_sbci1(Context& c, const SolverConfig& cfg, const std::function<void(const TraceRec&)>& trace,
                              Precond& pre, Deflation& defl, Seed seed, int alpha, bool track) {
    Driver dr(c, cfg, trace);
    return solve_state(dr, pre, defl, std::move(seed), alpha, track);
}

// init_guess_from_diagonal (sbci1.hpp:45-92)
std::vector<Seed> init_guess(Context& c, Ops& o, int n) {
    if (n < 1 || (int64_t)n > c.ndet) throw std::invalid_argument("init_guess_from_diagonal: need 1 <= n <= dim");
    const auto idx = o.lowest_diagonal(n);
    std::vector<DBuf> images;
    {
        DBuf e = c.vec();
        for (int k = 0; k < n; ++k) {
            o.set_unit(e, idx[k]);
            images.push_back(c.vec());
            o.apply(e, images.back());
        }
    }
    const int m = n;
    SmallMatrix proj(m);
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) proj(i, j) = o.read(images[j], idx[i]);
    for (int i = 0; i < m; ++i)
        for (int j = i + 1; j < m; ++j) {
            const double s = 0.5 * (proj(i, j) + proj(j, i));
            proj(i, j) = proj(j, i) = s;
        }
    const SmallEigResult eig = jacobi_symmetric_eig(proj);
    std::vector<Seed> seeds(m);
    for (int a = 0; a < m; ++a) {
        Seed& s = seeds[a];
        s.x = c.vec();
        s.hx = c.vec();
        for (int i = 0; i < m; ++i) {
            const int64_t gi = idx[i];
            const int64_t row = gi / c.NB, col = gi % c.NB;
            if (row >= c.row_lo && row < c.row_hi) {
                launch_set_element(s.x.p, (row - c.row_lo) * c.ld + col, eig.eigenvectors(i, a), c.st);
                c.launches++;
            }
        }
        // hx = sum_i v_ia images_i, accumulated in order (axpy chain)
        for (int i0 = 0; i0 < m; i0 += kMaxIn - 1) {
            Lin L;
            LinArgs& A = L.a;
            const int j = A.nout++;
            A.out[j] = s.hx.p;
            if (i0 > 0) A.coef[j][L.in(s.hx.p)] = 1.0;
            for (int i = i0; i < std::min(m, i0 + kMaxIn - 1); ++i) A.coef[j][L.in(images[i].p)] = eig.eigenvectors(i, a);
            L.run(c);
        }
        s.energy = eig.eigenvalues[a];
    }
    return seeds;
}

// select_seed (sbci1.hpp:501-519): lowest Rayleigh quotient after deflation
Seed select_seed(Context& c, Ops& o, std::vector<const Seed*> cands, Deflation& defl, double lindep) {
    std::optional<Seed> best;
    for (const Seed* cand : cands) {
        Seed s;
        s.x = o.clone(cand->x);
        s.hx = o.clone(cand->hx);
        defl.project_out_pair(o, s.x, s.hx);
        const double nm = o.norm(s.x);
        if (nm < std::max(lindep, 1e-8)) continue;
        o.scale2(s.x, s.hx, 1.0 / nm);
        s.energy = o.dot(s.x, s.hx);
        if (!best || s.energy < best->energy) best = std::move(s);
    }
    (void)c;
    if (!best) throw std::runtime_error("all seed candidates collapsed under deflation");
    return std::move(*best);
}

}  // namespace detail

using namespace detail;

// solve_n_states_sbci1 (sbci1.hpp:526-579)
MultiStateResult solve_n_states_sbci1(Context& c, int n, const SolverConfig& cfg,
                                      const std::function<void(const TraceRec&)>& trace) {
    cfg.validate();
    if (n < 1) throw std::invalid_argument("solve_n_states_sbci1: n must be >= 1");
    const auto t0 = std::chrono::steady_clock::now();
    const uint64_t applies_before = c.applies().load();
    Ops o(c);
    Driver dr(c, cfg, trace);
    g_lin_ms = 0;
    g_lin_n = 0;
    for (double& v : g_ph) v = 0;
    auto tp = Clk::now();
    std::vector<Seed> guesses = init_guess(c, o, n);
    const double t_init = ms_since(tp);
    Precond pre{&c.diagonal(), guesses.front().energy, cfg.clamp_delta};
    if (!(pre.clamp > 0.0)) throw std::invalid_argument("clamp_delta must be positive");
    Deflation defl;
    MultiStateResult out;
    std::optional<Seed> carried;
    for (int alpha = 0; alpha < n; ++alpha) {
        std::vector<const Seed*> cands;
        if (carried) cands.push_back(&*carried);
        for (int b = alpha; b < (int)guesses.size(); ++b) cands.push_back(&guesses[b]);
        for (int b = 0; b < alpha && b < (int)guesses.size(); ++b) cands.push_back(&guesses[b]);
        tp = Clk::now();
        Seed seed = select_seed(c, o, cands, defl, cfg.lindep);
        g_ph[7] += ms_since(tp);
        carried.reset();
        Sbci1Result res = solve_state(dr, pre, defl, std::move(seed), alpha, alpha == 0);
        if (alpha == 0) pre.update_shift(res.pair.energy);
        out.total_iterations += res.pair.iterations;
        out.total_restarts += res.pair.restarts;
        out.hx_refreshes += res.hx_refreshes;
        // the deflation set keeps its own copy of the converged vector
        DBuf keep = o.clone(res.pair.vector);
        defl.add_with_image(o, std::move(keep), std::move(res.converged_image), res.pair.energy);
        out.pairs.push_back(std::move(res.pair));
        carried = std::move(res.next_seed);
    }
    std::stable_sort(out.pairs.begin(), out.pairs.end(),
                     [](const StateResult& a, const StateResult& b) { return a.energy < b.energy; });
    out.matvecs = c.applies().load() - applies_before;
    out.peak_vectors = 7 + (int)defl.size();
    SBG_CUDA(cudaStreamSynchronize(c.st));
    out.wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (std::getenv("SBG_SOLVER_TIMING"))
        std::fprintf(stderr,
                     "[sbg timing] wall %.3f ms init %.3f | make_z %.3f apply %.3f subspace %.3f jacobi %.3f "
                     "guard+commit %.3f trace %.3f restart %.3f select %.3f | lincomb calls %ld %.3f ms\n",
                     out.wall_time_s * 1e3, t_init, g_ph[0], g_ph[1], g_ph[2], g_ph[3], g_ph[4], g_ph[5], g_ph[6], g_ph[7], g_lin_n, g_lin_ms);
    return out;
}

}  // namespace sbg
