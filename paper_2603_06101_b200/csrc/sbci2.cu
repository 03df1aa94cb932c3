// sbci2.cu — the SBCI2 pair driver on device-resident vectors (reference: sbci2.hpp:20-623).
// Scalar logic (coefficient formulas, guards, restart predicate, seed handling) follows the
// reference line by line on the host; every length-n_det operation is a fused pass:
//   precondition (x2)         precondition_and_deflate of z'_a, z'_b (+ |x_a|, |z_a| for the
//                             vanished-residual test)
//   sigma (x2)                H z_a, H z_b
//   gram                      all overlaps of the 4/6 stored vectors (norms + the overlap matrix of
//                             their unit-scaled copies, sbci2.hpp:141-158)
//   pair_subspace             the r x r cross dots of the materialized orthonormal basis and its
//                             images (sbci2.hpp:160-176)
//   guard                     |y'_a|, |y'_b|, |x'_a|, |x'_b|, |x_a|, |x_b| without writing
//   commit (2 passes)         y', x' in place; Hy', Hx', z'_a, z'_b(next) in place + |z'_a|^2
// Element arithmetic matches the reference's axpy/combine order (round(c*v) then add, input order).
#include "solver_detail.hpp"

#include <array>

namespace sbg {
namespace detail {

namespace {

struct PairCoefficients {  // sbci2.hpp:20-27
    double a_ab = 0.0, a_ba = 0.0;
    double b_aa = 1.0, b_ab = 0.0, b_ba = 0.0, b_bb = 1.0;
    double c_aa = 0.0, c_ab = 0.0, c_ba = 0.0, c_bb = 0.0;
    double k0 = 1.0, k1 = 1.0;
};

struct Sbci2State {  // sbci2.hpp:29-41
    int alpha = 0, t = 0;
    DBuf xa, hxa, xb, hxb, ya, hya, yb, hyb, zra, zrb;
    double ea = 0.0, eb = 0.0;
    PairCoefficients coeffs;
    int restart_count = 0;
    long total_iterations = 0;
};

// sbci2.hpp:45-56 (no alpha > 0 guard on the stall test, unlike the single-state rule)
std::optional<RestartReason> check_restart_sbci2(double b_aa, double b_bb, double dE, double xa_norm, double xb_norm,
                                                 double dz, int t, const SolverConfig& cfg, int max_cycle) {
    if ((std::abs(b_aa) < cfg.b_th || std::abs(b_bb) < cfg.b_th) && dE < cfg.eps1) return RestartReason::StallSmallB;
    if (xa_norm < cfg.x_th1 || xb_norm < cfg.x_th1 || xa_norm > cfg.x_th2 || xb_norm > cfg.x_th2)
        return RestartReason::NormOutOfRange;
    if (dz > cfg.r1 && t > 0) return RestartReason::ResidualBlowup;
    if (t + 1 >= max_cycle) return RestartReason::MaxCycle;
    return std::nullopt;
}

// u += a v (axpy, vector_ops.hpp:47-50) on device
void axpy(Context& c, double a, const DBuf& v, DBuf& u) {
    Lin L;
    const int su = L.in(u.p), sv = L.in(v.p);
    L.out(u.p, {{su, 1.0}, {sv, a}});
    L.run(c);
}

double rayleigh(Ops& o, const DBuf& x, const DBuf& hx) {  // operator.hpp:107-111
    Lin L;
    const int sx = L.in(x.p), sh = L.in(hx.p);
    L.dot(sx, sx);
    L.dot(sx, sh);
    const auto r = L.run(o.c_);
    if (r[0] == 0.0) throw std::invalid_argument("rayleigh_quotient: zero vector");
    return r[1] / r[0];
}

// init_pair (sbci2.hpp:63-103)
Sbci2State init_pair(Context& c, Ops& o, Deflation& defl, Seed lower, Seed upper, double lindep, int alpha) {
    defl.project_out_pair(o, lower.x, lower.hx);
    double nm = o.norm(lower.x);
    if (nm < lindep) throw std::invalid_argument("init_pair: lower seed collapsed under deflation");
    o.scale2(lower.x, lower.hx, 1.0 / nm);

    defl.project_out_pair(o, upper.x, upper.hx);
    const double ov = o.dot(lower.x, upper.x);
    axpy(c, -ov, lower.x, upper.x);
    axpy(c, -ov, lower.hx, upper.hx);
    nm = o.norm(upper.x);
    if (nm < lindep) throw std::invalid_argument("init_pair: upper seed collapsed against the lower one");
    o.scale2(upper.x, upper.hx, 1.0 / nm);

    Sbci2State st;
    st.alpha = alpha;
    st.ea = o.dot(lower.x, lower.hx);
    st.eb = o.dot(upper.x, upper.hx);
    st.xa = std::move(lower.x);
    st.hxa = std::move(lower.hx);
    st.xb = std::move(upper.x);
    st.hxb = std::move(upper.hx);
    st.ya = c.vec();
    st.hya = c.vec();
    st.yb = c.vec();
    st.hyb = c.vec();
    st.zra = c.vec();
    st.zrb = c.vec();
    o.combine(st.zra, 1.0, st.hxa, -st.ea, st.xa);
    o.combine(st.zrb, 1.0, st.hxb, -st.eb, st.xb);
    return st;
}

// pair_subspace_solve (sbci2.hpp:131-181) over device vectors
struct SubspaceSolve {
    bool ok = false;
    int rank = 0;
    std::vector<double> eigenvalues;
    std::vector<std::vector<double>> vprime;  // vprime[i][col]
};

SubspaceSolve pair_subspace_solve(Context& c, const std::vector<const DBuf*>& vecs,
                                  const std::vector<const DBuf*>& images, double lindep) {
    const int m = (int)vecs.size();
    std::vector<const double*> vp(m);
    for (int i = 0; i < m; ++i) vp[i] = vecs[i]->p;
    launch_gram(vp.data(), m, c.padded_len(), c.rws, c.st);
    c.launches += 1;
    const double* h = c.finish_dots(m * (m + 1) / 2);
    SmallMatrix raw(m);
    for (int i = 0, d = 0; i < m; ++i)
        for (int j = i; j < m; ++j, ++d) raw(i, j) = raw(j, i) = h[d];
    std::vector<double> norms(m, 0.0);
    for (int i = 0; i < m; ++i) {
        const double nm = std::sqrt(raw(i, i));
        norms[i] = nm <= lindep ? 0.0 : nm;  // zero vectors stay zero (sbci2.hpp:144-149)
    }
    // overlaps of the unit-scaled copies w_i = v_i / |v_i|
    SmallMatrix s(m);
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j)
            s(i, j) = (norms[i] == 0.0 || norms[j] == 0.0) ? 0.0 : raw(i, j) / (norms[i] * norms[j]);
    SubspaceSolve out;
    OrthoTransform trans;
    try {
        trans = canonical_orthogonalize_overlap(s, 1e-14);
    } catch (const std::runtime_error&) {
        return out;  // empty basis
    }
    if (trans.rank < 2) return out;

    PairSubArgs pa{};
    pa.n = c.padded_len();
    pa.m = m;
    pa.r = trans.rank;
    for (int i = 0; i < m; ++i) {
        pa.v[i] = vecs[i]->p;
        pa.h[i] = images[i]->p;
        pa.inv_n[i] = norms[i] == 0.0 ? 0.0 : 1.0 / norms[i];
        for (int col = 0; col < trans.rank; ++col) pa.P[i][col] = trans.coeff(i, col);
    }
    launch_pair_subspace(pa, c.rws, c.st);
    c.launches += 1;
    const int r = trans.rank;
    const double* x = c.finish_dots(r * r);
    SmallMatrix g(r);
    for (int i = 0; i < r; ++i)
        for (int j = i; j < r; ++j) g(i, j) = g(j, i) = 0.5 * (x[i * r + j] + x[j * r + i]);
    const SmallEigResult eig = jacobi_symmetric_eig(g);

    out.ok = true;
    out.rank = r;
    out.eigenvalues = eig.eigenvalues;
    out.vprime.assign(m, std::vector<double>(r, 0.0));
    for (int i = 0; i < m; ++i) {
        if (norms[i] == 0.0) continue;
        for (int col = 0; col < r; ++col) {
            double acc = 0.0;
            for (int mm = 0; mm < r; ++mm) acc += trans.coeff(i, mm) * eig.eigenvectors(mm, col);
            out.vprime[i][col] = acc / norms[i];
        }
    }
    return out;
}

struct Sbci2StepData {
    StepOutcome outcome;
    double dE = 0.0, dz = 0.0;
    bool committed = false;
    double xa_norm = 0.0, xb_norm = 0.0, zrb_norm = 0.0;  // valid when committed
    bool have_kinetic = false;  // kinetic scalar of the committed y'_a (traced solves, fused in the commit pass)
    double kinetic = 0.0;
};

class PairDriver {
public:
    PairDriver(Context& c, const SolverConfig& cfg)
        : c_(c), o_(c), cfg_(cfg), za_(c.vec()), zb_(c.vec()), hza_(c.vec()), hzb_(c.vec()), zrb_next_(c.vec()) {}

    // sbci2_step_impl (sbci2.hpp:186-333)
    Sbci2StepData step(Sbci2State& st, const Precond& pre, const Deflation& defl, int max_cycle) {
        Sbci2StepData out;
        const auto da = precondition(c_, st.zra, pre, defl, za_, st.xa, nullptr);
        precondition_post(c_, st.zrb, pre, defl, zb_, st.xb, nullptr);  // z_b's dots are not used: no wait
        if (std::sqrt(da[2]) < cfg_.lindep * std::sqrt(da[0])) {
            st.ea = rayleigh(o_, st.xa, st.hxa);
            out.outcome = StepOutcome::converged();
            out.dz = o_.norm(st.zra);
            return out;
        }
        o_.apply_multi({&za_, &zb_}, {&hza_, &hzb_});  // the pair's two sigma builds in one pass (sbci2.hpp:209-210)

        const bool first = st.t == 0;
        SubspaceSolve sub;
        if (first)
            sub = pair_subspace_solve(c_, {&st.xa, &st.xb, &za_, &zb_}, {&st.hxa, &st.hxb, &hza_, &hzb_}, cfg_.lindep);
        else
            sub = pair_subspace_solve(c_, {&st.xa, &st.xb, &st.ya, &st.yb, &za_, &zb_},
                                      {&st.hxa, &st.hxb, &st.hya, &st.hyb, &hza_, &hzb_}, cfg_.lindep);
        if (!sub.ok) {
            out.outcome = StepOutcome::restart(RestartReason::StallSmallB);
            return out;
        }
        const auto& vp = sub.vprime;
        PairCoefficients co;
        constexpr double tiny = 1e-14;
        if (first) {  // x rows 0/1, z rows 2/3
            if (std::abs(vp[0][0]) < tiny || std::abs(vp[1][1]) < tiny) {
                out.outcome = StepOutcome::restart(RestartReason::StallSmallB);
                return out;
            }
            co.k0 = 1.0 / vp[0][0];
            co.a_ab = vp[1][0] / vp[0][0];
            co.c_aa = -vp[2][0] / vp[0][0];
            co.c_ab = -vp[3][0] / vp[0][0];
            co.k1 = 1.0 / vp[1][1];
            co.a_ba = vp[0][1] / vp[1][1];
            co.c_ba = -vp[2][1] / vp[1][1];
            co.c_bb = -vp[3][1] / vp[1][1];
            co.b_aa = co.b_bb = 1.0;
            co.b_ab = co.b_ba = 0.0;
        } else {  // x rows 0/1, y rows 2/3, z rows 4/5
            if (std::abs(vp[2][0]) < tiny || std::abs(vp[3][1]) < tiny) {
                out.outcome = StepOutcome::restart(RestartReason::StallSmallB);
                return out;
            }
            co.a_ab = vp[1][0] / vp[2][0];
            co.a_ba = vp[0][1] / vp[3][1];
            const double k0_den = vp[0][0] - vp[3][0] * co.a_ba;
            const double k1_den = vp[1][1] - vp[2][1] * co.a_ab;
            if (std::abs(k0_den) < tiny || std::abs(k1_den) < tiny) {
                out.outcome = StepOutcome::restart(RestartReason::StallSmallB);
                return out;
            }
            co.k0 = 1.0 / k0_den;
            co.k1 = 1.0 / k1_den;
            co.b_aa = co.k0 * vp[2][0];
            co.b_ab = co.k0 * vp[3][0];
            co.b_ba = co.k1 * vp[2][1];
            co.b_bb = co.k1 * vp[3][1];
            const double m00 = vp[2][0], m01 = vp[3][0], m10 = vp[2][1], m11 = vp[3][1];
            const double det = m00 * m11 - m01 * m10;
            const double scale_sq = std::sqrt((m00 * m00 + m01 * m01) * (m10 * m10 + m11 * m11));
            if (std::abs(det) < tiny * std::max(scale_sq, 1e-30)) {
                out.outcome = StepOutcome::restart(RestartReason::StallSmallB);
                return out;
            }
            const double r00 = vp[4][0], r01 = vp[5][0], r10 = vp[4][1], r11 = vp[5][1];
            co.c_aa = -(m11 * r00 - m01 * r10) / det;
            co.c_ab = -(m11 * r01 - m01 * r11) / det;
            co.c_ba = -(-m10 * r00 + m00 * r10) / det;
            co.c_bb = -(-m10 * r01 + m00 * r11) / det;
        }
        const double e_new_a = sub.eigenvalues[0];
        const double e_new_b = sub.eigenvalues[1];

        // y'_a = y_a - c_aa z_a - c_ab z_b + a_ab x_b ; y'_b = y_b - c_ba z_a - c_bb z_b + a_ba x_a ;
        // x'_a = x_a + b_aa y'_a + b_ab y'_b ; x'_b = x_b + b_ba y'_a + b_bb y'_b   (sbci2.hpp:265-297)
        // guard + commit in one pass: y', x' of both states go into spare buffers with the six norms
        // the cancellation guard (sbci2.hpp:299-306) needs; the spares are swapped in only if it
        // passes, so a rejected step leaves the state untouched as in the reference
        {
            // with the four spares: guard + commit in one pass; without room for them (or with
            // SBG_GUARD_TWO_PASS=1): a read-only pass for the norms, then the commit in place
            const bool merged = spares();
            Lin L;
            const int sya = L.in(st.ya.p), syb = L.in(st.yb.p), sza = L.in(za_.p), szb = L.in(zb_.p),
                      sxa = L.in(st.xa.p), sxb = L.in(st.xb.p);
            const int ya = L.out(merged ? sp_ya_.p : nullptr, {{sya, 1.0}, {sza, -co.c_aa}, {szb, -co.c_ab}, {sxb, co.a_ab}});
            const int yb = L.out(merged ? sp_yb_.p : nullptr, {{syb, 1.0}, {sza, -co.c_ba}, {szb, -co.c_bb}, {sxa, co.a_ba}});
            const int xa = L.out(merged ? sp_xa_.p : nullptr, {{sxa, 1.0}, {ya, co.b_aa}, {yb, co.b_ab}});
            const int xb = L.out(merged ? sp_xb_.p : nullptr, {{sxb, 1.0}, {ya, co.b_ba}, {yb, co.b_bb}});
            for (int k : {ya, yb, xa, xb, sxa, sxb}) L.dot(k, k);
            if (want_kinetic) L.kinetic(ya, pre.D->p, pre.shift);
            const auto r = L.run(c_);
            if (want_kinetic) {
                out.have_kinetic = true;
                out.kinetic = r[6];
            }
            const double ya_nm = std::sqrt(r[0]), yb_nm = std::sqrt(r[1]);
            const double ingredients_a = std::sqrt(r[4]) + std::abs(co.b_aa) * ya_nm + std::abs(co.b_ab) * yb_nm;
            const double ingredients_b = std::sqrt(r[5]) + std::abs(co.b_ba) * ya_nm + std::abs(co.b_bb) * yb_nm;
            if (ingredients_a > 1e6 * std::max(std::sqrt(r[2]), 1e-300) ||
                ingredients_b > 1e6 * std::max(std::sqrt(r[3]), 1e-300)) {
                out.outcome = StepOutcome::restart(RestartReason::StallSmallB);
                return out;
            }
            if (merged) {
                std::swap(st.ya, sp_ya_);
                std::swap(st.yb, sp_yb_);
                std::swap(st.xa, sp_xa_);
                std::swap(st.xb, sp_xb_);
            } else {
                Lin W;
                const int wya = W.in(st.ya.p), wyb = W.in(st.yb.p), wza = W.in(za_.p), wzb = W.in(zb_.p),
                          wxa = W.in(st.xa.p), wxb = W.in(st.xb.p);
                const int ya2 = W.out(st.ya.p, {{wya, 1.0}, {wza, -co.c_aa}, {wzb, -co.c_ab}, {wxb, co.a_ab}});
                const int yb2 = W.out(st.yb.p, {{wyb, 1.0}, {wza, -co.c_ba}, {wzb, -co.c_bb}, {wxa, co.a_ba}});
                W.out(st.xa.p, {{wxa, 1.0}, {ya2, co.b_aa}, {yb2, co.b_ab}});
                W.out(st.xb.p, {{wxb, 1.0}, {ya2, co.b_ba}, {yb2, co.b_bb}});
                W.run(c_);
            }
            out.xa_norm = std::sqrt(r[2]);
            out.xb_norm = std::sqrt(r[3]);
        }
        double zz;
        std::vector<double> ovl;
        {  // images, then z'_a = (Hx'_a - E'_a x'_a)/k0 and z'_b likewise (sbci2.hpp:317, 329)
            Lin L;
            const int sya = L.in(st.hya.p), syb = L.in(st.hyb.p), sza = L.in(hza_.p), szb = L.in(hzb_.p),
                      sxa = L.in(st.hxa.p), sxb = L.in(st.hxb.p), xa = L.in(st.xa.p), xb = L.in(st.xb.p);
            std::vector<int> sxc;
            const bool fused_ovl = L.fits((int)defl.size());
            if (fused_ovl)
                for (auto& mm : defl.m) sxc.push_back(L.in(mm.x.p));
            const int ya = L.out(st.hya.p, {{sya, 1.0}, {sza, -co.c_aa}, {szb, -co.c_ab}, {sxb, co.a_ab}});
            const int yb = L.out(st.hyb.p, {{syb, 1.0}, {sza, -co.c_ba}, {szb, -co.c_bb}, {sxa, co.a_ba}});
            const int ha = L.out(st.hxa.p, {{sxa, 1.0}, {ya, co.b_aa}, {yb, co.b_ab}});
            const int hb = L.out(st.hxb.p, {{sxb, 1.0}, {ya, co.b_ba}, {yb, co.b_bb}});
            const int za = L.out(st.zra.p, {{ha, 1.0 / co.k0}, {xa, -e_new_a / co.k0}});
            const int zb = L.out(zrb_next_.p, {{hb, 1.0 / co.k1}, {xb, -e_new_b / co.k1}});
            L.dot(za, za);
            L.dot(zb, zb);
            for (int sc : sxc) L.dot(sc, za);
            const auto r = L.run(c_);
            zz = r[0];
            out.zrb_norm = std::sqrt(r[1]);
            ovl.assign(r.begin() + 2, r.end());
            if (!fused_ovl) ovl = deflation_overlaps(c_, defl, st.zra);
            ovl = defl.sequential(std::move(ovl));
        }
        out.committed = true;
        st.coeffs = co;
        out.dE = std::abs(e_new_a - st.ea);
        out.dz = std::sqrt(zz);
        double dz_defl = out.dz;
        if (!defl.empty()) {  // |(1 - sum x_c x_c^T) z'_a| (sbci2.hpp:323-327)
            Lin L;
            const int sz = L.in(st.zra.p);
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
        if (out.dE < cfg_.eps0 && std::min(out.dz, dz_defl) < cfg_.r0) {
            st.ea = e_new_a;
            st.eb = e_new_b;
            out.outcome = StepOutcome::converged();
            return out;  // z'_b keeps its previous value, as in the reference
        }
        std::swap(st.zrb, zrb_next_);
        st.ea = e_new_a;
        st.eb = e_new_b;
        if (auto reason = check_restart_sbci2(co.b_aa, co.b_bb, out.dE, out.xa_norm, out.xb_norm, out.dz, st.t, cfg_,
                                              max_cycle)) {
            out.outcome = StepOutcome::restart(*reason);
            return out;
        }
        out.outcome = StepOutcome::cont();
        return out;
    }

    Context& c_;
    Ops o_;
    SolverConfig cfg_;
    DBuf za_, zb_, hza_, hzb_, zrb_next_;
    DBuf sp_ya_, sp_yb_, sp_xa_, sp_xb_;  // candidate y', x' of the merged guard + commit pass
    bool want_kinetic = false;            // traced solve: the commit pass also forms y'_a^T (D - E0) y'_a
    bool two_pass_ = std::getenv("SBG_GUARD_TWO_PASS") && std::atoi(std::getenv("SBG_GUARD_TWO_PASS")) != 0;
    bool spares() {
        if (two_pass_) return false;
        if (!sp_ya_.empty()) return true;
        try {
            sp_ya_ = c_.vec();
            sp_yb_ = c_.vec();
            sp_xa_ = c_.vec();
            sp_xb_ = c_.vec();
            return true;
        } catch (const DeviceError&) {
            cudaGetLastError();
            for (DBuf* b : {&sp_ya_, &sp_yb_, &sp_xa_, &sp_xb_}) *b = DBuf();
            two_pass_ = true;
            return false;
        }
    }
};

struct Sbci2PairResult {
    StateResult pair;
    DBuf converged_image;
    Seed carry;
    int hx_refreshes = 0;
};

// solve_pair (sbci2.hpp:388-513)
Sbci2PairResult solve_pair(PairDriver& dr, Precond& pre, Deflation& defl, Seed lower, Seed upper, int alpha,
                           const std::function<void(const TraceRec&)>& trace, bool track) {
    Context& c = dr.c_;
    Ops& o = dr.o_;
    const SolverConfig& cfg = dr.cfg_;
    cfg.validate();
    const int max_cycle = cfg.effective_max_cycle(kSbci2DefaultMaxCycle);
    Sbci2State st = init_pair(c, o, defl, std::move(lower), std::move(upper), cfg.lindep, alpha);
    if (track) pre.update_shift(st.ea);
    dr.want_kinetic = (bool)trace;
    Sbci2PairResult result;
    {  // lower seed already converged: no update step, the upper seed carries over untouched
        const auto d = precondition(c, st.zra, pre, defl, dr.za_, st.xa, nullptr);
        if (std::sqrt(d[2]) < cfg.lindep) {
            result.pair.state = alpha;
            result.pair.energy = st.ea;
            result.pair.final_residual = o.norm(st.zra);
            result.pair.vector = std::move(st.xa);
            result.converged_image = std::move(st.hxa);
            result.carry.x = std::move(st.xb);
            result.carry.hx = std::move(st.hxb);
            result.carry.energy = st.eb;
            return result;
        }
    }
    while (st.total_iterations < cfg.t_max) {
        Sbci2StepData step = dr.step(st, pre, defl, max_cycle);
        ++st.total_iterations;
        if (trace) {  // sbci2.hpp:419-446
            TraceRec rec;
            rec.method = 2;
            rec.state = alpha;
            rec.pair_partner = alpha + 1;
            rec.t = st.t;
            rec.energy = st.ea;
            rec.dE = step.dE;
            rec.res_norm = step.dz;
            rec.x_norm = step.committed ? step.xa_norm : o.norm(st.xa);
            if (step.committed && step.have_kinetic) {
                rec.kinetic = step.kinetic;
            } else {
                launch_kinetic(st.ya.p, pre.D->p, pre.shift, c.padded_len(), c.rws, c.st);
                c.launches += 1;
                rec.kinetic = c.finish_dots(1)[0];
            }
            rec.matvecs = c.applies().load();
            rec.b = st.coeffs.b_aa;
            rec.c = st.coeffs.c_aa;
            rec.b_ab = st.coeffs.b_ab;
            rec.b_ba = st.coeffs.b_ba;
            rec.b_bb = st.coeffs.b_bb;
            rec.c_ab = st.coeffs.c_ab;
            rec.c_ba = st.coeffs.c_ba;
            rec.c_bb = st.coeffs.c_bb;
            rec.a_ab = st.coeffs.a_ab;
            rec.a_ba = st.coeffs.a_ba;
            rec.energy_partner = st.eb;
            rec.x_norm_partner = step.committed ? step.xb_norm : o.norm(st.xb);
            rec.res_norm_partner = o.norm(st.zrb);
            rec.restart_reason = step.outcome.kind == StepOutcome::Kind::Restart ? (int)step.outcome.reason : -1;
            trace(rec);
        }
        if (track) pre.update_shift(st.ea);
        switch (step.outcome.kind) {
            case StepOutcome::Kind::Converged: {
                StateResult pair;
                pair.state = alpha;
                pair.energy = rayleigh(o, st.xa, st.hxa);
                const double na = o.norm(st.xa);
                pair.vector = std::move(st.xa);
                if (na > 0.0) o.scale(pair.vector, 1.0 / na);
                for (auto& mm : defl.m)
                    if (std::abs(o.dot(mm.x, pair.vector)) > 1e-9) throw NonConvergenceError(alpha, pair.energy, step.dz);
                pair.iterations = (int)st.total_iterations;
                pair.restarts = st.restart_count;
                pair.final_residual = step.dz;
                result.pair = std::move(pair);
                o.scale(st.hxa, na > 0.0 ? 1.0 / na : 1.0);
                result.converged_image = std::move(st.hxa);
                const double nb = o.norm(st.xb);
                if (nb < cfg.lindep) throw NonConvergenceError(alpha + 1, st.eb, o.norm(st.zrb));
                o.scale2(st.xb, st.hxb, 1.0 / nb);
                result.carry.x = std::move(st.xb);
                result.carry.hx = std::move(st.hxb);
                result.carry.energy = rayleigh(o, result.carry.x, result.carry.hx);
                return result;
            }
            case StepOutcome::Kind::Restart: {  // sbci2.hpp:466-503
                double na = o.norm(st.xa), nb = o.norm(st.xb);
                if (na < cfg.lindep || nb < cfg.lindep) throw NonConvergenceError(alpha, st.ea, step.dz);
                o.scale2(st.xa, st.hxa, 1.0 / na);
                o.scale2(st.xb, st.hxb, 1.0 / nb);
                if (!defl.empty()) {
                    defl.project_out_pair(o, st.xa, st.hxa);
                    defl.project_out_pair(o, st.xb, st.hxb);
                    na = o.norm(st.xa);
                    nb = o.norm(st.xb);
                    if (na < cfg.lindep || nb < cfg.lindep) throw NonConvergenceError(alpha, st.ea, step.dz);
                    o.scale2(st.xa, st.hxa, 1.0 / na);
                    o.scale2(st.xb, st.hxb, 1.0 / nb);
                    st.ea = o.dot(st.xa, st.hxa);
                    st.eb = o.dot(st.xb, st.hxb);
                }
                o.zero(st.ya);
                o.zero(st.hya);
                o.zero(st.yb);
                o.zero(st.hyb);
                ++st.restart_count;
                if (cfg.hx_refresh_restarts > 0 && st.restart_count % cfg.hx_refresh_restarts == 0) {
                    o.apply_multi({&st.xa, &st.xb}, {&st.hxa, &st.hxb});
                    result.hx_refreshes += 2;
                }
                o.combine(st.zra, 1.0, st.hxa, -st.ea, st.xa);
                o.combine(st.zrb, 1.0, st.hxb, -st.eb, st.xb);
                st.coeffs = PairCoefficients{};
                st.t = 0;
                break;
            }
            case StepOutcome::Kind::Continue:
                ++st.t;
                break;
        }
    }
    throw NonConvergenceError(alpha, st.ea, o.norm(st.zra));
}

}  // namespace
}  // namespace detail

using namespace detail;

// solve_n_states_sbci2 (sbci2.hpp:527-623)
MultiStateResult solve_n_states_sbci2(Context& c, int n, const SolverConfig& cfg,
                                      const std::function<void(const TraceRec&)>& trace) {
    cfg.validate();
    if (n < 1) throw std::invalid_argument("solve_n_states_sbci2: n must be >= 1");
    if (n == 1) return solve_n_states_sbci1(c, 1, cfg, trace);
    const auto t0 = std::chrono::steady_clock::now();
    const uint64_t applies_before = c.applies().load();
    Ops o(c);
    std::vector<Seed> guesses = init_guess(c, o, n);
    Precond pre{&c.diagonal(), guesses.front().energy, cfg.clamp_delta};
    if (!(pre.clamp > 0.0)) throw std::invalid_argument("clamp_delta must be positive");
    Deflation defl;
    MultiStateResult out;
    std::optional<PairDriver> pdr;
    pdr.emplace(c, cfg);
    PairDriver& dr = *pdr;

    Seed lower;
    lower.x = o.clone(guesses.front().x);
    lower.hx = o.clone(guesses.front().hx);
    lower.energy = guesses.front().energy;
    for (int alpha = 0; alpha + 1 < n; ++alpha) {
        // the lower seed against the converged set
        defl.project_out_pair(o, lower.x, lower.hx);
        double nm = o.norm(lower.x);
        if (nm < std::max(cfg.lindep, 1e-8)) throw std::runtime_error("sbci2: carried seed collapsed under deflation");
        o.scale2(lower.x, lower.hx, 1.0 / nm);
        lower.energy = o.dot(lower.x, lower.hx);
        // upper seed: rotated guesses projected against the converged set and the lower seed;
        // the lowest surviving Rayleigh quotient wins
        std::optional<Seed> upper;
        for (int off = 0; off < (int)guesses.size(); ++off) {
            const int idx = (alpha + 1 + off) % (int)guesses.size();
            Seed cand;
            cand.x = o.clone(guesses[idx].x);
            cand.hx = o.clone(guesses[idx].hx);
            defl.project_out_pair(o, cand.x, cand.hx);
            const double ov = o.dot(lower.x, cand.x);
            axpy(c, -ov, lower.x, cand.x);
            axpy(c, -ov, lower.hx, cand.hx);
            const double cn = o.norm(cand.x);
            if (cn < std::max(cfg.lindep, 1e-8)) continue;
            o.scale2(cand.x, cand.hx, 1.0 / cn);
            cand.energy = o.dot(cand.x, cand.hx);
            if (!upper || cand.energy < upper->energy) upper = std::move(cand);
        }
        if (!upper) throw std::runtime_error("sbci2: no usable upper seed remained");
        Sbci2PairResult res = solve_pair(dr, pre, defl, std::move(lower), std::move(*upper), alpha, trace, alpha == 0);
        if (alpha == 0) pre.update_shift(res.pair.energy);
        out.total_iterations += res.pair.iterations;
        out.total_restarts += res.pair.restarts;
        out.hx_refreshes += res.hx_refreshes;
        DBuf keep = o.clone(res.pair.vector);
        defl.add_with_image(o, std::move(keep), std::move(res.converged_image), res.pair.energy);
        out.pairs.push_back(std::move(res.pair));
        lower = std::move(res.carry);
    }
    // highest state: the single-state procedure. The pair driver's buffers and the rotated guesses
    // go back to the pool first, so the SBCI1 driver reuses them instead of adding its own
    pdr.reset();
    guesses.clear();
    Sbci1Result last = solve_state_sbci1(c, cfg, trace, pre, defl, std::move(lower), n - 1, false);
    out.total_iterations += last.pair.iterations;
    out.total_restarts += last.pair.restarts;
    out.hx_refreshes += last.hx_refreshes;
    {
        DBuf keep = o.clone(last.pair.vector);
        defl.add_with_image(o, std::move(keep), std::move(last.converged_image), last.pair.energy);
    }
    out.pairs.push_back(std::move(last.pair));
    std::stable_sort(out.pairs.begin(), out.pairs.end(),
                     [](const StateResult& a, const StateResult& b) { return a.energy < b.energy; });
    out.matvecs = c.applies().load() - applies_before;
    out.peak_vectors = 14 + (int)defl.size();
    SBG_CUDA(cudaStreamSynchronize(c.st));
    out.wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return out;
}

}  // namespace sbg
