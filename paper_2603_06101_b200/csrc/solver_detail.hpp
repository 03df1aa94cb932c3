// solver_detail.hpp — device-vector plumbing shared by the SBCI1 (solver.cu) and SBCI2 (sbci2.cu)
// drivers: fused-pass builder, vector ops (vector_ops.hpp:27-79), GroundShiftPreconditioner and
// DeflationSet (precond.hpp:19-111), seeds (sbci1.hpp:45-92, 501-519). Internal to libsbg.
#pragma once

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <optional>
#include <stdexcept>
#include <vector>

#include "solver.hpp"

namespace sbg {
namespace detail {

constexpr int kSbci1DefaultMaxCycle = 20;
constexpr int kSbci2DefaultMaxCycle = 10;
// env-gated host phase timers (SBG_SOLVER_TIMING=1 prints them at solve end)
inline double g_lin_ms = 0, g_ph[8] = {0};
inline long g_lin_n = 0;
using Clk = std::chrono::steady_clock;
inline double ms_since(Clk::time_point t) { return std::chrono::duration<double, std::milli>(Clk::now() - t).count(); }

// ------------------------------------------------------------------ fused pass builder
struct Lin {
    LinArgs a{};
    Lin() {
        std::memset(&a, 0, sizeof(a));
        a.kdot = -1;
    }
    // sum_i s[slot]_i^2 (D_i - shift) as one more dot of the pass (the trace's kinetic scalar)
    int kinetic(int slot, const double* D, double shift) {
        const int d = dot(slot, slot);
        a.kdot = d;
        a.kD = D;
        a.kshift = shift;
        return d;
    }
    bool fits(int more_in) const { return a.nin + more_in <= kMaxIn; }
    int in(const double* p) {
        if (a.nin >= kMaxIn) throw std::invalid_argument("fused pass: too many inputs");
        a.in[a.nin] = p;
        return a.nin++;
    }
    // out = sum coef*slot, returns slot id of the output
    int out(double* p, std::initializer_list<std::pair<int, double>> terms) {
        if (a.nout >= kMaxOut) throw std::invalid_argument("fused pass: too many outputs");
        const int j = a.nout++;
        a.out[j] = p;
        for (auto& t : terms) a.coef[j][t.first] = t.second;
        return kMaxIn + j;
    }
    int dot(int s1, int s2) {
        if (a.ndot >= kMaxDot) throw std::invalid_argument("fused pass: too many dot products");
        a.da[a.ndot] = (unsigned char)s1;
        a.db[a.ndot] = (unsigned char)s2;
        return a.ndot++;
    }
    std::vector<double> run(Context& c) {
        a.n = c.padded_len();
        const auto t0 = std::chrono::steady_clock::now();
        launch_lincomb(a, c.rws, c.st);
        c.launches += 1;  // the dots are finished inside the pass
        std::vector<double> r(a.ndot);
        if (a.ndot > 0) {
            const double* h = c.finish_dots(a.ndot);
            std::copy(h, h + a.ndot, r.begin());
        }
        g_lin_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        g_lin_n++;
        return r;
    }
};

struct Seed {
    DBuf x, hx;
    double energy = 0.0;
};

class Ops {
public:
    explicit Ops(Context& c) : c_(c) {}
    Context& c_;

    double dot(const DBuf& u, const DBuf& v) {
        Lin L;
        const int a = L.in(u.p), b = L.in(v.p);
        L.dot(a, b);
        return L.run(c_)[0];
    }
    double norm(const DBuf& u) { return std::sqrt(dot(u, u)); }
    void scale(DBuf& u, double s) {  // u *= s (vector_ops.hpp:42-44)
        Lin L;
        const int a = L.in(u.p);
        L.out(u.p, {{a, s}});
        L.run(c_);
    }
    void scale2(DBuf& u, DBuf& v, double s) {
        Lin L;
        const int a = L.in(u.p), b = L.in(v.p);
        L.out(u.p, {{a, s}});
        L.out(v.p, {{b, s}});
        L.run(c_);
    }
    void copy(DBuf& dst, const DBuf& src) {
        SBG_CUDA(cudaMemcpyAsync(dst.p, src.p, c_.padded_len() * 8, cudaMemcpyDeviceToDevice, c_.st));
    }
    DBuf clone(const DBuf& src) {
        DBuf d = c_.vec();
        copy(d, src);
        return d;
    }
    void zero(DBuf& u) { SBG_CUDA(cudaMemsetAsync(u.p, 0, c_.padded_len() * 8, c_.st)); }
    // r = a*u + b*v (combine, vector_ops.hpp:53-58)
    void combine(DBuf& r, double a, const DBuf& u, double b, const DBuf& v) {
        Lin L;
        const int su = L.in(u.p), sv = L.in(v.p);
        L.out(r.p, {{su, a}, {sv, b}});
        L.run(c_);
    }
    void apply(const DBuf& x, DBuf& y) { c_.sigma(x, y); }
    // several sigma builds at once (Context::sigma_multi; batches of kMaxSigmaVec)
    void apply_multi(const std::vector<const DBuf*>& xs, const std::vector<DBuf*>& ys) {
        for (size_t v0 = 0; v0 < xs.size(); v0 += kMaxSigmaVec) {
            const double* xp[kMaxSigmaVec];
            double* yp[kMaxSigmaVec];
            const int n = (int)std::min<size_t>(kMaxSigmaVec, xs.size() - v0);
            for (int v = 0; v < n; ++v) {
                xp[v] = xs[v0 + v]->p;
                yp[v] = ys[v0 + v]->p;
            }
            c_.sigma_multi(xp, yp, n, c_.st);
        }
    }

    // global element read / unit vector (rank-aware)
    double read(const DBuf& v, int64_t gidx) {
        const int64_t row = gidx / c_.NB, col = gidx % c_.NB;
        double* r = c_.rws.result;
        if (row >= c_.row_lo && row < c_.row_hi)
            SBG_CUDA(cudaMemcpyAsync(r, v.p + (row - c_.row_lo) * c_.ld + col, 8, cudaMemcpyDeviceToDevice, c_.st));
        else
            SBG_CUDA(cudaMemsetAsync(r, 0, 8, c_.st));
        if (c_.rws.zc) c_.rws.zc->fresh = false;  // written by a copy, not by a pass
        return c_.finish_dots(1)[0];
    }
    void set_unit(DBuf& v, int64_t gidx) {
        zero(v);
        const int64_t row = gidx / c_.NB, col = gidx % c_.NB;
        if (row >= c_.row_lo && row < c_.row_hi) {
            launch_set_element(v.p, (row - c_.row_lo) * c_.ld + col, 1.0, c_.st);
            c_.launches++;
        }
    }
    // n smallest diagonal entries, ties by index (the stable_sort of sbci1.hpp:50-53)
    std::vector<int64_t> lowest_diagonal(int n) {
        const int grid = c_.rws.grid;
        double* pv;
        int64_t* pi;
        SBG_CUDA(cudaMalloc(&pv, grid * 8));
        SBG_CUDA(cudaMalloc(&pi, grid * 8));
        std::vector<double> hv(grid);
        std::vector<int64_t> hi(grid);
        std::vector<int64_t> out;
        double prev_v = -std::numeric_limits<double>::infinity();
        int64_t prev_i = -1;
        for (int k = 0; k < n; ++k) {
            launch_argmin_after(c_.diagonal().p, c_.nrows, c_.NB, c_.ld, c_.row_lo, prev_v, prev_i, nullptr, nullptr,
                                pv, pi, grid, c_.st);
            c_.launches++;
            SBG_CUDA(cudaMemcpyAsync(hv.data(), pv, grid * 8, cudaMemcpyDeviceToHost, c_.st));
            SBG_CUDA(cudaMemcpyAsync(hi.data(), pi, grid * 8, cudaMemcpyDeviceToHost, c_.st));
            SBG_CUDA(cudaStreamSynchronize(c_.st));
            double bv = std::numeric_limits<double>::max();
            int64_t bi = std::numeric_limits<int64_t>::max();
            for (int b = 0; b < grid; ++b)
                if (hv[b] < bv || (hv[b] == bv && hi[b] < bi)) {
                    bv = hv[b];
                    bi = hi[b];
                }
            if (c_.world > 1) {
                // all ranks' candidates: gather (value, index) through the dot buffer
                std::vector<double> all(2 * c_.world, 0.0);
                all[2 * c_.rank] = bv;
                all[2 * c_.rank + 1] = (double)bi;
                // sum-allreduce of a one-hot layout == allgather
                SBG_CUDA(cudaMemcpyAsync(c_.rws.result, all.data(), all.size() * 8, cudaMemcpyHostToDevice, c_.st));
                if (c_.rws.zc) c_.rws.zc->fresh = false;
                const double* h = c_.finish_dots((int)all.size());
                for (int r = 0; r < c_.world; ++r) {
                    const double v = h[2 * r];
                    const int64_t i = (int64_t)h[2 * r + 1];
                    if (v < bv || (v == bv && i < bi)) {
                        bv = v;
                        bi = i;
                    }
                }
            }
            out.push_back(bi);
            prev_v = bv;
            prev_i = bi;
        }
        cudaFree(pv);
        cudaFree(pi);
        return out;
    }
};

// ------------------------------------------------------------------ preconditioner & deflation
struct Precond {  // GroundShiftPreconditioner (precond.hpp:19-47)
    const DBuf* D;
    double shift, clamp;
    void update_shift(double e) {
        if (!std::isfinite(e)) throw std::invalid_argument("update_shift: E must be finite");
        shift = e;
    }
};

struct Deflation {  // DeflationSet (precond.hpp:54-102) with cached images
    struct Member {
        DBuf x, hx;
        double e;
    };
    std::vector<Member> m;
    std::vector<std::vector<double>> gram;  // gram[i][j] = x_i . x_j for j < i (|.| <= 1e-10 by add)
    bool empty() const { return m.empty(); }
    size_t size() const { return m.size(); }

    void add_with_image(Ops& o, DBuf x, DBuf hx, double e) {
        const double n = o.norm(x);
        if (std::abs(n - 1.0) > 1e-12) throw std::invalid_argument("DeflationSet::add: vector must be unit norm");
        std::vector<double> g;
        for (auto& mm : m) {
            const double d = o.dot(mm.x, x);
            if (std::abs(d) > 1e-10) throw std::invalid_argument("DeflationSet::add: vector not orthogonal to stored set");
            g.push_back(d);
        }
        m.push_back({std::move(x), std::move(hx), e});
        gram.push_back(std::move(g));
    }
    // The fused passes compute every overlap x_c . v from the unprojected v at once; the reference
    // projects member by member (project_out, precond.hpp:78-80: axpy(-dot(x_c, v), x_c, v)), so
    // member c sees v already stripped of members j < c. In exact arithmetic that overlap is
    // o'_c = x_c . v - sum_{j<c} o'_j (x_c . x_j): this turns the one-pass overlaps into the
    // sequential projection's, which then runs as v - sum_c o'_c x_c in one pass.
    std::vector<double> sequential(std::vector<double> o) const {
        for (size_t c = 1; c < o.size() && c < gram.size(); ++c)
            for (size_t j = 0; j < c; ++j) o[c] -= o[j] * gram[c][j];
        return o;
    }
    // v -= x_i (x_i . v), sequentially over members (precond.hpp:78-80)
    void project_out(Ops& o, DBuf& v) {
        for (auto& mm : m) {
            const double ov = o.dot(mm.x, v);
            Lin L;
            const int sv = L.in(v.p), sx = L.in(mm.x.p);
            L.out(v.p, {{sv, 1.0}, {sx, -ov}});
            L.run(o.c_);
        }
    }
    // precond.hpp:84-93
    void project_out_pair(Ops& o, DBuf& v, DBuf& hv) {
        for (auto& mm : m) {
            const double ov = o.dot(mm.x, v);
            Lin L;
            const int sv = L.in(v.p), sx = L.in(mm.x.p), sh = L.in(hv.p), shx = L.in(mm.hx.p);
            L.out(v.p, {{sv, 1.0}, {sx, -ov}});
            L.out(hv.p, {{sh, 1.0}, {shx, -ov}});
            L.run(o.c_);
        }
    }
};

// deflation overlaps x_c . v for every stored state (chunks of kMaxIn - 1 per pass)
inline std::vector<double> deflation_overlaps(Context& c, const Deflation& defl, const DBuf& v) {
    std::vector<double> out;
    for (size_t c0 = 0; c0 < defl.size(); c0 += kMaxIn - 1) {
        Lin L;
        const int sv = L.in(v.p);
        for (size_t i = c0; i < std::min(defl.size(), c0 + kMaxIn - 1); ++i) L.dot(L.in(defl.m[i].x.p), sv);
        const auto r = L.run(c);
        out.insert(out.end(), r.begin(), r.end());
    }
    return out;
}

constexpr int kMaxDeflated = 8;  // precondition() folds up to 8 deflated states into one pass

// z = (1 - sum x_c x_c^T)(D - E0)^-1 zres (precondition_and_deflate, precond.hpp:106-111) with the
// dots xx, xz, zz [, xy, yy, yz] of x (and y when given) against the new z
std::vector<double> precondition(Context& c, const DBuf& zres, const Precond& pre, const Deflation& defl, DBuf& z,
                                 const DBuf& x, const DBuf* y);
// the same without waiting: the dots are posted (Context::post_dots / wait_dots); returns their count
int precondition_post(Context& c, const DBuf& zres, const Precond& pre, const Deflation& defl, DBuf& z,
                      const DBuf& x, const DBuf* y);

struct Sbci1Result {
    StateResult pair;
    DBuf converged_image;
    std::optional<Seed> next_seed;
    int hx_refreshes = 0;
};

// init_guess_from_diagonal (sbci1.hpp:45-92)
std::vector<Seed> init_guess(Context& c, Ops& o, int n);
// select_seed (sbci1.hpp:501-519)
Seed select_seed(Context& c, Ops& o, std::vector<const Seed*> cands, Deflation& defl, double lindep);
// solve_state_sbci1 (sbci1.hpp:357-473)
Sbci1Result solve_state_sbci1(Context& c, const SolverConfig& cfg, const std::function<void(const TraceRec&)>& trace,
                              Precond& pre, Deflation& defl, Seed seed, int alpha, bool track);

}  // namespace detail
}  // namespace sbg
