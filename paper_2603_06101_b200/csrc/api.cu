// api.cu — the extern "C" boundary (include/sbg.h). Translates C++ exceptions into the
// reference's error classes' codes and keeps a thread-local message (sbg_last_error).
#include <nccl.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <random>
#include <string>

#include "../../include/sbg.h"
#include "context.hpp"
#include "solver.hpp"
#include "solver_detail.hpp"

// One operator handle. The reference's apply is const and callable from several threads at once
// (operator.hpp:14-18, 47; test_operator.cpp:49-64): every entry point that touches the context's
// streams, staging slots, scratch or profile ring holds `mu`, and Context chains its sigma builds on
// the device (ev_order_), so concurrent callers are serialised host-side and device-side while
// apply_count stays an atomic counter.
struct sbg_ctx {
    std::unique_ptr<sbg::Context> c;
    std::mutex mu;
};

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return SBG_OK;
    } catch (const sbg::NonConvergenceError& e) {
        g_err = e.what();
        return SBG_ENONCONV;
    } catch (const sbg::DeviceError& e) {
        g_err = e.what();
        return SBG_EDEVICE;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SBG_EINVAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SBG_ERUNTIME;
    }
}

uint64_t binomial_u64(int n, int k) {  // determinants.hpp:17-31
    if (k < 0 || k > n) return 0;
    k = std::min(k, n - k);
    uint64_t r = 1;
    for (int i = 1; i <= k; ++i) {
        const uint64_t num = (uint64_t)(n - k + i);
        const uint64_t g = std::gcd(r, (uint64_t)i);
        r = (r / g) * num / ((uint64_t)i / g);
    }
    return r;
}

sbg::SolverConfig to_cfg(const sbg_config* c) {
    sbg::SolverConfig s;
    if (!c) return s;
    s.eps0 = c->eps0;
    s.r0 = c->r0;
    s.b_th = c->b_th;
    s.eps1 = c->eps1;
    s.x_th1 = c->x_th1;
    s.x_th2 = c->x_th2;
    s.r1 = c->r1;
    s.max_cycle = c->max_cycle;
    s.t_max = (long)c->t_max;
    s.lindep = c->lindep;
    s.clamp_delta = c->clamp_delta;
    s.hx_refresh_restarts = c->hx_refresh_restarts;
    return s;
}

// every context entry point runs on the context's device (the calling thread may be a different
// one than the creating thread, e.g. the ranks of a local group)
void require_ctx(const sbg_ctx* ctx) {
    if (!ctx || !ctx->c) throw std::invalid_argument("null sbg_ctx");
    SBG_CUDA(cudaSetDevice(ctx->c->device));
}
// the same, holding the context's lock for the rest of the call
[[nodiscard]] std::unique_lock<std::mutex> lock_ctx(sbg_ctx* ctx) {
    if (!ctx || !ctx->c) throw std::invalid_argument("null sbg_ctx");
    std::unique_lock<std::mutex> lk(ctx->mu);
    SBG_CUDA(cudaSetDevice(ctx->c->device));
    return lk;
}

// sbg::TraceRec -> sbg_trace_record callback (empty when trace is NULL)
std::function<void(const sbg::TraceRec&)> make_trace(sbg_trace_fn trace, void* trace_user) {
    if (!trace) return {};
    return [trace, trace_user](const sbg::TraceRec& r) {
        sbg_trace_record rec{};
        rec.state = r.state;
        rec.t = r.t;
        rec.energy = r.energy;
        rec.dE = r.dE;
        rec.res_norm = r.res_norm;
        rec.x_norm = r.x_norm;
        rec.kinetic = r.kinetic;
        rec.matvecs = r.matvecs;
        rec.restart_reason = r.restart_reason;
        rec.b = r.b;
        rec.c = r.c;
        rec.method = r.method;
        rec.pair_partner = r.pair_partner;
        rec.b_ab = r.b_ab;
        rec.b_ba = r.b_ba;
        rec.b_bb = r.b_bb;
        rec.c_ab = r.c_ab;
        rec.c_ba = r.c_ba;
        rec.c_bb = r.c_bb;
        rec.a_ab = r.a_ab;
        rec.a_ba = r.a_ba;
        rec.energy_partner = r.energy_partner;
        rec.x_norm_partner = r.x_norm_partner;
        rec.res_norm_partner = r.res_norm_partner;
        trace(&rec, trace_user);
    };
}
}  // namespace

namespace sbg {
void shard_range(int64_t n, int rank, int world, int64_t* lo, int64_t* hi);
}

extern "C" {

const char* sbg_last_error(void) { return g_err.c_str(); }
const char* sbg_version(void) { return "sbg 0.1 (sm_100a)"; }
uint64_t sbg_binomial(int n, int k) { return binomial_u64(n, k); }

int sbg_determinant_count(int norb, int n_alpha, int n_beta, uint64_t* out) {
    return guarded([&] {
        if (norb < 0 || norb > 64) throw std::invalid_argument("determinant_count: norb out of range");
        if (n_alpha < 0 || n_beta < 0 || n_alpha > norb || n_beta > norb)
            throw std::invalid_argument("determinant_count: electron count out of range");
        *out = binomial_u64(norb, n_alpha) * binomial_u64(norb, n_beta);
    });
}

int sbg_ab_plan_info(int norb, int n_alpha, int n_beta, int64_t* out) {
    return guarded([&] {
        if (norb < 1 || norb > sbg::kMaxOrb || n_alpha < 0 || n_beta < 0 || n_alpha > norb || n_beta > norb)
            throw std::invalid_argument("ab_plan_info: sector out of range");
        if (n_alpha == 0 || n_beta == 0) throw std::invalid_argument("ab_plan_info: no opposite-spin term");
        const int64_t NA = (int64_t)binomial_u64(norb, n_alpha), NB = (int64_t)binomial_u64(norb, n_beta);
        const int64_t ld = sbg::round_up(NB, 32);
        const sbg::AbPlan pl = sbg::plan_sigma_ab(norb, n_alpha, n_beta, NA, NB, ld, 148);
        const int64_t v[16] = {pl.KS, pl.nt, pl.mb16, pl.extra, pl.k0e, pl.tall, pl.xs, pl.dc, pl.tma, pl.npass,
                               (int64_t)pl.smem, pl.grows ? pl.grows : pl.npad, pl.gstride ? pl.gstride : pl.nt + 8,
                               pl.maxE, pl.threads, pl.red};
        for (int i = 0; i < 16; ++i) out[i] = v[i];
    });
}

sbg_config sbg_config_default(void) {
    sbg::SolverConfig s;
    sbg_config c{};
    c.eps0 = s.eps0;
    c.r0 = s.r0;
    c.b_th = s.b_th;
    c.eps1 = s.eps1;
    c.x_th1 = s.x_th1;
    c.x_th2 = s.x_th2;
    c.r1 = s.r1;
    c.max_cycle = s.max_cycle;
    c.hx_refresh_restarts = s.hx_refresh_restarts;
    c.t_max = s.t_max;
    c.lindep = s.lindep;
    c.clamp_delta = s.clamp_delta;
    return c;
}

int sbg_config_validate(const sbg_config* cfg) {
    return guarded([&] { to_cfg(cfg).validate(); });
}

// Pinned BASELINE.json generator; bit-identical to oracle/sbci_oracle.cpp:or_synthetic.
int sbg_synthetic_integrals(int norb, uint64_t seed, double offdiag_scale, double* h1, double* eri) {
    return guarded([&] {
        if (norb < 1 || norb > 32) throw std::invalid_argument("synthetic: norb out of range");
        std::mt19937_64 eng(seed);
        auto uni = [&]() { return (double)(eng() >> 11) * 0x1.0p-53; };
        auto normal = [&]() {
            const double u1 = uni(), u2 = uni();
            return std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(6.283185307179586476925286766559 * u2);
        };
        for (int p = 0; p < norb; ++p)
            for (int q = p; q < norb; ++q) {
                const double base = (p == q) ? (-1.0 + 2.0 * p / norb) : 0.0;
                const double v = base + 0.05 * normal();
                h1[p * norb + q] = v;
                h1[q * norb + p] = v;
            }
        const size_t no2 = (size_t)norb * norb;
        std::vector<double> L((size_t)norb * no2);
        for (int k = 0; k < norb; ++k)
            for (int p = 0; p < norb; ++p)
                for (int q = p; q < norb; ++q) {
                    const double v = (p == q) ? 0.5 + 0.1 * normal() : offdiag_scale * normal();
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

int sbg_shard_range(int64_t n, int rank, int world, int64_t* lo, int64_t* hi) {
    return guarded([&] {
        if (world < 1 || rank < 0 || rank >= world || n < 0) throw std::invalid_argument("shard_range: bad arguments");
        sbg::shard_range(n, rank, world, lo, hi);
    });
}

int sbg_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int sbg_create(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri, int device,
               uint64_t max_det, sbg_ctx** out) {
    return sbg_create_dist(norb, nelec, ms2, e_core, h1, eri, device, max_det, 0, 1, nullptr, out);
}

int sbg_create_dist(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri, int device,
                    uint64_t max_det, int rank, int world, const void* nccl_unique_id, sbg_ctx** out) {
    return guarded([&] {
        if (!out || !h1 || !eri) throw std::invalid_argument("sbg_create: null argument");
        if (world > 1 && !nccl_unique_id) throw std::invalid_argument("sbg_create_dist: missing NCCL unique id");
        auto* c = new sbg_ctx;
        try {
            c->c = std::make_unique<sbg::Context>(norb, nelec, ms2, e_core, h1, eri, device, max_det, rank, world,
                                                  nccl_unique_id);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

int sbg_local_group_create(int world, sbg_local_group** out) {
    return guarded([&] {
        if (!out || world < 1) throw std::invalid_argument("sbg_local_group_create: bad arguments");
        *out = reinterpret_cast<sbg_local_group*>(new sbg::LocalGroup(world));
    });
}

void sbg_local_group_destroy(sbg_local_group* g) { delete reinterpret_cast<sbg::LocalGroup*>(g); }

int sbg_create_local(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri, int device,
                     uint64_t max_det, sbg_local_group* group, int rank, sbg_ctx** out) {
    return guarded([&] {
        if (!out || !h1 || !eri || !group) throw std::invalid_argument("sbg_create_local: null argument");
        auto* g = reinterpret_cast<sbg::LocalGroup*>(group);
        auto* c = new sbg_ctx;
        try {
            c->c = std::make_unique<sbg::Context>(norb, nelec, ms2, e_core, h1, eri, device, max_det, rank, g->world,
                                                  nullptr, g);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

int sbg_nccl_unique_id(void* out128) {
    return guarded([&] {
        ncclUniqueId id;
        if (ncclGetUniqueId(&id) != ncclSuccess) throw sbg::DeviceError("ncclGetUniqueId failed");
        std::memcpy(out128, &id, sizeof(id));
    });
}

void sbg_destroy(sbg_ctx* ctx) { delete ctx; }

int64_t sbg_dim(const sbg_ctx* ctx) { return ctx && ctx->c ? ctx->c->ndet : -1; }

int sbg_sector(const sbg_ctx* ctx, int* norb, int* n_alpha, int* n_beta, int64_t* nas, int64_t* nbs) {
    return guarded([&] {
        require_ctx(ctx);
        const auto& c = *ctx->c;
        if (norb) *norb = c.norb;
        if (n_alpha) *n_alpha = c.na_el;
        if (n_beta) *n_beta = c.nb_el;
        if (nas) *nas = c.NA;
        if (nbs) *nbs = c.NB;
    });
}

int sbg_local_rows(const sbg_ctx* ctx, int64_t* lo, int64_t* hi) {
    return guarded([&] {
        require_ctx(ctx);
        *lo = ctx->c->row_lo;
        *hi = ctx->c->row_hi;
    });
}

int sbg_diagonal(sbg_ctx* ctx, double* out) {
    return guarded([&] {
        auto lk = lock_ctx(ctx);
        auto& c = *ctx->c;
        c.download_local(c.diagonal().p, out + c.row_lo * c.NB, c.st);
        SBG_CUDA(cudaStreamSynchronize(c.st));
    });
}

int sbg_table_sizes(const sbg_ctx* ctx, int spin, int64_t* n_strings, int64_t* row_len) {
    return guarded([&] {
        require_ctx(ctx);
        if (spin != 0 && spin != 1) throw std::invalid_argument("spin must be 0 or 1");
        if (n_strings) *n_strings = spin == 0 ? ctx->c->NA : ctx->c->NB;
        if (row_len) *row_len = ctx->c->row_len(spin);
    });
}

int sbg_string_tables(sbg_ctx* ctx, int spin, uint64_t* strings, sbg_excitation* links) {
    return guarded([&] {
        auto lk = lock_ctx(ctx);
        if (spin != 0 && spin != 1) throw std::invalid_argument("spin must be 0 or 1");
        ctx->c->string_tables(spin, strings, reinterpret_cast<sbg::Excitation*>(links));
    });
}

int sbg_sigma(sbg_ctx* ctx, const double* x, double* y, int nvec) {
    return guarded([&] {
        auto lk = lock_ctx(ctx);
        if (nvec < 0 || (!x && nvec) || (!y && nvec)) throw std::invalid_argument("sbg_sigma: bad arguments");
        auto& c = *ctx->c;
        if (nvec == 0) return;
        // Host-fed pipeline. Vectors alternate between two device slots; H2D of vector v+1 and D2H of
        // vector v-1 run on their own copy streams while sigma(v) runs on the compute stream. On one
        // GPU each vector also moves in row blocks (Context::sigma_rowblocks): the row-local beta-beta
        // term of block i starts as soon as block i has landed, and block i of y is copied out as
        // soon as its alpha-beta launch is done — so the first upload and the last download overlap
        // the sigma they feed instead of standing alone.
        static const int io_blocks = [] {
            const char* e = std::getenv("SBG_IO_BLOCKS");
            return e ? std::max(1, std::min(64, std::atoi(e))) : 4;
        }();
        const int nb = c.rowblocks_ok() ? io_blocks : 1;
        cudaStream_t cin = c.copy_stream(0), cout = c.copy_stream(1);
        std::vector<cudaEvent_t> up((size_t)nvec * nb), yd((size_t)nvec * nb), down(nvec);
        auto mk = [](cudaEvent_t& e) { SBG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)); };
        struct Cleanup {
            std::vector<cudaEvent_t>* v[3];
            ~Cleanup() {
                for (auto* l : v)
                    for (auto e : *l)
                        if (e) cudaEventDestroy(e);
            }
        } cleanup{{&up, &yd, &down}};
        for (auto& e : up) mk(e);
        for (auto& e : yd) mk(e);
        for (auto& e : down) mk(e);
        for (int v = 0; v < nvec; ++v) {
            const int slot = v & 1;
            double *dx = c.io_x(slot), *dy = c.io_y(slot);
            cudaEvent_t* upv = &up[(size_t)v * nb];
            cudaEvent_t* ydv = &yd[(size_t)v * nb];
            // sigma(v-2) released dx once its last alpha-beta block is done
            if (v >= 2) SBG_CUDA(cudaStreamWaitEvent(cin, yd[(size_t)(v - 2) * nb + nb - 1], 0));
            if (v >= 2) SBG_CUDA(cudaStreamWaitEvent(c.st, down[v - 2], 0));  // D2H(v-2) released dy
            if (nb == 1) {
                c.upload_local(x + (size_t)v * c.ndet, dx, cin);
                SBG_CUDA(cudaEventRecord(upv[0], cin));
                SBG_CUDA(cudaStreamWaitEvent(c.st, upv[0], 0));
                c.sigma(dx, dy, c.st);
                SBG_CUDA(cudaEventRecord(ydv[0], c.st));
                SBG_CUDA(cudaStreamWaitEvent(cout, ydv[0], 0));
                c.download_local(dy, y + (size_t)v * c.ndet + c.row_lo * c.NB, cout);
            } else {
                for (int i = 0; i < nb; ++i) {
                    int64_t lo, hi;
                    c.chunk_rows(nb, i, &lo, &hi);
                    c.upload_rows(x + (size_t)v * c.ndet, dx, lo, hi, cin);
                    SBG_CUDA(cudaEventRecord(upv[i], cin));
                }
                c.sigma_rowblocks(dx, dy, c.st, nb, upv, ydv);
                for (int i = 0; i < nb; ++i) {
                    int64_t lo, hi;
                    c.chunk_rows(nb, i, &lo, &hi);
                    SBG_CUDA(cudaStreamWaitEvent(cout, ydv[i], 0));
                    c.download_rows(dy, y + (size_t)v * c.ndet + c.row_lo * c.NB, lo, hi, cout);
                }
            }
            SBG_CUDA(cudaEventRecord(down[v], cout));
        }
        SBG_CUDA(cudaStreamSynchronize(cout));
        SBG_CUDA(cudaStreamSynchronize(cin));
        SBG_CUDA(cudaStreamSynchronize(c.st));
    });
}

int64_t sbg_padded_len(const sbg_ctx* ctx) { return ctx && ctx->c ? ctx->c->padded_len() : -1; }

int sbg_pack(sbg_ctx* ctx, const double* d_dense_full, double* d_padded_local, void* stream) {
    return guarded([&] {
        auto lk = lock_ctx(ctx);
        auto& c = *ctx->c;
        cudaStream_t s = stream ? (cudaStream_t)stream : c.st;
        SBG_CUDA(cudaMemsetAsync(d_padded_local, 0, c.padded_len() * 8, s));
        c.pack_device(d_dense_full, d_padded_local, s);
    });
}

int sbg_unpack(sbg_ctx* ctx, const double* d_padded_local, double* d_dense_local, void* stream) {
    return guarded([&] {
        auto lk = lock_ctx(ctx);
        auto& c = *ctx->c;
        c.unpack_device(d_padded_local, d_dense_local, stream ? (cudaStream_t)stream : c.st);
    });
}

int sbg_sigma_padded(sbg_ctx* ctx, const double* dx, double* dy, void* stream) {
    return guarded([&] {
        auto lk = lock_ctx(ctx);
        auto& c = *ctx->c;
        c.sigma(dx, dy, stream ? (cudaStream_t)stream : c.st);
    });
}

int sbg_sigma_padded_multi(sbg_ctx* ctx, int nvec, const double* const* dx, double* const* dy, void* stream) {
    return guarded([&] {
        auto lk = lock_ctx(ctx);
        if (nvec < 0 || (nvec > 0 && (!dx || !dy))) throw std::invalid_argument("sbg_sigma_padded_multi: bad arguments");
        auto& c = *ctx->c;
        cudaStream_t s = stream ? (cudaStream_t)stream : c.st;
        for (int v0 = 0; v0 < nvec; v0 += sbg::kMaxSigmaVec)
            c.sigma_multi(dx + v0, dy + v0, std::min(sbg::kMaxSigmaVec, nvec - v0), s);
    });
}

int sbg_sigma_device(sbg_ctx* ctx, const double* d_x, double* d_y, void* stream) {
    return guarded([&] {
        auto lk = lock_ctx(ctx);
        auto& c = *ctx->c;
        cudaStream_t s = stream ? (cudaStream_t)stream : c.st;
        double *px = c.io_x(), *py = c.io_y();
        c.pack_device(d_x, px, s);
        c.sigma(px, py, s);
        c.unpack_device(py, d_y + c.row_lo * c.NB, s);
        SBG_CUDA(cudaStreamSynchronize(s));
    });
}

uint64_t sbg_apply_count(const sbg_ctx* ctx) { return ctx && ctx->c ? ctx->c->applies().load() : 0; }
void sbg_reset_apply_count(sbg_ctx* ctx) {
    if (ctx && ctx->c) ctx->c->applies().store(0);
}
uint64_t sbg_kernel_launches(const sbg_ctx* ctx) { return ctx && ctx->c ? ctx->c->launches.load() : 0; }

int sbg_profile_reset(sbg_ctx* ctx) {
    return guarded([&] {
        auto lk = lock_ctx(ctx);
        ctx->c->profile_reset();
    });
}

int sbg_profile_read(sbg_ctx* ctx, double* ms, int64_t* calls) {
    return guarded([&] {
        auto lk = lock_ctx(ctx);
        ctx->c->profile_read(ms, calls);
    });
}

int sbg_sigma_flops(const sbg_ctx* ctx, double* ab, double* ss, double* total) {
    return guarded([&] {
        require_ctx(ctx);
        if (ab) *ab = ctx->c->flops_ab;
        if (ss) *ss = ctx->c->flops_ss;
        if (total) *total = ctx->c->flops_ab + ctx->c->flops_ss;
    });
}

int sbg_spin_squared(sbg_ctx* ctx, const double* x, double* out) {
    return guarded([&] {
        auto lk = lock_ctx(ctx);
        if (!x || !out) throw std::invalid_argument("sbg_spin_squared: null argument");
        auto& c = *ctx->c;
        double* dx = c.io_x();
        c.upload_local(x, dx, c.st);
        *out = c.spin_squared(dx);
    });
}

int sbg_spin_squared_padded(sbg_ctx* ctx, const double* d_x, double* out) {
    return guarded([&] {
        auto lk = lock_ctx(ctx);
        if (!d_x || !out) throw std::invalid_argument("sbg_spin_squared_padded: null argument");
        *out = ctx->c->spin_squared(d_x);
    });
}

static int solve_impl(sbg_ctx* ctx, int method, int nroots, int max_space, const sbg_config* cfg, double* energies,
                      double* vectors, sbg_stats* stats, sbg_trace_fn trace, void* trace_user) {
    return guarded([&] {
        auto lk = lock_ctx(ctx);
        if (method < 1 || method > 3)
            throw std::invalid_argument("sbg_solve: method must be 1 (sbci1), 2 (sbci2) or 3 (davidson)");
        if (nroots < 1 || nroots > sbg::detail_max_roots)
            throw std::invalid_argument("sbg_solve: nroots must be in 1..9 (at most 8 deflated states)");
        auto& c = *ctx->c;
        const std::function<void(const sbg::TraceRec&)> tf = make_trace(trace, trace_user);
        const uint64_t launches0 = c.launches;
        c.pool().reset_peak();
        try {
            sbg::MultiStateResult r = method == 1   ? sbg::solve_n_states_sbci1(c, nroots, to_cfg(cfg), tf)
                                      : method == 2 ? sbg::solve_n_states_sbci2(c, nroots, to_cfg(cfg), tf)
                                                    : sbg::davidson_solve(c, nroots, to_cfg(cfg), tf, max_space);
            std::vector<double> s2(nroots);
            for (int k = 0; k < nroots; ++k) s2[k] = c.spin_squared(r.pairs[k].vector.p);
            for (int k = 0; k < nroots; ++k) {
                energies[k] = r.pairs[k].energy;
                if (vectors) c.download_local(r.pairs[k].vector.p, vectors + (size_t)k * c.ndet + c.row_lo * c.NB, c.st);
            }
            SBG_CUDA(cudaStreamSynchronize(c.st));
            if (stats) {
                std::memset(stats, 0, sizeof(*stats));
                stats->nroots = nroots;
                for (int k = 0; k < nroots; ++k) {
                    stats->iterations[k] = r.pairs[k].iterations;
                    stats->restarts[k] = r.pairs[k].restarts;
                    stats->final_residual[k] = r.pairs[k].final_residual;
                }
                stats->matvecs = r.matvecs;
                stats->total_iterations = r.total_iterations;
                stats->total_restarts = r.total_restarts;
                stats->hx_refreshes = r.hx_refreshes;
                stats->peak_vectors = r.peak_vectors;
                stats->wall_time_s = r.wall_time_s;
                stats->failed_state = -1;
                stats->kernel_launches = c.launches - launches0;
                stats->device_vectors_peak = c.pool().peak;
                for (int k = 0; k < nroots; ++k) stats->s_squared[k] = s2[k];
            }
        } catch (const sbg::NonConvergenceError& e) {
            if (stats) {
                std::memset(stats, 0, sizeof(*stats));
                stats->failed_state = e.state;
                stats->best_energy = e.best_energy;
                stats->best_residual = e.best_residual;
            }
            throw;
        }
    });
}

int sbg_solve(sbg_ctx* ctx, int method, int nroots, const sbg_config* cfg, double* energies, double* vectors,
              sbg_stats* stats, sbg_trace_fn trace, void* trace_user) {
    return solve_impl(ctx, method, nroots, 0, cfg, energies, vectors, stats, trace, trace_user);
}

int sbg_solve_davidson(sbg_ctx* ctx, int nroots, int max_space, const sbg_config* cfg, double* energies,
                       double* vectors, sbg_stats* stats, sbg_trace_fn trace, void* trace_user) {
    return solve_impl(ctx, 3, nroots, max_space, cfg, energies, vectors, stats, trace, trace_user);
}

int sbg_solve_state_sbci1(sbg_ctx* ctx, const double* x0, double e0, double* shift, int alpha, int ndefl,
                          const double* defl_x, const double* defl_hx, const double* defl_e, const sbg_config* cfg,
                          double* energy, double* vector, double* image, sbg_stats* stats, sbg_trace_fn trace,
                          void* trace_user) {
    return guarded([&] {
        auto lk = lock_ctx(ctx);
        if (!x0 || !shift || !energy) throw std::invalid_argument("sbg_solve_state_sbci1: null argument");
        if (ndefl < 0 || ndefl > sbg::detail_max_roots - 1 || (ndefl > 0 && (!defl_x || !defl_e)))
            throw std::invalid_argument("sbg_solve_state_sbci1: bad deflation set");
        if (alpha < 0) throw std::invalid_argument("sbg_solve_state_sbci1: alpha must be >= 0");
        auto& c = *ctx->c;
        const sbg::SolverConfig scfg = to_cfg(cfg);
        scfg.validate();
        sbg::detail::Ops o(c);
        // deflation set: stored vectors (+ images, rebuilt by sigma when not given; those builds are
        // not applications of the caller's solve)
        sbg::detail::Deflation defl;
        for (int i = 0; i < ndefl; ++i) {
            sbg::DBuf xv = c.vec(), hv = c.vec();
            c.upload_local(defl_x + (size_t)i * c.ndet, xv.p, c.st);
            if (defl_hx) {
                c.upload_local(defl_hx + (size_t)i * c.ndet, hv.p, c.st);
            } else {
                o.apply(xv, hv);
                c.applies().fetch_sub(1);
            }
            defl.add_with_image(o, std::move(xv), std::move(hv), defl_e[i]);
        }
        const uint64_t applies1 = c.applies().load();
        c.pool().reset_peak();
        // Seed{x0, H x0, E0} (sbci1.hpp:481-485)
        sbg::detail::Seed seed;
        seed.x = c.vec();
        seed.hx = c.vec();
        c.upload_local(x0, seed.x.p, c.st);
        if (o.norm(seed.x) == 0.0) throw std::invalid_argument("solve_state_sbci1: x0 must be nonzero");
        o.apply(seed.x, seed.hx);
        seed.energy = e0;
        sbg::detail::Precond pre{&c.diagonal(), *shift, scfg.clamp_delta};
        if (!(pre.clamp > 0.0)) throw std::invalid_argument("clamp_delta must be positive");
        sbg::detail::Sbci1Result r;
        const auto t0 = std::chrono::steady_clock::now();
        try {
            r = sbg::detail::solve_state_sbci1(c, scfg, make_trace(trace, trace_user), pre, defl, std::move(seed), alpha,
                                               alpha == 0);
        } catch (const sbg::NonConvergenceError& e) {
            if (stats) {
                std::memset(stats, 0, sizeof(*stats));
                stats->failed_state = e.state;
                stats->best_energy = e.best_energy;
                stats->best_residual = e.best_residual;
            }
            throw;
        }
        if (alpha == 0) pre.update_shift(r.pair.energy);
        *shift = pre.shift;
        *energy = r.pair.energy;
        if (vector) c.download_local(r.pair.vector.p, vector + c.row_lo * c.NB, c.st);
        if (image) c.download_local(r.converged_image.p, image + c.row_lo * c.NB, c.st);
        SBG_CUDA(cudaStreamSynchronize(c.st));
        if (stats) {
            std::memset(stats, 0, sizeof(*stats));
            stats->nroots = 1;
            stats->iterations[0] = r.pair.iterations;
            stats->restarts[0] = r.pair.restarts;
            stats->final_residual[0] = r.pair.final_residual;
            stats->matvecs = c.applies().load() - applies1;
            stats->total_iterations = r.pair.iterations;
            stats->total_restarts = r.pair.restarts;
            stats->hx_refreshes = r.hx_refreshes;
            stats->peak_vectors = 7 + ndefl;
            stats->device_vectors_peak = c.pool().peak;
            stats->wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            stats->failed_state = -1;
            stats->s_squared[0] = c.spin_squared(r.pair.vector.p);
        }
    });
}

int sbg_selftest(void) {
    int bad = -1;
    const int rc = guarded([&] {
        SBG_CUDA(cudaSetDevice(0));
        bad = sbg::run_mma_selftest();
    });
    if (rc != SBG_OK) return rc;
    if (bad != 0) {
        g_err = "DMMA fragment layout mismatch in " + std::to_string(bad) + " entries";
        return SBG_EDEVICE;
    }
    return SBG_OK;
}

int sbg_selftest_nccl(void) {
    int bad = -1;
    const int rc = guarded([&] {
        bad = sbg::run_nccl_selftest();  // on the calling thread's current device
    });
    if (rc != SBG_OK) return rc;
    if (bad != 0) {
        g_err = "NCCL collective self test: " + std::to_string(bad) + " wrong entries";
        return SBG_EDEVICE;
    }
    return SBG_OK;
}

}  // extern "C"
