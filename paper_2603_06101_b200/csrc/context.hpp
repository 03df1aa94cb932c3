// context.hpp — device-resident FCI operator: the B200 replacement of sbci::fci::FciOperator
// (fci_operator.hpp:60-86). Owns the string tables, folded integrals, scatter codes, the exact
// diagonal and the sigma workspaces in HBM; sigma() is SymmetricOperator::apply (operator.hpp:25-31)
// on device vectors.
//
// HBM layout of every length-n_det vector: row-major [rows][ld] with rows = the
// alpha strings owned by this rank (contiguous block) and ld = n_beta_strings rounded
// up to 32 (256-byte rows, so 16-byte cp.async / TMA-sized gathers never straddle a row); the
// padding columns are kept at exactly zero by every kernel.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <atomic>
#include <memory>
#include <string>
#include <vector>

#include "comm.hpp"
#include "common.cuh"
#include "kernels.cuh"

namespace sbg {

// Recycles the padded solver vectors of one Context (all the same length). cudaMalloc/cudaFree of
// ~100 MB vectors cost milliseconds and cudaFree synchronises the device, so the solver's per-state
// allocations (sbci1.hpp keeps 7 + n_deflated vectors live) come from here instead. Buffers are
// reused in stream order: every user of a pooled buffer works on the Context stream.
struct VecPool {
    std::vector<double*> free_;
    int64_t n = 0;
    int live = 0, peak = 0;  // pooled vectors in use now / at most since reset_peak
    ~VecPool();
    double* take(int64_t count);
    void give(double* p) {
        free_.push_back(p);
        --live;
    }
    void reset_peak() { peak = live; }
};

struct DBuf {
    double* p = nullptr;
    int64_t n = 0;
    VecPool* pool = nullptr;
    DBuf() = default;
    explicit DBuf(int64_t count);                          // cudaMalloc + zero fill, synchronous
    DBuf(VecPool& vp, int64_t count, cudaStream_t zero_on);  // pooled, zero fill ordered on zero_on
    ~DBuf();
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), pool(o.pool) {
        o.p = nullptr;
        o.n = 0;
        o.pool = nullptr;
    }
    DBuf& operator=(DBuf&& o) noexcept;
    bool empty() const { return p == nullptr; }

private:
    void release();
};


class Context {
public:
    Context(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri, int device,
            uint64_t max_det, int rank, int world, const void* nccl_id, LocalGroup* local_group = nullptr);
    ~Context();

    // sector
    int norb, nelec, ms2, na_el, nb_el;
    double e_core;
    int64_t NA, NB, ndet, ld, ldT;  // ldT: leading dimension of the transposed local rows [NB][ldT]
    int64_t row_lo, row_hi, nrows;  // alpha rows owned by this rank
    int rank, world, device, nsm;
    cudaStream_t st = nullptr;

    int64_t padded_len() const { return nrows * ld; }
    DBuf alloc_vec() const;  // zero-initialised padded local vector
    // pooled zero-initialised padded local vector; the zero fill is ordered on st (solver work)
    DBuf vec() { return DBuf(*pool_, padded_len(), st); }
    VecPool& pool() { return *pool_; }
    // persistent staging vectors of the host-pointer entry points (sbg_sigma, sbg_sigma_device)
    double* io_x(int slot = 0) {
        if (io_x_[slot].empty()) io_x_[slot] = alloc_vec();
        return io_x_[slot].p;
    }
    double* io_y(int slot = 0) {
        if (io_y_[slot].empty()) io_y_[slot] = alloc_vec();
        return io_y_[slot].p;
    }
    // host <-> device copy streams (0: H2D, 1: D2H) of the batched host-pointer entry points
    cudaStream_t copy_stream(int which);

    // y = H x on padded local vectors (counts one application)
    void sigma(const double* x_local, double* y_local, cudaStream_t s);
    // single GPU, host-fed: the same sigma with the rows in nchunks blocks so that copies overlap
    // it. The beta-beta term of block i (row-local) waits only for x_ready[i]; the alpha-alpha and
    // alpha-beta terms wait for every block; y_done[i] is recorded once rows of block i are final.
    void sigma_rowblocks(const double* x_local, double* y_local, cudaStream_t s, int nchunks,
                         const cudaEvent_t* x_ready, const cudaEvent_t* y_done);
    void chunk_rows(int nchunks, int i, int64_t* lo, int64_t* hi) const;  // rows of block i
    bool rowblocks_ok() const { return world == 1 && have_ab_ && !direct_ab_ && !ss_csr_[0] && !ss_csr_[1]; }
    // host <-> padded device copies of local rows [lo, hi) (host pointers: dense full / dense local)
    void upload_rows(const double* host_dense_full, double* d_padded, int64_t lo, int64_t hi, cudaStream_t s) const;
    void download_rows(const double* d_padded, double* host_dense_local, int64_t lo, int64_t hi, cudaStream_t s) const;
    void sigma(const DBuf& x, DBuf& y) { sigma(x.p, y.p, st); }
    // y_v = H x_v for nvec vectors; single GPU with the reduction kernels: the alpha-beta and
    // alpha-alpha kernels take all vectors in one launch (per-row / per-K set-up paid once), the
    // beta-beta term runs per vector; anything else: one sigma per vector. Counts nvec applications.
    void sigma_multi(const double* const* x, double* const* y, int nvec, cudaStream_t s);
    // <S^2> of a padded local vector (fci/spin.hpp:17-51); collective over ranks
    double spin_squared(const double* x_local);

    // host <-> padded device conversions (dense local rows = rows [row_lo,row_hi) of the n_det vector)
    void upload_local(const double* host_dense_full, double* d_padded, cudaStream_t s) const;
    void download_local(const double* d_padded, double* host_dense_local, cudaStream_t s) const;
    void pack_device(const double* d_dense_full, double* d_padded, cudaStream_t s) const;
    void unpack_device(const double* d_padded, double* d_dense_local, cudaStream_t s) const;

    // tables
    const DBuf& diagonal() const { return diag_; }
    void string_tables(int spin, uint64_t* strings, Excitation* links);
    int64_t row_len(int spin) const;

    // reductions: dot buffer all-reduced over ranks and copied to host
    ReduceWs rws;
    const double* finish_dots(int ndot);  // sync; returns host pointer
    // the same split in two: post_dots enqueues the all-reduce and the copy to the host and records
    // an event; wait_dots waits for that event only — kernels enqueued in between keep running
    void post_dots(int ndot);
    const double* wait_dots();
    void allreduce_inplace_device(double* d, int count);

    // per-phase CUDA-event profile of sigma calls (sbg_profile_*)
    void profile_reset();
    void profile_read(double* ms, int64_t* calls);

    std::atomic<uint64_t>& applies() { return applies_; }
    std::atomic<uint64_t> launches{0};
    double sigma_ms = 0.0;  // accumulated device time of sigma calls (events)
    double flops_ab = 0, flops_ss = 0;

private:
    std::unique_ptr<VecPool> pool_ = std::make_unique<VecPool>();  // declared first: destroyed last
    void build_tables(const double* h1, const double* eri);
    void ensure_links();
    void gather_full(const double* x_local, cudaStream_t s);

    std::atomic<uint64_t> applies_{0};
    std::unique_ptr<Comm> comm_;
    // device tables
    uint64_t *d_sa_ = nullptr, *d_sb_ = nullptr;
    Excitation *d_la_ = nullptr, *d_lb_ = nullptr;
    double *d_h1_ = nullptr, *d_eri_ = nullptr, *d_Vp_ = nullptr, *d_Va_ = nullptr, *d_Vb_ = nullptr;
    uint16_t* d_codes_ = nullptr;
    uint32_t *d_sc_tgt_ = nullptr, *d_sc_tt_ = nullptr, *d_sc_te_ = nullptr;
    uint32_t *d_red_ent_ = nullptr, *d_red_te_ = nullptr;
    uint16_t* d_sc_ent_ = nullptr;
    DBuf diag_;
    // sigma workspaces
    DBuf xfull_, xT_, sT_, saa_, a2a_send_, a2a_recv_, io_x_[2], io_y_[2];
    cudaStream_t cs_[2] = {nullptr, nullptr};
    AbPlan ab_{};
    SsPlan ssa_{}, ssb_{};
    bool have_ab_ = false;
    // generic fallbacks for sectors outside the tensor-core kernels' limits
    bool direct_ab_ = false;
    bool ss_csr_[2] = {false, false};
    SsCsrDev csr_dev_[2];
    void* csr_mem_[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};
    double csr_nnz_[2] = {0.0, 0.0};
    bool has_ss(int spin) const { return ss_csr_[spin] || (spin ? ssb_.P : ssa_.P) > 0; }
    // same-spin term of one spin on a column window (x, y: rows = that spin's strings)
    // col_pad: see launch_sigma_ss (zero padding columns of x past col_hi inside y's rows)
    void run_ss(int spin, const double* x, double* y, int64_t ldx, int64_t col_lo, int64_t col_hi, cudaStream_t s,
                int64_t ldy = 0, int64_t ycol0 = 0, int64_t col_pad = 0);
    // world > 1: the alpha-alpha term's beta-column window [aa_lo_, aa_hi_) lives in saa_ as
    // [NA][ldw_] starting at the aligned column aa_c0_
    int64_t aa_lo_ = 0, aa_hi_ = 0, aa_c0_ = 0, ldw_ = 0;
    void run_ab(const double* x_full, double* y_rows, int64_t lo, int64_t hi, cudaStream_t s);
    std::vector<std::pair<uint32_t*, uint32_t*>> red_pass_;  // reduction lists per pair-row block
    cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
    // device-side order of sigma builds issued on different streams (they share xT_, sT_, xfull_, the
    // alpha-alpha buffers): every build waits for the previous one's completion event
    cudaEvent_t ev_order_ = nullptr;
    cudaEvent_t ev_dots_ = nullptr;  // post_dots -> wait_dots
    std::unique_ptr<ReduceWs::ZeroCopy> zc_;  // single GPU: dots read from mapped host memory
    unsigned long long post_seq_ = 0;
    int post_n_ = 0;
    bool poll_zero_copy(unsigned long long seq);
    bool order_recorded_ = false;
    void order_begin(cudaStream_t s);
    void order_end(cudaStream_t s);
    // world > 1: the collectives run on their own stream, overlapped with the kernels that do not
    // need their result (beta-beta term during the all-gather, alpha-beta during the alpha-alpha
    // exchange)
    cudaStream_t comm_st_ = nullptr;
    cudaEvent_t ev_in_ = nullptr, ev_gathered_ = nullptr, ev_aa_ = nullptr, ev_xdone_ = nullptr, ev_ab_ = nullptr;
    // the alpha-beta kernel reduces into y with red.global.add (so the exchanged alpha-alpha blocks
    // may be added beside it); the direct and deterministic forms read-modify-write y rows instead
    bool ab_reduces() const { return have_ab_ && !direct_ab_ && ab_.red; }
    struct EvSet {
        cudaEvent_t e[5];
    };
    std::vector<EvSet> ev_pool_;
    size_t ev_used_ = 0;
    double prof_ms_[4] = {0, 0, 0, 0};
    int64_t prof_calls_ = 0;
    EvSet* next_evset();
};

}  // namespace sbg
