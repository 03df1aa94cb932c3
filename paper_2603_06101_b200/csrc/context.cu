// context.cu — construction of the device-resident FCI operator and the sigma orchestration.
#include "context.hpp"

#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

namespace sbg {

// ------------------------------------------------------------------ buffers
DBuf::DBuf(int64_t count) : n(count) {
    if (count > 0) {
        SBG_CUDA(cudaMalloc(&p, (size_t)count * sizeof(double)));
        // the library works on a non-blocking stream, which does not order against the legacy
        // default stream a plain cudaMemset runs on: finish the zero-fill before handing out p
        SBG_CUDA(cudaMemsetAsync(p, 0, (size_t)count * sizeof(double), cudaStreamLegacy));
        SBG_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
    }
}
DBuf::DBuf(VecPool& vp, int64_t count, cudaStream_t zero_on) : n(count), pool(&vp) {
    if (count > 0) {
        p = vp.take(count);
        SBG_CUDA(cudaMemsetAsync(p, 0, (size_t)count * sizeof(double), zero_on));
    }
}
void DBuf::release() {
    if (p) {
        if (pool) pool->give(p);
        else cudaFree(p);
    }
    p = nullptr;
    n = 0;
    pool = nullptr;
}
DBuf::~DBuf() { release(); }
DBuf& DBuf::operator=(DBuf&& o) noexcept {
    if (this != &o) {
        release();
        p = o.p;
        n = o.n;
        pool = o.pool;
        o.p = nullptr;
        o.n = 0;
        o.pool = nullptr;
    }
    return *this;
}

double* VecPool::take(int64_t count) {
    if (n == 0) n = count;
    if (count != n) throw std::invalid_argument("VecPool: all pooled vectors have the padded local length");
    double* p = nullptr;
    if (!free_.empty()) {
        p = free_.back();
        free_.pop_back();
    } else {
        SBG_CUDA(cudaMalloc(&p, (size_t)count * sizeof(double)));
    }
    peak = std::max(peak, ++live);
    return p;
}
VecPool::~VecPool() {
    for (double* p : free_) cudaFree(p);
}

// ------------------------------------------------------------------ collectives (comm.hpp)
#define SBG_NCCL(x)                                                                                     \
    do {                                                                                                \
        ncclResult_t r_ = (x);                                                                          \
        if (r_ != ncclSuccess) throw DeviceError(std::string("NCCL error ") + ncclGetErrorString(r_) + \
                                                 " in " #x);                                            \
    } while (0)

namespace {

class NcclComm final : public Comm {
public:
    NcclComm(int world, int rank, const void* id_bytes) {
        ncclUniqueId id;
        std::memcpy(&id, id_bytes, sizeof(id));
        SBG_NCCL(ncclCommInitRank(&comm_, world, id, rank));
    }
    ~NcclComm() override {
        if (comm_) ncclCommDestroy(comm_);
    }
    void all_gather(const double* send, double* recv, size_t count, cudaStream_t s) override {
        SBG_NCCL(ncclAllGather(send, recv, count, ncclDouble, comm_, s));
    }
    void all_reduce_sum(double* buf, size_t count, cudaStream_t s) override {
        SBG_NCCL(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, comm_, s));
    }
    void exchange(const std::vector<CommBlock>& sends, const std::vector<CommBlock>& recvs, cudaStream_t s) override {
        // the group is always closed, even when a send/recv fails inside it (an open group would
        // make the next collective hang); the first failure is reported after ncclGroupEnd
        SBG_NCCL(ncclGroupStart());
        ncclResult_t first = ncclSuccess;
        const char* what = "";
        for (const auto& b : sends) {
            const ncclResult_t r = ncclSend(b.ptr, b.count, ncclDouble, b.peer, comm_, s);
            if (r != ncclSuccess && first == ncclSuccess) first = r, what = "ncclSend";
        }
        for (const auto& b : recvs) {
            const ncclResult_t r = ncclRecv(b.ptr, b.count, ncclDouble, b.peer, comm_, s);
            if (r != ncclSuccess && first == ncclSuccess) first = r, what = "ncclRecv";
        }
        const ncclResult_t end = ncclGroupEnd();
        if (first != ncclSuccess)
            throw DeviceError(std::string("NCCL error ") + ncclGetErrorString(first) + " in " + what);
        if (end != ncclSuccess) throw DeviceError(std::string("NCCL error ") + ncclGetErrorString(end) + " in ncclGroupEnd");
    }

private:
    ncclComm_t comm_ = nullptr;
};

// ranks = threads of one process; every collective: finish my stream, publish, barrier, copy, barrier
class LocalComm final : public Comm {
public:
    LocalComm(LocalGroup* g, int rank) : g_(g), rank_(rank) {}
    void all_gather(const double* send, double* recv, size_t count, cudaStream_t s) override {
        SBG_CUDA(cudaStreamSynchronize(s));
        g_->ptr[rank_] = send;
        g_->barrier();
        for (int r = 0; r < g_->world; ++r)
            if (recv + r * count != g_->ptr[r])
                SBG_CUDA(cudaMemcpyAsync(recv + r * count, g_->ptr[r], count * 8, cudaMemcpyDeviceToDevice, s));
        SBG_CUDA(cudaStreamSynchronize(s));
        g_->barrier();  // nobody reads my send buffer any more
    }
    void all_reduce_sum(double* buf, size_t count, cudaStream_t s) override {
        SBG_CUDA(cudaStreamSynchronize(s));
        g_->ptr[rank_] = buf;
        g_->barrier();
        std::vector<double> acc(count, 0.0), part(count);
        for (int r = 0; r < g_->world; ++r) {  // rank order: every rank forms the identical sum
            SBG_CUDA(cudaMemcpy(part.data(), g_->ptr[r], count * 8, cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < count; ++i) acc[i] += part[i];
        }
        g_->barrier();  // all reads done before anyone overwrites its buffer
        SBG_CUDA(cudaMemcpyAsync(buf, acc.data(), count * 8, cudaMemcpyHostToDevice, s));
        SBG_CUDA(cudaStreamSynchronize(s));
    }
    void exchange(const std::vector<CommBlock>& sends, const std::vector<CommBlock>& recvs, cudaStream_t s) override {
        SBG_CUDA(cudaStreamSynchronize(s));
        g_->sends[rank_] = sends;
        g_->barrier();
        for (const auto& rb : recvs) {
            const CommBlock* sb = nullptr;
            for (const auto& b : g_->sends[rb.peer])
                if (b.peer == rank_) sb = &b;
            if (!sb || sb->count != rb.count) throw DeviceError("local exchange: unmatched block");
            SBG_CUDA(cudaMemcpyAsync(rb.ptr, sb->ptr, rb.count * 8, cudaMemcpyDeviceToDevice, s));
        }
        SBG_CUDA(cudaStreamSynchronize(s));
        g_->barrier();
    }

private:
    LocalGroup* g_;
    int rank_;
};

}  // namespace

std::unique_ptr<Comm> make_nccl_comm(int world, int rank, const void* nccl_unique_id) {
    return std::make_unique<NcclComm>(world, rank, nccl_unique_id);
}
std::unique_ptr<Comm> make_local_comm(LocalGroup* group, int rank) {
    if (!group || rank < 0 || rank >= group->world) throw InvalidArgument("local group: bad rank");
    return std::make_unique<LocalComm>(group, rank);
}

namespace {

template <class T>
T* dmalloc(size_t n) {
    T* p = nullptr;
    SBG_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    return p;
}

// dst += src on a column window, as fp64 reductions: it runs beside the alpha-beta kernel, which
// reduces into the same rows of y
__global__ void k_add_block(double* dst, int64_t ldd, const double* src, int64_t rows, int64_t cols) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= rows * cols) return;
    const int64_t r = i / cols, c = i % cols;
    red_add_f64(dst + r * ldd + c, src[i]);
}

}  // namespace

// rows [lo,hi) of a block partition with equal block sizes ceil(n/world); the last
// ranks may own fewer (or zero) rows.
void shard_range(int64_t n, int rank, int world, int64_t* lo, int64_t* hi) {
    const int64_t per = (n + world - 1) / world;
    *lo = std::min<int64_t>(n, (int64_t)rank * per);
    *hi = std::min<int64_t>(n, *lo + per);
}

// ------------------------------------------------------------------ context
Context::Context(int norb_, int nelec_, int ms2_, double e_core_, const double* h1, const double* eri, int device_,
                 uint64_t max_det, int rank_, int world_, const void* nccl_id, LocalGroup* local_group)
    : norb(norb_), nelec(nelec_), ms2(ms2_), e_core(e_core_), rank(rank_), world(world_), device(device_) {
    if (norb < 1 || norb > kMaxOrb) throw InvalidArgument("FciProblem: norb must be in [1, 32]");
    if (nelec < 0 || nelec > 2 * norb) throw InvalidArgument("as_operator: NELEC out of range");
    if ((nelec + ms2) % 2 != 0) throw InvalidArgument("as_operator: MS2 parity mismatch");
    na_el = (nelec + ms2) / 2;
    nb_el = (nelec - ms2) / 2;
    if (na_el < 0 || nb_el < 0 || na_el > norb || nb_el > norb)
        throw InvalidArgument("determinant_count: electron count out of range");
    if (na_el + nb_el == 0) throw InvalidArgument("FciOperator: empty electron sector");
    NA = (int64_t)binom_host_calc(norb, na_el);
    NB = (int64_t)binom_host_calc(norb, nb_el);
    ndet = NA * NB;
    if ((uint64_t)ndet > max_det)
        throw std::runtime_error("as_operator: sector holds " + std::to_string(ndet) +
                                 " determinants, above the guard of " + std::to_string(max_det) +
                                 " (pass a larger bound to override)");
    if (world < 1 || rank < 0 || rank >= world) throw InvalidArgument("sbg_create_dist: bad rank/world");
    ld = round_up(NB, 32);
    shard_range(NA, rank, world, &row_lo, &row_hi);
    nrows = row_hi - row_lo;
    ldT = round_up(std::max<int64_t>(nrows, 1), 32);  // beta-beta: only this rank's alpha rows are transposed

    SBG_CUDA(cudaSetDevice(device));
    SBG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
    SBG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    SBG_CUDA(cudaEventCreate(&ev0_));
    SBG_CUDA(cudaEventCreate(&ev1_));
    SBG_CUDA(cudaEventCreateWithFlags(&ev_order_, cudaEventDisableTiming));
    SBG_CUDA(cudaEventCreateWithFlags(&ev_dots_, cudaEventDisableTiming));

    if (world > 1) {
        if (local_group && local_group->world != world) throw InvalidArgument("local group: world mismatch");
        comm_ = local_group ? make_local_comm(local_group, rank) : make_nccl_comm(world, rank, nccl_id);
        SBG_CUDA(cudaStreamCreateWithFlags(&comm_st_, cudaStreamNonBlocking));
        for (cudaEvent_t* e : {&ev_in_, &ev_gathered_, &ev_aa_, &ev_xdone_, &ev_ab_})
            SBG_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }

    rws.grid = 16 * nsm;
    rws.partial = dmalloc<double>((size_t)rws.grid * kMaxRed);
    rws.result = dmalloc<double>(kMaxRed);
    rws.ticket = dmalloc<unsigned int>(1);
    SBG_CUDA(cudaMemset(rws.ticket, 0, sizeof(unsigned int)));
    if (world == 1 && !(std::getenv("SBG_ZERO_COPY_DOTS") && std::atoi(std::getenv("SBG_ZERO_COPY_DOTS")) == 0)) {
        zc_ = std::make_unique<ReduceWs::ZeroCopy>();
        SBG_CUDA(cudaHostAlloc(&zc_->mirror, kMaxRed * sizeof(double), cudaHostAllocMapped));
        SBG_CUDA(cudaHostAlloc(&zc_->flag, sizeof(unsigned long long), cudaHostAllocMapped));
        *zc_->flag = 0;
        rws.zc = zc_.get();
    }
    SBG_CUDA(cudaMallocHost(&rws.host, kMaxRed * sizeof(double)));

    build_tables(h1, eri);
}

Context::~Context() {
    if (st) cudaStreamSynchronize(st);
    for (void* p : {(void*)d_sa_, (void*)d_sb_, (void*)d_la_, (void*)d_lb_, (void*)d_h1_, (void*)d_eri_, (void*)d_Vp_,
                    (void*)d_Va_, (void*)d_codes_, (void*)d_sc_tgt_, (void*)d_sc_ent_,
                    (void*)d_sc_tt_, (void*)d_sc_te_, (void*)rws.partial, (void*)rws.result, (void*)rws.ticket})
        if (p) cudaFree(p);
    if (rws.host) cudaFreeHost(rws.host);
    if (zc_) {
        cudaFreeHost(zc_->mirror);
        cudaFreeHost(zc_->flag);
    }
    for (auto& pr : red_pass_) {
        cudaFree(pr.first);
        cudaFree(pr.second);
    }
    for (auto& sp : csr_mem_)
        for (void* q : sp)
            if (q) cudaFree(q);
    comm_.reset();
    for (auto& es : ev_pool_)
        for (auto& e : es.e) cudaEventDestroy(e);
    for (auto& c : cs_)
        if (c) cudaStreamDestroy(c);
    if (ev0_) cudaEventDestroy(ev0_);
    if (ev1_) cudaEventDestroy(ev1_);
    if (ev_order_) cudaEventDestroy(ev_order_);
    if (ev_dots_) cudaEventDestroy(ev_dots_);
    for (cudaEvent_t e : {ev_in_, ev_gathered_, ev_aa_, ev_xdone_, ev_ab_})
        if (e) cudaEventDestroy(e);
    if (comm_st_) {
        cudaStreamSynchronize(comm_st_);
        cudaStreamDestroy(comm_st_);
    }
    if (st) cudaStreamDestroy(st);
}

DBuf Context::alloc_vec() const { return DBuf(padded_len()); }

cudaStream_t Context::copy_stream(int which) {
    if (!cs_[which]) SBG_CUDA(cudaStreamCreateWithFlags(&cs_[which], cudaStreamNonBlocking));
    return cs_[which];
}

void Context::build_tables(const double* h1, const double* eri) {
    const size_t n2 = (size_t)norb * norb, n4 = n2 * n2;
    d_h1_ = dmalloc<double>(n2);
    d_eri_ = dmalloc<double>(n4);
    SBG_CUDA(cudaMemcpyAsync(d_h1_, h1, n2 * 8, cudaMemcpyHostToDevice, st));
    SBG_CUDA(cudaMemcpyAsync(d_eri_, eri, n4 * 8, cudaMemcpyHostToDevice, st));
    d_sa_ = dmalloc<uint64_t>(NA);
    d_sb_ = dmalloc<uint64_t>(NB);
    launch_strings(d_sa_, NA, na_el, norb, st);
    launch_strings(d_sb_, NB, nb_el, norb, st);
    launches += 2;

    // exact diagonal (fci_operator.hpp:16-57)
    {
        double* ea = dmalloc<double>(NA);
        double* eb = dmalloc<double>(NB);
        launch_string_energy(d_sa_, NA, norb, d_h1_, d_eri_, ea, st);
        launch_string_energy(d_sb_, NB, norb, d_h1_, d_eri_, eb, st);
        diag_ = alloc_vec();
        launch_diag(d_sa_, d_sb_, ea, eb, row_lo, nrows, NB, ld, norb, d_eri_, e_core, diag_.p, st);
        launches += 3;
        SBG_CUDA(cudaStreamSynchronize(st));
        cudaFree(ea);
        cudaFree(eb);
    }

    auto g = [&](int p, int q, int r, int s) { return eri[((size_t)(p * norb + q) * norb + r) * norb + s]; };
    // alpha-beta integrals with both one-body terms folded (sigma_ab.cu header)
    have_ab_ = na_el > 0 && nb_el > 0;
    if (have_ab_) {
        const int np = norb * (norb + 1) / 2;
        std::vector<double> Vp((size_t)np * np);
        for (int p = 0; p < norb; ++p)
            for (int q = 0; q <= p; ++q)
                for (int r = 0; r < norb; ++r)
                    for (int s = 0; s <= r; ++s) {
                        double v = g(p, q, r, s);
                        if (r == s) v += h1[p * norb + q] / nb_el;
                        if (p == q) v += h1[r * norb + s] / na_el;
                        Vp[(size_t)pair_sym(p, q) * np + pair_sym(r, s)] = v;
                    }
        d_Vp_ = dmalloc<double>(Vp.size());
        SBG_CUDA(cudaMemcpyAsync(d_Vp_, Vp.data(), Vp.size() * 8, cudaMemcpyHostToDevice, st));
        SBG_CUDA(cudaStreamSynchronize(st));  // the host Vp buffer ends with this block
        try {
            ab_ = plan_sigma_ab(norb, na_el, nb_el, NA, NB, ld, nsm);
        } catch (const InvalidArgument&) {
            direct_ab_ = true;  // outside the tensor-core kernel's limits: link-table kernel
        }
    }
    if (have_ab_ && direct_ab_) {
        ensure_links();
    } else if (have_ab_) {
        d_codes_ = dmalloc<uint16_t>((size_t)ld * ab_.code_ld);
        launch_scatter_codes(d_sb_, NB, ld, norb, ab_.npair, ab_.code_ld, d_codes_, st);
        launches += 1;
        std::vector<uint16_t> codes((size_t)ld * ab_.code_ld);
        SBG_CUDA(cudaMemcpyAsync(codes.data(), d_codes_, codes.size() * 2, cudaMemcpyDeviceToHost, st));
        SBG_CUDA(cudaStreamSynchronize(st));  // Vp host buffer, codes
        std::vector<uint32_t> tgt, tt, te;
        std::vector<uint16_t> ent;
        build_ab_scatter(ab_, codes, tgt, ent, tt, te);
        d_sc_tgt_ = dmalloc<uint32_t>(tgt.size());
        d_sc_ent_ = dmalloc<uint16_t>(ent.size());
        d_sc_tt_ = dmalloc<uint32_t>(tt.size());
        d_sc_te_ = dmalloc<uint32_t>(te.size());
        SBG_CUDA(cudaMemcpyAsync(d_sc_tgt_, tgt.data(), tgt.size() * 4, cudaMemcpyHostToDevice, st));
        SBG_CUDA(cudaMemcpyAsync(d_sc_ent_, ent.data(), ent.size() * 2, cudaMemcpyHostToDevice, st));
        SBG_CUDA(cudaMemcpyAsync(d_sc_tt_, tt.data(), tt.size() * 4, cudaMemcpyHostToDevice, st));
        SBG_CUDA(cudaMemcpyAsync(d_sc_te_, te.data(), te.size() * 4, cudaMemcpyHostToDevice, st));
        if (ab_.red) {
            for (int pass = 0; pass < ab_.npass; ++pass) {  // one reduction list per pair-row block
                std::vector<uint32_t> e32, t32;
                build_ab_red_list(ab_, codes, e32, t32, pass * 128);
                uint32_t* de = dmalloc<uint32_t>(e32.size());
                uint32_t* dt = dmalloc<uint32_t>(t32.size());
                SBG_CUDA(cudaMemcpyAsync(de, e32.data(), e32.size() * 4, cudaMemcpyHostToDevice, st));
                SBG_CUDA(cudaMemcpyAsync(dt, t32.data(), t32.size() * 4, cudaMemcpyHostToDevice, st));
                SBG_CUDA(cudaStreamSynchronize(st));
                red_pass_.push_back({de, dt});
            }
            d_red_ent_ = red_pass_[0].first;
            d_red_te_ = red_pass_[0].second;
        }
        SBG_CUDA(cudaStreamSynchronize(st));
    }
    // same-spin antisymmetrized pair integrals W(pr,qs) = (pq|rs) - (ps|rq), p<r, q<s
    std::vector<double> Va_host;
    if (norb >= 2) {
        const int npa = norb * (norb - 1) / 2;
        std::vector<double>& Va = Va_host;
        Va.assign((size_t)npa * npa, 0.0);
        for (int r = 1; r < norb; ++r)
            for (int p = 0; p < r; ++p)
                for (int s = 1; s < norb; ++s)
                    for (int q = 0; q < s; ++q)
                        Va[(size_t)pair_strict(p, r) * npa + pair_strict(q, s)] = g(p, q, r, s) - g(p, s, r, q);
        d_Va_ = dmalloc<double>(Va.size());
        SBG_CUDA(cudaMemcpyAsync(d_Va_, Va.data(), Va.size() * 8, cudaMemcpyHostToDevice, st));
        SBG_CUDA(cudaStreamSynchronize(st));
    }
    for (int spin = 0; spin < 2; ++spin) {
        const int nel = spin ? nb_el : na_el;
        SsPlan& pl = spin ? ssb_ : ssa_;
        try {
            pl = plan_sigma_ss(norb, nel);
        } catch (const InvalidArgument&) {
            // more pair rows than the tensor-core kernel holds: CSR of the one-spin operator
            pl = SsPlan{};
            SsCsr m;
            build_ss_csr(norb, nel, Va_host.data(), m);
            int64_t* rp = dmalloc<int64_t>(m.rowptr.size());
            int* cl = dmalloc<int>(m.col.size());
            double* vl = dmalloc<double>(m.val.size());
            SBG_CUDA(cudaMemcpy(rp, m.rowptr.data(), m.rowptr.size() * 8, cudaMemcpyHostToDevice));
            if (!m.col.empty()) {
                SBG_CUDA(cudaMemcpy(cl, m.col.data(), m.col.size() * 4, cudaMemcpyHostToDevice));
                SBG_CUDA(cudaMemcpy(vl, m.val.data(), m.val.size() * 8, cudaMemcpyHostToDevice));
            }
            csr_mem_[spin][0] = rp;
            csr_mem_[spin][1] = cl;
            csr_mem_[spin][2] = vl;
            csr_dev_[spin] = SsCsrDev{m.nstr, rp, cl, vl};
            ss_csr_[spin] = true;
            csr_nnz_[spin] = (double)m.col.size();
        }
    }
    if (!have_ab_) ensure_links();

    // flop accounting: useful (unpadded) multiply-adds x 2
    flops_ab = !have_ab_ ? 0.0
               : direct_ab_ ? 2.0 * (double)row_len(0) * (double)row_len(1) * (double)ndet
                            : 2.0 * ab_.npair * ab_.K * (double)ndet;
    flops_ss = (ss_csr_[0] ? 2.0 * csr_nnz_[0] * NB : 2.0 * ssa_.P * ssa_.P * (double)ssa_.NK * NB) +
               (ss_csr_[1] ? 2.0 * csr_nnz_[1] * NA : 2.0 * ssb_.P * ssb_.P * (double)ssb_.NK * NA);

    // workspaces
    // workspaces beyond the shards: the gathered x is full size by construction; the
    // alpha-alpha window (all rows x this rank's beta-column window) and its send buffer are
    // NA x window, the transposed beta-beta operands nrows wide
    if (world > 1) {
        const int64_t per = (NA + world - 1) / world;
        xfull_ = DBuf(per * world * ld);
        shard_range(NB, rank, world, &aa_lo_, &aa_hi_);
        aa_c0_ = aa_lo_ / 32 * 32;
        ldw_ = round_up(std::max<int64_t>(aa_hi_ - aa_c0_, 1), 32);
        saa_ = DBuf(NA * ldw_);
        a2a_send_ = DBuf(NA * std::max<int64_t>(aa_hi_ - aa_lo_, 1));
        a2a_recv_ = DBuf(nrows * ld);
    }
    if (has_ss(1)) {
        xT_ = DBuf(NB * ldT);
        sT_ = DBuf(NB * ldT);
    }
    SBG_CUDA(cudaStreamSynchronize(st));
}

void Context::ensure_links() {
    if (d_la_) return;
    d_la_ = dmalloc<Excitation>((size_t)NA * row_len(0));
    d_lb_ = dmalloc<Excitation>((size_t)NB * row_len(1));
    launch_links(d_sa_, NA, norb, (int)row_len(0), d_la_, st);
    launch_links(d_sb_, NB, norb, (int)row_len(1), d_lb_, st);
    launches += 2;
    SBG_CUDA(cudaStreamSynchronize(st));
}

int64_t Context::row_len(int spin) const {
    const int k = spin == 0 ? na_el : nb_el;
    return (int64_t)k * (norb - k + 1);
}

void Context::string_tables(int spin, uint64_t* strings, Excitation* links) {
    const int64_t n = spin == 0 ? NA : NB;
    if (strings)
        SBG_CUDA(cudaMemcpyAsync(strings, spin == 0 ? d_sa_ : d_sb_, n * 8, cudaMemcpyDeviceToHost, st));
    if (links) {
        ensure_links();
        SBG_CUDA(cudaMemcpyAsync(links, spin == 0 ? d_la_ : d_lb_, (size_t)n * row_len(spin) * sizeof(Excitation),
                                 cudaMemcpyDeviceToHost, st));
    }
    SBG_CUDA(cudaStreamSynchronize(st));
}

void Context::upload_local(const double* host_dense_full, double* d_padded, cudaStream_t s) const {
    if (nrows == 0) return;
    SBG_CUDA(cudaMemcpy2DAsync(d_padded, ld * 8, host_dense_full + row_lo * NB, NB * 8, NB * 8, nrows,
                               cudaMemcpyHostToDevice, s));
}
void Context::download_local(const double* d_padded, double* host_dense_local, cudaStream_t s) const {
    if (nrows == 0) return;
    SBG_CUDA(cudaMemcpy2DAsync(host_dense_local, NB * 8, d_padded, ld * 8, NB * 8, nrows, cudaMemcpyDeviceToHost, s));
}
void Context::upload_rows(const double* host_dense_full, double* d_padded, int64_t lo, int64_t hi,
                          cudaStream_t s) const {
    if (hi <= lo) return;
    SBG_CUDA(cudaMemcpy2DAsync(d_padded + lo * ld, ld * 8, host_dense_full + (row_lo + lo) * NB, NB * 8, NB * 8, hi - lo,
                               cudaMemcpyHostToDevice, s));
}
void Context::download_rows(const double* d_padded, double* host_dense_local, int64_t lo, int64_t hi,
                            cudaStream_t s) const {
    if (hi <= lo) return;
    SBG_CUDA(cudaMemcpy2DAsync(host_dense_local + lo * NB, NB * 8, d_padded + lo * ld, ld * 8, NB * 8, hi - lo,
                               cudaMemcpyDeviceToHost, s));
}
void Context::pack_device(const double* d_dense_full, double* d_padded, cudaStream_t s) const {
    if (nrows == 0) return;
    SBG_CUDA(cudaMemcpy2DAsync(d_padded, ld * 8, d_dense_full + row_lo * NB, NB * 8, NB * 8, nrows,
                               cudaMemcpyDeviceToDevice, s));
}
void Context::unpack_device(const double* d_padded, double* d_dense_local, cudaStream_t s) const {
    if (nrows == 0) return;
    SBG_CUDA(cudaMemcpy2DAsync(d_dense_local, NB * 8, d_padded, ld * 8, NB * 8, nrows, cudaMemcpyDeviceToDevice, s));
}

void Context::gather_full(const double* x_local, cudaStream_t s) {
    const int64_t per = (NA + world - 1) / world;
    // every rank contributes `per` rows (zero rows past NA on the last ranks)
    SBG_CUDA(cudaMemsetAsync(xfull_.p + (int64_t)rank * per * ld, 0, per * ld * 8, s));
    if (nrows > 0)
        SBG_CUDA(cudaMemcpyAsync(xfull_.p + (int64_t)rank * per * ld, x_local, nrows * ld * 8,
                                 cudaMemcpyDeviceToDevice, s));
    comm_->all_gather(xfull_.p + (int64_t)rank * per * ld, xfull_.p, (size_t)(per * ld), s);
}

double Context::spin_squared(const double* x_local) {
    const double* v[1] = {x_local};
    launch_gram(v, 1, padded_len(), rws, st);
    launches += 1;
    const double xx = finish_dots(1)[0];
    if (!(xx > 0.0)) throw std::invalid_argument("spin_squared: zero vector");
    const double sz = 0.5 * (na_el - nb_el);
    double raised_sq = 0.0;
    if (nb_el > 0 && na_el < norb) {
        const double* xf = x_local;
        if (world > 1) {
            gather_full(x_local, st);
            xf = xfull_.p;
        }
        int64_t lo, hi;
        shard_range((int64_t)binom_host_calc(norb, na_el + 1), rank, world, &lo, &hi);
        if (hi > lo) {
            launch_spin_raise(xf, ld, na_el, nb_el, norb, lo, hi, rws, st);
            launches += 2;
        } else {
            SBG_CUDA(cudaMemsetAsync(rws.result, 0, 8, st));
            if (zc_) zc_->fresh = false;
        }
        raised_sq = finish_dots(1)[0];
    }
    return raised_sq / xx + sz * (sz + 1.0);
}

void Context::allreduce_inplace_device(double* d, int count) {
    if (world > 1 && count > 0) comm_->all_reduce_sum(d, (size_t)count, st);
}

// Zero-copy wait: the finishing block of the latest pass with dots writes them into mapped host
// memory and then sets the flag to that pass's sequence number. Polls with a stream query every few
// thousand spins, so a stream that drained without setting the flag (cannot happen for the passes
// that advance the sequence) falls back to the copy path instead of hanging.
bool Context::poll_zero_copy(unsigned long long seq) {
    volatile unsigned long long* flag = zc_->flag;
    for (unsigned spins = 1;; ++spins) {
        if (*flag >= seq) return true;
        if ((spins & 4095u) == 0) {
            const cudaError_t q = cudaStreamQuery(st);
            if (q == cudaSuccess) return *flag >= seq;
            if (q != cudaErrorNotReady) SBG_CUDA(q);
        }
    }
}

void Context::post_dots(int ndot) {
    if (zc_ && zc_->fresh) {  // the flag is the completion signal: nothing to enqueue
        zc_->fresh = false;
        post_seq_ = zc_->seq;
        post_n_ = ndot;
        return;
    }
    post_seq_ = 0;
    allreduce_inplace_device(rws.result, ndot);
    SBG_CUDA(cudaMemcpyAsync(rws.host, rws.result, ndot * 8, cudaMemcpyDeviceToHost, st));
    SBG_CUDA(cudaEventRecord(ev_dots_, st));
}

const double* Context::wait_dots() {
    if (post_seq_ && poll_zero_copy(post_seq_)) {
        std::memcpy(rws.host, (const void*)zc_->mirror, post_n_ * sizeof(double));
        return rws.host;
    }
    if (post_seq_) {  // fallback: the copy path
        SBG_CUDA(cudaMemcpyAsync(rws.host, rws.result, post_n_ * 8, cudaMemcpyDeviceToHost, st));
        SBG_CUDA(cudaStreamSynchronize(st));
        return rws.host;
    }
    SBG_CUDA(cudaEventSynchronize(ev_dots_));
    return rws.host;
}

const double* Context::finish_dots(int ndot) {
    if (zc_ && zc_->fresh) {
        zc_->fresh = false;
        if (poll_zero_copy(zc_->seq)) {
            std::memcpy(rws.host, (const void*)zc_->mirror, ndot * sizeof(double));
            return rws.host;
        }
    }
    allreduce_inplace_device(rws.result, ndot);
    SBG_CUDA(cudaMemcpyAsync(rws.host, rws.result, ndot * 8, cudaMemcpyDeviceToHost, st));
    SBG_CUDA(cudaStreamSynchronize(st));
    return rws.host;
}

// y = H x (SymmetricOperator::apply, operator.hpp:25-31). Kernel sequence:
//   1. [world>1] all-gather x over NVLink (the only data-path collective of a sigma build)
//   2. beta-beta: transpose x -> x^T, same-spin kernel on x^T, transpose back into y (local rows)
//   3. alpha-alpha: same-spin kernel on x, fp64 reductions into y (world>1: column window +
//      all-to-all of the blocks)
//   4. alpha-beta + one-body + e_core: sigma_ab, accumulating into y
// the tensor-core opposite-spin kernel on rows [lo, hi), one launch per pair-row block
void Context::run_ab(const double* x_full, double* y_rows, int64_t lo, int64_t hi, cudaStream_t s) {
    for (int pass = 0; pass < ab_.npass; ++pass) {
        const uint32_t* re = red_pass_.empty() ? nullptr : red_pass_[pass].first;
        const uint32_t* rt = red_pass_.empty() ? nullptr : red_pass_[pass].second;
        launch_sigma_ab(ab_, AbScatter{d_sc_tgt_, d_sc_ent_, d_sc_tt_, d_sc_te_, re, rt}, x_full, y_rows, d_Vp_, lo, hi,
                        e_core, 1, nsm, s, pass);
        launches += 1;
    }
}

void Context::run_ss(int spin, const double* x, double* y, int64_t ldx, int64_t col_lo, int64_t col_hi,
                     cudaStream_t s, int64_t ldy, int64_t ycol0, int64_t col_pad) {
    if (ss_csr_[spin]) launch_sigma_ss_csr(csr_dev_[spin], x, y, ldx, col_lo, col_hi, s, ldy, ycol0);
    else launch_sigma_ss(spin ? ssb_ : ssa_, x, y, d_Va_, ldx, col_lo, col_hi, s, ldy, ycol0, col_pad);
}

// rows [lo, hi) of block i of nchunks: equal blocks on a 32-row grid
void Context::chunk_rows(int nchunks, int i, int64_t* lo, int64_t* hi) const {
    const int64_t per = round_up((nrows + nchunks - 1) / nchunks, 32);
    *lo = std::min<int64_t>(nrows, (int64_t)i * per);
    *hi = std::min<int64_t>(nrows, *lo + per);
}

void Context::sigma_rowblocks(const double* x_local, double* y_local, cudaStream_t s, int nchunks,
                              const cudaEvent_t* x_ready, const cudaEvent_t* y_done) {
    if (world != 1 || !have_ab_ || nchunks < 1) throw InvalidArgument("sigma_rowblocks: single-GPU two-spin sectors only");
    order_begin(s);
    EvSet* ev = next_evset();
    if (ev) {
        SBG_CUDA(cudaEventRecord(ev->e[0], s));
        SBG_CUDA(cudaEventRecord(ev->e[1], s));
    }
    // ---- beta-beta, block by block as the rows arrive (transpose -> same-spin -> transpose back)
    for (int i = 0; i < nchunks; ++i) {
        int64_t lo, hi;
        chunk_rows(nchunks, i, &lo, &hi);
        SBG_CUDA(cudaStreamWaitEvent(s, x_ready[i], 0));
        if (hi <= lo) continue;
        if (ssb_.P > 0) {
            launch_transpose(x_local + lo * ld, hi - lo, NB, ld, xT_.p + lo, ldT, NB, hi - lo, 0, s);
            SBG_CUDA(cudaMemset2DAsync(sT_.p + lo, ldT * 8, 0, (hi - lo) * 8, NB, s));
            launch_sigma_ss(ssb_, xT_.p, sT_.p, d_Va_, ldT, lo, hi, s, 0, 0, hi == nrows ? ldT : 0);
            launch_transpose(sT_.p + lo, NB, hi - lo, ldT, y_local + lo * ld, ld, hi - lo, ld, 0, s);
            launches += 3;
        } else {
            SBG_CUDA(cudaMemsetAsync(y_local + lo * ld, 0, (size_t)(hi - lo) * ld * 8, s));
        }
    }
    // ---- alpha-alpha (all rows: x complete)
    if (ssa_.P > 0) {
        launch_sigma_ss(ssa_, x_local, y_local, d_Va_, ld, 0, NB, s, 0, 0, ld);
        launches += 1;
    }
    if (ev) {
        SBG_CUDA(cudaEventRecord(ev->e[2], s));
        SBG_CUDA(cudaEventRecord(ev->e[3], s));
    }
    // ---- alpha-beta per block: rows of block i are final after its launch
    for (int i = 0; i < nchunks; ++i) {
        int64_t lo, hi;
        chunk_rows(nchunks, i, &lo, &hi);
        if (hi > lo) run_ab(x_local, y_local + lo * ld, lo, hi, s);
        SBG_CUDA(cudaEventRecord(y_done[i], s));
    }
    if (ev) SBG_CUDA(cudaEventRecord(ev->e[4], s));
    order_end(s);
    applies_.fetch_add(1, std::memory_order_relaxed);
}

void Context::order_begin(cudaStream_t s) {
    if (order_recorded_) SBG_CUDA(cudaStreamWaitEvent(s, ev_order_, 0));
}
void Context::order_end(cudaStream_t s) {
    SBG_CUDA(cudaEventRecord(ev_order_, s));
    order_recorded_ = true;
}

void Context::sigma_multi(const double* const* x, double* const* y, int nvec, cudaStream_t s) {
    const bool fused = nvec > 1 && nvec <= kMaxSigmaVec && world == 1 && have_ab_ && !direct_ab_ && ab_.tma &&
                       ab_.npass == 1 && !ss_csr_[0] && !ss_csr_[1] && (ssa_.P == 0 || ssa_.bulk);
    if (!fused) {
        for (int v = 0; v < nvec; ++v) sigma(x[v], y[v], s);
        return;
    }
    order_begin(s);
    EvSet* ev = next_evset();
    if (ev) {
        SBG_CUDA(cudaEventRecord(ev->e[0], s));
        SBG_CUDA(cudaEventRecord(ev->e[1], s));
    }
    // beta-beta per vector (the transposed operands are one vector's worth of scratch)
    for (int v = 0; v < nvec; ++v) {
        if (has_ss(1)) {
            launch_transpose(x[v], nrows, NB, ld, xT_.p, ldT, NB, ldT, 0, s);
            SBG_CUDA(cudaMemsetAsync(sT_.p, 0, (size_t)NB * ldT * 8, s));
            run_ss(1, xT_.p, sT_.p, ldT, 0, nrows, s, 0, 0, ldT);
            launch_transpose(sT_.p, NB, nrows, ldT, y[v], ld, nrows, ld, 0, s);
            launches += 3;
        } else {
            SBG_CUDA(cudaMemsetAsync(y[v], 0, (size_t)nrows * ld * 8, s));
        }
    }
    // alpha-alpha: every vector in one launch
    if (ssa_.P > 0) {
        launch_sigma_ss_multi(ssa_, x, y, nvec, d_Va_, ld, 0, NB, s, 0, 0, ld);
        launches += 1;
    }
    if (ev) {
        SBG_CUDA(cudaEventRecord(ev->e[2], s));
        SBG_CUDA(cudaEventRecord(ev->e[3], s));
    }
    // alpha-beta + one-body + e_core: every vector in one launch
    launch_sigma_ab_multi(ab_, AbScatter{d_sc_tgt_, d_sc_ent_, d_sc_tt_, d_sc_te_, red_pass_[0].first, red_pass_[0].second},
                          x, y, nvec, d_Vp_, row_lo, row_hi, e_core, 1, nsm, s, 0);
    launches += 1;
    if (ev) SBG_CUDA(cudaEventRecord(ev->e[4], s));
    order_end(s);
    applies_.fetch_add((uint64_t)nvec, std::memory_order_relaxed);
}

Context::EvSet* Context::next_evset() {
    if (ev_used_ == ev_pool_.size()) {
        if (ev_pool_.size() >= 256) return nullptr;  // profile ring full: stop recording until read/reset
        EvSet es;
        for (auto& e : es.e) SBG_CUDA(cudaEventCreate(&e));
        ev_pool_.push_back(es);
    }
    return &ev_pool_[ev_used_++];
}

void Context::profile_reset() {
    SBG_CUDA(cudaStreamSynchronize(st));
    ev_used_ = 0;
    prof_calls_ = 0;
    for (double& v : prof_ms_) v = 0.0;
}

void Context::profile_read(double* ms, int64_t* calls) {
    SBG_CUDA(cudaDeviceSynchronize());
    for (size_t i = 0; i < ev_used_; ++i) {
        float t[4];
        const auto& e = ev_pool_[i].e;
        SBG_CUDA(cudaEventElapsedTime(&t[0], e[3], e[4]));  // alpha-beta (+ the exchange it hides)
        SBG_CUDA(cudaEventElapsedTime(&t[1], e[0], e[3]));  // same-spin + transposes (+ all-gather wait)
        SBG_CUDA(cudaEventElapsedTime(&t[2], e[0], e[1]));  // all-gather (overlapped with beta-beta)
        SBG_CUDA(cudaEventElapsedTime(&t[3], e[0], e[4]));  // whole sigma
        for (int k = 0; k < 4; ++k) prof_ms_[k] += t[k];
        ++prof_calls_;
    }
    ev_used_ = 0;
    for (int k = 0; k < 4; ++k) ms[k] = prof_ms_[k];
    *calls = prof_calls_;
}

void Context::sigma(const double* x_local, double* y_local, cudaStream_t s) {
    order_begin(s);
    EvSet* ev = next_evset();
    if (ev) SBG_CUDA(cudaEventRecord(ev->e[0], s));
    const double* xf = x_local;
    if (world > 1) {
        // (1) all-gather of x on the comm stream, beside the beta-beta term (row-local)
        SBG_CUDA(cudaEventRecord(ev_in_, s));
        SBG_CUDA(cudaStreamWaitEvent(comm_st_, ev_in_, 0));
        xf = xfull_.p;
    } else if (ev) {
        SBG_CUDA(cudaEventRecord(ev->e[1], s));
    }
    bool y_written = false;
    // ---- beta-beta via the transpose: only this rank's alpha rows (columns of x^T) are needed
    if (has_ss(1)) {
        // x^T of the local rows: [NB][ldT], column r = local alpha row r
        launch_transpose(x_local, nrows, NB, ld, xT_.p, ldT, NB, ldT, 0, s);
        SBG_CUDA(cudaMemsetAsync(sT_.p, 0, (size_t)NB * ldT * 8, s));
        run_ss(1, xT_.p, sT_.p, ldT, 0, nrows, s, 0, 0, ldT);
        // y[r][c] = sT[c][r]
        launch_transpose(sT_.p, NB, nrows, ldT, y_local, ld, nrows, ld, 0, s);
        launches += 3;
        y_written = true;
    }
    if (!y_written) SBG_CUDA(cudaMemsetAsync(y_local, 0, (size_t)nrows * ld * 8, s));
    if (world > 1) {
        // enqueued after the beta-beta kernels: a host-synchronous comm (LocalComm) then overlaps them
        gather_full(x_local, comm_st_);
        if (ev) SBG_CUDA(cudaEventRecord(ev->e[1], comm_st_));
        SBG_CUDA(cudaEventRecord(ev_gathered_, comm_st_));
        SBG_CUDA(cudaStreamWaitEvent(s, ev_gathered_, 0));
    }
    // ---- alpha-alpha
    bool exchange = false;
    if (has_ss(0)) {
        if (world == 1) {
            run_ss(0, xf, y_local, ld, 0, NB, s, 0, 0, ld);
            launches += 1;
        } else {
            const int64_t clo = aa_lo_, chi = aa_hi_;
            if (chi > clo) SBG_CUDA(cudaMemset2DAsync(saa_.p + (clo - aa_c0_), ldw_ * 8, 0, (chi - clo) * 8, NA, s));
            run_ss(0, xf, saa_.p, ld, clo, chi, s, ldw_, aa_c0_, chi == NB ? ld : 0);
            launches += 1;
            SBG_CUDA(cudaEventRecord(ev_aa_, s));
            exchange = true;
        }
    }
    if (ev) {
        SBG_CUDA(cudaEventRecord(ev->e[2], s));
        SBG_CUDA(cudaEventRecord(ev->e[3], s));
    }
    // ---- alpha-beta (+ one-body folded, + e_core); with world > 1 it runs while the alpha-alpha
    // blocks are exchanged on the comm stream (both reduce into y)
    if (have_ab_ && direct_ab_) {
        launch_sigma_ab_direct(xf, y_local, d_Vp_, norb * (norb + 1) / 2, d_la_, (int)row_len(0), d_lb_,
                               (int)row_len(1), row_lo, row_hi, NB, ld, e_core, s);
        launches += 1;
    } else if (have_ab_) {
        run_ab(xf, y_local, row_lo, row_hi, s);
    } else {
        ensure_links();
        // rows of this rank: the one-body kernel works on full-height buffers; single GPU only
        if (world > 1) throw InvalidArgument("single-spin sectors are not supported across ranks");
        launch_onebody(xf, y_local, d_la_, (int)row_len(0), d_lb_, (int)row_len(1), d_h1_, norb, NA, NB, ld, e_core,
                       1, s);
        launches += 1;
    }
    if (exchange) SBG_CUDA(cudaEventRecord(ev_ab_, s));
    if (exchange) {
        // all-to-all of the alpha-alpha column window: send rows of rank r' restricted to my column
        // window; receive my rows of every rank's window
        cudaStream_t cs = comm_st_;
        SBG_CUDA(cudaStreamWaitEvent(cs, ev_aa_, 0));
        const int64_t clo = aa_lo_, chi = aa_hi_;
        const int64_t wl = chi - clo;
        std::vector<int64_t> rlo(world), rhi(world), cwl(world), cwh(world);
        for (int r = 0; r < world; ++r) {
            shard_range(NA, r, world, &rlo[r], &rhi[r]);
            shard_range(NB, r, world, &cwl[r], &cwh[r]);
        }
        int64_t off = 0;
        for (int r = 0; r < world; ++r) {
            const int64_t nr = rhi[r] - rlo[r];
            if (nr > 0 && wl > 0)
                SBG_CUDA(cudaMemcpy2DAsync(a2a_send_.p + off, wl * 8, saa_.p + rlo[r] * ldw_ + (clo - aa_c0_), ldw_ * 8, wl * 8, nr,
                                           cudaMemcpyDeviceToDevice, cs));
            off += nr * wl;
        }
        std::vector<CommBlock> sends, recvs;
        off = 0;
        int64_t roff = 0;
        for (int r = 0; r < world; ++r) {
            const int64_t nr = rhi[r] - rlo[r];
            const int64_t rw = cwh[r] - cwl[r];
            if (r != rank) {
                if (nr * wl > 0) sends.push_back({a2a_send_.p + off, (size_t)(nr * wl), r});
                if (nrows * rw > 0) recvs.push_back({a2a_recv_.p + roff, (size_t)(nrows * rw), r});
            } else if (nrows * rw > 0) {
                SBG_CUDA(cudaMemcpyAsync(a2a_recv_.p + roff, a2a_send_.p + off, nrows * rw * 8, cudaMemcpyDeviceToDevice,
                                         cs));
            }
            off += nr * wl;
            roff += nrows * rw;
        }
        comm_->exchange(sends, recvs, cs);
        // the blocks travel beside the alpha-beta kernel; adding them into y may too only when that
        // kernel reduces atomically — otherwise after it (its plain row updates would lose ours)
        if (!ab_reduces()) SBG_CUDA(cudaStreamWaitEvent(cs, ev_ab_, 0));
        roff = 0;
        for (int r = 0; r < world; ++r) {
            const int64_t rw = cwh[r] - cwl[r];
            if (nrows * rw > 0) {
                const int64_t n = nrows * rw;
                k_add_block<<<(unsigned)((n + 255) / 256), 256, 0, cs>>>(y_local + cwl[r], ld, a2a_recv_.p + roff, nrows,
                                                                         rw);
                SBG_LAUNCH_CHECK();
                launches += 1;
            }
            roff += nrows * rw;
        }
        SBG_CUDA(cudaEventRecord(ev_xdone_, cs));
        SBG_CUDA(cudaStreamWaitEvent(s, ev_xdone_, 0));
    }
    if (ev) SBG_CUDA(cudaEventRecord(ev->e[4], s));
    order_end(s);
    applies_.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace sbg
