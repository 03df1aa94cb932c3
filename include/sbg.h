/*
 * sbg.h — C ABI of the B200-native SBCI sigma / update hot path (libsbg.so).
 *
 * This is the drop-in boundary for the reference's operator plugin API
 * (/root/reference/proj/include/sbci/operator.hpp:19-48, fci/fci_operator.hpp:60-120) and its
 * solver entry points (sbci1.hpp:526-579, sbci2.hpp:527-623). Plain pointers and sizes only:
 * no C++ or torch types cross this line. Every call returns an error code; the message of the
 * last failure on the calling thread is available from sbg_last_error().
 *
 *   SBG_OK            0
 *   SBG_EINVAL        1   maps to std::invalid_argument in the reference (operator.hpp:26, sigma.hpp:92, ...)
 *   SBG_ENONCONV      2   maps to sbci::NonConvergenceError (config.hpp:92-100); CLI exit code 2
 *   SBG_EDEVICE       3   CUDA / NCCL failure (no reference equivalent; never silently downgraded)
 *   SBG_ERUNTIME      4   maps to std::runtime_error (e.g. the determinant guard, fci_operator.hpp:107-109)
 *
 * Vectors crossing the ABI are dense, alpha-major (det = ia * n_beta_strings + ib,
 * determinants.hpp:73), fp64, length sbg_dim(). Inside the library they live in HBM as padded
 * row blocks; the padding never crosses the ABI.
 */
#ifndef SBG_H
#define SBG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define SBG_OK 0
#define SBG_EINVAL 1
#define SBG_ENONCONV 2
#define SBG_EDEVICE 3
#define SBG_ERUNTIME 4

typedef struct sbg_ctx sbg_ctx;

/* One single-excitation table entry: a+_p a_q |source> = sign |target>.
 * Mirrors sbci::fci::Excitation (fci/sigma.hpp:19-23) byte for byte (16 bytes). */
typedef struct sbg_excitation {
    uint16_t p, q;
    uint32_t target;
    double sign;
} sbg_excitation;

/* Mirrors sbci::SolverConfig (config.hpp:10-60); sbg_config_default() gives the reference defaults. */
typedef struct sbg_config {
    double eps0, r0, b_th, eps1, x_th1, x_th2, r1;
    int32_t max_cycle;          /* 0 = method default (20 sbci1, 10 sbci2) */
    int32_t hx_refresh_restarts;
    int64_t t_max;
    double lindep, clamp_delta;
} sbg_config;

/* Per-state and per-run results (ConvergedEigenpair sbci1.hpp:27-34, RunSummary trace.hpp:212-221). */
#define SBG_MAX_ROOTS 64
typedef struct sbg_stats {
    int32_t nroots;
    int32_t iterations[SBG_MAX_ROOTS];
    int32_t restarts[SBG_MAX_ROOTS];
    double final_residual[SBG_MAX_ROOTS];
    uint64_t matvecs;
    int64_t total_iterations;
    int32_t total_restarts;
    int32_t hx_refreshes;
    int32_t peak_vectors;
    double wall_time_s;
    /* filled on SBG_ENONCONV (NonConvergenceError{state, best_energy, best_residual}) */
    int32_t failed_state;
    double best_energy, best_residual;
    /* device-side accounting for the bench */
    double sigma_seconds;       /* summed sigma time (CUDA events) */
    uint64_t kernel_launches;   /* kernels launched by the library during the call */
    /* <S^2> of each returned state (fci/spin.hpp:17-51, the CLI summary's s_squared column) */
    double s_squared[SBG_MAX_ROOTS];
    /* length-n_det solver vectors resident in HBM at once during the call (peak_vectors keeps the
     * reference's own formula, 7 + deflated states for SBCI1) */
    int32_t device_vectors_peak;
} sbg_stats;

/* Per-iteration trace record (TraceRecord trace.hpp:22-44). Fields a method does not produce are NaN. */
typedef struct sbg_trace_record {
    int32_t state, t;
    double energy, dE, res_norm, x_norm, kinetic;
    uint64_t matvecs;
    int32_t restart_reason; /* -1 none, else RestartReason (0 stall_small_b, 1 norm_out_of_range, 2 residual_blowup, 3 max_cycle) */
    double b, c;            /* sbci2: the diagonal (alpha,alpha) coefficients */
    int32_t method;         /* 1 sbci1, 2 sbci2, 3 davidson */
    int32_t pair_partner;   /* alpha+1 for sbci2 rows, else -1 */
    double b_ab, b_ba, b_bb, c_ab, c_ba, c_bb, a_ab, a_ba;
    double energy_partner, x_norm_partner, res_norm_partner;
} sbg_trace_record;
typedef void (*sbg_trace_fn)(const sbg_trace_record* rec, void* user);

/* ---- host-only helpers (no GPU needed) ---- */
const char* sbg_last_error(void);
const char* sbg_version(void);
uint64_t sbg_binomial(int n, int k);                                  /* determinants.hpp:17-31 */
/* Diagnostics (host logic only, no GPU needed): the launch plan of the opposite-spin kernel for a
 * sector. out[0..15] = k-steps, tile columns, m16 blocks, extra-row block, rank-1 epilogue (K0E),
 * TALL, uniform stream (0/1/2), D stages of the mbarrier hand-offs (0 = named barriers), bulk-copied
 * lists, pair-row passes, dynamic shared memory in bytes, staged G rows, G row stride, list buffer
 * (u16 slots), threads, reduction mode. SBG_EINVAL when the sector is outside the tensor-core
 * kernel's limits (the operator then uses the link-table kernel). */
int sbg_ab_plan_info(int norb, int n_alpha, int n_beta, int64_t* out16);
int sbg_determinant_count(int norb, int n_alpha, int n_beta, uint64_t* out); /* determinants.hpp:33-37 */
sbg_config sbg_config_default(void);                                  /* config.hpp:11-22 */
int sbg_config_validate(const sbg_config* cfg);                       /* config.hpp:26-43 */
/* BASELINE.json synthetic integrals (pinned generator). h1[norb^2], eri[norb^4]. */
int sbg_synthetic_integrals(int norb, uint64_t seed, double offdiag_scale, double* h1, double* eri);
/* alpha-string block owned by `rank` of `world` (SURVEY §8e partition). */
int sbg_shard_range(int64_t n_alpha_strings, int rank, int world, int64_t* lo, int64_t* hi);
int sbg_device_count(void);

/* ---- operator (replaces as_operator + FciOperator, fci_operator.hpp:60-120) ----
 * nelec/ms2 define the sector as in FciProblem (n_alpha = (nelec+ms2)/2). eri must hold all eight
 * permutations (fcidump.hpp:53-65). max_det is the determinant guard (kDefaultDeterminantGuard =
 * 5,000,000 in the reference); the guard message matches the reference's. */
int sbg_create(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri,
               int device, uint64_t max_det, sbg_ctx** out);
/* Distributed variant: one rank per GPU, CI vector sharded by alpha-string blocks.
 * nccl_unique_id points at the 128-byte ncclUniqueId created on rank 0 (world > 1). */
int sbg_create_dist(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri,
                    int device, uint64_t max_det, int rank, int world, const void* nccl_unique_id,
                    sbg_ctx** out);
int sbg_nccl_unique_id(void* out128);
/* Testing aid for the sharded path without several GPUs: the ranks of a group are threads of one
 * process (each calls the collective entry points — sbg_sigma*, sbg_solve, sbg_spin_squared — on
 * its own context concurrently); collectives run through host barriers and device copies. Same
 * partition and kernels as sbg_create_dist. */
typedef struct sbg_local_group sbg_local_group;
int sbg_local_group_create(int world, sbg_local_group** out);
void sbg_local_group_destroy(sbg_local_group* group);
int sbg_create_local(int norb, int nelec, int ms2, double e_core, const double* h1, const double* eri,
                     int device, uint64_t max_det, sbg_local_group* group, int rank, sbg_ctx** out);
void sbg_destroy(sbg_ctx* ctx);

int64_t sbg_dim(const sbg_ctx* ctx);                                 /* SymmetricOperator::dim */
int sbg_sector(const sbg_ctx* ctx, int* norb, int* n_alpha, int* n_beta, int64_t* n_alpha_strings,
               int64_t* n_beta_strings);
int sbg_local_rows(const sbg_ctx* ctx, int64_t* lo, int64_t* hi);    /* alpha rows owned by this rank */
/* Exact diagonal <D|H|D> (fci_operator.hpp:16-57), bit-identical to the reference. Host buffer, n_det. */
int sbg_diagonal(sbg_ctx* ctx, double* out);
/* Strings (u64[n_strings]) and link table (sbg_excitation[n_strings * L], row-major, reference order)
 * of one spin channel (0 = alpha, 1 = beta). Either pointer may be NULL. */
int sbg_table_sizes(const sbg_ctx* ctx, int spin, int64_t* n_strings, int64_t* row_len);
int sbg_string_tables(sbg_ctx* ctx, int spin, uint64_t* strings, sbg_excitation* links);

/* sigma = H x for nvec vectors (host buffers, each n_det). Counts nvec applications
 * (SymmetricOperator::apply, operator.hpp:25-31). x and y may not alias. nvec > 1 pipelines the
 * uploads and downloads of neighbouring vectors behind the sigma builds (pinned buffers overlap). */
int sbg_sigma(sbg_ctx* ctx, const double* x, double* y, int nvec);
/* Same on dense device buffers (n_det each) on the given cudaStream_t (NULL = library stream).
 * Inputs already resident in HBM; used by the bench's device-resident leg. */
int sbg_sigma_device(sbg_ctx* ctx, const double* d_x, double* d_y, void* stream);
/* Padded-layout device entry points (no pack/unpack), for the throughput bench:
 * buffers of sbg_padded_len() doubles in the library's internal layout (local rows only). */
int64_t sbg_padded_len(const sbg_ctx* ctx);
int sbg_pack(sbg_ctx* ctx, const double* d_dense_full, double* d_padded_local, void* stream);
int sbg_unpack(sbg_ctx* ctx, const double* d_padded_local, double* d_dense_local, void* stream);
int sbg_sigma_padded(sbg_ctx* ctx, const double* d_x_padded_local, double* d_y_padded_local, void* stream);
/* nvec sigma builds in one pass (padded device buffers, counts nvec applications): on one GPU the
 * opposite-spin and alpha-alpha kernels take every vector in one launch, paying their per-row /
 * per-string set-up once; SBCI2's pair and Davidson's expansion block use it. Any nvec >= 1. */
int sbg_sigma_padded_multi(sbg_ctx* ctx, int nvec, const double* const* d_x_padded_local,
                           double* const* d_y_padded_local, void* stream);
uint64_t sbg_apply_count(const sbg_ctx* ctx);
void sbg_reset_apply_count(sbg_ctx* ctx);
uint64_t sbg_kernel_launches(const sbg_ctx* ctx);
/* Device-time profile of the sigma calls since the last reset, measured with CUDA events recorded on
 * the launching stream around each phase: ms[0] alpha-beta kernel, ms[1] same-spin kernels +
 * transposes, ms[2] collectives (world > 1), ms[3] whole sigma. *calls = sigma calls profiled. */
int sbg_profile_reset(sbg_ctx* ctx);
int sbg_profile_read(sbg_ctx* ctx, double* ms, int64_t* calls);
/* Flop count of one sigma (algorithm actually executed), split by kernel. */
int sbg_sigma_flops(const sbg_ctx* ctx, double* alpha_beta, double* same_spin, double* total);

/* ---- solvers (drivers of sbci1.hpp:526-579 / sbci2.hpp:527-623 on device-resident vectors) ----
 * method: 1 = SBCI1 (solve_n_states_sbci1), 2 = SBCI2 (solve_n_states_sbci2), 3 = block Davidson
 * (davidson_solve(op, nroots, cfg), davidson.hpp:228-244); nroots <= 9. energies[nroots] ascending; vectors (nullable) nroots x n_det host buffer,
 * unit norm. trace may be NULL. */
/* <S^2> = |S+ x|^2/|x|^2 + S_z(S_z+1) (fci/spin.hpp:17-51). x: full n_det host vector. */
int sbg_spin_squared(sbg_ctx* ctx, const double* x, double* out);
/* same on a padded local device vector (every rank passes its rows; collective when world > 1) */
int sbg_spin_squared_padded(sbg_ctx* ctx, const double* d_x_padded_local, double* out);
int sbg_solve(sbg_ctx* ctx, int method, int nroots, const sbg_config* cfg, double* energies,
              double* vectors, sbg_stats* stats, sbg_trace_fn trace, void* trace_user);
/* Davidson with an explicit subspace cap: DavidsonConfig::max_space (davidson.hpp:19-38; the CLI's
 * --max-space, sbci_cli.cpp:49,125). 0 = 12*nroots; otherwise it must be >= 2*nroots. */
int sbg_solve_davidson(sbg_ctx* ctx, int nroots, int max_space, const sbg_config* cfg, double* energies,
                       double* vectors, sbg_stats* stats, sbg_trace_fn trace, void* trace_user);

/* Plain-vector warm start of one SBCI1 state (solve_state_sbci1(op, pre, defl, x0, E0, cfg, alpha, sink),
 * sbci1.hpp:477-486): seed x0 (host, n_det, nonzero) with image H x0 (one counted sigma) and energy label
 * e0; the preconditioner shift is *shift (GroundShiftPreconditioner, precond.hpp:19-47; cfg->clamp_delta
 * is its clamp); with alpha == 0 the shift tracks the Rayleigh quotient and its final value is written
 * back to *shift (sbci1.hpp:381, 416). Deflated against ndefl unit, mutually orthogonal vectors defl_x
 * (host, ndefl x n_det) with energies defl_e; their images defl_hx may be NULL, then they are rebuilt
 * with one (uncounted) sigma each. Outputs: *energy, vector (unit, nullable), image (H vector, nullable),
 * stats (nroots = 1). Errors as sbg_solve. */
int sbg_solve_state_sbci1(sbg_ctx* ctx, const double* x0, double e0, double* shift, int alpha, int ndefl,
                          const double* defl_x, const double* defl_hx, const double* defl_e, const sbg_config* cfg,
                          double* energy, double* vector, double* image, sbg_stats* stats, sbg_trace_fn trace,
                          void* trace_user);

/* self test of the DMMA fragment layouts used by the sigma kernels (GPU) */
int sbg_selftest(void);

/* self test of the NCCL collectives used by the sharded path (all-gather, all-reduce, grouped
 * send/recv) on a one-rank communicator (GPU) */
int sbg_selftest_nccl(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* SBG_H */
