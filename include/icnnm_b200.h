/*
 * icnnm_b200.h — C ABI of the B200-native ICNNM hot path.
 *
 * This is the drop-in boundary for the reference's C++ solver/operator API
 * (/root/reference/proj/core/include/icnnm/*.hpp).  Every entry point takes
 * plain host pointers and sizes (no C++ or torch types), f64 data in the
 * reference's layouts:
 *   - tensors: row-major, last index fastest            (tensor.hpp:64-68)
 *   - m x k operator matrices: column-major (Eigen)    (conv_op.hpp:76)
 *   - basis K: k x k column-major, column j = row-major
 *     flattened eigen-kernel j                          (spectral.hpp:30-44,
 *                                                        tensor_io.cpp:111-112)
 * Device memory is owned by the library; host buffers are owned by the caller.
 * Supported tensor order: 1..3 (the reference tests use order <= 3).
 *
 * Status codes mirror the reference's exception classes:
 *   ICNNM_OK                 0
 *   ICNNM_INVALID_ARGUMENT   1   std::invalid_argument (solver.cpp:26-40,66-72;
 *                                tensor.hpp:100-107; spectral.cpp:25-41)
 *   ICNNM_RUNTIME_ERROR      2   std::runtime_error
 *   ICNNM_CUDA_ERROR         3   CUDA / NCCL failure (no reference analogue)
 * The message of the last failure on the calling thread is returned by
 * icnnm_last_error().
 */
#ifndef ICNNM_B200_H_
#define ICNNM_B200_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ICNNM_OK 0
#define ICNNM_INVALID_ARGUMENT 1
#define ICNNM_RUNTIME_ERROR 2
#define ICNNM_CUDA_ERROR 3

#define ICNNM_INIT_ZERO 0
#define ICNNM_INIT_MEAN 1

#define ICNNM_TERM_MAX_ITERS 0
#define ICNNM_TERM_CONVERGED 1

/* GEMM engine of the two per-iteration contractions. */
#define ICNNM_ENGINE_FFMA 0     /* exact fp32 FFMA implicit GEMM            */
#define ICNNM_ENGINE_TF32X3 1   /* tcgen05 kind::tf32, 3-term split (sm_100a) */
#define ICNNM_ENGINE_F16X3 2    /* tcgen05 kind::f16, 3-term split of power-of-2
                                   scaled operands (sm_100a; half the MMA time) */
#define ICNNM_ENGINE_F64 3      /* literal fp64 loop on the GPU (cuBLAS DGEMM
                                   contractions): resolves the reference's default
                                   tolerances; not the hot path                   */
#define ICNNM_ENGINE_AUTO 4     /* default: F16X3 when both tolerances are disabled
                                   (<= 1e-200, fixed iteration counts) or resolvable in
                                   fp32 (tol_change >= 1e-6; tol_primal >= 1e-4, then with
                                   exact_residual); F64 otherwise, so that the default
                                   SolverConfig stops where solver.cpp:136-139 does      */

/* Field-for-field mirror of icnnm::SolverConfig (solver.hpp:29-43). */
typedef struct icnnm_solver_config {
  double lambda;        /* 1000                                       */
  int has_theta0;       /* std::optional<double> theta0               */
  double theta0;
  double theta_growth;  /* 1.05                                       */
  double theta_max;     /* 1e10                                       */
  int max_iters;        /* 1000                                       */
  double tol_primal;    /* 1e-7                                       */
  double tol_change;    /* 1e-8                                       */
  double rank_tol;      /* 1e-8 (unused by the solver, as upstream)   */
  int init_fill;        /* ICNNM_INIT_ZERO | ICNNM_INIT_MEAN          */
  int engine;           /* ICNNM_ENGINE_* (extension; default AUTO)  */
  int exact_residual;   /* extension: 1 = exact primal_residual trace
                           (one extra forward contraction per iteration);
                           0 = fp32 identity estimate (NaN once unresolved) */
} icnnm_solver_config;

/* Mirror of icnnm::SolveReport (solver.hpp:46-52).  objective and
 * primal_residual are caller-allocated arrays of >= max_iters doubles (or
 * NULL); the library writes `iterations` entries. */
typedef struct icnnm_solve_report {
  int iterations;
  double* objective;
  double* primal_residual;
  double* l_change;          /* extension: per-iteration ||dL||/||L|| */
  int termination;           /* ICNNM_TERM_*                          */
  double wall_time_seconds;
  double loop_seconds;       /* extension: device time of the ADMM loop */
  double device_seconds;     /* extension: device time of the whole run
                                (setup kernels + loop), CUDA events      */
} icnnm_solve_report;

/* Defaults of SolverConfig (solver.hpp:29-43). */
void icnnm_default_config(icnnm_solver_config* cfg);

/* Replaces SolverConfig::validate (solver.cpp:26-40). */
int icnnm_validate_config(const icnnm_solver_config* cfg);

/* Message of the last failed call on this thread ("" if none). */
const char* icnnm_last_error(void);

/* Library / device information. */
const char* icnnm_version(void);
int icnnm_device_count(void);
/* Device blocks freed by finished calls are cached per device and reused by
 * later calls (no cudaMalloc/cudaFree per solve); this hands them back to the
 * driver.  ICNNM_DEVCACHE=0 disables the cache.  (No reference counterpart.) */
int icnnm_empty_cache(void);

/* ------------------------------------------------------------------------
 * Solver.  Replaces
 *   std::pair<DenseTensor,SolveReport> icnnm_solve(const DenseTensor& M_obs,
 *     const SamplingMask& mask, const EigenBasis& basis, const SolverConfig&)
 * (solver.hpp:64-67, solver.cpp:150-159 -> admm_solve solver.cpp:62-146).
 * `eigenvalues` may be NULL (then only K's orthogonality is validated, as
 * EigenBasis::validate does at spectral.cpp:31-34).
 * ---------------------------------------------------------------------- */
int icnnm_cuda_solve(int order, const int64_t* dims, const double* M_obs,
                     const double* mask, const int64_t* kdims,
                     const double* K_colmajor, const double* eigenvalues,
                     const icnnm_solver_config* cfg, int device, double* L_out,
                     icnnm_solve_report* report);

/* Batch of independent solves (BASELINE config 4: 64 tensors, one shared
 * basis and config).  Each problem i is exactly icnnm_cuda_solve on
 * (M_obs[i], masks[i]) -- its own theta0 (solver.cpp:88-91), res_scale
 * (:97) and stopping test -- the reference's "concurrent independent solves"
 * contract (solver.hpp:64-67) as one call.  Problems are split
 * into contiguous blocks over the n_devices GPUs in `devices` (one host
 * thread, stream and solver state per device, no inter-GPU communication);
 * the basis is validated once for the whole batch.  reports may be NULL or
 * an array of n reports (each with its own caller-allocated trace arrays).
 * On failure the status of the first failing problem is returned and
 * icnnm_last_error() names it. */
int icnnm_cuda_solve_batch(int n, int order, const int64_t* dims,
                           const double* const* M_obs,
                           const double* const* masks, const int64_t* kdims,
                           const double* K_colmajor, const double* eigenvalues,
                           const icnnm_solver_config* cfg, const int* devices,
                           int n_devices, double* const* L_out,
                           icnnm_solve_report* reports);

/* Handle API mirroring BasisConvolver's precompute-once pattern
 * (conv_op.hpp:61-81): create binds dims, kernel box and K to a device;
 * upload stages one problem in HBM; run solves it from HBM; download
 * returns L.  run() is the device-resident hot path timed by bench.py. */
typedef struct icnnm_solver_s* icnnm_solver_t;

int icnnm_solver_create(int order, const int64_t* dims, const int64_t* kdims,
                        const double* K_colmajor, const double* eigenvalues,
                        int device, icnnm_solver_t* out);
int icnnm_solver_upload(icnnm_solver_t h, const double* M_obs,
                        const double* mask);
int icnnm_solver_run(icnnm_solver_t h, const icnnm_solver_config* cfg,
                     icnnm_solve_report* report);
int icnnm_solver_download(icnnm_solver_t h, double* L_out);
/* Kernel launches issued by the last run() (for bench accounting). */
int64_t icnnm_solver_last_launches(icnnm_solver_t h);
/* Bytes of device memory held by the handle. */
int64_t icnnm_solver_device_bytes(icnnm_solver_t h);
/* Average device time (ms) of each kernel family over the last run() when
 * profiling was enabled with icnnm_solver_set_profile(h, 1):
 * out[0]=forward, out[1]=adjoint, out[2]=update, out[3]=coef. */
int icnnm_solver_set_profile(icnnm_solver_t h, int enable);
int icnnm_solver_kernel_times(icnnm_solver_t h, double* out_ms4);
/* tcgen05 pipeline counters of the last run() with set_profile(h, 2):
 * 2 x 10 cycle sums (forward, adjoint): builder wait/work, MMA wait on A /
 * B / accumulator, epilogue wait/work, loader wait, MMA-thread total,
 * builder per-brick preparation (halo, operand scale).  The counters are
 * compiled into the experiments build only (make EXPERIMENTS=1); the product
 * library reports zeros. */
int icnnm_solver_tc_counters(icnnm_solver_t h, unsigned long long* out20);
void icnnm_solver_destroy(icnnm_solver_t h);

/* ------------------------------------------------------------------------
 * Operator-level entry points (parity surface).
 * ---------------------------------------------------------------------- */

/* BasisConvolver(dims, ks, K).apply(L) (conv_op.cpp:100-114):
 * out (m x k, column-major) = A_k(L) K. */
int icnnm_cuda_conv_forward(int order, const int64_t* dims, const double* L,
                            const int64_t* kdims, const double* K_colmajor,
                            int device, double* out_colmajor);

/* conv_adjoint(W, ks, dims) (conv_op.cpp:57-77):
 * out[i] = sum_s W[(i+s) mod dims, s], W m x k column-major. */
int icnnm_cuda_conv_adjoint(int order, const int64_t* dims,
                            const int64_t* kdims, const double* W_colmajor,
                            int device, double* out);

/* Same operators with an explicit GEMM engine (ICNNM_ENGINE_*). */
int icnnm_cuda_conv_forward_ex(int order, const int64_t* dims, const double* L,
                               const int64_t* kdims, const double* K_colmajor,
                               int engine, int device, double* out_colmajor);
int icnnm_cuda_conv_adjoint_ex(int order, const int64_t* dims,
                               const int64_t* kdims, const double* W_colmajor,
                               int engine, int device, double* out);

/* prox_l21(W, tau) (solver.cpp:42-50), W rows x cols column-major. */
int icnnm_cuda_prox_l21(int64_t rows, int64_t cols, const double* W_colmajor,
                        double tau, int device, double* Z_colmajor);

/* conv_gram(L, ks) (spectral.cpp:54-81): k x k Gram A_k(L)^T A_k(L). */
int icnnm_cuda_conv_gram(int order, const int64_t* dims, const double* L,
                         const int64_t* kdims, int device, double* G_colmajor);

/* learn_ensemble_basis(refs, ks) (spectral.cpp:133-161): GPU Gram
 * accumulation over the references, host eigensolve (descending order,
 * eigenvalues clamped >= 0, column signs fixed, sigma = sqrt(lambda)).
 * refs: n_refs pointers to m doubles each.  degenerate: 1 when the Gram is
 * identically zero (K = I, eigenvalues 0). */
int icnnm_cuda_learn_basis(int n_refs, int order, const int64_t* dims,
                           const double* const* refs, const int64_t* kdims,
                           int device, double* K_colmajor_out,
                           double* eigenvalues_out, int* degenerate);

/* Host eigensolver used by learn_basis (exported for tests):
 * symmetric G (n x n, column-major) -> eigenvalues descending and
 * eigenvectors (column-major), Householder tridiagonalisation + implicit QL. */
int icnnm_host_symeig(int n, const double* G_colmajor, double* evals_desc,
                      double* evecs_colmajor);

/* objective_icnnm(L, M, mask, basis, lambda) (solver.cpp:172-187). */
int icnnm_cuda_objective(int order, const int64_t* dims, const double* L,
                         const double* M_obs, const double* mask,
                         const int64_t* kdims, const double* K_colmajor,
                         double lambda, int device, double* out);

/* ------------------------------------------------------------------------
 * CNNM baseline.  Replaces
 *   std::pair<DenseTensor,SolveReport> cnnm_solve(const DenseTensor& M_obs,
 *     const SamplingMask& mask, const KernelShape& ks, const SolverConfig&)
 * (solver.hpp:71-75, solver.cpp:161-170): the same ADMM loop with K = I and
 * singular-value thresholding (svt, solver.cpp:52-57) as the Z-update, in
 * fp64 on the GPU (Gram + cuSOLVER eigensolve + DGEMM per iteration).
 * cfg->engine and cfg->exact_residual are ignored (the trace is exact).
 * ---------------------------------------------------------------------- */
int icnnm_cuda_cnnm_solve(int order, const int64_t* dims, const double* M_obs,
                          const double* mask, const int64_t* kdims,
                          const icnnm_solver_config* cfg, int device, double* L_out,
                          icnnm_solve_report* report);

/* ------------------------------------------------------------------------
 * Recovery-theory diagnostics (`analyze`), replacing
 * /root/reference/proj/core/include/icnnm/analysis.hpp:25-99 and
 * core/src/analysis.cpp.  Matrix-free on the GPU in fp64: the m x k
 * convolution matrix the reference builds for its SVD (analysis.cpp:111-135)
 * is never formed.  `evals` may be NULL (the reference's basis_from_matrix
 * test bases carry zero eigenvalues); when given it is validated like
 * EigenBasis::validate (spectral.cpp:25-41).  rank_tol default: 1e-8
 * (kDefaultRankTol, spectral.hpp:25).
 * ---------------------------------------------------------------------- */
#define ICNNM_DEFAULT_RANK_TOL 1e-8

/* ConvCoherence (analysis.hpp:62-67). */
typedef struct icnnm_conv_coherence {
  double mu1, mu2, tau;
  int64_t rank;
} icnnm_conv_coherence;

/* ThresholdInputs / Thresholds (analysis.hpp:72-93). */
typedef struct icnnm_threshold_inputs {
  int64_t r_K;
  double alpha_K, mu_K_I, mu1, mu2;
  int64_t r0, k, m;
  double rho0;
} icnnm_threshold_inputs;

typedef struct icnnm_threshold_values {
  double rho_min_noiseless, rho_min_noisy, error_bound_factor, cnnm_bound,
      icnnm_ideal_bound;
  int certified;
} icnnm_threshold_values;

/* RecoveryDiagnostics (analysis.hpp:29-44).  support_I: caller-owned array
 * of k entries (or NULL); the first r_K are written. */
typedef struct icnnm_recovery_diagnostics {
  int64_t r_K;
  int64_t* support_I;
  double alpha_K, mu_K_I, mu1, mu2, tau;
  int64_t r0;
  double rho0, rho_min_noiseless, rho_min_noisy, error_bound_factor, cnnm_bound,
      icnnm_ideal_bound;
  int certified;
} icnnm_recovery_diagnostics;

/* sigma^K_i = ||A(L0) K_i|| for i < k (relative_eigenvalues,
 * analysis.cpp:29-38). */
int icnnm_cuda_relative_eigenvalues(int order, const int64_t* dims, const double* L0,
                                    const int64_t* kdims, const double* K_colmajor,
                                    const double* evals, int device, double* sigma);
/* relative_conv_rank (analysis.hpp:45-51): r_K and the support (k entries). */
int icnnm_cuda_relative_conv_rank(int order, const int64_t* dims, const double* L0,
                                  const int64_t* kdims, const double* K_colmajor,
                                  const double* evals, double rank_tol, int device,
                                  int64_t* r_K, int64_t* support);
/* spectral_corr_coeff (analysis.hpp:53-57); r_K = 0 is an error. */
int icnnm_cuda_spectral_corr_coeff(int order, const int64_t* dims, const double* L0,
                                   const int64_t* kdims, const double* K_colmajor,
                                   const double* evals, double rank_tol, int device,
                                   double* alpha);
/* active_coherence (analysis.hpp:59-60); host only. */
int icnnm_active_coherence(int64_t k, const double* K_colmajor, int64_t n_support,
                           const int64_t* support, double* out);
/* conv_coherence (analysis.hpp:68-70); zero tensor is an error. */
int icnnm_cuda_conv_coherence(int order, const int64_t* dims, const double* L0,
                              const int64_t* kdims, double rank_tol, int device,
                              icnnm_conv_coherence* out);
/* thresholds (analysis.hpp:94); host only. */
int icnnm_thresholds(const icnnm_threshold_inputs* in, icnnm_threshold_values* out);
/* analyze_recovery (analysis.hpp:96-99). */
int icnnm_cuda_analyze_recovery(int order, const int64_t* dims, const double* L0,
                                const int64_t* kdims, const double* K_colmajor,
                                const double* evals, const double* mask, double rank_tol,
                                int device, icnnm_recovery_diagnostics* out);

/* ------------------------------------------------------------------------
 * Sharded solve of one large tensor, split over H into G slabs (one slab per
 * rank of a NCCL communicator, optionally several virtual slabs per process;
 * BASELINE config 5).  Periodic halos of kh-1 rows travel from rank g-1 to g
 * before the forward pass, adjoint partial sums travel back, and the
 * k-length column-norm vector (+ scalars) is all-reduced once per
 * iteration.  The result equals the unsharded solve up to fp32 rounding.
 * ---------------------------------------------------------------------- */
#define ICNNM_NCCL_UNIQUE_ID_BYTES 128

int icnnm_dist_unique_id(char* out128);

/* Solve with `local_slabs` slabs per process and `world` processes
 * (G = local_slabs * world slabs), every process passing the FULL tensor
 * (M_obs, mask: m doubles); each process reads only its own rows and
 * receives them in L_out (rows [row0, row0 + nrows) of the H axis, written
 * to L_out[0 .. nrows*W*T)).  world == 1 needs no NCCL id (pass NULL: the
 * exchange is device copies); world == 1 WITH an id (icnnm_dist_unique_id)
 * runs the exchange through a one-rank NCCL communicator (self send/recv,
 * all-reduce) -- the multi-process transport, exercised on one GPU.
 * Each call builds (and destroys) its communicator, so each call needs a fresh
 * id from icnnm_dist_unique_id (an id bootstraps exactly one communicator).
 * row0/nrows may be NULL. */
int icnnm_sharded_solve(int order, const int64_t* dims, const double* M_obs,
                        const double* mask, const int64_t* kdims,
                        const double* K_colmajor,
                        const icnnm_solver_config* cfg, int local_slabs,
                        int world, int rank, const char* nccl_id128,
                        int device, double* L_out, int64_t* row0,
                        int64_t* nrows, icnnm_solve_report* report);

/* The rows [row0, row0 + nrows) of the H axis that rank `rank` owns (its
 * local_slabs consecutive slabs of the G-slab plan). */
int icnnm_sharded_rows(int order, const int64_t* dims, const int64_t* kdims,
                       int local_slabs, int world, int rank, int64_t* row0,
                       int64_t* nrows);

/* The same solve with slab-local inputs: M_rows / mask_rows hold only this
 * rank's rows [row0, row0 + nrows) (nrows*W*T doubles each, as
 * icnnm_sharded_rows returns them) -- no process holds the full tensor.  The
 * global setup scalars (theta0 from max|pm|, solver.cpp:88-91; res_scale
 * from ||pm||, :97; the mean fill, :83-86; the empty-set check, :70-71)
 * are all-reduced over the ranks, and an invalid slab fails every rank. */
int icnnm_sharded_solve_local(int order, const int64_t* dims, int64_t row0,
                              int64_t nrows, const double* M_rows,
                              const double* mask_rows, const int64_t* kdims,
                              const double* K_colmajor,
                              const icnnm_solver_config* cfg, int local_slabs,
                              int world, int rank, const char* nccl_id128,
                              int device, double* L_out,
                              icnnm_solve_report* report);

/* Slab plan (host logic, exported for CPU tests): slab g of G over H rows
 * gets rows [start, start+count); returns 1 (invalid) when a slab would be
 * thinner than kh-1 rows. */
int icnnm_shard_plan(int64_t H, int G, int64_t kh, int g, int64_t* start,
                     int64_t* count);

/* ------------------------------------------------------------------------
 * Reference file formats (tensor_io.cpp:86-128, report_io.cpp:39-68), used
 * by the GPU CLI drop-in (bin: paper_2604_17001_b200/icnnm_b200).
 * ---------------------------------------------------------------------- */
const char* icnnm_io_last_error(void);
int icnnm_write_tnsr(const char* path, int order, const int64_t* dims,
                     const double* values);
/* values == NULL: header only (order, dims16[0..order)) */
int icnnm_read_tnsr(const char* path, int* order, int64_t* dims16,
                    double* values);
int icnnm_write_ebas(const char* path, int order, const int64_t* kdims,
                     const double* eigenvalues, const double* K_colmajor);
/* eigenvalues/K NULL: header only */
int icnnm_read_ebas(const char* path, int* order, int64_t* kdims16,
                    double* eigenvalues, double* K_colmajor);
/* solver_config_from_json: flat object, absent keys keep the defaults,
 * "theta0": null = automatic; validates (SolverConfig::validate). */
int icnnm_config_from_json(const char* text, icnnm_solver_config* cfg);
/* solve_report_to_json; returns the byte length, writes <= cap bytes. */
int64_t icnnm_report_to_json(const icnnm_solve_report* rep, char* out,
                             int64_t cap);
/* diagnostics_to_json (report_io.cpp:70-88): same contract as
 * icnnm_report_to_json. */
int64_t icnnm_diagnostics_to_json(const icnnm_recovery_diagnostics* d, char* out,
                                  int64_t cap);

/* ------------------------------------------------------------------------
 * Probes used by bench.py for roofline denominators (device microbenches).
 * ---------------------------------------------------------------------- */
/* FP32 FFMA throughput in TFLOP/s measured with a register-resident kernel. */
int icnnm_probe_ffma_tflops(int device, double* out);
/* FP64 DFMA throughput in TFLOP/s (the Gram kernel's roofline denominator). */
int icnnm_probe_dfma_tflops(int device, double* out);

#ifdef __cplusplus
}
#endif
#endif /* ICNNM_B200_H_ */
