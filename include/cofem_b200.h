/*
 * cofem_b200.h -- C ABI of the B200-native CoFEM hot path.
 *
 * Plain pointers and sizes only (no torch / CUDA types), so any FFI can bind
 * it (ctypes here; see INTEGRATION.md for the binding the reference would
 * add).  Every entry point names the reference interface it replaces; paths
 * are relative to the reference package /root/reference/pkg/src/sbl/.
 *
 * Conventions
 *   - Phi (the dictionary) is N x D float32, row-major (C order), exactly the
 *     (N, D) numpy layout of operators.DenseOperator.matrix (operators.py:104).
 *     Under column sharding a context holds its local D_r columns.
 *   - Column blocks ("D x Q" in the reference, e.g. the PCG right-hand sides
 *     B of cg.solve, cg.py:155) are float64 row-major D x Q on the host side:
 *     coordinate j's Q entries are contiguous, as numpy (D, Q) C-order.
 *   - Every function returns 0 on success and a negative COFEM_E* code on
 *     failure; cofem_last_error() returns the message of the last failure on
 *     the calling thread.  No entry point ever falls back to the CPU.
 */
#ifndef COFEM_B200_H
#define COFEM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COFEM_ABI_VERSION 1

enum cofem_status {
  COFEM_OK = 0,
  COFEM_EINVAL = -1,      /* bad argument (ShapeMismatchError / ValueError in the reference) */
  COFEM_ECUDA = -2,       /* CUDA runtime failure */
  COFEM_ENOMEM = -3,      /* device allocation failed */
  COFEM_EDIVERGED = -4,   /* non-finite residual: DivergenceError (cg.py:17) */
  COFEM_ENCCL = -5,       /* NCCL failure / NCCL not loadable */
  COFEM_ESTATE = -6       /* call order violated (e.g. no dictionary set) */
};

/* Arithmetic of the column blocks and of the Phi contractions.
 * FP32: fp32 vectors, fp32 contraction accumulators, fp64 scalar reductions
 *       (the north_star's "GPU runs fp32").
 * FP64: CUDA-core DFMA contractions over the dictionary as given (float32
 *       entries, or the exact float64 ones of cofem_set_dictionary_f64);
 *       vectors, accumulators and scalars fp64: the reference's float64
 *       arithmetic up to summation order.
 * OZAKI: fp64 vectors and scalars; the two Phi contractions run on the int8
 *       tensor cores (tcgen05.mma.kind::i8) over a 32-bit fixed-point copy of
 *       Phi (four signed digit planes, 4 B / entry) with exact int32
 *       accumulation -- float64-grade results at tensor-core rate.
 * OZAKI24: OZAKI over a 24-bit fixed-point Phi (three digit planes, 3 B /
 *       entry: a quarter less HBM traffic per PCG step on dense
 *       dictionaries); the operands stay 32-bit.  Structured dictionaries
 *       (convolution, 2-D DCT) treat it as OZAKI. */
enum cofem_precision { COFEM_FP32 = 0, COFEM_FP64 = 1, COFEM_OZAKI = 2, COFEM_OZAKI24 = 3 };

/* Preconditioner policy, cg.py:79-108 make_preconditioner(policy, ...). */
enum cofem_theta { COFEM_THETA_ALL_ONES = 0, COFEM_THETA_JACOBI = 1, COFEM_THETA_NONE = 2,
                   COFEM_THETA_CUSTOM = 3 };

/* M-step variant, cofem.py:103 m_step / cofem.py:120 m_step_nonneg. */
enum cofem_variant { COFEM_STANDARD = 0, COFEM_NONNEG = 1 };

typedef struct cofem_ctx cofem_ctx;

/* CgConfig, cg.py:48-67 (theta lives in cofem_em_config / the minv argument). */
typedef struct {
  int32_t max_steps;          /* U >= 1 */
  int32_t printed_recursion;  /* 0: P <- W + eta P (standard PCG); 1: P <- R + eta P */
  double tolerance;           /* Frobenius ||R||_F / ||B||_F stopping threshold > 0 */
} cofem_cg_config;

/* CgReport, cg.py:70-76. */
typedef struct {
  int32_t steps_taken;
  int32_t converged;
  int32_t diverged;            /* 1 => residual turned non-finite at step `steps_taken` */
  int32_t n_breakdown;         /* number of columns frozen by pi_q == 0 */
  double final_relative_residual;
} cofem_cg_report;

/* CofemConfig, cofem.py:30-47 (+ the CG part in a cofem_cg_config). */
typedef struct {
  int32_t iterations;   /* T >= 1 */
  int32_t probes;       /* K >= 1 */
  int32_t variant;      /* cofem_variant */
  int32_t theta_policy; /* cofem_theta */
  double clamp_max;     /* 1e12 */
  double floor_eps;     /* 1e-12 */
} cofem_em_config;

/* ---- library ---------------------------------------------------------- */
int cofem_abi_version(void);
const char* cofem_last_error(void);
int cofem_device_count(int* out);

/* ---- context: one dense dictionary shard on one GPU --------------------
 * Replaces operators.DenseOperator (operators.py:104-129) + the workspace
 * that cg._pcg_loop (cg.py:111-152) allocates per call.               */
int cofem_create(cofem_ctx** out, int device, int64_t n_rows, int64_t n_cols, int precision);
int cofem_destroy(cofem_ctx* ctx);

/* Causal convolution dictionary (operators.ConvolutionOperator,
 * operators.py:182-225; BASELINE config 3): the D x D lower-triangular
 * Toeplitz matrix Phi_ij = taps[i - j] for 0 <= i - j < ntaps.  COFEM_OZAKI:
 * banded int8 tensor-core contractions (Phi and Phi^T; any filter length up to
 * 32512 taps; the reference's filter (1 - rho)^m is passed truncated where it
 * falls below the fixed-point resolution).  COFEM_FP64: float64 overlap-save
 * FFT passes (filters up to 512 taps, one GPU). */
int cofem_create_convolution(cofem_ctx** out, int device, int64_t dim, const double* taps, int64_t ntaps,
                             int precision);

/* 2-D partial DCT dictionary (BASELINE config 5; the 2-D analogue of
 * operators.SubsampledDctOperator, operators.py:132-179): z is an n x n image
 * (row-major, D = n^2), Phi z = the coefficients `mask` (flat k n + l) of its
 * orthonormal 2-D DCT-II.  Phi^T Phi runs as three fused float64 FFT passes
 * (row DCT-II; column DCT-II, mask, DCT-III; row DCT-III + PCG combine);
 * n a power of two in [64, 1024]; precision COFEM_FP64 (COFEM_OZAKI is
 * accepted as an alias: the passes are float64 either way). */
int cofem_create_dct2(cofem_ctx** out, int device, int64_t n, const int64_t* mask, int64_t nmask, int precision);

/* 1-D subsampled DCT dictionary: operators.SubsampledDctOperator
 * (operators.py:132-179), Phi = the rows `mask` of the orthonormal inverse
 * DCT-II (DCT-III) of length `dim` (any dim >= 2).  O(D log D): Makhoul's
 * reduction, two real columns per complex length-D FFT (cuFFT double
 * complex, loaded at run time), fused float64 pre / mask / post passes;
 * Phi^T Phi = DCT-II(mask .* DCT-III(.)).  Precision COFEM_FP64 (the int8
 * modes are accepted as aliases). */
int cofem_create_dct1(cofem_ctx** out, int device, int64_t dim, const int64_t* mask, int64_t nmask, int precision);

/* Upload Phi (N x D_local float32, row stride `ld` elements) from host
 * memory (or adopt a device pointer when `on_device` != 0; the caller keeps
 * it alive).  operators.DenseOperator.__init__, operators.py:109-117. */
int cofem_set_dictionary(cofem_ctx* ctx, const float* phi, int64_t ld, int on_device);

/* Upload a float64 Phi from host memory (row stride `ld`).  COFEM_FP64 keeps
 * the exact float64 entries in HBM and multiplies them (the reference's
 * float64 DenseOperator, operators.py:109-117); COFEM_OZAKI builds its
 * fixed-point digit planes from the exact float64 values; COFEM_FP32 uses the
 * float32 rounding.  (A sharded context joins its communicator / group
 * first: the digit planes of a column shard use row scales shared across
 * the ranks, so the call is collective there.) */
int cofem_set_dictionary_f64(cofem_ctx* ctx, const double* phi, int64_t ld);

/* Declare this context's place in a column-sharded dictionary: it holds
 * global columns [col_offset, col_offset + n_cols) of `global_cols`.  Used by
 * the device generators so every shard draws the same global Phi / probes.
 * Convolution contexts are time shards: samples [col_offset, col_offset +
 * dim) of a length-global_cols sequence (rows = columns); col_offset is a
 * multiple of 256, every shard but the last holds a multiple of 256 samples
 * and at least the filter halo.  2-D DCT contexts are not sharded. */
int cofem_set_shard(cofem_ctx* ctx, int64_t col_offset, int64_t global_cols);

/* Generate Phi on the device: entries scale * N(0,1) from a counter-based
 * generator keyed by `seed` (synthetic benchmark dictionaries,
 * operators.build_dense_gaussian, operators.py:227-232, with a device RNG). */
int cofem_generate_gaussian_dictionary(cofem_ctx* ctx, uint64_t seed, double scale);

/* Copy Phi back to the host (n_rows x n_cols, row stride n_cols). */
int cofem_get_dictionary(cofem_ctx* ctx, float* out);

/* ---- multi-GPU: Phi column-sharded across `nranks` processes ----------
 * 128-byte NCCL unique id from rank 0, broadcast by the host.  With
 * nranks == 1 the collectives are real single-rank NCCL calls.        */
int cofem_nccl_get_unique_id(void* out128);
int cofem_set_comm(cofem_ctx* ctx, const void* unique_id128, int nranks, int rank);
/* Exchanges per PCG step (call cofem_set_shard first):
 *   dense:        all-reduce(sum) of the N x (K+1) partial Phi_r P_r; pi and
 *                 (rho, ||R||^2) all-reduces.
 *   convolution:  all-reduce(max) of the operand column maxima (common int8
 *                 scales), then a neighbour halo send/recv of lpad operand rows
 *                 (int8 digit planes) before each banded contraction -- Phi P
 *                 takes the left neighbour's last rows, Phi^T V the right
 *                 neighbour's first rows; pi and (rho, ||R||^2) all-reduces.
 *
 * In-process shard group: the same exchanges between contexts driven from
 * host threads of one process (one thread per rank, each calling the usual
 * entry points on its context).  The ranks' buffers are read directly (same
 * device or peer memory) after stream-ordered events; a rank that fails
 * breaks the group so the others return an error instead of waiting.
 * A context joins either an NCCL communicator or a group, once.        */
typedef struct cofem_group cofem_group;
int cofem_group_create(cofem_group** out, int nranks);  /* 1 <= nranks <= 8 */
int cofem_group_destroy(cofem_group* group);            /* after its contexts */
int cofem_group_abort(cofem_group* group);              /* a host-side failure: release the ranks */
int cofem_set_group(cofem_ctx* ctx, cofem_group* group, int rank);

/* ---- operator applications (host float64 buffers) ---------------------
 * LinearOperator.apply / apply_adjoint, operators.py:61-71.            */
int cofem_apply(cofem_ctx* ctx, const double* V, int64_t q, double* out);          /* (D,q)->(N,q) */
int cofem_apply_adjoint(cofem_ctx* ctx, const double* U, int64_t q, double* out);  /* (N,q)->(D,q) */
/* SystemMatrix.apply, operators.py:267-272: out = beta Phi^T Phi V + alpha .* V */
int cofem_system_apply(cofem_ctx* ctx, double beta, const double* alpha, const double* V,
                       int64_t q, double* out);
/* LinearOperator.column_sq_norms for the dense kind, operators.py:128-129. */
int cofem_column_sq_norms(cofem_ctx* ctx, double* out);

/* ---- blocked PCG --------------------------------------------------------
 * cg.solve / cg.solve_blocked (cg.py:155-234) on the dense system
 * A = beta Phi^T Phi + diag(alpha).  minv is the inverse preconditioner
 * diagonal, D x n_groups row-major, and group_of_col (length q, may be NULL
 * when n_groups == 1) maps each column to its group (cg.py:225-228).
 * B, X: host D x q float64.  breakdown (length q, may be NULL) receives 1 for
 * columns frozen by pi_q == 0.  Returns COFEM_EDIVERGED with rep->diverged
 * set when the residual turns non-finite. */
int cofem_pcg_solve(cofem_ctx* ctx, double beta, const double* alpha, const double* minv,
                    int32_t n_groups, const int32_t* group_of_col, const double* B, int64_t q,
                    const cofem_cg_config* cg, double* X, cofem_cg_report* rep,
                    uint8_t* breakdown);

/* ---- the CoFEM EM loop ---------------------------------------------------
 * cofem.run_cofem (cofem.py:136-157): T E-steps (cofem.e_step, cofem.py:76)
 * each solving A X = [p_1..p_K | Phi^T y] by blocked PCG, reading
 * mu = beta x_{K+1} and s_j = (1/K) sum_k p_jk x_jk (probes.py:28), and the
 * closed-form M-step (cofem.py:103 / :120) between E-steps.
 *   y            N float64 observation
 *   probes       T x D_local x K int8 (+1/-1), the host-drawn Rademacher
 *                blocks (probes.draw_rademacher, probes.py:13), iteration
 *                major; NULL => the device draws them (no host parity).
 *   theta        D_local custom theta (COFEM_THETA_CUSTOM) or NULL
 * Outputs (host, may be NULL): alpha (the precision used by the final
 * E-step), mu, s (length D_local), and per-iteration CG steps / residuals
 * (length T).  On divergence returns COFEM_EDIVERGED and *failed_iteration
 * / *failed_step name the EM iteration and CG step. */
int cofem_run(cofem_ctx* ctx, const double* y, double beta, const cofem_em_config* em,
              const cofem_cg_config* cg, const double* theta, const int8_t* probes,
              uint64_t device_probe_seed, double* alpha, double* mu, double* s,
              int32_t* cg_steps, double* cg_residuals, int32_t* failed_iteration,
              int32_t* failed_step);

/* The CgReport of the last cofem_run's final E-step and its per-iteration
 * wall times (cofem.py:97-100 PosteriorEstimate.cg_report, cofem.py:127-133
 * _iteration_record's wall_time).  Any output may be NULL:
 *   wall_times  length `iterations` (must equal the run's T), seconds
 *   solution    D x (K+1) float64, the final block X = [X_probes | x_mean]
 *   breakdown   K+1 flags of columns frozen by pi_q == 0
 *   rep         steps / convergence / residual of the final solve */
int cofem_last_run_report(cofem_ctx* ctx, int32_t iterations, double* wall_times, double* solution,
                          uint8_t* breakdown, cofem_cg_report* rep);

/* cg.solve_blocked (cg.py:201-234) over DISTINCT systems: block l solves
 * (beta_l Phi_l^T Phi_l + diag(alpha_l)) X_l = B_l (D x q_l host float64,
 * row-major) with inverse preconditioner minv_l (length D), all blocks in ONE
 * lockstep PCG whose Frobenius stopping rule aggregates every block.  One
 * context per block (same D, precision and device; a dictionary shared by
 * two blocks needs two contexts).  breakdowns (may be NULL, or hold NULL
 * entries) receive the per-column freeze flags. */
int cofem_pcg_solve_multi(cofem_ctx* const* ctxs, int n_blocks, const double* betas, const double* const* alphas,
                          const double* const* minvs, const double* const* Bs, const int64_t* qs,
                          const cofem_cg_config* cg, double* const* Xs, cofem_cg_report* rep,
                          uint8_t* const* breakdowns);

/* ---- the reference's probe stream on the device ---------------------------------
 * probes.draw_rademacher (probes.py:13-17) over numpy's PCG64 generator
 * substream(seed, 3) (cofem.py:143): cofem_set_probe_stream(ctx, state, inc)
 * hands the generator's 128-bit state and increment ({hi, lo} words, as in
 * Generator.bit_generator.state) to the context; a later cofem_run with
 * probes == NULL then draws EM iteration t's D x K signs on the device from
 * the 32-bit halves [(t - 1) D K, t D K) of the generator's output -- bit for
 * bit the reference's probes, with no host draw or upload (the generator
 * must not hold a buffered half: has_uint32 == 0).  NULL state restores host
 * / dseed probes.  cofem_pcg64_rademacher draws rows [row0, row0 + rows) of
 * the D x K draw starting at half half_offset into host memory (a checker). */
int cofem_set_probe_stream(cofem_ctx* ctx, const uint64_t* state, const uint64_t* inc);
/* the same with an explicit layout: iteration t's draw starts at half
 * first_half + (t - 1) halves_per_iteration (0: D K).  Task l of L in
 * run_cofem_multitask (cofem.py:178-184) uses first_half = l D K,
 * halves_per_iteration = L D K; with share_probes, 0 and D K. */
int cofem_set_probe_stream_ex(cofem_ctx* ctx, const uint64_t* state, const uint64_t* inc, uint64_t first_half,
                              uint64_t halves_per_iteration);
int cofem_pcg64_rademacher(int device, const uint64_t* state, const uint64_t* inc, uint64_t half_offset, int64_t row0,
                           int64_t rows, int32_t k, int8_t* out);

/* ---- multi-task CoFEM ----------------------------------------------------------
 * cofem.run_cofem_multitask (cofem.py:160-214): L tasks (one context each,
 * same D and precision, one GPU) share alpha; every EM iteration solves all
 * L (K+1)-column systems in ONE lockstep PCG whose stopping rule aggregates
 * the residual over all tasks (cg.solve_blocked, cg.py:201-234), then the
 * pooled M-step alpha = L / sum_l (mu_l^2 + s_l).  betas: one noise precision
 * per task (task.beta).  theta (custom policy only): L x D, row l for task l.
 * probes: T x L x D x K int8
 * in the reference's draw order; mus / ss: L host pointers of length D. */
int cofem_run_multitask(cofem_ctx* const* ctxs, int n_tasks, const double* const* ys, const double* betas,
                        const cofem_em_config* em, const cofem_cg_config* cg, const double* theta,
                        const int8_t* probes, double* alpha, double* const* mus, double* const* ss,
                        int32_t* cg_steps, double* cg_residuals, int32_t* failed_iteration, int32_t* failed_step);

/* ---- device-timed benchmark hooks ----------------------------------------
 * Run `n_iter` EM iterations continuing the context's resident state
 * (bench.py "value": inputs already in HBM), returning device milliseconds
 * for the whole call and for the dominant kernels of the last call.     */
typedef struct {
  double total_ms;          /* CUDA-event time of the n_iter iterations */
  double fwd_ms;            /* summed device time of Phi X launches */
  double bwd_ms;            /* summed device time of Phi^T U launches */
  int64_t fwd_launches;
  int64_t bwd_launches;
  int64_t pcg_steps;        /* PCG steps executed */
  int64_t kernel_launches;  /* all kernels launched by the library */
  double solve_ms;          /* CUDA-event time of the one-launch PCG solves (dense, one GPU) */
  int64_t solve_launches;   /* their launches (fwd_ms / bwd_ms then hold their contraction phases) */
} cofem_timing;

int cofem_bench_prepare(cofem_ctx* ctx, const double* y, double beta, const cofem_em_config* em,
                        const cofem_cg_config* cg, uint64_t device_probe_seed);
int cofem_bench_iterations(cofem_ctx* ctx, int n_iter, int time_kernels, cofem_timing* out);

#ifdef __cplusplus
}
#endif
#endif /* COFEM_B200_H */
