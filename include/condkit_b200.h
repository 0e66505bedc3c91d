/*
 * condkit_b200.h -- C ABI of the B200-native Projected-Adam kappa_2 estimator.
 *
 * Drop-in boundary for the reference estimator / error-bound interface
 * (condkit, /root/reference/proj/include/condkit). Every entry point names the
 * reference symbol (file:line) it replaces. Plain pointers and sizes only; no
 * C++ or torch types cross this boundary and no exception escapes it.
 *
 * Conventions
 *  - Every function returns a ck_status; on failure ck_last_error() returns a
 *    thread-local message. Status values map 1:1 onto the reference's
 *    exception types (see ck_status).
 *  - Matrices are CSR: int64 row offsets (nrows+1, starting at 0), int32 column
 *    indices strictly increasing within a row, finite double values -- the
 *    invariants of SparseMatrix (sparse.hpp:47-52, validated at 129-145).
 *  - Vectors passed as `const double*` / `double*` are HOST buffers unless the
 *    name ends in `_dev`. Host buffers may be registered with
 *    ck_host_register() so transfers run at pinned-memory speed.
 *  - A handle is bound to the device current at its creation and owns one
 *    CUDA stream. Calls on distinct handles are thread-safe; calls on one
 *    handle must be serialised by the caller (the reference's objects are
 *    likewise single-threaded per run).
 */
#ifndef CONDKIT_B200_H
#define CONDKIT_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CK_OK = 0,
  CK_ERR_DIMENSION = 1,        /* DimensionMismatch          sparse.hpp:25-27 */
  CK_ERR_INVALID_ARGUMENT = 2, /* std::invalid_argument      condest.hpp:187,303 */
  CK_ERR_LOGIC = 3,            /* std::logic_error (witness)  condest.hpp:286-289 */
  CK_ERR_STRUCT_SINGULAR = 4,  /* StructurallySingular        lu.hpp:24-30 */
  CK_ERR_NUM_SINGULAR = 5,     /* NumericallySingular         lu.hpp:32-40 */
  CK_ERR_ZERO_RHS = 6,         /* ZeroRHS                     error_bounds.hpp:33-35 */
  CK_ERR_ZERO_SOLUTION = 7,    /* ZeroSolution                error_bounds.hpp:37-39 */
  CK_ERR_ZERO_COLUMN = 8,      /* ZeroColumn                  sparse.hpp:29-33 */
  CK_ERR_ZERO_ROW = 9,         /* ZeroRow                     sparse.hpp:35-39 */
  CK_ERR_CUDA = 20,            /* CUDA runtime failure (no reference analogue) */
  CK_ERR_NO_DEVICE = 21,       /* no sm_100 device visible */
  CK_ERR_UNSUPPORTED = 22,     /* input outside this build's limits (e.g. nnz >= 2^32) */
  CK_ERR_OUT_OF_MEMORY = 23
} ck_status;

/* AdamConfig, condest.hpp:39-48 (same fields, same defaults via ck_adam_default). */
typedef struct {
  double alpha, beta1, beta2, eps_stab;
  uint64_t max_iter, seed;
  double rel_tol;
  uint64_t patience;
} ck_adam_cfg;

/* NormEstimate, condest.hpp:69-74 (the witness is returned through a separate buffer). */
typedef struct {
  double value;
  uint64_t iterations;
  int32_t converged;
  int32_t _pad;
} ck_norm_result;

/* Per-iteration scalars of AdamStepInfo (condest.hpp:61-65) plus the AdamState
 * scalars (condest.hpp:51-56) for observer mode. */
typedef struct {
  uint64_t t;
  double loss, loss_min;
  double x_dot_delta, delta_norm;
  int32_t phase; /* 0 running, 1 restarted this step, 2 finished */
  int32_t _pad;
} ck_step_info;

typedef struct {
  int64_t nrows, ncols, nnz;
  int64_t sell_entries_a, sell_entries_at; /* stored entries incl. slice padding */
  int64_t device_bytes;
  int32_t device;
  /* column-index format of the device layouts: bit0 = A narrow, bit1 = A^T
   * narrow (uint16 offsets from a per-slice base, 10 B per stored entry with
   * the value; otherwise int32, 12 B); bit2 / bit3 = the narrow offsets of A /
   * A^T come from a dictionary of repeating slice patterns (stencil operators:
   * 8 B per stored entry from HBM). Same columns in the same order in every
   * format. */
  int32_t col_format;
} ck_matrix_info;

typedef struct ck_matrix_s* ck_matrix;
typedef struct ck_session_s* ck_session;
typedef struct ck_lu_s* ck_lu;

/* ----------------------------------------------------------------- runtime */
const char* ck_last_error(void);
int32_t ck_abi_version(void);
ck_status ck_device_count(int32_t* count);
/* Free / total memory and SM count of the current device (sizing of ensemble waves). */
ck_status ck_device_memory(uint64_t* free_bytes, uint64_t* total_bytes, int32_t* sm_count);
/* Select the device for handles created by this thread (cudaSetDevice). */
ck_status ck_set_device(int32_t device);
ck_status ck_device_synchronize(void);
ck_status ck_host_register(void* ptr, uint64_t bytes);
ck_status ck_host_unregister(void* ptr);
/* Start drawing random_unit_vector(n) from mt19937_64(seed) (rng.hpp:68-77) on a
 * host thread, so that the draw overlaps the matrix upload that precedes a
 * session. The next ck_session_create whose first column has this seed and
 * dimension takes the vector and the engine state (bit-identical to drawing it
 * there); anything else ignores it. One slot per process; a new call replaces
 * (and first joins) the previous one. No reference counterpart: the reference
 * draws inside projected_adam (condest.hpp:191). */
ck_status ck_start_vector_prefetch(uint64_t seed, int64_t n);
/* Drops the pending prefetch (joins its thread, frees its pinned buffer): for a
 * caller whose session creation failed after requesting one. A session that
 * finds a slot for another seed or size drops it too. */
ck_status ck_start_vector_prefetch_cancel(void);
/* Slots taken by a session and slots dropped, since the library was loaded. */
ck_status ck_start_vector_prefetch_stats(uint64_t* taken, uint64_t* dropped);
void ck_adam_default(ck_adam_cfg* cfg);

/* --------------------------------------------------- rng.hpp mirror (host) */
/* mix_seed, rng.hpp:23-28 */
uint64_t ck_mix_seed(uint64_t base, uint64_t stream);
/* `count` successive random_unit_vector(n, gen) draws from one mt19937_64(seed),
 * rng.hpp:68-77; bit-identical to the reference. */
ck_status ck_random_unit_vectors(uint64_t seed, int64_t n, int64_t count, double* out);

/* `count` uniform_in(gen, lo, hi) draws of one mt19937_64(seed), rng.hpp:36-38
 * (make_known_solution's x*, bench.hpp:141-150). */
ck_status ck_uniform_in(uint64_t seed, int64_t count, double lo, double hi, double* out);

/* ------------------------------------------ error_bounds.hpp scalar formulas */
ck_status ck_loose_bounds(double residual_norm, double b_norm, double kappa, double* lower,
                          double* upper);                               /* :59-68 */
ck_status ck_tight_bounds(double residual_norm, double a_norm, double xhat_norm, double kappa,
                          double* lower, double* upper);                /* :71-80 */
ck_status ck_propagate_bound(double eps_tight, double* out);           /* :84-88 */
ck_status ck_singularity_bound(double kappa, double eps_mach, double* out); /* :93-99 */

/* --------------------------------------------------- device-resident operator */
/* Uploads A (SparseMatrix, sparse.hpp:52-152) and builds, on the device, the
 * sliced-ELL layouts of A and A^T used by every kernel. Validates the CSR
 * invariants like SparseMatrix::validate (sparse.hpp:129-145). */
ck_status ck_matrix_upload(int64_t nrows, int64_t ncols, const int64_t* row_offsets,
                           const int32_t* col_indices, const double* values, ck_matrix* out);
ck_status ck_matrix_free(ck_matrix a);
ck_status ck_matrix_get_info(ck_matrix a, ck_matrix_info* info);
/* y = A x, matvec sparse.hpp:212-226 (stored-order row sums: bit-identical). */
ck_status ck_spmv(ck_matrix a, const double* x, double* y);
/* y = A^T x, transpose_matvec sparse.hpp:230-242 (increasing-row accumulation per
 * output: bit-identical). */
ck_status ck_spmv_t(ck_matrix a, const double* x, double* y);
/* ||A x - b||, ||x||, ||b|| (verify_solution residual, error_bounds.hpp:176-183). */
ck_status ck_residual_norms(ck_matrix a, const double* x, const double* b, double* r_norm,
                            double* x_norm, double* b_norm);
/* loss_explicit / grad_explicit (condest.hpp:88-107) on the device. */
ck_status ck_loss_explicit(ck_matrix a, const double* x, double* loss);
ck_status ck_grad_explicit(ck_matrix a, const double* x, double* g);

/* ------------------------------------------ Projected Adam (ExplicitOracle) */
/* projected_adam(ExplicitOracle(A), cfg), condest.hpp:184-297 and norm2 :315-317.
 * witness (ncols doubles) may be NULL. */
ck_status ck_projected_adam(ck_matrix a, const ck_adam_cfg* cfg, ck_norm_result* res,
                            double* witness);
/* estimate_norm(ExplicitOracle(A), cfg, restarts), condest.hpp:301-312. The
 * restarts run concurrently as columns of one multi-vector iteration; each is
 * bit-identical to running it alone. */
ck_status ck_estimate_norm(ck_matrix a, const ck_adam_cfg* cfg, uint64_t restarts,
                           ck_norm_result* res, double* witness);

/* Batched ensemble (config 5): S independent square operators packed
 * block-diagonally into one uploaded matrix, member g at rows/cols
 * [off_g, off_g + n_g) with off_g = sum over h < g of round_up(n_h, 256).
 * estimate_norm for every member: restarts with member_seeds[g] (r = 0) or
 * mix_seed(member_seeds[g], r); results[g] is the best of member g. */
ck_status ck_estimate_norm_batch(ck_matrix packed, const int64_t* seg_n, int32_t nseg,
                                 const ck_adam_cfg* cfg, const uint64_t* member_seeds,
                                 uint64_t restarts, ck_norm_result* results);
/* Session over a packed batch: nseg members x ncols restart columns; column
 * k = g * ncols + c in ck_session_result. seeds has nseg * ncols entries. */
ck_status ck_session_create_batch(ck_matrix packed, const int64_t* seg_n, int32_t nseg,
                                  const ck_adam_cfg* cfg, const uint64_t* seeds, int32_t ncols,
                                  ck_session* out);

/* Session: the device-resident loop with explicit control (bench, observer).
 * `ncols` independent runs with seeds[c]; each follows projected_adam exactly. */
ck_status ck_session_create(ck_matrix a, const ck_adam_cfg* cfg, const uint64_t* seeds,
                            int32_t ncols, ck_session* out);
/* Runs until every column finished (max_steps == 0) or for at most max_steps
 * loop trips. *finished = 1 when all columns are done. */
ck_status ck_session_run(ck_session s, uint64_t max_steps, int32_t* finished);
/* One loop trip with per-step scalars for column 0 (AdamObserver mode). */
ck_status ck_session_step_observed(ck_session s, ck_step_info* info, double* x, double* x_min);
/* Device-timed steps (CUDA events on the session stream): runs `steps` loop trips.
 * mode 0: one event between every kernel -> total plus per-kernel milliseconds;
 * mode 1: CUDA-graph chunks, total only (per-kernel outputs set to -1).
 * Columns must not finish inside the timed region (max_iter/patience large enough). */
ck_status ck_session_time(ck_session s, uint64_t steps, int32_t mode, double* ms_total,
                          double* ms_apply, double* ms_transpose);
ck_status ck_session_result(ck_session s, int32_t column, ck_norm_result* res, double* witness);
ck_status ck_session_free(ck_session s);

/* ------------------------------------------- LU factors and the InverseOracle */
/* lu_factorize(A, pivot_tol), lu.hpp:55-177, on the device: band LU with row
 * partial pivoting and the reference's pivot rule -- the largest candidate,
 * ties to the first row in the elimination's touched order (lu.hpp:88-124) --
 * and its singularity tests: StructurallySingular when no unpivoted row of the
 * column is touched (lu.hpp:126), NumericallySingular when the best pivot is 0
 * or < pivot_tol * column max (:127-129). On failure *fail_col / *fail_pivot
 * (may be NULL) are set. Limits (CK_ERR_UNSUPPORTED / CK_ERR_OUT_OF_MEMORY,
 * reported before any allocation): kl + ku <= 16319 (the solve window) and
 * ~(3 kl + ku) * n * 8 bytes of device memory. */
ck_status ck_lu_factorize(ck_matrix a, double pivot_tol, ck_lu* out, int64_t* fail_col,
                          double* fail_pivot);
/* lu_factorize of nmem matrices at once (run_bench's per-matrix cond2 over an
 * ensemble, bench.hpp:430-442): one panel loop for the whole batch. status[g] is
 * CK_OK with out[g] the factors, or the member's error (out[g] = NULL) with
 * fail_col / fail_pivot (optional arrays) as for ck_lu_factorize. */
ck_status ck_lu_factorize_batch(const ck_matrix* a, int32_t nmem, double pivot_tol, ck_lu* out,
                                int32_t* status, int64_t* fail_col, double* fail_pivot);
ck_status ck_lu_free(ck_lu f);
/* n, band widths, LUFactors::pivot_min (lu.hpp:46), device bytes. */
ck_status ck_lu_get_info(ck_lu f, int64_t* n, int64_t* kl, int64_t* ku, double* pivot_min,
                         int64_t* device_bytes);
/* LAPACK band layout (ldab = 2kl+ku+1, column major, n columns) and 0-based ipiv. */
ck_status ck_lu_export(ck_lu f, double* ab, int32_t* ipiv);
/* LUFactors in the reference's shape (lu.hpp:42-47, 144-176): L strictly lower
 * in pivot coordinates, U upper with the diagonal first in each row, CSR with
 * ascending columns, row_perm[k] = original row pivoted at step k. Built on the
 * device on first request. ck_lu_csr_info gives the entry counts; any output
 * pointer of ck_lu_export_csr may be NULL. */
ck_status ck_lu_csr_info(ck_lu f, int64_t* nnz_l, int64_t* nnz_u);
ck_status ck_lu_export_csr(ck_lu f, int64_t* l_rp, int32_t* l_ci, double* l_va, int64_t* u_rp,
                           int32_t* u_ci, double* u_va, int64_t* row_perm);
/* lu_solve (lu.hpp:180-202): x = A^-1 b; lu_transpose_solve (lu.hpp:207-227): x = A^-T b. */
ck_status ck_lu_solve(ck_lu f, const double* b, double* x);
ck_status ck_lu_transpose_solve(ck_lu f, const double* b, double* x);
/* Restart columns that share one sweep of the operator in ck_estimate_norm (batch = 0)
 * and ck_estimate_norm_batch (batch = 1): estimate_norm's restarts (condest.hpp:301-312)
 * are independent runs, grouped for throughput only. */
ck_status ck_restart_group(ck_matrix a, uint64_t restarts, int32_t batch, int32_t* group);
/* The dense-block sweeps the InverseOracle loop runs on narrow bands
 * (max(kl, kl + ku) <= 192; same solves as ck_lu_solve / ck_lu_transpose_solve,
 * lu.hpp:180-227, with the 32 x 32 head triangles of every block inverted once
 * per factorisation). available = 0: the band is too wide or a head's growth
 * factor || |Hinv| |H| || exceeds 1e4, and the loop keeps the substitution
 * sweeps; ck_lu_dense_solve then returns CK_ERR_UNSUPPORTED. */
ck_status ck_lu_dense_info(ck_lu f, int32_t* available, double* growth);
ck_status ck_lu_dense_solve(ck_lu f, int32_t transpose, const double* b, double* x);
/* InverseOracle::loss / grad_inverse (condest.hpp:112-123, 142-146) on the device. */
ck_status ck_loss_inverse(ck_lu f, const double* x, double* loss);
ck_status ck_grad_inverse(ck_lu f, const double* x, double* g);
/* projected_adam(InverseOracle(f), cfg) / inv_norm2 (condest.hpp:138-152, 184-297, 320-322). */
ck_status ck_inv_projected_adam(ck_lu f, const ck_adam_cfg* cfg, ck_norm_result* res,
                                double* witness);
/* estimate_norm(InverseOracle(f), cfg, restarts), condest.hpp:301-312. */
ck_status ck_inv_estimate_norm(ck_lu f, const ck_adam_cfg* cfg, uint64_t restarts,
                               ck_norm_result* res, double* witness);
ck_status ck_session_create_inverse(ck_lu f, const ck_adam_cfg* cfg, const uint64_t* seeds,
                                    int32_t ncols, ck_session* out);
/* Column / row scaling (sparse.hpp:244-313) on the device, for the `cond
 * --scale column|row` path (condkit_cli.cpp:151-160). Norms are bit-identical
 * to column_norms / two_norm per row. The CSR arrays are the ones `a` was
 * uploaded from (host); va_out receives the scaled values in CSR order.
 * ZeroColumn / ZeroRow report the first zero-norm index in *zero_index. */
ck_status ck_column_norms(ck_matrix a, double* norms);
ck_status ck_row_norms(ck_matrix a, double* norms);
ck_status ck_column_scale(ck_matrix a, const int32_t* col_indices, const double* values,
                          double* values_out, double* norms, int64_t* zero_index);
ck_status ck_row_scale(ck_matrix a, const int64_t* row_offsets, const double* values,
                       double* values_out, const double* b, double* b_out, double* norms,
                       int64_t* zero_index);
/* unscale_solution (sparse.hpp:287-293): x = y / d componentwise. */
ck_status ck_unscale_solution(int64_t n, const double* y, const double* d, double* x);

/* Row-block partition of one operator across ranks (replaces
 * running projected_adam on the whole matrix, condest.hpp:184-297, for grids
 * that are split across GPUs). Rank p owns global rows/columns
 * [g0, g0 + n_loc). Its extended local operator (CSR, ext_rows x ext_cols)
 * orders both index spaces by global index as [left halo | own block, padded
 * to whole 256-row tiles | right halo]; the own block is tiles [tile0, tile1).
 * Rows: the own rows of A (complete) and the halo rows -- rows of A outside
 * the block with entries in own columns, restricted to those columns.
 * Halo lists (per peer q, offsets [q], [q+1] into the index arrays):
 *   xs: own columns q needs (extended column positions), xr: where the
 *   values from q land (extended halo column positions), ys/yr: the same for
 *   rows (y' = A x~). ext_global[e]: global column of extended position e, or
 *   -1 for padding (start vectors are drawn globally and sliced).
 * nccl_id != NULL: NCCL backend, one rank per process (ck_dist_nccl_id on
 * rank 0, broadcast by the caller). nccl_id == NULL: every rank in this
 * process on the current device, stepped in lockstep. */
typedef struct ck_dist_part {
  int64_t n_global;
  int64_t tile0, tile1;
  int64_t ext_rows, ext_cols;
  const int64_t* rp;
  const int32_t* ci;
  const double* va;
  const int64_t* xs_off;
  const int32_t* xs_idx;
  const int64_t* xr_off;
  const int32_t* xr_idx;
  const int64_t* ys_off;
  const int32_t* ys_idx;
  const int64_t* yr_off;
  const int32_t* yr_idx;
  const int64_t* ext_global;
} ck_dist_part;
typedef struct ck_dist_s* ck_dist;
ck_status ck_dist_nccl_id(void* id128);
ck_status ck_dist_create(const ck_dist_part* parts, int32_t nparts, int32_t rank0, int32_t nranks,
                         const void* nccl_id, const ck_adam_cfg* cfg, const uint64_t* seeds,
                         int32_t ncols, ck_dist* out);
ck_status ck_dist_run(ck_dist d, uint64_t max_steps, int32_t* finished);
/* device time of `steps` iterations (graph replay on the NCCL backend) */
ck_status ck_dist_time(ck_dist d, uint64_t steps, double* ms);
/* NormEstimate of restart column col; witness = local rank `part`'s
 * extended-order slice (ext_cols doubles), NULL to skip. Collective. */
ck_status ck_dist_result(ck_dist d, int32_t col, int32_t part, ck_norm_result* res,
                         double* witness);
/* Device layout of part `part`'s extended local operator (ck_matrix_get_info). */
ck_status ck_dist_part_info(ck_dist d, int32_t part, ck_matrix_info* info);
ck_status ck_dist_free(ck_dist d);

/* Ensembles on A^-1 (the sigma_min half of cond2 per member, config 5): nmem
 * independent factorisations, one device CTA per member per step. Column
 * k = g * ncols + c in ck_session_result; seeds has nmem * ncols entries.
 * Replaces running InverseOracle/estimate_norm (condest.hpp:156-175, 301-312)
 * once per matrix as run_bench does (bench.hpp:435). */
ck_status ck_session_create_inverse_batch(const ck_lu* lus, int32_t nmem, const ck_adam_cfg* cfg,
                                          const uint64_t* seeds, int32_t ncols, ck_session* out);
/* estimate_norm on every A_g^-1; member g's restarts seeded as in
 * ck_estimate_norm_batch; results[g] is the best of member g. */
ck_status ck_inv_estimate_norm_batch(const ck_lu* lus, int32_t nmem, const ck_adam_cfg* cfg,
                                     const uint64_t* member_seeds, uint64_t restarts,
                                     ck_norm_result* results);
/* cond2(A, cfg, restarts, pivot_tol), condest.hpp:341-365 (Cond2Result without the
 * factors: has_factors reports whether they were formed). */
ck_status ck_cond2(ck_matrix a, const ck_adam_cfg* cfg, uint64_t restarts, double pivot_tol,
                   double* kappa, ck_norm_result* fwd, ck_norm_result* inv, int32_t* has_factors);

/* ----------------------------------------------------- synthetic inputs (host) */
/* Operators of the BASELINE.json configurations (no reference counterpart for
 * kinds 2-5; kind 1 follows acceptance.cpp:240-254 plus BASELINE row scaling).
 * kind 1 Laplacian grid^2, 2 Stokes 3*grid^2, 3 hydro-mechanical 6*grid^2,
 * 5 banded (grid = n, param = bandwidth). Call with row_offsets == NULL to get
 * *nrows / *nnz, then with buffers of those sizes. */
ck_status ck_generate(int32_t kind, int64_t grid, int64_t param, uint64_t seed, int64_t* nrows,
                      int64_t* nnz, int64_t* row_offsets, int32_t* col_indices, double* values);

#ifdef __cplusplus
}
#endif
#endif
