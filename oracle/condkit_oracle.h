/*
 * condkit_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference CPU path (condkit, arXiv 2409.11515,
 * /root/reference/proj/include/condkit/ headers) used as the parity checker for
 * the B200 implementation. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it. The product library
 * (paper_2409_11515_b200/) never links or calls anything in this directory.
 *
 * The same entry points (prefix `ckref_` instead of `cko_`) are exported by
 * oracle/_ref/libcondkit_ref.so, which is the UNMODIFIED reference headers
 * compiled in place by oracle/Makefile; tests pin this restatement to it
 * bit-for-bit (tests/test_oracle.py).
 *
 * Status codes (shared with include/condkit_b200.h):
 *   0 ok, 1 DimensionMismatch, 2 invalid_argument, 3 logic_error,
 *   4 StructurallySingular, 5 NumericallySingular, 6 ZeroRHS, 7 ZeroSolution.
 * Matrices are CSR: int64 row offsets (nrows+1), int32 column indices,
 * double values, columns strictly increasing within a row.
 */
#ifndef CONDKIT_ORACLE_H
#define CONDKIT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double alpha, beta1, beta2, eps_stab;
  uint64_t max_iter, seed;
  double rel_tol;
  uint64_t patience;
} cko_adam_cfg;

typedef struct {
  double value;
  uint64_t iterations;
  int32_t converged;
  int32_t _pad;
} cko_norm_result;

typedef struct {
  double residual_norm, b_norm, a_norm, xhat_norm, kappa;
  int32_t kappa_supplied, verdict; /* verdict: 0 accepted, 1 rejected, 2 numerically_singular */
  double loose_lower, loose_upper, tight_lower, tight_upper;
  double true_error_cap, singularity_cap, threshold, eps_mach;
} cko_bounds_report;

typedef struct {
  double threshold;
  int32_t has_kappa, has_a_norm;
  double kappa, a_norm, eps_mach;
  cko_adam_cfg adam;
  uint64_t restarts;
  double pivot_tol;
} cko_verify_options;

typedef struct cko_lu cko_lu;

/* rng.hpp */
uint64_t cko_mix_seed(uint64_t base, uint64_t stream);
void cko_mt_draws(uint64_t seed, int64_t count, uint64_t* out);
void cko_random_unit_vectors(uint64_t seed, int64_t n, int64_t count, double* out);
void cko_uniform_in(uint64_t seed, int64_t count, double lo, double hi, double* out);

/* sparse.hpp */
double cko_two_norm(int64_t n, const double* v);
double cko_dot(int64_t n, const double* a, const double* b);
double cko_compensated_norm(int64_t n, const double* v);
void cko_matvec(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci,
                const double* va, const double* x, double* y);
void cko_column_norms(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci,
                      const double* va, double* out);
void cko_row_norms(int64_t nrows, const int64_t* rp, const double* va, double* out);
void cko_transpose_matvec(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci,
                          const double* va, const double* x, double* y);

/* condest.hpp, explicit oracle */
int cko_loss_explicit(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci,
                      const double* va, const double* x, double* loss);
int cko_grad_explicit(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci,
                      const double* va, const double* x, double* g);
int cko_projected_adam_explicit(int64_t nrows, int64_t ncols, const int64_t* rp,
                                const int32_t* ci, const double* va, const cko_adam_cfg* cfg,
                                cko_norm_result* res, double* witness, double* loss_trace);
int cko_estimate_norm_explicit(int64_t nrows, int64_t ncols, const int64_t* rp,
                               const int32_t* ci, const double* va, const cko_adam_cfg* cfg,
                               uint64_t restarts, cko_norm_result* res, double* witness);

/* lu.hpp */
int cko_lu_factorize(int64_t n, const int64_t* rp, const int32_t* ci, const double* va,
                     double pivot_tol, cko_lu** out, int64_t* fail_col, double* fail_pivot);
void cko_lu_free(cko_lu* f);
void cko_lu_info(const cko_lu* f, int64_t* n, int64_t* nnz_l, int64_t* nnz_u, double* pivot_min);
void cko_lu_export(const cko_lu* f, int64_t* l_rp, int32_t* l_ci, double* l_va, int64_t* u_rp,
                   int32_t* u_ci, double* u_va, int64_t* row_perm);
int cko_lu_solve(const cko_lu* f, const double* b, double* x);
int cko_lu_transpose_solve(const cko_lu* f, const double* b, double* x);

/* condest.hpp, inverse oracle and cond2 */
int cko_loss_inverse(const cko_lu* f, const double* x, double* loss);
int cko_grad_inverse(const cko_lu* f, const double* x, double* g);
int cko_projected_adam_inverse(const cko_lu* f, const cko_adam_cfg* cfg, cko_norm_result* res,
                               double* witness, double* loss_trace);
int cko_estimate_norm_inverse(const cko_lu* f, const cko_adam_cfg* cfg, uint64_t restarts,
                              cko_norm_result* res, double* witness);
int cko_cond2(int64_t n, const int64_t* rp, const int32_t* ci, const double* va,
              const cko_adam_cfg* cfg, uint64_t restarts, double pivot_tol, double* kappa,
              cko_norm_result* fwd, cko_norm_result* inv, int32_t* has_factors);

/* error_bounds.hpp */
int cko_loose_bounds(double residual_norm, double b_norm, double kappa, double* lower,
                     double* upper);
int cko_tight_bounds(double residual_norm, double a_norm, double xhat_norm, double kappa,
                     double* lower, double* upper);
int cko_propagate_bound(double eps_tight, double* out);
int cko_singularity_bound(double kappa, double eps_mach, double* out);
int cko_verify_solution(int64_t n, const int64_t* rp, const int32_t* ci, const double* va,
                        const double* xhat, const double* b, const cko_verify_options* opt,
                        cko_bounds_report* rep);

#ifdef __cplusplus
}
#endif
#endif
