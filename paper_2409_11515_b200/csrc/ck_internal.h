// Cross-translation-unit internals (host side).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>

#include "ck_common.h"

struct ck_lu_s;

namespace ck {

constexpr int kNormParts = 296;  // partial blocks of the standalone norm (2 x 148 SMs)

void matrix_info(const ck_matrix_s* a, ck_matrix_info* info);
// Batched band LU (ck_lu.cu): codes[g] = CK_OK or the member's error status.
void lu_factorize_batch(ck_lu_s* const* fs, ck_matrix_s* const* ms, int S, double pivot_tol,
                        int32_t* codes, int64_t* fail_cols, double* fail_pivots);
void matrix_upload(ck_matrix_s* m, int64_t nrows, int64_t ncols, const int64_t* rp,
                   const int32_t* ci, const double* va);
void matrix_apply_host(ck_matrix_s* m, bool transpose, const double* x, double* y);
void matrix_apply_perm(ck_matrix_s* m, const double* x_perm, double* y_perm, cudaStream_t st);
void gather_perm(const int32_t* perm, int64_t n_out, const double* in, double* out,
                 cudaStream_t st);
void scatter_perm(const int32_t* perm, int64_t n_in, const double* in, double* out,
                  cudaStream_t st);
double device_norm(const double* v, int64_t n, double* scratch, cudaStream_t st);
void residual_norms(ck_matrix_s* m, const double* x, const double* b, double* rn, double* xn,
                    double* bn);
double loss_explicit_dev(ck_matrix_s* m, const double* x, bool* degenerate);
void grad_explicit_dev(ck_matrix_s* m, const double* x, double* g, bool* degenerate);

// Column / row norms and scalings (ck_scale.cu).
void matrix_norms(ck_matrix_s* m, bool column, double* out_dev);
void csr_divide(ck_matrix_s* m, bool column, const int64_t* h_rp, const int32_t* h_ci,
                const double* h_va, const double* d_norms, double* h_out);
void vector_divide(int64_t n, const double* h_y, const double* h_d, double* h_out, cudaStream_t st);

// Host mirror of random_unit_vector (rng.hpp:68-77) on a caller-owned engine
// state; bit-identical to the reference, Box-Muller transform multithreaded.
struct Mt64;
void random_unit_vector_host(void* engine /* std::mt19937_64* */, int64_t n, double* out,
                             const std::function<double*()>& dst = {});

// The prefetched start vector for (seed, n), if ck_start_vector_prefetch made
// one: *hx adopts the pinned buffer holding the normalised vector, *engine
// takes the engine state after the draw. False (nothing touched) otherwise.
bool take_start_prefetch(uint64_t seed, int64_t n, void* engine /* std::mt19937_64* */,
                         PinnedBuf<double>* hx);

}  // namespace ck
