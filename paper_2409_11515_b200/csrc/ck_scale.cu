// Column / row norms and scalings on the device (sparse.hpp:173-186,
// 244-313): the preprocessing behind `cond --scale column|row`
// (condkit_cli.cpp:151-160).
//
// Norms run one thread per SELL row: a column of A is a row of A^T, whose
// entries the device copy keeps in increasing row order -- the order in which
// column_norms (sparse.hpp:246-268) accumulates -- so every norm is
// bit-identical to the reference. Scaled values are plain IEEE divisions.
#include <cmath>

#include "ck_common.h"
#include "ck_device.cuh"
#include "ck_internal.h"

namespace ck {

// kColumn: column_norms semantics (no non-finite early exit);
// otherwise two_norm (sparse.hpp:175-186).
template <bool kColumn>
__global__ void __launch_bounds__(256) k_sell_norms(int64_t nrows_pad, SellView s, double* out) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= nrows_pad) return;
  const int64_t base = sell_rowbase(s.sp[r / kSlice], r);
  const int len = s.len[r];
  double amax = 0.0;
  for (int j = 0; j < len; ++j) {
    const double a = fabs(s.val[sell_at(base, j)]);
    amax = amax < a ? a : amax;  // std::max(amax, |x|)
  }
  if (amax == 0.0) {
    out[r] = 0.0;
    return;
  }
  if (!kColumn && !isfinite(amax)) {
    out[r] = amax;
    return;
  }
  double sum = 0.0;
  for (int j = 0; j < len; ++j) {
    const double q = __ddiv_rn(s.val[sell_at(base, j)], amax);
    sum = __dadd_rn(sum, __dmul_rn(q, q));
  }
  out[r] = __dmul_rn(amax, __dsqrt_rn(sum));
}

__global__ void k_div_by_col(int64_t nnz, const int32_t* __restrict__ ci, const double* __restrict__ va,
                             const double* __restrict__ d, double* out) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < nnz) out[k] = __ddiv_rn(va[k], d[ci[k]]);
}

__global__ void k_div_by_row(int64_t nrows, const int64_t* __restrict__ rp, const double* __restrict__ va,
                             const double* __restrict__ d, double* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  const double di = d[i];
  for (int64_t k = rp[i]; k < rp[i + 1]; ++k) out[k] = __ddiv_rn(va[k], di);
}

__global__ void k_vec_div(int64_t n, const double* __restrict__ y, const double* __restrict__ d,
                          double* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = __ddiv_rn(y[i], d[i]);
}

static unsigned blocks(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + 255) / 256); }

// Norms of A's columns (column = true) or rows, in original index order, into
// the device buffer `out` (ncols or nrows doubles).
void matrix_norms(ck_matrix_s* m, bool column, double* out) {
  cudaStream_t st = m->stream;
  const Sell& s = column ? m->at : m->a;
  const int64_t n = column ? m->ncols : m->nrows;
  DBuf<double> perm_order(std::max<int64_t>(1, s.nrows_pad));
  if (column)
    k_sell_norms<true><<<blocks(s.nrows_pad), 256, 0, st>>>(s.nrows_pad, view(s), perm_order.p);
  else
    k_sell_norms<false><<<blocks(s.nrows_pad), 256, 0, st>>>(s.nrows_pad, view(s), perm_order.p);
  CK_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * std::max<int64_t>(1, n), st));
  scatter_perm(s.perm.p, s.nrows_pad, perm_order.p, out, st);
  CK_CUDA(cudaGetLastError());
  CK_CUDA(cudaStreamSynchronize(st));
}

void csr_divide(ck_matrix_s* m, bool column, const int64_t* h_rp, const int32_t* h_ci,
                const double* h_va, const double* d_norms, double* h_out) {
  cudaStream_t st = m->stream;
  const int64_t nnz = m->nnz;
  if (nnz == 0) return;
  DBuf<double> va(nnz), out(nnz);
  CK_CUDA(cudaMemcpyAsync(va.p, h_va, sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
  if (column) {
    DBuf<int32_t> ci(nnz);
    CK_CUDA(cudaMemcpyAsync(ci.p, h_ci, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st));
    k_div_by_col<<<blocks(nnz), 256, 0, st>>>(nnz, ci.p, va.p, d_norms, out.p);
    CK_CUDA(cudaGetLastError());
    CK_CUDA(cudaMemcpyAsync(h_out, out.p, sizeof(double) * nnz, cudaMemcpyDeviceToHost, st));
    CK_CUDA(cudaStreamSynchronize(st));
  } else {
    DBuf<int64_t> rp(m->nrows + 1);
    CK_CUDA(cudaMemcpyAsync(rp.p, h_rp, sizeof(int64_t) * (m->nrows + 1), cudaMemcpyHostToDevice, st));
    k_div_by_row<<<blocks(m->nrows), 256, 0, st>>>(m->nrows, rp.p, va.p, d_norms, out.p);
    CK_CUDA(cudaGetLastError());
    CK_CUDA(cudaMemcpyAsync(h_out, out.p, sizeof(double) * nnz, cudaMemcpyDeviceToHost, st));
    CK_CUDA(cudaStreamSynchronize(st));
  }
}

void vector_divide(int64_t n, const double* h_y, const double* h_d, double* h_out, cudaStream_t st) {
  if (n == 0) return;
  DBuf<double> y(n), d(n), out(n);
  CK_CUDA(cudaMemcpyAsync(y.p, h_y, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  CK_CUDA(cudaMemcpyAsync(d.p, h_d, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  k_vec_div<<<blocks(n), 256, 0, st>>>(n, y.p, d.p, out.p);
  CK_CUDA(cudaGetLastError());
  CK_CUDA(cudaMemcpyAsync(h_out, out.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  CK_CUDA(cudaStreamSynchronize(st));
}

}  // namespace ck
