// Dense-block sweeps for NARROW band factors (max(kl, kl + ku) <= kDenseMaxBand,
// e.g. BASELINE config 1: kl = ku = 64): the single-system latency path of the
// InverseOracle loop (lu.hpp:180-227 inside condest.hpp:112-152).
//
// The blocked substitution sweeps (ck_lu_sweeps.cuh) spend ~2-3.5k cycles per
// 32-row block in the 32 dependent steps of the head triangle. Here every block
// step is ONE matrix-vector product with a composite matrix built once per
// factorisation (k_dense_blocks, ck_lu.cu):
//
//   L forward    [ h ; t' ] = [ Linv ; -(Tl Linv) ] w_head + [ 0 ; t ]   after the
//                block's composite interchange (window of 32 + kl rows)
//   U backward   [ t' ; x ] = [ -(Tu Uinv) ; Uinv ] y_head + [ t ; 0 ]  (kv + 32 rows)
//   U^T forward  [ w ; t' ] = [ Uinv^T ; -(G Uinv^T) ] b_head + [ 0 ; t ]
//   L^T backward h = [ Linv^T | -(Tl Linv)^T ] [ v_head ; v_tail ], then the
//                inverse interchange
//
// with Linv / Uinv the inverses of the block's 32 x 32 head triangles and Tl,
// Tu, G the band coefficients the block reaches. One thread per window row
// accumulates 32 products (coefficients prefetched one block ahead into
// registers, the 32 head values broadcast from shared memory) and the window
// slides through two shared-memory buffers: one CTA barrier per block (two for
// L^T, whose 32 outputs are reductions over the window).
//
// Accuracy: the inverses replace substitution, so a solve is no longer
// componentwise backward stable; its error is bounded by eps * || |Hinv| |H| ||
// per block. k_dense_blocks measures that growth factor and the path is used
// only when it stays below kDenseMaxGrowth (solves then agree with the
// substitution sweeps to ~1e-13 relative); otherwise the session keeps the
// substitution sweeps.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "ck_device.cuh"

namespace ck {

constexpr int kDenseThreads = 256;
constexpr int kDenseMaxBand = kDenseThreads - 2 * 32;  // window rows + 32 loader threads <= 256
constexpr double kDenseMaxGrowth = 1.0e4;

struct DenseView {
  int64_t n;
  int nb;      // 32-row blocks
  int kl, kv;  // band below the diagonal of L, above the diagonal of U
  int wl, wu;  // window rows: 32 + kl, 32 + kv
  const double* clf;  // [nb][32][wl]  L forward: column c, window row r
  const double* clt;  // [nb][wl][32]  L^T backward: window input k, output c
  const double* cub;  // [nb][32][wu]  U backward: rows [0, kv) tail, [kv, wu) head
  const double* cut;  // [nb][32][wu]  U^T forward: rows [0, 32) head, [32, wu) tail
  // composite interchange of each L block: the value at window position q moves
  // to pinv[q]; position q receives the value of psrc[q]
  const uint8_t* pinv;  // [nb][wl]
  const uint8_t* psrc;  // [nb][wl]
};

// 32 products in four independent chains, merged in a fixed order.
__device__ __forceinline__ double dense_dot32(const double* cf, const double* h) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
  for (int c = 0; c < 32; c += 4) {
    a0 = __fma_rn(cf[c], h[c], a0);
    a1 = __fma_rn(cf[c + 1], h[c + 1], a1);
    a2 = __fma_rn(cf[c + 2], h[c + 2], a2);
    a3 = __fma_rn(cf[c + 3], h[c + 3], a3);
  }
  return __dadd_rn(__dadd_rn(a0, a1), __dadd_rn(a2, a3));
}

// Forward push sweep (L forward with PERM, U^T forward without): window rows
// [J, J + W), head = positions [0, 32). x is solved in place.
template <bool PERM>
__device__ void dense_forward(const DenseView& d, const double* __restrict__ C, int W, double* x,
                              double* wa, double* wb) {
  const int tid = threadIdx.x;
  const int64_t n = d.n;
  double* in = wa;
  double* out = wb;
  for (int q = tid; q < W; q += kDenseThreads) {
    const int pos = PERM ? d.pinv[q] : q;
    CK_DASSERT(pos >= 0 && pos < W);
    in[pos] = q < n ? x[q] : 0.0;
  }
  double cf[32];
  if (tid < W) {
#pragma unroll
    for (int c = 0; c < 32; ++c) cf[c] = C[(int64_t)c * W + tid];
  }
  __syncthreads();
  for (int blk = 0; blk < d.nb; ++blk) {
    const int64_t J = (int64_t)blk * 32;
    const bool more = blk + 1 < d.nb;
    double cn[32];
    double fresh = 0.0;
    if (more && tid < W) {
      const double* Cn = C + (int64_t)(blk + 1) * 32 * W;
#pragma unroll
      for (int c = 0; c < 32; ++c) cn[c] = Cn[(int64_t)c * W + tid];
    }
    if (tid >= W && tid < W + 32) {  // the 32 rows entering the next window
      const int64_t g = J + W + (tid - W);
      fresh = g < n ? x[g] : 0.0;
    }
    if (tid < W) {
      const double acc = dense_dot32(cf, in);
      if (tid < 32) {
        if (J + tid < n) x[J + tid] = acc;  // head rows are final
      } else if (more) {
        const int q = tid - 32;
        const int pos = PERM ? d.pinv[(int64_t)(blk + 1) * d.wl + q] : q;
        CK_DASSERT(pos >= 0 && pos < W);
        out[pos] = __dadd_rn(in[tid], acc);
      }
    } else if (tid < W + 32 && more) {
      const int q = W - 32 + (tid - W);
      const int pos = PERM ? d.pinv[(int64_t)(blk + 1) * d.wl + q] : q;
      CK_DASSERT(pos >= 0 && pos < W);
      out[pos] = fresh;
    }
    __syncthreads();
    double* t = in;
    in = out;
    out = t;
#pragma unroll
    for (int c = 0; c < 32; ++c) cf[c] = cn[c];
  }
}

// U backward: window rows [J - kv, J + 32), head = positions [kv, kv + 32).
static __device__ void dense_u_backward(const DenseView& d, double* x, double* wa, double* wb) {
  const int tid = threadIdx.x;
  const int64_t n = d.n;
  const int W = d.wu, kv = d.kv;
  const double* __restrict__ C = d.cub;
  double* in = wa;
  double* out = wb;
  {
    const int64_t J = (int64_t)(d.nb - 1) * 32;
    for (int q = tid; q < W; q += kDenseThreads) {
      const int64_t row = J - kv + q;
      in[q] = (row >= 0 && row < n) ? x[row] : 0.0;
    }
  }
  double cf[32];
  if (tid < W) {
    const double* C0 = C + (int64_t)(d.nb - 1) * 32 * W;
#pragma unroll
    for (int c = 0; c < 32; ++c) cf[c] = C0[(int64_t)c * W + tid];
  }
  __syncthreads();
  for (int blk = d.nb - 1; blk >= 0; --blk) {
    const int64_t J = (int64_t)blk * 32;
    const bool more = blk > 0;
    double cn[32];
    double fresh = 0.0;
    if (more && tid < W) {
      const double* Cn = C + (int64_t)(blk - 1) * 32 * W;
#pragma unroll
      for (int c = 0; c < 32; ++c) cn[c] = Cn[(int64_t)c * W + tid];
    }
    if (tid >= W && tid < W + 32) {  // rows entering below: J - 32 - kv + t
      const int64_t g = J - 32 - kv + (tid - W);
      fresh = g >= 0 ? x[g] : 0.0;
    }
    if (tid < W) {
      const double acc = dense_dot32(cf, in + kv);
      if (tid >= kv) {
        const int64_t row = J + (tid - kv);
        if (row < n) x[row] = acc;
      } else if (more) {
        out[tid + 32] = __dadd_rn(in[tid], acc);
      }
    } else if (tid < W + 32 && more) {
      out[tid - W] = fresh;
    }
    __syncthreads();
    double* t = in;
    in = out;
    out = t;
#pragma unroll
    for (int c = 0; c < 32; ++c) cf[c] = cn[c];
  }
}

// L^T backward: window rows [J, J + wl); the 32 head outputs are reductions
// over the whole window (parts of 32 inputs per warp, merged in part order),
// then the block's inverse interchange. part: [8][32] doubles of scratch.
static __device__ void dense_lt_backward(const DenseView& d, double* x, double* wa, double* wb, double* part) {
  const int tid = threadIdx.x, p = tid >> 5, c = tid & 31;
  const int64_t n = d.n;
  const int W = d.wl, kl = d.kl;
  const int P = (W + 31) >> 5;
  const double* __restrict__ C = d.clt;
  double* in = wa;
  double* out = wb;
  {
    const int64_t J = (int64_t)(d.nb - 1) * 32;
    for (int q = tid; q < W; q += kDenseThreads) in[q] = J + q < n ? x[J + q] : 0.0;
  }
  auto load_cf = [&](int blk, double* cf) {
    const double* Cb = C + ((int64_t)blk * W + p * 32) * 32 + c;
#pragma unroll
    for (int kk = 0; kk < 32; ++kk) cf[kk] = (p < P && p * 32 + kk < W) ? Cb[(int64_t)kk * 32] : 0.0;
  };
  double cf[32];
  load_cf(d.nb - 1, cf);
  __syncthreads();
  for (int blk = d.nb - 1; blk >= 0; --blk) {
    const int64_t J = (int64_t)blk * 32;
    const bool more = blk > 0;
    double cn[32];
    double fresh = 0.0;
    if (more) load_cf(blk - 1, cn);
    if (more && tid < 32) fresh = x[J - 32 + tid];  // rows entering above (J >= 32 here)
    if (p < P) part[p * 32 + c] = dense_dot32(cf, in + p * 32);
    __syncthreads();
    if (tid < W) {
      double v;
      if (tid < 32) {
        v = part[tid];
        for (int pp = 1; pp < P; ++pp) v = __dadd_rn(v, part[pp * 32 + tid]);
      } else {
        v = in[tid];
      }
      const int pos = d.psrc[(int64_t)blk * d.wl + tid];  // inverse interchange: q -> psrc[q]
      CK_DASSERT(pos >= 0 && pos < W);
      if (more && pos < kl) {
        out[pos + 32] = v;
      } else if (J + pos < n) {
        x[J + pos] = v;  // the row leaves the window: final
      }
    }
    if (more && tid < 32) out[tid] = fresh;
    __syncthreads();
    double* t = in;
    in = out;
    out = t;
#pragma unroll
    for (int kk = 0; kk < 32; ++kk) cf[kk] = cn[kk];
  }
}

// x := U^-1 L^-1 P x  (transpose: x := P^T L^-T U^-T x), one CTA of
// kDenseThreads threads; smem: 2 * 256 + 256 doubles.
__device__ __forceinline__ void dense_solve(const DenseView& d, double* x, double* smem, bool transpose) {
  double* wa = smem;
  double* wb = smem + kDenseThreads;
  double* part = smem + 2 * kDenseThreads;
  // positions past a window are read against zero coefficients: keep them finite
  wa[threadIdx.x] = 0.0;
  wb[threadIdx.x] = 0.0;
  __syncthreads();
  if (!transpose) {
    dense_forward<true>(d, d.clf, d.wl, x, wa, wb);
    __syncthreads();
    dense_u_backward(d, x, wa, wb);
  } else {
    dense_forward<false>(d, d.cut, d.wu, x, wa, wb);
    __syncthreads();
    dense_lt_backward(d, x, wa, wb, part);
  }
  __syncthreads();
}

}  // namespace ck
