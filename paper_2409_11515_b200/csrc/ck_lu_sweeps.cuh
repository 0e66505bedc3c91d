// Triangular sweeps over the device band LU (ck_lu.cu) -- shared by the
// standalone solves (ck_lu.cu) and the inverse Projected-Adam step
// (ck_inverse.cu). See ck_lu.cu for the layout and the algorithm.
#pragma once
#include "ck_device.cuh"
#include "ck_lu.h"

namespace ck {

__device__ __forceinline__ double& AB(const BandView& b, int64_t i, int64_t j) {
  return b.ab[(b.kv + i - j) + j * b.ldab];
}

// ----------------------------------------------------------- solves
// Ring-buffer view of the active rows of one right-hand side.
struct Ring {
  double* w;
  int mask;
  __device__ __forceinline__ double& operator[](int64_t row) const { return w[row & mask]; }
};

// x := (L-part)^{-1} x, i.e. LAPACK gbtrs 'N' first half: for every step j
// interchange rows j, ipiv[j], then eliminate below j. x is read/written in
// global memory; rows are staged through the ring.
template <int R>
__device__ void sweep_l_forward(const BandView& b, double* const* x, Ring* ring) {
  const int64_t n = b.n;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  int64_t hi = 0;  // rows [0, hi) have been loaded into the ring
  for (int64_t J = 0; J < n; J += kLUBlock) {
    const int jb = (int)lmin(kLUBlock, n - J);
    const int64_t wend = lmin(n, J + kLUBlock + b.kl);
    for (int64_t i = hi + tid; i < wend; i += nt)
#pragma unroll
      for (int r = 0; r < R; ++r) ring[r][i] = x[r][i];
    hi = lmax(hi, wend);
    __syncthreads();
    // block interchanges, in step order (one thread per column)
    if (tid < R)
      for (int c = 0; c < jb; ++c) {
        const int64_t p = b.ipiv[J + c];
        if (p != J + c) {
          double t = ring[tid][J + c];
          ring[tid][J + c] = ring[tid][p];
          ring[tid][p] = t;
        }
      }
    __syncthreads();
    const double* lb = b.lb + (J / kLUBlock) * kLUBlock * b.lb_ld;
    // head: 32x32 unit-lower solve in warp 0
    if (warp == 0) {
      double h[R];
#pragma unroll
      for (int r = 0; r < R; ++r) h[r] = lane < jb ? ring[r][J + lane] : 0.0;
      for (int c = 0; c < jb; ++c) {
        const double l = lane > c && lane < jb ? lb[(int64_t)c * b.lb_ld + lane] : 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double y = __shfl_sync(0xffffffffu, h[r], c);
          if (lane > c && lane < jb) h[r] = __dsub_rn(h[r], __dmul_rn(l, y));
        }
      }
      if (lane < jb)
#pragma unroll
        for (int r = 0; r < R; ++r) ring[r][J + lane] = h[r];
    }
    __syncthreads();
    // tail: rows J+jb .. wend-1 minus the block's contributions (column order)
    for (int64_t i = J + jb + tid; i < wend; i += nt) {
      double acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = ring[r][i];
      for (int c = 0; c < jb; ++c) {
        const double l = lb[(int64_t)c * b.lb_ld + (i - J)];
        if (l != 0.0)
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r] = __dsub_rn(acc[r], __dmul_rn(l, ring[r][J + c]));
      }
#pragma unroll
      for (int r = 0; r < R; ++r) ring[r][i] = acc[r];
    }
    // head rows are final
    for (int q = tid; q < jb * R; q += nt) {
      const int r = q / jb, c = q % jb;
      x[r][J + c] = ring[r][J + c];
    }
    __syncthreads();
  }
}

// x := U^{-1} x (backward), U of bandwidth kv above the diagonal.
template <int R>
__device__ void sweep_u_backward(const BandView& b, double* const* x, Ring* ring) {
  const int64_t n = b.n;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int64_t nblk = (n + kLUBlock - 1) / kLUBlock;
  int64_t lo = n;  // rows [lo, n) loaded
  for (int64_t blk = nblk - 1; blk >= 0; --blk) {
    const int64_t J = blk * kLUBlock;
    const int jb = (int)lmin(kLUBlock, n - J);
    const int64_t wbeg = lmax(0, J - b.kv);
    for (int64_t i = wbeg + tid; i < lo; i += nt)
#pragma unroll
      for (int r = 0; r < R; ++r) ring[r][i] = x[r][i];
    lo = lmin(lo, wbeg);
    __syncthreads();
    if (warp == 0) {
      double h[R];
#pragma unroll
      for (int r = 0; r < R; ++r) h[r] = lane < jb ? ring[r][J + lane] : 0.0;
      for (int c = jb - 1; c >= 0; --c) {
        const double d = AB(b, J + c, J + c);
        const double u = (lane < c && c - lane <= b.kv) ? AB(b, J + lane, J + c) : 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double y = __ddiv_rn(__shfl_sync(0xffffffffu, h[r], c), d);
          if (lane == c) h[r] = y;
          if (lane < c) h[r] = __dsub_rn(h[r], __dmul_rn(u, y));
        }
      }
      if (lane < jb)
#pragma unroll
        for (int r = 0; r < R; ++r) ring[r][J + lane] = h[r];
    }
    __syncthreads();
    for (int64_t i = wbeg + tid; i < J; i += nt) {
      double acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = ring[r][i];
      for (int c = 0; c < jb; ++c) {
        const int64_t k = J + c;
        if (i < k - b.kv) continue;
        const double u = AB(b, i, k);
        if (u != 0.0)
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r] = __dsub_rn(acc[r], __dmul_rn(u, ring[r][k]));
      }
#pragma unroll
      for (int r = 0; r < R; ++r) ring[r][i] = acc[r];
    }
    for (int q = tid; q < jb * R; q += nt) {
      const int r = q / jb, c = q % jb;
      x[r][J + c] = ring[r][J + c];
    }
    __syncthreads();
  }
}

// x := U^{-T} x (forward): w_k = (x_k - sum_{i<k} U(i,k) w_i) / U(k,k).
template <int R>
__device__ void sweep_ut_forward(const BandView& b, double* const* x, Ring* ring, double* s_dot) {
  const int64_t n = b.n;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = nt >> 5;
  for (int64_t J = 0; J < n; J += kLUBlock) {
    const int jb = (int)lmin(kLUBlock, n - J);
    for (int q = tid; q < jb * R; q += nt) {
      const int r = q / jb, c = q % jb;
      ring[r][J + c] = x[r][J + c];
    }
    __syncthreads();
    // dots over earlier (final) rows: one warp per head row
    for (int c = warp; c < jb; c += nwarps) {
      const int64_t k = J + c;
      const int64_t i0 = lmax(0, k - b.kv);
      double s[R];
#pragma unroll
      for (int r = 0; r < R; ++r) s[r] = 0.0;
      for (int64_t i = i0 + lane; i < J; i += 32) {
        const double u = AB(b, i, k);
#pragma unroll
        for (int r = 0; r < R; ++r) s[r] = __fma_rn(u, ring[r][i], s[r]);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double t = warp_sum(s[r]);
        if (lane == 0) s_dot[r * kLUBlock + c] = t;
      }
    }
    __syncthreads();
    if (warp == 0) {
      double h[R];
#pragma unroll
      for (int r = 0; r < R; ++r)
        h[r] = lane < jb ? __dsub_rn(ring[r][J + lane], s_dot[r * kLUBlock + lane]) : 0.0;
      for (int c = 0; c < jb; ++c) {
        const double d = AB(b, J + c, J + c);
        // U(J+c, J+lane) for lane > c lives in column J+lane
        const double u = (lane > c && lane < jb && lane - c <= b.kv) ? AB(b, J + c, J + lane) : 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double w = __ddiv_rn(__shfl_sync(0xffffffffu, h[r], c), d);
          if (lane == c) h[r] = w;
          if (lane > c) h[r] = __dsub_rn(h[r], __dmul_rn(u, w));
        }
      }
      if (lane < jb)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          ring[r][J + lane] = h[r];
          x[r][J + lane] = h[r];
        }
    }
    __syncthreads();
  }
}

// x := (L-part)^{-T} x: LAPACK gbtrs 'T' second half, blocks in reverse.
template <int R>
__device__ void sweep_l_backward(const BandView& b, double* const* x, Ring* ring, double* s_dot) {
  const int64_t n = b.n;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = nt >> 5;
  const int64_t nblk = (n + kLUBlock - 1) / kLUBlock;
  int64_t lo = n;  // rows [lo, n) are in the ring
  for (int64_t blk = nblk - 1; blk >= 0; --blk) {
    const int64_t J = blk * kLUBlock;
    const int jb = (int)lmin(kLUBlock, n - J);
    const int64_t wend = lmin(n, J + kLUBlock + b.kl);
    for (int64_t i = J + tid; i < lo; i += nt)
#pragma unroll
      for (int r = 0; r < R; ++r) ring[r][i] = x[r][i];
    lo = J;
    __syncthreads();
    const double* lb = b.lb + blk * kLUBlock * b.lb_ld;
    // head column c: minus the tail dot
    for (int c = warp; c < jb; c += nwarps) {
      double s[R];
#pragma unroll
      for (int r = 0; r < R; ++r) s[r] = 0.0;
      for (int64_t i = J + jb + lane; i < wend; i += 32) {
        const double l = lb[(int64_t)c * b.lb_ld + (i - J)];
#pragma unroll
        for (int r = 0; r < R; ++r) s[r] = __fma_rn(l, ring[r][i], s[r]);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double t = warp_sum(s[r]);
        if (lane == 0) s_dot[r * kLUBlock + c] = t;
      }
    }
    __syncthreads();
    if (warp == 0) {
      double h[R];
#pragma unroll
      for (int r = 0; r < R; ++r)
        h[r] = lane < jb ? __dsub_rn(ring[r][J + lane], s_dot[r * kLUBlock + lane]) : 0.0;
      for (int c = jb - 1; c >= 0; --c) {
        // u_c is final; push -l(c, lane) u_c into the columns lane < c
        const double l = lane < c ? lb[(int64_t)lane * b.lb_ld + c] : 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double u = __shfl_sync(0xffffffffu, h[r], c);
          if (lane < c) h[r] = __dsub_rn(h[r], __dmul_rn(l, u));
        }
      }
      if (lane < jb)
#pragma unroll
        for (int r = 0; r < R; ++r) ring[r][J + lane] = h[r];
    }
    __syncthreads();
    // inverse block permutation: interchanges in reverse step order
    if (tid < R)
      for (int c = jb - 1; c >= 0; --c) {
        const int64_t p = b.ipiv[J + c];
        if (p != J + c) {
          double t = ring[tid][J + c];
          ring[tid][J + c] = ring[tid][p];
          ring[tid][p] = t;
        }
      }
    __syncthreads();
    // rows that no later (lower) step can touch any more are final: steps
    // j < J only read or interchange rows <= j + kl < J + kl
    for (int64_t i = J + b.kl + tid; i < wend; i += nt)
#pragma unroll
      for (int r = 0; r < R; ++r) x[r][i] = ring[r][i];
    __syncthreads();
  }
  for (int64_t i = tid; i < lmin(n, b.kl); i += nt)
#pragma unroll
    for (int r = 0; r < R; ++r) x[r][i] = ring[r][i];
  __syncthreads();
}

// x := A^{-1} x (transpose = false) or A^{-T} x, for R right-hand sides, by the
// calling CTA; smem holds R rings of ring_size doubles plus R*32 dot scratch.
template <int R>
__device__ __forceinline__ void inv_solve(const BandView& b, double* const* x, double* smem,
                                          int ring_size, bool transpose) {
  Ring ring[R];
#pragma unroll
  for (int r = 0; r < R; ++r) ring[r] = Ring{smem + (int64_t)r * ring_size, ring_size - 1};
  double* s_dot = smem + (int64_t)R * ring_size;
  if (!transpose) {
    sweep_l_forward<R>(b, x, ring);
    sweep_u_backward<R>(b, x, ring);
  } else {
    sweep_ut_forward<R>(b, x, ring, s_dot);
    sweep_l_backward<R>(b, x, ring, s_dot);
  }
}

}  // namespace ck
