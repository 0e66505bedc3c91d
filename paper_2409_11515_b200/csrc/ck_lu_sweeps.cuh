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

// 32x32 staging buffer for a block's head triangle (shared by the sweeps).
struct Head {
  double v[kLUBlock][kLUBlock + 1];
};

// Composite interchange of block blk, precomputed by k_convert_l_blocks:
// window position dst (relative to the block start) receives the value of
// position src; at most 64 moved positions per block.
__device__ __forceinline__ void block_perm(const BandView& b, int64_t blk, int& np,
                                           const int32_t*& pairs) {
  const int32_t* p = b.perm + blk * (1 + 2 * 2 * kLUBlock);
  np = p[0];
  pairs = p + 1;
}

// x := (L-part)^{-1} x, i.e. LAPACK gbtrs 'N' first half: for every step j
// interchange rows j, ipiv[j], then eliminate below j. Rows are staged through
// the ring. Per block, warp 0 applies the block's composite interchange and
// solves the 32x32 unit-lower head; then all warps update the tail while the
// next block's head multipliers and incoming rows are already being loaded --
// two CTA barriers per block.
template <int R>
__device__ void sweep_l_forward(const BandView& b, double* const* x, Ring* ring, Head& H) {
  const int64_t n = b.n;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  // initial window: rows [0, min(n, 32 + kl)) and block 0's head
  int64_t hi = lmin(n, kLUBlock + b.kl);
  for (int64_t i = tid; i < hi; i += nt)
#pragma unroll
    for (int r = 0; r < R; ++r) ring[r][i] = x[r][i];
  for (int q = tid; q < kLUBlock * kLUBlock; q += nt) H.v[q >> 5][q & 31] = b.lb[(int64_t)(q >> 5) * b.lb_ld + (q & 31)];
  __syncthreads();
  for (int64_t J = 0; J < n; J += kLUBlock) {
    const int64_t blk = J / kLUBlock;
    const int jb = (int)lmin(kLUBlock, n - J);
    const int64_t wend = lmin(n, J + kLUBlock + b.kl);
    const double* lb = b.lb + blk * kLUBlock * b.lb_ld;
    if (warp == 0) {
      int np;
      const int32_t* pairs;
      block_perm(b, blk, np, pairs);
      double pv[2][R];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int t = lane + 32 * h;
        if (t < np)
#pragma unroll
          for (int r = 0; r < R; ++r) pv[h][r] = ring[r][J + pairs[2 * t + 1]];
      }
      __syncwarp();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int t = lane + 32 * h;
        if (t < np)
#pragma unroll
          for (int r = 0; r < R; ++r) ring[r][J + pairs[2 * t]] = pv[h][r];
      }
      __syncwarp();
      double hv[R];
#pragma unroll
      for (int r = 0; r < R; ++r) hv[r] = lane < jb ? ring[r][J + lane] : 0.0;
      for (int c = 0; c < jb; ++c) {
        const double l = lane > c && lane < jb ? H.v[c][lane] : 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double y = __shfl_sync(0xffffffffu, hv[r], c);
          if (lane > c && lane < jb) hv[r] = __dsub_rn(hv[r], __dmul_rn(l, y));
        }
      }
      if (lane < jb)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          ring[r][J + lane] = hv[r];
          x[r][J + lane] = hv[r];  // head rows are final
        }
    }
    __syncthreads();
    // prefetch: the next block's head multipliers and its incoming rows
    const bool more = J + kLUBlock < n;
    const int64_t nend = lmin(n, J + 2 * kLUBlock + b.kl);
    double pf_h = 0.0, pf_x[R];
    if (more) {
      const int q = tid;
      if (q < kLUBlock * kLUBlock) pf_h = lb[(int64_t)kLUBlock * b.lb_ld + (int64_t)(q >> 5) * b.lb_ld + (q & 31)];
      if (hi + tid < nend)
#pragma unroll
        for (int r = 0; r < R; ++r) pf_x[r] = x[r][hi + tid];
    }
    // tail: rows J+jb .. wend-1 minus the block's contributions (column order)
    for (int64_t i = J + jb + tid; i < wend; i += nt) {
      double acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = ring[r][i];
      for (int c = 0; c < jb; ++c) {
        const double l = lb[(int64_t)c * b.lb_ld + (i - J)];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = __dsub_rn(acc[r], __dmul_rn(l, ring[r][J + c]));
      }
#pragma unroll
      for (int r = 0; r < R; ++r) ring[r][i] = acc[r];
    }
    if (more) {
      if (tid < kLUBlock * kLUBlock) H.v[tid >> 5][tid & 31] = pf_h;
      if (hi + tid < nend)
#pragma unroll
        for (int r = 0; r < R; ++r) ring[r][hi + tid] = pf_x[r];
      hi = nend;
    }
    __syncthreads();
  }
}

// Element q (0..1023) of U's 32x32 diagonal block of block J, staged as
// H.v[c][r] = U(J+r, J+c) for r <= c (zero elsewhere).
__device__ __forceinline__ double u_head_elem(const BandView& b, int64_t J, int jb, int q) {
  const int c = q >> 5, r = q & 31;
  return (r <= c && c < jb && c - r <= b.kv) ? AB(b, J + r, J + c) : 0.0;
}

// x := U^{-1} x (backward), U of bandwidth kv above the diagonal. Same
// two-barrier pipeline as sweep_l_forward, blocks in reverse.
template <int R>
__device__ void sweep_u_backward(const BandView& b, double* const* x, Ring* ring, Head& H) {
  const int64_t n = b.n;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int64_t nblk = (n + kLUBlock - 1) / kLUBlock;
  if (nblk == 0) return;
  int64_t lo;  // rows [lo, n) are in the ring
  {
    const int64_t J = (nblk - 1) * kLUBlock;
    lo = lmax(0, J - b.kv);
    for (int64_t i = lo + tid; i < n; i += nt)
#pragma unroll
      for (int r = 0; r < R; ++r) ring[r][i] = x[r][i];
    H.v[tid >> 5][tid & 31] = u_head_elem(b, J, (int)(n - J), tid);
  }
  __syncthreads();
  for (int64_t blk = nblk - 1; blk >= 0; --blk) {
    const int64_t J = blk * kLUBlock;
    const int jb = (int)lmin(kLUBlock, n - J);
    const int64_t wbeg = lmax(0, J - b.kv);
    if (warp == 0) {
      double h[R];
#pragma unroll
      for (int r = 0; r < R; ++r) h[r] = lane < jb ? ring[r][J + lane] : 0.0;
      for (int c = jb - 1; c >= 0; --c) {
        const double d = H.v[c][c];
        const double u = lane < c ? H.v[c][lane] : 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double y = __ddiv_rn(__shfl_sync(0xffffffffu, h[r], c), d);
          if (lane == c) h[r] = y;
          if (lane < c) h[r] = __dsub_rn(h[r], __dmul_rn(u, y));
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
    const bool more = blk > 0;
    const int64_t nlo = lmax(0, J - kLUBlock - b.kv);
    double pf_h = 0.0, pf_x[R];
    if (more) {
      pf_h = u_head_elem(b, J - kLUBlock, kLUBlock, tid);
      if (nlo + tid < lo)
#pragma unroll
        for (int r = 0; r < R; ++r) pf_x[r] = x[r][nlo + tid];
    }
    for (int64_t i = wbeg + tid; i < J; i += nt) {
      double acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = ring[r][i];
      const int cend = (int)lmin(jb, i + b.kv - J + 1);  // U(i, J+c) in band
      for (int c = 0; c < cend; ++c) {
        const int64_t k = J + c;
        const double u = AB(b, i, k);
        if (u != 0.0)
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r] = __dsub_rn(acc[r], __dmul_rn(u, ring[r][k]));
      }
#pragma unroll
      for (int r = 0; r < R; ++r) ring[r][i] = acc[r];
    }
    if (more) {
      H.v[tid >> 5][tid & 31] = pf_h;
      if (nlo + tid < lo)
#pragma unroll
        for (int r = 0; r < R; ++r) ring[r][nlo + tid] = pf_x[r];
      lo = nlo;
    }
    __syncthreads();
  }
}

// x := U^{-T} x (forward): w_k = (x_k - sum_{i<k} U(i,k) w_i) / U(k,k).
// Phase 1: commit the block's staged head and rows, start loading the next
// block's, one warp per head row forms its dot over the final rows below J.
// Phase 2: warp 0 solves the head triangle.
template <int R>
__device__ void sweep_ut_forward(const BandView& b, double* const* x, Ring* ring, double* s_dot,
                                 Head& H) {
  const int64_t n = b.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double pf_h = 0.0, pf_x[R];
  if (n > 0) {
    pf_h = u_head_elem(b, 0, (int)lmin(kLUBlock, n), tid);
    if (tid < lmin(kLUBlock, n))
#pragma unroll
      for (int r = 0; r < R; ++r) pf_x[r] = x[r][tid];
  }
  for (int64_t J = 0; J < n; J += kLUBlock) {
    const int jb = (int)lmin(kLUBlock, n - J);
    H.v[tid >> 5][tid & 31] = pf_h;
    if (tid < jb)
#pragma unroll
      for (int r = 0; r < R; ++r) ring[r][J + tid] = pf_x[r];
    const int64_t J1 = J + kLUBlock;
    if (J1 < n) {
      const int jb1 = (int)lmin(kLUBlock, n - J1);
      pf_h = u_head_elem(b, J1, jb1, tid);
      if (tid < jb1)
#pragma unroll
        for (int r = 0; r < R; ++r) pf_x[r] = x[r][J1 + tid];
    }
    if (warp < jb) {
      const int c = warp;
      const int64_t k = J + c;
      const int64_t i0 = lmax(0, k - b.kv);
      double sm[R];
#pragma unroll
      for (int r = 0; r < R; ++r) sm[r] = 0.0;
      for (int64_t i = i0 + lane; i < J; i += 32) {
        const double u = AB(b, i, k);
#pragma unroll
        for (int r = 0; r < R; ++r) sm[r] = __fma_rn(u, ring[r][i], sm[r]);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double t = warp_sum(sm[r]);
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
        const double d = H.v[c][c];
        // U(J+c, J+lane) for lane > c: column J+lane, row J+c
        const double u = lane > c && lane < jb ? H.v[lane][c] : 0.0;
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
// Phase 1: commit the block's head multipliers and head rows, write out the
// rows the previous block finalised, start the next block's loads, one warp
// per head column forms its dot over the tail. Phase 2: warp 0 solves the
// head and applies the block's inverse interchange.
template <int R>
__device__ void sweep_l_backward(const BandView& b, double* const* x, Ring* ring, double* s_dot,
                                 Head& H) {
  const int64_t n = b.n;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int64_t nblk = (n + kLUBlock - 1) / kLUBlock;
  if (nblk == 0) return;
  double pf_h, pf_x[R];
  {
    const int64_t J = (nblk - 1) * kLUBlock;
    pf_h = b.lb[J * b.lb_ld + (int64_t)(tid >> 5) * b.lb_ld + (tid & 31)];
    if (J + tid < n)
#pragma unroll
      for (int r = 0; r < R; ++r) pf_x[r] = x[r][J + tid];
  }
  for (int64_t blk = nblk - 1; blk >= 0; --blk) {
    const int64_t J = blk * kLUBlock;
    const int jb = (int)lmin(kLUBlock, n - J);
    const int64_t wend = lmin(n, J + kLUBlock + b.kl);
    const double* lb = b.lb + blk * kLUBlock * b.lb_ld;
    H.v[tid >> 5][tid & 31] = pf_h;
    if (tid < jb)
#pragma unroll
      for (int r = 0; r < R; ++r) ring[r][J + tid] = pf_x[r];
    if (blk + 1 < nblk) {  // rows block blk+1 finalised: [J1 + kl, wend1)
      const int64_t J1 = J + kLUBlock;
      for (int64_t i = J1 + b.kl + tid; i < lmin(n, J1 + kLUBlock + b.kl); i += nt)
#pragma unroll
        for (int r = 0; r < R; ++r) x[r][i] = ring[r][i];
    }
    if (blk > 0) {
      pf_h = lb[-(int64_t)kLUBlock * b.lb_ld + (int64_t)(tid >> 5) * b.lb_ld + (tid & 31)];
      if (tid < kLUBlock)
#pragma unroll
        for (int r = 0; r < R; ++r) pf_x[r] = x[r][J - kLUBlock + tid];
    }
    if (warp < jb) {
      const int c = warp;
      double sm[R];
#pragma unroll
      for (int r = 0; r < R; ++r) sm[r] = 0.0;
      for (int64_t i = J + jb + lane; i < wend; i += 32) {
        const double l = lb[(int64_t)c * b.lb_ld + (i - J)];
#pragma unroll
        for (int r = 0; r < R; ++r) sm[r] = __fma_rn(l, ring[r][i], sm[r]);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double t = warp_sum(sm[r]);
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
        const double l = lane < c ? H.v[lane][c] : 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double u = __shfl_sync(0xffffffffu, h[r], c);
          if (lane < c) h[r] = __dsub_rn(h[r], __dmul_rn(l, u));
        }
      }
      if (lane < jb)
#pragma unroll
        for (int r = 0; r < R; ++r) ring[r][J + lane] = h[r];
      __syncwarp();
      // inverse block interchange as one warp-wide scatter
      int np;
      const int32_t* pairs;
      block_perm(b, blk, np, pairs);
      double pv[2][R];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int t = lane + 32 * q;
        if (t < np)
#pragma unroll
          for (int r = 0; r < R; ++r) pv[q][r] = ring[r][J + pairs[2 * t]];
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int t = lane + 32 * q;
        if (t < np)
#pragma unroll
          for (int r = 0; r < R; ++r) ring[r][J + pairs[2 * t + 1]] = pv[q][r];
      }
    }
    __syncthreads();
  }
  // rows no step can touch any more: everything below kl + 32
  for (int64_t i = tid; i < lmin(n, kLUBlock + b.kl); i += nt)
#pragma unroll
    for (int r = 0; r < R; ++r) x[r][i] = ring[r][i];
  __syncthreads();
}

// x := A^{-1} x (transpose = false) or A^{-T} x, for R right-hand sides, by the
// calling CTA; smem holds R rings of ring_size doubles plus R*32 dot scratch.
template <int R>
__device__ __forceinline__ void inv_solve(const BandView& b, double* const* x, double* smem,
                                          int ring_size, bool transpose) {
  __shared__ Head H;
  Ring ring[R];
#pragma unroll
  for (int r = 0; r < R; ++r) ring[r] = Ring{smem + (int64_t)r * ring_size, ring_size - 1};
  double* s_dot = smem + (int64_t)R * ring_size;
  if (!transpose) {
    sweep_l_forward<R>(b, x, ring, H);
    sweep_u_backward<R>(b, x, ring, H);
  } else {
    sweep_ut_forward<R>(b, x, ring, s_dot, H);
    sweep_l_backward<R>(b, x, ring, s_dot, H);
  }
}

}  // namespace ck
