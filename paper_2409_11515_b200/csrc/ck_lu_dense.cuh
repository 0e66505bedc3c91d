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

// ---------------------------------------------------------------- block ring
// The composite blocks of a sweep arrive by TMA bulk copies (cp.async.bulk, one
// thread, completion on an mbarrier per stage) in a ring of kDenseStages stages,
// issued kDenseStages blocks ahead of their use: a 24-57 KB block is several L2
// latencies of plain loads, and a one-block-ahead register prefetch left the
// sweep waiting (1640 cycles per block step against ~400 of shared-memory time).
constexpr int kDenseStagesMax = 4;

struct DenseRing {
  double* buf;           // [ns][stage] doubles, 16-byte aligned
  uint64_t* bar;         // [ns] mbarriers
  int ns;                // stages in use
  int64_t stage;         // doubles per stage (>= 32 * max(wl, wu))
  // the stage the next block arrives in and every stage's mbarrier phase
  // parity (bit s; same in every thread): the stages are used round robin
  // across sweeps, and a runtime modulo per block would sit on the critical path
  int cur;
  uint32_t pbits;
  __device__ __forceinline__ void advance() { cur = cur + 1 == ns ? 0 : cur + 1; }
};

// Shared memory of a dense CTA in doubles: window buffers, L^T partials, ring.
__host__ __device__ __forceinline__ int64_t dense_ring_stage(int wl, int wu) {
  return (int64_t)32 * (wl > wu ? wl : wu);
}

__device__ __forceinline__ void ring_init(const DenseRing& R) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < R.ns; ++s) {
      const uint32_t a = (uint32_t)__cvta_generic_to_shared(R.bar + s);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

// One thread: request `bytes` of block data into stage s.
__device__ __forceinline__ void ring_issue(const DenseRing& R, int s, const double* src, uint32_t bytes) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(R.bar + s);
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(R.buf + (int64_t)s * R.stage);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}

__device__ __forceinline__ void ring_wait(const DenseRing& R, int s, uint32_t parity) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(R.bar + s);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(b), "r"(parity)
        : "memory");
  }
}

// The k-th block a sweep visits is block first + k * step; its data is `bytes`
// at C + block * (bytes / 8). Prologue: the first ns blocks in flight.
struct RingFeed {
  const double* C;
  int first, step, nb;
  uint32_t bytes;
  // one thread requests block k of the sweep into stage s
  __device__ __forceinline__ void issue(const DenseRing& R, int k, int s) const {
    // the issuer sits in the last warp, which owns no window row for all but the widest
    // bands: the copy's address arithmetic stays off the head rows' warp
    if (threadIdx.x == kDenseThreads - 32 && k < nb)
      ring_issue(R, s, C + (int64_t)(first + k * step) * (bytes / 8), bytes);
  }
  // every stage is free here: the previous sweep waited for all it issued
  __device__ __forceinline__ void start(const DenseRing& R) const {
    int s = R.cur;
    for (int k = 0; k < R.ns; ++k) {
      issue(R, k, s);
      s = s + 1 == R.ns ? 0 : s + 1;
    }
  }
  // the current block's data (stage R.cur)
  __device__ __forceinline__ const double* wait(DenseRing& R) const {
    ring_wait(R, R.cur, (R.pbits >> R.cur) & 1u);
    R.pbits ^= 1u << R.cur;
    return R.buf + (int64_t)R.cur * R.stage;
  }
  // after the block's barrier: its stage takes block k + ns, the ring moves on
  __device__ __forceinline__ void next(DenseRing& R, int k) const {
    issue(R, k + R.ns, R.cur);
    R.advance();
  }
};

// 32 products in eight independent chains of four (the block step is one
// dependent chain per thread: fp64 FMA latency, not issue, bounds it), merged
// in a fixed order; the coefficients of this thread's row at cf[c * ld].
__device__ __forceinline__ double dense_dot32(const double* cf, int64_t ld, const double* h) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = __dmul_rn(cf[k * ld], h[k]);
#pragma unroll
  for (int c = 8; c < 32; c += 8) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = __fma_rn(cf[(c + k) * ld], h[c + k], a[k]);
  }
  return __dadd_rn(__dadd_rn(__dadd_rn(a[0], a[1]), __dadd_rn(a[2], a[3])),
                   __dadd_rn(__dadd_rn(a[4], a[5]), __dadd_rn(a[6], a[7])));
}

// Forward push sweep (L forward with PERM, U^T forward without): window rows
// [J, J + W), head = positions [0, 32). x is solved in place.
template <bool PERM>
__device__ void dense_forward(const DenseView& d, const double* __restrict__ C, int W, double* x,
                              double* wa, double* wb, DenseRing& R) {
  const int tid = threadIdx.x;
  const int64_t n = d.n;
  double* in = wa;
  double* out = wb;
  const RingFeed feed{C, 0, 1, d.nb, (uint32_t)(32 * W * sizeof(double))};
  feed.start(R);
  for (int q = tid; q < W; q += kDenseThreads) {
    const int pos = PERM ? d.pinv[q] : q;
    CK_DASSERT(pos >= 0 && pos < W);
    in[pos] = q < n ? x[q] : 0.0;
  }
  __syncthreads();
  for (int blk = 0; blk < d.nb; ++blk) {
    const int64_t J = (int64_t)blk * 32;
    const bool more = blk + 1 < d.nb;
    double fresh = 0.0;
    if (tid >= W && tid < W + 32) {  // the 32 rows entering the next window
      const int64_t g = J + W + (tid - W);
      fresh = g < n ? x[g] : 0.0;
    }
    // where this thread's value goes in the next window (the next block's
    // interchange folded in): requested before the block's data is waited for,
    // a global load here would sit on the block step's critical path
    int pos = tid < W ? tid - 32 : W - 32 + (tid - W);
    if (PERM && more && tid >= 32 && tid < W + 32) pos = d.pinv[(int64_t)(blk + 1) * d.wl + pos];
    const double* cf = feed.wait(R);
    if (tid < W) {
      const double acc = dense_dot32(cf + tid, W, in);
      if (tid < 32) {
        if (J + tid < n) x[J + tid] = acc;  // head rows are final
      } else if (more) {
        CK_DASSERT(pos >= 0 && pos < W);
        out[pos] = __dadd_rn(in[tid], acc);
      }
    } else if (tid < W + 32 && more) {
      CK_DASSERT(pos >= 0 && pos < W);
      out[pos] = fresh;
    }
    __syncthreads();
    feed.next(R, blk);  // the stage just read is free again
    double* t = in;
    in = out;
    out = t;
  }
}

// U backward: window rows [J - kv, J + 32), head = positions [kv, kv + 32).
static __device__ void dense_u_backward(const DenseView& d, double* x, double* wa, double* wb,
                                        DenseRing& R) {
  const int tid = threadIdx.x;
  const int64_t n = d.n;
  const int W = d.wu, kv = d.kv;
  double* in = wa;
  double* out = wb;
  const RingFeed feed{d.cub, d.nb - 1, -1, d.nb, (uint32_t)(32 * W * sizeof(double))};
  feed.start(R);
  {
    const int64_t J = (int64_t)(d.nb - 1) * 32;
    for (int q = tid; q < W; q += kDenseThreads) {
      const int64_t row = J - kv + q;
      in[q] = (row >= 0 && row < n) ? x[row] : 0.0;
    }
  }
  __syncthreads();
  for (int k = 0; k < d.nb; ++k) {
    const int blk = d.nb - 1 - k;
    const int64_t J = (int64_t)blk * 32;
    const bool more = blk > 0;
    double fresh = 0.0;
    if (tid >= W && tid < W + 32) {  // rows entering below: J - 32 - kv + t
      const int64_t g = J - 32 - kv + (tid - W);
      fresh = g >= 0 ? x[g] : 0.0;
    }
    const double* cf = feed.wait(R);
    if (tid < W) {
      const double acc = dense_dot32(cf + tid, W, in + kv);
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
    feed.next(R, k);
    double* t = in;
    in = out;
    out = t;
  }
}

// L^T backward: window rows [J, J + wl); the 32 head outputs are reductions
// over the whole window (parts of 32 inputs per warp, merged in part order),
// then the block's inverse interchange. part: [8][32] doubles of scratch.
static __device__ void dense_lt_backward(const DenseView& d, double* x, double* wa, double* wb, double* part,
                                         DenseRing& R) {
  const int tid = threadIdx.x, p = tid >> 5, c = tid & 31;
  const int64_t n = d.n;
  const int W = d.wl, kl = d.kl;
  const int P = (W + 31) >> 5;
  double* in = wa;
  double* out = wb;
  const RingFeed feed{d.clt, d.nb - 1, -1, d.nb, (uint32_t)(32 * W * sizeof(double))};
  feed.start(R);
  {
    const int64_t J = (int64_t)(d.nb - 1) * 32;
    for (int q = tid; q < W; q += kDenseThreads) in[q] = J + q < n ? x[J + q] : 0.0;
  }
  __syncthreads();
  for (int k = 0; k < d.nb; ++k) {
    const int blk = d.nb - 1 - k;
    const int64_t J = (int64_t)blk * 32;
    const bool more = blk > 0;
    double fresh = 0.0;
    if (more && tid < 32) fresh = x[J - 32 + tid];  // rows entering above (J >= 32 here)
    // the inverse interchange's target of this thread's row, requested ahead of the wait
    const int pos = tid < W ? d.psrc[(int64_t)blk * d.wl + tid] : 0;  // q -> psrc[q]
    const double* cf = feed.wait(R);
    if (p < P) {
      // inputs k' = p * 32 + kk of this part; coefficient (k', c) at cf[k' * 32 + c]
      const int kmax = W - p * 32 < 32 ? W - p * 32 : 32;
      const double* cp = cf + (int64_t)p * 32 * 32 + c;
      const double* ip = in + p * 32;
      double acc;
      if (kmax == 32) {
        acc = dense_dot32(cp, 32, ip);
      } else {  // the window's last, partial part: same chain assignment, missing terms are zeros
        double a[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = 0.0;
        for (int kk = 0; kk < kmax; ++kk) {
          const double t = __dmul_rn(cp[kk * 32], ip[kk]);
          a[kk & 7] = kk < 8 ? t : __fma_rn(cp[kk * 32], ip[kk], a[kk & 7]);
        }
        acc = __dadd_rn(__dadd_rn(__dadd_rn(a[0], a[1]), __dadd_rn(a[2], a[3])),
                        __dadd_rn(__dadd_rn(a[4], a[5]), __dadd_rn(a[6], a[7])));
      }
      part[p * 32 + c] = acc;
    }
    __syncthreads();
    if (tid < W) {
      double v;
      if (tid < 32) {
        v = part[tid];
        for (int pp = 1; pp < P; ++pp) v = __dadd_rn(v, part[pp * 32 + tid]);
      } else {
        v = in[tid];
      }
      CK_DASSERT(pos >= 0 && pos < W);
      if (more && pos < kl) {
        out[pos + 32] = v;
      } else if (J + pos < n) {
        x[J + pos] = v;  // the row leaves the window: final
      }
    }
    if (more && tid < 32) out[tid] = fresh;
    __syncthreads();
    feed.next(R, k);
    double* t = in;
    in = out;
    out = t;
  }
}

// x := U^-1 L^-1 P x  (transpose: x := P^T L^-T U^-T x), one CTA of
// kDenseThreads threads. smem: 3 * 256 doubles of window / partial scratch;
// R: the block ring (dynamic shared memory of the kernel).
__device__ __forceinline__ void dense_solve(const DenseView& d, double* x, double* smem, DenseRing& R,
                                            bool transpose) {
  double* wa = smem;
  double* wb = smem + kDenseThreads;
  double* part = smem + 2 * kDenseThreads;
  // positions past a window are read against zero coefficients: keep them finite
  wa[threadIdx.x] = 0.0;
  wb[threadIdx.x] = 0.0;
  __syncthreads();
  if (!transpose) {
    dense_forward<true>(d, d.clf, d.wl, x, wa, wb, R);
    __syncthreads();
    dense_u_backward(d, x, wa, wb, R);
  } else {
    dense_forward<false>(d, d.cut, d.wu, x, wa, wb, R);
    __syncthreads();
    dense_lt_backward(d, x, wa, wb, part, R);
  }
  __syncthreads();
}

// Ring of a dense CTA from its dynamic shared memory (dyn, 16-byte aligned,
// dyn_bytes long): the mbarriers first, then as many stages as fit (<= 4).
__device__ __forceinline__ DenseRing dense_ring(const DenseView& d, double* dyn, size_t dyn_bytes) {
  DenseRing R;
  R.bar = reinterpret_cast<uint64_t*>(dyn);
  R.buf = dyn + 8;  // 64 bytes of barriers
  R.stage = dense_ring_stage(d.wl, d.wu);
  const int64_t fit = ((int64_t)(dyn_bytes / sizeof(double)) - 8) / R.stage;
  R.ns = (int)(fit < kDenseStagesMax ? fit : kDenseStagesMax);
  R.cur = 0;
  R.pbits = 0;
  ring_init(R);
  return R;
}

// Dynamic shared memory (bytes) a dense CTA asks for: up to 4 stages within budget.
inline size_t dense_dyn_smem(int wl, int wu) {
  const size_t stage = (size_t)dense_ring_stage(wl, wu) * sizeof(double);
  const size_t budget = 200 * 1024;
  size_t ns = budget / stage;
  if (ns > (size_t)kDenseStagesMax) ns = kDenseStagesMax;
  if (ns < 2) ns = 2;
  return 64 + ns * stage;
}

}  // namespace ck
