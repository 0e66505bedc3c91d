// Triangular sweeps over the device band LU (ck_lu.cu) -- shared by the
// standalone solves (ck_lu.cu) and the inverse Projected-Adam step
// (ck_inverse.cu). See ck_lu.cu for the layout and the algorithm.
//
// One CTA of kSweepThreads threads walks the blocks of 32 steps in order,
// with two CTA barriers per block:
//   * warp 0 solves the block's 32x32 head (and applies the block's composite
//     interchange) -- the sequential critical path, fully unrolled;
//   * every warp folds the block into the rows it reaches (L, U: row tails),
//     or forms the head's dots over the final rows (U^T, L^T).
// The tail/dot coefficients of a block (32 columns x up to max(kl, kv)
// rows) are streamed from HBM into a shared-memory stage by TMA bulk copies
// (cp.async.bulk issued by one thread, completion on an mbarrier) while warp
// 0 is busy with a head, and the idle warps load the next head triangle,
// interchange pairs and incoming rows into registers at the same time. Rows
// beyond the stage capacity (very wide bands) are read directly.
#pragma once
#include <cooperative_groups.h>

#include "ck_device.cuh"
#include "ck_lu.h"

namespace ck {

// Phase timing of the sweeps (profiling build only, -DCK_SWEEP_PROF):
// thread 0 accumulates clock64 deltas per (sweep, phase) slot.
#ifdef CK_SWEEP_PROF
static __device__ unsigned long long g_sweep_prof[32];  // per translation unit
#define CK_PROF_INIT long long ck_prof_t = clock64()
#define CK_PROF(slot)                                                      \
  do {                                                                     \
    if (threadIdx.x == 0) {                                                \
      const long long t = clock64();                                       \
      atomicAdd(&g_sweep_prof[slot], (unsigned long long)(t - ck_prof_t)); \
      ck_prof_t = t;                                                       \
    }                                                                      \
  } while (0)
#else
#define CK_PROF_INIT
#define CK_PROF(slot)
#endif

constexpr int kSweepThreads = 1024;  // launch width of every sweep CTA
constexpr int kIssuer = 32;          // thread that drives the TMA stage (warp 1)

__device__ __forceinline__ double& AB(const BandView& b, int64_t i, int64_t j) {
  return b.ab[(b.kv + i - j) + j * b.ldab];
}

// Ring-buffer view of the active rows of one right-hand side.
struct Ring {
  double* w;
  int mask;
  __device__ __forceinline__ double& operator[](int64_t row) const { return w[row & mask]; }
};

// 32x32 staging buffer for a block's head triangle (+ the U diagonal's
// reciprocals for the U sweeps).
struct Head {
  double v[kLUBlock][kLUBlock + 1];
  double rd[kLUBlock];
};

// ------------------------------------------------------------ TMA stage
// Column c of a block's coefficients is a contiguous run of doubles in HBM
// starting at element first(c) (the two run kinds are below). The stage
// holds rows [0, srows) of each run at st[c * sld + (first(c) & 1) + m]: the
// bulk copy starts at the 16-byte boundary below the run.
struct Stage {
  double* st = nullptr;
  uint64_t* bar = nullptr;
  int64_t srows = 0, sld = 2;
  uint32_t parity = 0;

  __device__ void layout(int64_t cap, int64_t len, int64_t min_len) {
    const int64_t rows_fit = ((cap / kLUBlock) & ~(int64_t)1) - 2;
    srows = len < min_len ? 0 : lmax(0, lmin(len, rows_fit));
    sld = (srows + 3) & ~(int64_t)1;
  }
  __device__ __forceinline__ uint32_t copy_bytes(int64_t first) const {
    return srows == 0 ? 0u : (uint32_t)(8 * (((first & 1) + srows + 1) & ~(int64_t)1));
  }
  // One thread: arm the barrier and bulk-copy columns c < ncols of runs first(c).
  template <class First>
  __device__ void issue(const double* src, int ncols, First first) const {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
    uint32_t bytes = 0;
    for (int c = 0; c < ncols; ++c) bytes += copy_bytes(first(c));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    for (int c = 0; c < ncols; ++c) {
      const int64_t f = first(c);
      const uint32_t n8 = copy_bytes(f);
      if (n8 == 0) continue;
      const uint32_t d = (uint32_t)__cvta_generic_to_shared(st + (int64_t)c * sld);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
          "l"(src + (f & ~(int64_t)1)), "r"(n8), "r"(b)
          : "memory");
    }
  }
  // Every thread: wait for the stage issued last.
  __device__ void wait() {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
          : "=r"(done)
          : "r"(b), "r"(parity)
          : "memory");
    }
    parity ^= 1u;
  }
  __device__ __forceinline__ double at(int c, int off, int64_t m) const { return st[c * sld + off + m]; }
};

// L run of block blk, column c: lb rows 32 .. 32+kl-1 (the tail multipliers).
__device__ __forceinline__ int64_t l_run_first(const BandView& b, int64_t blk, int c) {
  return (blk * kLUBlock + c) * b.lb_ld + kLUBlock;
}
// U run of block J, column c: band entries of column J+c for rows
// J-kv+m, m in [0, kv); rows m < c lie outside the band (masked by users).
__device__ __forceinline__ int64_t u_run_first(const BandView& b, int64_t J, int c) {
  return (J + c) * b.ldab - c;
}

// ---------------------------------------------------------- interchanges
// Composite interchange of block blk (precomputed by k_convert_l_blocks):
// window position dst (relative to the block start) receives the value of
// position src; at most 64 moved positions, two per lane of warp 0.
struct Perm {
  int np;
  int2 p[2];  // (dst, src) for t = lane, lane + 32
};

__device__ __forceinline__ Perm load_perm(const BandView& b, int64_t blk, int lane) {
  const int32_t* p = b.perm + blk * (1 + 2 * 2 * kLUBlock);
  Perm q;
  q.np = p[0];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int t = lane + 32 * h;
    q.p[h] = t < q.np ? make_int2(p[1 + 2 * t], p[2 + 2 * t]) : make_int2(0, 0);
  }
  return q;
}

// Warp-wide gather: ring[J + dst] := ring[J + src] (inverse: roles swapped).
template <int R, bool kInverse>
__device__ __forceinline__ void apply_perm(const Perm& q, const Ring* ring, int64_t J, int lane) {
  double pv[2][R];
#pragma unroll
  for (int h = 0; h < 2; ++h)
    if (lane + 32 * h < q.np)
#pragma unroll
      for (int r = 0; r < R; ++r) pv[h][r] = ring[r][J + (kInverse ? q.p[h].x : q.p[h].y)];
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h)
    if (lane + 32 * h < q.np)
#pragma unroll
      for (int r = 0; r < R; ++r) ring[r][J + (kInverse ? q.p[h].y : q.p[h].x)] = pv[h][r];
  __syncwarp();
}

// a / d, correctly rounded, from rd = RN(1/d) (precomputed per pivot at
// factorisation): multiply plus one FMA correction (Markstein) -- a full
// division is ~380 cycles of dependent latency on the head solve's chain.
__device__ __forceinline__ double div_rcp(double a, double d, double rd) {
  const double q = __dmul_rn(a, rd);
  return __fma_rn(__fma_rn(-q, d, a), rd, q);
}

// Element q of the head triangles: U's 32x32 diagonal block of block J as
// H.v[c][r] = U(J+r, J+c) for r <= c (zero elsewhere); L's from lb.
// Columns c >= jb of a partial last block are padded with the identity, so
// the unrolled head solves need no bounds.
__device__ __forceinline__ double u_head_elem(const BandView& b, int64_t J, int jb, int q) {
  const int c = q >> 5, r = q & 31;
  if (c >= jb) return r == c ? 1.0 : 0.0;
  return (r <= c && c - r <= b.kv) ? AB(b, J + r, J + c) : 0.0;
}
__device__ __forceinline__ double u_head_rd(const BandView& b, int64_t J, int jb, int c) {
  return c < jb ? b.rdiag[J + c] : 1.0;
}
__device__ __forceinline__ double l_head_elem(const BandView& b, int64_t blk, int q) {
  return b.lb[(blk * kLUBlock + (q >> 5)) * b.lb_ld + (q & 31)];
}

// Next-block head prefetch by warps 1..31: elements q = tid-32 and, for
// warp 1, q + 992.
struct HeadPrefetch {
  double v[3];
  template <class F>
  __device__ __forceinline__ void load(F elem) {
    const int q = (int)threadIdx.x - 32;
    if (q >= 0) {
      v[0] = elem(q);
      if (q < 32) v[1] = elem(q + 992);
    }
  }
  template <class F, class G>
  __device__ __forceinline__ void load(F elem, G rd) {
    load(elem);
    const int q = (int)threadIdx.x - 32;
    if (q >= 0 && q < 32) v[2] = rd(q);
  }
  __device__ __forceinline__ void commit(Head& H, bool with_rd = false) const {
    const int q = (int)threadIdx.x - 32;
    if (q >= 0) {
      H.v[q >> 5][q & 31] = v[0];
      if (q < 32) {
        H.v[(q + 992) >> 5][(q + 992) & 31] = v[1];
        if (with_rd) H.rd[q] = v[2];
      }
    }
  }
};

// Incoming rows [r0, r1) (at most 32) by warp 1.
template <int R>
struct RowPrefetch {
  double v[R];
  __device__ __forceinline__ void load(double* const* x, int64_t r0, int64_t r1) {
    const int t = (int)threadIdx.x - 32;
    if (t >= 0 && t < 32 && r0 + t < r1)
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = x[r][r0 + t];
  }
  __device__ __forceinline__ void commit(const Ring* ring, int64_t r0, int64_t r1) const {
    const int t = (int)threadIdx.x - 32;
    if (t >= 0 && t < 32 && r0 + t < r1)
#pragma unroll
      for (int r = 0; r < R; ++r) ring[r][r0 + t] = v[r];
  }
};

// --------------------------------------------------------------- tails
// Lanes per row for a tail of `rows` rows: up to 4 (8 columns per lane)
// while the rows still fit one pass of the CTA. Fewer lanes per row keeps
// the issue count low -- warps without rows skip the tail altogether.
__device__ __forceinline__ int tail_log_lanes(int64_t rows) {
  int lg = 0;
  while (lg < 2 && ((int64_t)kSweepThreads >> (lg + 1)) >= rows) ++lg;
  return lg;
}

// ring[base + m] -= sum_{c < jb} coef(m, c) * ring[J + c] for m in [m0, m1):
// 2^lg lanes share a row (rows fastest within a warp), each summing every
// 2^lg-th column; the partial sums meet by shuffles.
template <int R, class Coef>
__device__ __forceinline__ void tail_update(int64_t base, int64_t m0, int64_t m1, int64_t J, int jb,
                                            int lg, const Ring* ring, Coef coef) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rs_bits = 5 - lg, G = 1 << lg;
  const int g = lane >> rs_bits, rs = lane & ((1 << rs_bits) - 1);
  const int64_t per_pass = (int64_t)kSweepThreads >> lg;
  for (int64_t mb = m0; mb < m1; mb += per_pass) {
    if (mb + ((int64_t)warp << rs_bits) >= m1) continue;  // warp-uniform
    const int64_t m = mb + ((int64_t)warp << rs_bits) + rs;
    const bool act = m < m1;
    double sm[R];
#pragma unroll
    for (int r = 0; r < R; ++r) sm[r] = 0.0;
    if (act) {
#pragma unroll 8
      for (int c = g; c < jb; c += G) {
        const double l = coef(m, c);
#pragma unroll
        for (int r = 0; r < R; ++r) sm[r] = __fma_rn(l, ring[r][J + c], sm[r]);
      }
    }
    for (int o = 16; o >= (1 << rs_bits); o >>= 1)
#pragma unroll
      for (int r = 0; r < R; ++r) sm[r] = __dadd_rn(sm[r], __shfl_xor_sync(0xffffffffu, sm[r], o));
    if (act && g == 0)
#pragma unroll
      for (int r = 0; r < R; ++r) ring[r][base + m] = __dsub_rn(ring[r][base + m], sm[r]);
  }
}

// Warp c's dot s_c = sum_m coef(m) * ring[base + m], m in [m0, m1).
template <int R, class Coef>
__device__ __forceinline__ void warp_dot(int64_t base, int64_t m0, int64_t m1, const Ring* ring,
                                         double* s_dot, int c, Coef coef) {
  const int lane = threadIdx.x & 31;
  double sm[R];
#pragma unroll
  for (int r = 0; r < R; ++r) sm[r] = 0.0;
#pragma unroll 4
  for (int64_t m = m0 + lane; m < m1; m += 32) {
    const double u = coef(m);
#pragma unroll
    for (int r = 0; r < R; ++r) sm[r] = __fma_rn(u, ring[r][base + m], sm[r]);
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const double t = warp_sum(sm[r]);
    if (lane == 0) s_dot[r * kLUBlock + c] = t;
  }
}

// ------------------------------------------------------ cluster split
// Wide bands on few systems: the sweep of one system runs on a cluster of
// CTAs. Rank 0 (the leader) keeps everything the single-CTA sweep has -- the
// solution ring, interchanges, head solves and prefetch -- and hands every
// block's tail rows / dot rows to ranks 1.. (helpers), split evenly. A helper
// loads its share of the block's coefficients before the barrier that releases
// the block, gets the head values pushed by the leader (tails) or reads the
// final ring rows it needs through DSMEM (dots), and writes its tail sums / dot
// partials back into the leader's shared memory. Two cluster barriers per
// block. Tail rows keep the single-CTA arithmetic (same per-row sum order for a
// given lanes-per-row); dot rows are summed per rank and combined in rank order.
struct Clu {
  int size, rank;
  double* tsum;   // leader smem: [R][ts] helper tail sums, by tail-relative row
  int64_t ts;
  double* dpart;  // leader smem: [size][R][32] dot partials per rank
  double* hy;     // helpers' smem (same offset in every CTA): [R][32] head values, pushed by the leader
};

// Leader, warp 0 after a head solve: lane c's solved values of the block go
// straight into every helper's head buffer (remote stores; the next cluster
// barrier publishes them), so the helpers need no DSMEM round trip.
template <int R>
__device__ __forceinline__ void clu_push_head(const Clu& C, int lane, int jb, const double* v, int slot = 0) {
  if (lane >= jb) return;
  auto cl = cooperative_groups::this_cluster();
  for (int k = 1; k < C.size; ++k) {
    double* d = cl.map_shared_rank(C.hy + slot * R * kLUBlock, k);
#pragma unroll
    for (int r = 0; r < R; ++r) d[r * kLUBlock + lane] = v[r];
  }
}

__device__ __forceinline__ void clu_sync() { cooperative_groups::this_cluster().sync(); }

template <class T>
__device__ __forceinline__ T* clu_leader(T* p) {
  return cooperative_groups::this_cluster().map_shared_rank(p, 0);
}

// Leader, after the CTA barrier that follows a head solve: warp k (1..size-1)
// copies the block's head values from the ring into helper k's head slot
// (remote stores, published by the next cluster barrier) -- all helpers at once.
template <int R>
__device__ __forceinline__ void clu_push_ring_head(const Clu& C, const Ring* ring, int64_t J, int jb,
                                                   int slot) {
  const int warp = (int)threadIdx.x >> 5, lane = (int)threadIdx.x & 31;
  if (warp < 1 || warp >= C.size || lane >= jb) return;
  double* d = cooperative_groups::this_cluster().map_shared_rank(C.hy + slot * R * kLUBlock, warp);
#pragma unroll
  for (int r = 0; r < R; ++r) d[r * kLUBlock + lane] = ring[r][J + lane];
}

// Rows [lo, hi) of share k out of `size` of the row range [m0, m1).
// (32-bit arithmetic: the range is at most a band width, k < 16 -- a 64-bit
// division is ~100 instructions on every helper's path, twice per block)
__device__ __forceinline__ int64_t clu_cut(int64_t m0, int64_t m1, int k, int size) {
  return m0 + (int64_t)(((uint32_t)(m1 - m0) * (uint32_t)k) / (uint32_t)size);
}

// Helper: the coefficients of a share, cf[c * (hi - lo) + (m - lo)] = coef(m, c)
// for m in [lo, hi), c < jb -- loaded before the cluster barrier that releases
// the head values, so their latency hides behind the leader's head solve. Warp
// c loads column c, 32 consecutive rows per step, 8 steps in flight (TMA bulk
// copies of the 32 runs, one thread issuing, measured slower: 164 vs 134 ms per
// config-2 iteration).
template <class Coef>
__device__ __forceinline__ void helper_fetch(int64_t lo, int64_t hi, int jb, double* cf, Coef coef) {
  constexpr int U = 8;
  const int sh = (int)(hi - lo);
  const int c = (int)threadIdx.x >> 5, l = (int)threadIdx.x & 31;
  if (c >= jb) return;
  for (int m0 = l; m0 < sh; m0 += 32 * U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int mm = m0 + 32 * u;
      v[u] = mm < sh ? coef(lo + mm, c) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int mm = m0 + 32 * u;
      if (mm < sh) cf[c * sh + mm] = v[u];
    }
  }
}

// Helper: the same share copied asynchronously (cp.async, 8 bytes per element,
// warp c -> column c, 32 consecutive rows per step): the copies proceed while
// the helper works on the previous block; cp_async_wait<0>() + a CTA barrier
// before use. Element (m, c) of the share is src[first(c) + (m - lo)].
template <class First>
__device__ __forceinline__ void helper_fetch_async(int64_t lo, int64_t hi, int jb, double* cf,
                                                   const double* src, First first) {
  const int sh = (int)(hi - lo);
  const int c = (int)threadIdx.x >> 5, l = (int)threadIdx.x & 31;
  if (c < jb) {
    const double* s0 = src + first(c);
    for (int mm = l; mm < sh; mm += 32) cp_async_elem(cf + c * sh + mm, s0 + mm);
  }
  cp_async_commit();
}

// Helper: sums of rows m in [lo, hi) of a block tail, sum_c cf(m, c) * y_c,
// written to the leader's tsum (same lane split and order as tail_update).
template <int R>
__device__ __forceinline__ void helper_tail(int64_t lo, int64_t hi, int jb, const double* hy,
                                            const double* cf, const Clu& C, bool umask = false) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lg = tail_log_lanes(hi - lo);
  const int rs_bits = 5 - lg, G = 1 << lg;
  const int g = lane >> rs_bits, rs = lane & ((1 << rs_bits) - 1);
  const int64_t per_pass = (int64_t)kSweepThreads >> lg;
  double* ts = clu_leader(C.tsum);
  for (int64_t mb = lo; mb < hi; mb += per_pass) {
    if (mb + ((int64_t)warp << rs_bits) >= hi) continue;  // warp-uniform
    const int64_t m = mb + ((int64_t)warp << rs_bits) + rs;
    const bool act = m < hi;
    double sm[R];
#pragma unroll
    for (int r = 0; r < R; ++r) sm[r] = 0.0;
    if (act) {
#pragma unroll 8
      for (int c = g; c < jb; c += G) {
        const double l = (umask && m < c) ? 0.0 : cf[(int64_t)c * (hi - lo) + (m - lo)];
#pragma unroll
        for (int r = 0; r < R; ++r) sm[r] = __fma_rn(l, hy[r * kLUBlock + c], sm[r]);
      }
    }
    for (int o = 16; o >= (1 << rs_bits); o >>= 1)
#pragma unroll
      for (int r = 0; r < R; ++r) sm[r] = __dadd_rn(sm[r], __shfl_xor_sync(0xffffffffu, sm[r], o));
    if (act && g == 0)
#pragma unroll
      for (int r = 0; r < R; ++r) ts[r * C.ts + m] = sm[r];
  }
}

// Helper: dot partials of rows m in [lo, hi) (ring rows base + m, copied from
// the leader into hl) for every head column c < jb, into the leader's dpart.
template <int R>
__device__ __forceinline__ void helper_dots(const Ring* lring, int64_t base, int64_t lo, int64_t hi, int jb,
                                            int64_t cmin_off, double* hl, const double* cf, const Clu& C) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int64_t m = lo + tid; m < hi; m += kSweepThreads)
#pragma unroll
    for (int r = 0; r < R; ++r) hl[r * (hi - lo) + (m - lo)] = lring[r][base + m];
  __syncthreads();
  double* dp = clu_leader(C.dpart) + (int64_t)C.rank * R * kLUBlock;
  const int c = warp;
  double sm[R];
#pragma unroll
  for (int r = 0; r < R; ++r) sm[r] = 0.0;
  if (c < jb) {
    const int64_t s0 = lmax(lo, cmin_off >= 0 ? (int64_t)c + cmin_off : lo);
#pragma unroll 4
    for (int64_t m = s0 + lane; m < hi; m += 32) {
      const double u = cf[(int64_t)c * (hi - lo) + (m - lo)];
#pragma unroll
      for (int r = 0; r < R; ++r) sm[r] = __fma_rn(u, hl[r * (hi - lo) + (m - lo)], sm[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const double t = warp_sum(sm[r]);
    if (lane == 0) dp[r * kLUBlock + c] = t;
  }
  __syncthreads();  // hl is reused by the next block
}

// ------------------------------------------------------------ L forward
// x := (L-part)^{-1} x, i.e. LAPACK gbtrs 'N' first half: for every step j
// interchange rows j, ipiv[j], then eliminate below j.
template <int R, bool CLU = false>
__device__ void sweep_l_forward(const BandView& b, double* const* x, Ring* ring, Head& H, Stage& S,
                                const Clu& C) {
  const int64_t n = b.n;
  const int tid = threadIdx.x, nt = kSweepThreads, lane = tid & 31, warp = tid >> 5;
  if (n == 0) return;
  const int lg = tail_log_lanes(CLU ? (b.kl + C.size - 1) / C.size : b.kl);
  Perm pq;
  HeadPrefetch ph;
  RowPrefetch<R> px;
  int64_t hi = lmin(n, kLUBlock + b.kl);  // rows [.., hi) are in the ring
  for (int64_t i = tid; i < hi; i += nt)
#pragma unroll
    for (int r = 0; r < R; ++r) ring[r][i] = x[r][i];
  H.v[tid >> 5][tid & 31] = l_head_elem(b, 0, tid);
  if (warp == 0) pq = load_perm(b, 0, lane);
  __syncthreads();
  CK_PROF_INIT;
  for (int64_t J = 0; J < n; J += kLUBlock) {
    const int64_t blk = J / kLUBlock;
    const int jb = (int)lmin(kLUBlock, n - J);
    const int64_t wend = lmin(n, J + kLUBlock + b.kl);
    const int64_t nend = lmin(n, J + 2 * kLUBlock + b.kl);
    const bool more = J + kLUBlock < n;
    const bool tail = wend > J + jb;
    if (warp == 0) {
      apply_perm<R, false>(pq, ring, J, lane);
      if (more) pq = load_perm(b, blk + 1, lane);
      double hv[R];
#pragma unroll
      for (int r = 0; r < R; ++r) hv[r] = lane < jb ? ring[r][J + lane] : 0.0;
      // branch-free: lanes <= c subtract 0 * y (lb is zero past the block)
#pragma unroll
      for (int c = 0; c < kLUBlock; ++c) {
        const double l = lane > c ? H.v[c][lane] : 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) hv[r] = __dsub_rn(hv[r], __dmul_rn(l, __shfl_sync(0xffffffffu, hv[r], c)));
      }
      if (lane < jb)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          ring[r][J + lane] = hv[r];
          x[r][J + lane] = hv[r];  // head rows are final
        }

    } else {
      if (tid == kIssuer && tail) S.issue(b.lb, jb, [&](int c) { return l_run_first(b, blk, c); });
      if (more) {
        ph.load([&](int q) { return l_head_elem(b, blk + 1, q); });
        px.load(x, hi, nend);
      }
    }
    CK_PROF(0);
    __syncthreads();
    CK_PROF(1);
    if (CLU && tail) clu_push_ring_head<R>(C, ring, J, jb, 0);
    if (CLU) clu_sync();  // head values pushed to the helpers
    const int64_t M = wend - J - kLUBlock;  // tail rows
    const int64_t mh = CLU ? 0 : M;  // the leader's own tail rows (none with helpers)
    if (tail) {
      S.wait();
      const double* lbk = b.lb + blk * kLUBlock * b.lb_ld;
      tail_update<R>(J + kLUBlock, 0, mh, J, jb, lg, ring, [&](int64_t m, int c) {
        return m < S.srows ? S.at(c, (int)((c * b.lb_ld) & 1), m) : lbk[c * b.lb_ld + kLUBlock + m];
      });
    }
    if (CLU) {
      clu_sync();  // helper sums in tsum
      for (int64_t m = mh + tid; m < M; m += nt)
#pragma unroll
        for (int r = 0; r < R; ++r)
          ring[r][J + kLUBlock + m] = __dsub_rn(ring[r][J + kLUBlock + m], C.tsum[r * C.ts + m]);
    }
    if (more) {
      ph.commit(H);
      px.commit(ring, hi, nend);
      hi = nend;
    }
    CK_PROF(4);
    __syncthreads();
    CK_PROF(5);
  }
}

// ----------------------------------------------------------- U backward
// x := U^{-1} x (backward), U of bandwidth kv above the diagonal; blocks in
// reverse, same two phases as sweep_l_forward.
template <int R>
__device__ void sweep_u_backward(const BandView& b, double* const* x, Ring* ring, Head& H, Stage& S) {
  const int64_t n = b.n;
  const int tid = threadIdx.x, nt = kSweepThreads, lane = tid & 31, warp = tid >> 5;
  const int64_t nblk = (n + kLUBlock - 1) / kLUBlock;
  if (nblk == 0) return;
  const int lg = tail_log_lanes(b.kv);
  HeadPrefetch ph;
  RowPrefetch<R> px;
  int64_t lo;  // rows [lo, n) are in the ring
  {
    const int64_t J = (nblk - 1) * kLUBlock;
    lo = lmax(0, J - b.kv);
    for (int64_t i = lo + tid; i < n; i += nt)
#pragma unroll
      for (int r = 0; r < R; ++r) ring[r][i] = x[r][i];
    H.v[tid >> 5][tid & 31] = u_head_elem(b, J, (int)(n - J), tid);
    if (tid < kLUBlock) H.rd[tid] = u_head_rd(b, J, (int)(n - J), tid);
  }
  __syncthreads();
  CK_PROF_INIT;
  for (int64_t blk = nblk - 1; blk >= 0; --blk) {
    const int64_t J = blk * kLUBlock;
    const int jb = (int)lmin(kLUBlock, n - J);
    const int64_t wbeg = lmax(0, J - b.kv);
    const int64_t nlo = lmax(0, J - kLUBlock - b.kv);
    const bool more = blk > 0;
    const bool tail = J > wbeg;
    if (warp == 0) {
      double h[R];
#pragma unroll
      for (int r = 0; r < R; ++r) h[r] = lane < jb ? ring[r][J + lane] : 0.0;
#pragma unroll
      for (int c = kLUBlock - 1; c >= 0; --c) {
        const double d = H.v[c][c], rd = H.rd[c];
        const double u = lane < c ? H.v[c][lane] : 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double y = div_rcp(__shfl_sync(0xffffffffu, h[r], c), d, rd);
          const double t = __dsub_rn(h[r], __dmul_rn(u, y));
          h[r] = lane == c ? y : t;
        }
      }
      if (lane < jb)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          ring[r][J + lane] = h[r];
          x[r][J + lane] = h[r];
        }
    } else {
      if (tid == kIssuer && tail) S.issue(b.ab, jb, [&](int c) { return u_run_first(b, J, c); });
      if (more) {
        ph.load([&](int q) { return u_head_elem(b, J - kLUBlock, kLUBlock, q); },
                [&](int c) { return u_head_rd(b, J - kLUBlock, kLUBlock, c); });
        px.load(x, nlo, lo);
      }
    }
    CK_PROF(8);
    __syncthreads();
    CK_PROF(9);
    const int64_t m0 = wbeg - (J - b.kv);  // first tail row (relative)
    if (tail) {
      S.wait();
      // tail row i = J - kv + m; U(i, J+c) lies in the band for m >= c
      tail_update<R>(J - b.kv, m0, b.kv, J, jb, lg, ring, [&](int64_t m, int c) {
        if (m < c) return 0.0;
        const int64_t f = u_run_first(b, J, c);
        return m < S.srows ? S.at(c, (int)(f & 1), m) : b.ab[f + m];
      });
    }
    if (more) {
      ph.commit(H, true);
      px.commit(ring, nlo, lo);
      lo = nlo;
    }
    CK_PROF(12);
    __syncthreads();
    CK_PROF(13);
  }
}

// U backward on a cluster: one cluster barrier per block. The helpers' share of
// block J's tail -- every row above the next head block ("far" rows) -- is
// computed while the leader solves the next head, and folded in by the leader
// one block later; the next head block's rows ("near": J-32 .. J-1) the leader
// does itself right after the barrier, after the pending far rows of block J+32
// (per-row order: blocks in sweep order, as in the single-CTA sweep). Tail sums
// and head values are double-buffered by block parity.
template <int R>
__device__ void sweep_u_backward_clu(const BandView& b, double* const* x, Ring* ring, Head& H,
                                     const Clu& C) {
  __shared__ double s_un[kLUBlock][kLUBlock + 1];  // near coefficients [m - (kv-32)][c]
  const int64_t n = b.n;
  const int tid = threadIdx.x, nt = kSweepThreads, lane = tid & 31, warp = tid >> 5;
  const int64_t nblk = (n + kLUBlock - 1) / kLUBlock;
  if (nblk == 0) return;
  HeadPrefetch ph;
  RowPrefetch<R> px;
  int64_t lo;  // rows [lo, n) are in the ring
  {
    const int64_t J = (nblk - 1) * kLUBlock;
    lo = lmax(0, J - b.kv);
    for (int64_t i = lo + tid; i < n; i += nt)
#pragma unroll
      for (int r = 0; r < R; ++r) ring[r][i] = x[r][i];
    H.v[tid >> 5][tid & 31] = u_head_elem(b, J, (int)(n - J), tid);
    if (tid < kLUBlock) H.rd[tid] = u_head_rd(b, J, (int)(n - J), tid);
  }
  __syncthreads();
  int64_t pend_J = -1, pend_m0 = 0, pend_m1 = 0;  // far rows of the previous block, in flight
  double un[2] = {0.0, 0.0};                      // near coefficients loaded during the head
  CK_PROF_INIT;
  for (int64_t blk = nblk - 1; blk >= 0; --blk) {
    const int64_t J = blk * kLUBlock;
    const int jb = (int)lmin(kLUBlock, n - J);
    const int64_t wbeg = lmax(0, J - b.kv);
    const int64_t nlo = lmax(0, J - kLUBlock - b.kv);
    const bool more = blk > 0;
    const bool tail = J > wbeg;
    const int64_t m0 = wbeg - (J - b.kv);        // first tail row (relative)
    const int64_t mn = lmax(m0, b.kv - kLUBlock);  // first near row
    if (warp == 0) {
      double h[R];
#pragma unroll
      for (int r = 0; r < R; ++r) h[r] = lane < jb ? ring[r][J + lane] : 0.0;
#pragma unroll
      for (int c = kLUBlock - 1; c >= 0; --c) {
        const double d = H.v[c][c], rd = H.rd[c];
        const double u = lane < c ? H.v[c][lane] : 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double y = div_rcp(__shfl_sync(0xffffffffu, h[r], c), d, rd);
          const double t = __dsub_rn(h[r], __dmul_rn(u, y));
          h[r] = lane == c ? y : t;
        }
      }
      if (lane < jb)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          ring[r][J + lane] = h[r];
          x[r][J + lane] = h[r];
        }

    } else {
      // near coefficients U(J - kv + m, J + c), m in [mn, kv): thread q -> (row, column)
      if (tail) {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int q = tid - 32 + k * (kSweepThreads - 32);
          if (q < kLUBlock * kLUBlock) {
            const int rr = q >> 5, c = q & 31;
            const int64_t m = b.kv - kLUBlock + rr;
            un[k] = (m >= mn && m >= c && c < jb) ? b.ab[u_run_first(b, J, c) + m] : 0.0;
          }
        }
      }
      if (more) {
        ph.load([&](int q) { return u_head_elem(b, J - kLUBlock, kLUBlock, q); },
                [&](int c) { return u_head_rd(b, J - kLUBlock, kLUBlock, c); });
        px.load(x, nlo, lo);
      }
    }
    if (warp != 0 && tail) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int q = tid - 32 + k * (kSweepThreads - 32);
        if (q < kLUBlock * kLUBlock) s_un[q >> 5][q & 31] = un[k];
      }
    }
    CK_PROF(8);
    __syncthreads();
    CK_PROF(9);
    if (tail) clu_push_ring_head<R>(C, ring, J, jb, (int)(blk & 1));
    clu_sync();  // head values pushed; the far sums of block J+32 are in their slot
    if (pend_J >= 0) {  // far rows of block J+32: rows pend_J - kv + m, m in [pend_m0, pend_m1)
      const double* ts = C.tsum + (int64_t)(((pend_J / kLUBlock) & 1) * R) * C.ts;
      for (int64_t m = pend_m0 + tid; m < pend_m1; m += nt)
#pragma unroll
        for (int r = 0; r < R; ++r)
          ring[r][pend_J - b.kv + m] = __dsub_rn(ring[r][pend_J - b.kv + m], ts[r * C.ts + m]);
      __syncthreads();
    }
    if (tail && tid < b.kv - mn) {  // near rows, one thread each, columns in order
      const int rr = (int)(mn - (b.kv - kLUBlock)) + tid;
      const int64_t i = J - kLUBlock + rr;
      double sm[R];
#pragma unroll
      for (int r = 0; r < R; ++r) sm[r] = 0.0;
      for (int c = 0; c < jb; ++c) {
        const double u = s_un[rr][c];
#pragma unroll
        for (int r = 0; r < R; ++r) sm[r] = __fma_rn(u, ring[r][J + c], sm[r]);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) ring[r][i] = __dsub_rn(ring[r][i], sm[r]);
    }
    pend_J = tail ? J : -1;
    pend_m0 = m0;
    pend_m1 = b.kv - kLUBlock;
    if (more) {
      ph.commit(H, true);
      px.commit(ring, nlo, lo);
      lo = nlo;
    }
    CK_PROF(12);
    __syncthreads();
    CK_PROF(13);
  }
}

// ---------------------------------------------------------- U^T forward
// x := U^{-T} x (forward): w_k = (x_k - sum_{i<k} U(i,k) w_i) / U(k,k).
// Phase 1: warp c forms head row c's dot over the final rows below J (from
// the stage). Phase 2: warp 0 solves the head triangle while the stage and
// the idle warps fetch the next block.
template <int R>
__device__ void sweep_ut_forward(const BandView& b, double* const* x, Ring* ring, double* s_dot,
                                 Head& H, Stage& S) {
  const int64_t n = b.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (n == 0) return;
  HeadPrefetch ph;
  RowPrefetch<R> px;
  // block 0: head and rows straight in
  H.v[tid >> 5][tid & 31] = u_head_elem(b, 0, (int)lmin(kLUBlock, n), tid);
  if (tid < kLUBlock) H.rd[tid] = u_head_rd(b, 0, (int)lmin(kLUBlock, n), tid);
  if (tid < lmin(kLUBlock, n))
#pragma unroll
    for (int r = 0; r < R; ++r) ring[r][tid] = x[r][tid];
  __syncthreads();
  CK_PROF_INIT;
  for (int64_t J = 0; J < n; J += kLUBlock) {
    const int jb = (int)lmin(kLUBlock, n - J);
    const int64_t J1 = J + kLUBlock;
    const bool dots = J > 0;
    if (dots) {
      S.wait();
      if (warp < jb) {
        const int c = warp;
        // rows i = J - kv + m of column J+c: in the band for m >= c, i >= 0
        const int64_t f = u_run_first(b, J, c);
        warp_dot<R>(J - b.kv, lmax(c, b.kv - J), b.kv, ring, s_dot, c, [&](int64_t m) {
          return m < S.srows ? S.at(c, (int)(f & 1), m) : b.ab[f + m];
        });
      }
    }
    CK_PROF(16);
    __syncthreads();
    CK_PROF(17);
    if (warp == 0) {
      double h[R];
#pragma unroll
      for (int r = 0; r < R; ++r)
        h[r] = lane < jb ? (dots ? __dsub_rn(ring[r][J + lane], s_dot[r * kLUBlock + lane])
                                 : ring[r][J + lane])
                         : 0.0;
#pragma unroll
      for (int c = 0; c < kLUBlock; ++c) {
        const double d = H.v[c][c], rd = H.rd[c];
        // U(J+c, J+lane) for lane > c: column J+lane, row J+c
        const double u = lane > c ? H.v[lane][c] : 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double w = div_rcp(__shfl_sync(0xffffffffu, h[r], c), d, rd);
          const double t = __dsub_rn(h[r], __dmul_rn(u, w));
          h[r] = lane == c ? w : t;
        }
      }
      if (lane < jb)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          ring[r][J + lane] = h[r];
          x[r][J + lane] = h[r];
        }
    } else if (J1 < n) {
      const int jb1 = (int)lmin(kLUBlock, n - J1);
      if (tid == kIssuer) S.issue(b.ab, jb1, [&](int c) { return u_run_first(b, J1, c); });
      ph.load([&](int q) { return u_head_elem(b, J1, jb1, q); },
              [&](int c) { return u_head_rd(b, J1, jb1, c); });
      px.load(x, J1, J1 + jb1);
    }
    CK_PROF(20);
    __syncthreads();
    CK_PROF(21);
    if (J1 < n) {
      ph.commit(H, true);
      px.commit(ring, J1, lmin(n, J1 + kLUBlock));
    }
  }
  __syncthreads();
}

// U^T forward on a cluster: one cluster barrier per block. The dots of block J
// over rows below J - 32 ("far") are the helpers', computed one block ahead
// (those rows are final once head J - 64 is done) into a slot by block parity;
// the rows of the previous head block ("near", J - 32 .. J - 1) the leader
// folds in itself, with coefficients loaded during that head.
template <int R>
__device__ void sweep_ut_forward_clu(const BandView& b, double* const* x, Ring* ring, double* s_dot,
                                     Head& H, const Clu& C) {
  __shared__ double s_un[kLUBlock][kLUBlock + 1];  // U(J - 32 + k, J + c) for the next block
  const int64_t n = b.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (n == 0) return;
  HeadPrefetch ph;
  RowPrefetch<R> px;
  H.v[tid >> 5][tid & 31] = u_head_elem(b, 0, (int)lmin(kLUBlock, n), tid);
  if (tid < kLUBlock) H.rd[tid] = u_head_rd(b, 0, (int)lmin(kLUBlock, n), tid);
  if (tid < lmin(kLUBlock, n))
#pragma unroll
    for (int r = 0; r < R; ++r) ring[r][tid] = x[r][tid];
  __syncthreads();
  CK_PROF_INIT;
  for (int64_t J = 0; J < n; J += kLUBlock) {
    const int jb = (int)lmin(kLUBlock, n - J);
    const int64_t J1 = J + kLUBlock;
    const bool dots = J > 0;
    if (dots && tid < R * kLUBlock) {  // thread (r, c): far partials, then the near rows
      const int r = tid >> 5, c = tid & 31;
      double t = 0.0;
      if (J > kLUBlock) {
        const double* dp = C.dpart + (int64_t)((J / kLUBlock) & 1) * C.size * R * kLUBlock;
        for (int k = 1; k < C.size; ++k) t = __dadd_rn(t, dp[((int64_t)k * R + r) * kLUBlock + c]);
      }
      double sn = 0.0;
      for (int k = 0; k < kLUBlock; ++k) sn = __fma_rn(s_un[k][c], ring[r][J - kLUBlock + k], sn);
      s_dot[tid] = __dadd_rn(t, sn);
    }
    CK_PROF(16);
    __syncthreads();
    CK_PROF(17);
    if (warp == 0) {
      double h[R];
#pragma unroll
      for (int r = 0; r < R; ++r)
        h[r] = lane < jb ? (dots ? __dsub_rn(ring[r][J + lane], s_dot[r * kLUBlock + lane])
                                 : ring[r][J + lane])
                         : 0.0;
#pragma unroll
      for (int c = 0; c < kLUBlock; ++c) {
        const double d = H.v[c][c], rd = H.rd[c];
        const double u = lane > c ? H.v[lane][c] : 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double w = div_rcp(__shfl_sync(0xffffffffu, h[r], c), d, rd);
          const double t = __dsub_rn(h[r], __dmul_rn(u, w));
          h[r] = lane == c ? w : t;
        }
      }
      if (lane < jb)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          ring[r][J + lane] = h[r];
          x[r][J + lane] = h[r];
        }
    } else if (J1 < n) {
      const int jb1 = (int)lmin(kLUBlock, n - J1);
      ph.load([&](int q) { return u_head_elem(b, J1, jb1, q); },
              [&](int c) { return u_head_rd(b, J1, jb1, c); });
      px.load(x, J1, J1 + jb1);
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {  // near coefficients of block J1: rows J + k
        const int q = tid - 32 + kk * (kSweepThreads - 32);
        if (q < kLUBlock * kLUBlock) {
          const int k = q >> 5, c = q & 31;
          const bool in = c < jb1 && c + kLUBlock - k <= b.kv;
          s_un[k][c] = in ? b.ab[u_run_first(b, J1, c) + (b.kv - kLUBlock + k)] : 0.0;
        }
      }
    }
    CK_PROF(20);
    __syncthreads();
    CK_PROF(21);
    clu_sync();  // block J final: the helpers go on with the far dots of block J + 64
    if (J1 < n) {
      ph.commit(H, true);
      px.commit(ring, J1, lmin(n, J1 + kLUBlock));
    }
  }
  __syncthreads();
}

// --------------------------------------------------------- L^T backward
// x := (L-part)^{-T} x: LAPACK gbtrs 'T' second half, blocks in reverse.
// Phase 1: warp c forms head column c's dot over the block's tail (from the
// stage) and the rows the previous block finalised go out. Phase 2: warp 0
// solves the head and applies the block's inverse interchange while the
// stage and the idle warps fetch the next block.
template <int R, bool CLU = false>
__device__ void sweep_l_backward(const BandView& b, double* const* x, Ring* ring, double* s_dot,
                                 Head& H, Stage& S, const Clu& C) {
  const int64_t n = b.n;
  const int tid = threadIdx.x, nt = kSweepThreads, lane = tid & 31, warp = tid >> 5;
  const int64_t nblk = (n + kLUBlock - 1) / kLUBlock;
  if (nblk == 0) return;
  Perm pq;
  HeadPrefetch ph;
  RowPrefetch<R> px;
  {
    const int64_t J = (nblk - 1) * kLUBlock;
    H.v[tid >> 5][tid & 31] = l_head_elem(b, nblk - 1, tid);
    if (J + tid < n)
#pragma unroll
      for (int r = 0; r < R; ++r) ring[r][J + tid] = x[r][J + tid];
    if (warp == 0) pq = load_perm(b, nblk - 1, lane);
  }
  __syncthreads();
  CK_PROF_INIT;
  for (int64_t blk = nblk - 1; blk >= 0; --blk) {
    const int64_t J = blk * kLUBlock;
    const int jb = (int)lmin(kLUBlock, n - J);
    const int64_t wend = lmin(n, J + kLUBlock + b.kl);
    const bool dots = wend > J + jb;
    if (blk + 1 < nblk) {  // rows block blk+1 finalised: [J1 + kl, wend1)
      const int64_t J1 = J + kLUBlock;
      for (int64_t i = J1 + b.kl + tid; i < lmin(n, J1 + kLUBlock + b.kl); i += nt)
#pragma unroll
        for (int r = 0; r < R; ++r) x[r][i] = ring[r][i];
    }
    const int64_t M = wend - J - kLUBlock;
    const int64_t mh = CLU ? 0 : M;  // the leader's own dot rows (none with helpers)
    if (dots) {
      S.wait();
      if (warp < jb) {
        const int c = warp;
        const double* col = b.lb + l_run_first(b, blk, c);
        const int off = (int)((c * b.lb_ld) & 1);
        warp_dot<R>(J + kLUBlock, 0, mh, ring, CLU ? C.dpart : s_dot, c,
                    [&](int64_t m) { return m < S.srows ? S.at(c, off, m) : col[m]; });
      }
    }
    CK_PROF(24);
    if (CLU) {
      clu_sync();  // every rank's partials in dpart
      if (dots && tid < R * kLUBlock) {
        double t = 0.0;
        for (int k = 0; k < C.size; ++k) t = __dadd_rn(t, C.dpart[(int64_t)k * R * kLUBlock + tid]);
        s_dot[tid] = t;
      }
    }
    __syncthreads();
    CK_PROF(25);
    if (warp == 0) {
      double h[R];
#pragma unroll
      for (int r = 0; r < R; ++r)
        h[r] = lane < jb ? (dots ? __dsub_rn(ring[r][J + lane], s_dot[r * kLUBlock + lane])
                                 : ring[r][J + lane])
                         : 0.0;
#pragma unroll
      for (int c = kLUBlock - 1; c >= 0; --c) {
        // u_c is final; push -l(c, lane) u_c into the columns lane < c
        const double l = lane < c ? H.v[lane][c] : 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) h[r] = __dsub_rn(h[r], __dmul_rn(l, __shfl_sync(0xffffffffu, h[r], c)));
      }
      if (lane < jb)
#pragma unroll
        for (int r = 0; r < R; ++r) ring[r][J + lane] = h[r];
      __syncwarp();
      apply_perm<R, true>(pq, ring, J, lane);
      if (blk > 0) pq = load_perm(b, blk - 1, lane);
    } else if (blk > 0) {
      const int64_t Jp = J - kLUBlock;
      if (tid == kIssuer && lmin(n, Jp + kLUBlock + b.kl) > J)
        S.issue(b.lb, kLUBlock, [&](int c) { return l_run_first(b, blk - 1, c); });
      ph.load([&](int q) { return l_head_elem(b, blk - 1, q); });
      px.load(x, Jp, J);
    }
    CK_PROF(28);
    __syncthreads();
    CK_PROF(29);
    if (CLU) clu_sync();  // the block's rows are final for the helpers
    if (blk > 0) {
      ph.commit(H);
      px.commit(ring, J - kLUBlock, J);
    }
  }
  // rows no step can touch any more: everything below kl + 32
  for (int64_t i = tid; i < lmin(n, kLUBlock + b.kl); i += nt)
#pragma unroll
    for (int r = 0; r < R; ++r) x[r][i] = ring[r][i];
  __syncthreads();
}

// x := A^{-1} x (transpose = false) or A^{-T} x, for R right-hand sides, by the
// calling CTA of kSweepThreads threads (CLU: the cluster's leader, see Clu).
template <int R, bool CLU = false>
__device__ __forceinline__ void inv_solve(const BandView& b, double* const* x, double* smem,
                                          int ring_size, bool transpose, const Clu& C = Clu{1, 0, nullptr, 0, nullptr, nullptr}) {
  __shared__ Head H;
  __shared__ alignas(8) uint64_t mbar;
  Ring ring[R];
#pragma unroll
  for (int r = 0; r < R; ++r) ring[r] = Ring{smem + (int64_t)r * ring_size, ring_size - 1};
  double* s_dot = smem + (int64_t)R * ring_size;
  if (threadIdx.x == 0) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(&mbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  Stage S;
  S.st = smem + stage_offset(R, ring_size);
  S.bar = &mbar;
  // the leader works on no tail / dot rows itself in cluster mode: no stage
  const int64_t kl = CLU ? 0 : b.kl;
  const int64_t kv = CLU ? 0 : b.kv;
  if (!transpose) {
    S.layout(b.stage_cap, kl, b.stage_min);
    sweep_l_forward<R, CLU>(b, x, ring, H, S, C);
    if (CLU) {
      sweep_u_backward_clu<R>(b, x, ring, H, C);
    } else {
      S.layout(b.stage_cap, kv, b.stage_min);
      sweep_u_backward<R>(b, x, ring, H, S);
    }
  } else {
    if (CLU) {
      sweep_ut_forward_clu<R>(b, x, ring, s_dot, H, C);
    } else {
      S.layout(b.stage_cap, kv, b.stage_min);
      sweep_ut_forward<R>(b, x, ring, s_dot, H, S);
    }
    S.layout(b.stage_cap, kl, b.stage_min);
    sweep_l_backward<R, CLU>(b, x, ring, s_dot, H, S, C);
  }
}

// The helper side of inv_solve (cluster rank > 0): the same block sequence and
// cluster barriers as the leader's four sweeps; `local` is this CTA's dynamic
// shared memory (head copy, then copied ring rows).
template <int R>
__device__ void helper_solve(const BandView& b, double* local, int ring_size, bool transpose, const Clu& C) {
  const int64_t n = b.n;
  const int64_t nblk = (n + kLUBlock - 1) / kLUBlock;
  const Clu& c = C;
  Ring lring[R];  // the leader's rings (DSMEM)
#pragma unroll
  for (int r = 0; r < R; ++r) lring[r] = Ring{clu_leader(local + (int64_t)r * ring_size), ring_size - 1};
  const int64_t shmax = (lmax(b.kl, b.kv) + c.size - 2) / (c.size - 1) + 2;
  double* hy = local;                            // [2][R][32] head values (block parity)
  double* hl = hy + (int64_t)2 * R * kLUBlock;   // [R][share] ring rows of a dot share
  double* cf = hl + (int64_t)R * shmax;         // [32][share] coefficients of a share
  auto share = [&](int64_t m0, int64_t m1, int64_t& lo, int64_t& hi) {  // helpers only
    lo = clu_cut(m0, m1, c.rank - 1, c.size - 1);
    hi = clu_cut(m0, m1, c.rank, c.size - 1);
  };
  if (n == 0) return;
  if (!transpose) {
    for (int64_t J = 0; J < n; J += kLUBlock) {  // L forward
      const int64_t blk = J / kLUBlock;
      const int jb = (int)lmin(kLUBlock, n - J);
      const int64_t wend = lmin(n, J + kLUBlock + b.kl);
      const bool tail = wend > J + jb;
      int64_t lo = 0, hi = 0;
      if (tail) {
        share(0, wend - J - kLUBlock, lo, hi);
        const double* lbk = b.lb + blk * kLUBlock * b.lb_ld;
        helper_fetch(lo, hi, jb, cf, [&](int64_t m, int cc) { return lbk[cc * b.lb_ld + kLUBlock + m]; });
      }
      clu_sync();  // head values pushed by the leader, cf complete
      if (tail) helper_tail<R>(lo, hi, jb, hy, cf, c);
      clu_sync();
    }
    // U backward (sweep_u_backward_clu): one barrier per block; far rows of
    // block J (above J - 32) while the leader solves the next head. Coefficient
    // shares double-buffered, copied asynchronously one block ahead (U runs are
    // masked above the band, m < c, at use).
    auto u_share = [&](int64_t blk, int64_t& lo, int64_t& hi) {
      const int64_t J = blk * kLUBlock;
      const int64_t wbeg = lmax(0, J - b.kv);
      if (!(J > wbeg)) return false;
      share(wbeg - (J - b.kv), lmax(wbeg - (J - b.kv), b.kv - kLUBlock), lo, hi);
      return true;
    };
    double* cfs[2] = {cf, cf + (int64_t)kLUBlock * shmax};
    auto u_fetch = [&](int64_t blk) {
      int64_t lo, hi;
      if (blk < 0 || !u_share(blk, lo, hi)) {
        cp_async_commit();
        return;
      }
      const int64_t J = blk * kLUBlock;
      helper_fetch_async(lo, hi, (int)lmin(kLUBlock, n - J), cfs[blk & 1], b.ab,
                         [&](int cc) { return u_run_first(b, J, cc) + lo; });
    };
    u_fetch(nblk - 1);
    for (int64_t blk = nblk - 1; blk >= 0; --blk) {
      const int64_t J = blk * kLUBlock;
      const int jb = (int)lmin(kLUBlock, n - J);
      clu_sync();  // head values of block J pushed
      cp_async_wait<0>();
      __syncthreads();  // the share of block J is in
      u_fetch(blk - 1);  // the next block's share streams in meanwhile
      int64_t lo, hi;
      if (u_share(blk, lo, hi)) {
        Clu cs = c;
        cs.tsum = c.tsum + (int64_t)((blk & 1) * R) * c.ts;
        helper_tail<R>(lo, hi, jb, hy + (blk & 1) * R * kLUBlock, cfs[blk & 1], cs, true);
      }
    }
    cp_async_wait<0>();
    __syncthreads();
  } else {
    // U^T forward (sweep_ut_forward_clu): after barrier B(J) the rows below
    // J + 32 are final; the far dots of block J + 64 (rows below J + 32) go
    // into the partial slot of that block's parity. The coefficient shares are
    // double-buffered and copied asynchronously one block ahead.
    auto ut_share = [&](int64_t Jd, int64_t& lo, int64_t& hi) {
      share(lmax(0, b.kv - Jd), lmax(lmax(0, b.kv - Jd), b.kv - kLUBlock), lo, hi);
    };
    double* cfs[2] = {cf, cf + (int64_t)kLUBlock * shmax};
    auto ut_fetch = [&](int64_t Jd) {
      if (Jd >= n) {
        cp_async_commit();
        return;
      }
      int64_t lo, hi;
      ut_share(Jd, lo, hi);
      helper_fetch_async(lo, hi, (int)lmin(kLUBlock, n - Jd), cfs[(Jd / kLUBlock) & 1], b.ab,
                         [&](int cc) { return u_run_first(b, Jd, cc) + lo; });
    };
    ut_fetch(2 * kLUBlock);
    for (int64_t J = 0; J < n; J += kLUBlock) {
      clu_sync();  // B(J)
      const int64_t Jd = J + 2 * kLUBlock;
      if (Jd < n) {
        int64_t lo, hi;
        ut_share(Jd, lo, hi);
        cp_async_wait<0>();
        __syncthreads();  // the share of block Jd is in
        ut_fetch(Jd + kLUBlock);  // next block's share streams in meanwhile
        Clu cs = c;
        cs.dpart = c.dpart + (int64_t)((Jd / kLUBlock) & 1) * c.size * R * kLUBlock;
        helper_dots<R>(lring, Jd - b.kv, lo, hi, (int)lmin(kLUBlock, n - Jd), 0, hl,
                       cfs[(Jd / kLUBlock) & 1], cs);
      }
    }
    cp_async_wait<0>();
    __syncthreads();
    auto lt_dots = [&](int64_t blk, int64_t& lo, int64_t& hi) {
      const int64_t J = blk * kLUBlock;
      const int jb = (int)lmin(kLUBlock, n - J);
      const int64_t wend = lmin(n, J + kLUBlock + b.kl);
      if (!(wend > J + jb)) return false;
      share(0, wend - J - kLUBlock, lo, hi);
      return true;
    };
    auto lt_fetch = [&](int64_t blk) {
      int64_t lo, hi;
      if (blk < 0 || !lt_dots(blk, lo, hi)) return;
      helper_fetch(lo, hi, (int)lmin(kLUBlock, n - blk * kLUBlock), cf,
                   [&](int64_t m, int cc) { return b.lb[l_run_first(b, blk, cc) + m]; });
    };
    lt_fetch(nblk - 1);
    for (int64_t blk = nblk - 1; blk >= 0; --blk) {  // L^T backward
      const int64_t J = blk * kLUBlock;
      const int jb = (int)lmin(kLUBlock, n - J);
      int64_t lo, hi;
      if (lt_dots(blk, lo, hi)) {
        __syncthreads();  // cf complete
        helper_dots<R>(lring, J + kLUBlock, lo, hi, jb, -1, hl, cf, c);
      }
      clu_sync();
      lt_fetch(blk - 1);
      clu_sync();
    }
  }
}

}  // namespace ck
