// Device-side building blocks: deterministic fp64 reductions and the
// sliced-ELL row kernel shared by every operator application.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "ck_common.h"

// Device-side index checks of the checked build (-DCK_CHECKED, scripts/
// checked_build.sh): compute-sanitizer is not available on every pool, so the
// kernels carry their own bounds assertions, compiled out of the product build.
#ifdef CK_CHECKED
#include <cstdio>
#define CK_DASSERT(c)                                                     \
  do {                                                                    \
    if (!(c)) {                                                           \
      printf("CK_DASSERT failed: %s (%s:%d)\n", #c, __FILE__, __LINE__);   \
      __trap();                                                           \
    }                                                                     \
  } while (0)
#else
#define CK_DASSERT(c) ((void)0)
#endif

namespace ck {

__host__ __device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t lmax(int64_t a, int64_t b) { return a > b ? a : b; }

// ---------------------------------------------------------------------------
// Overflow-safe sum of squares in one pass (the two-pass amax/scale scheme of
// two_norm, sparse.hpp:175-186, folded into a running power-of-two scale):
// value^2 = s * 2^(2e), every partial term is (x * 2^-e)^2 < 1, and scales are
// exact powers of two, so no overflow or spurious underflow for finite input.
// flags: bit0 = saw +-inf, bit1 = saw NaN (two_norm returns inf / NaN then).
struct ES {
  double s;
  int e;
  int flags;
};

__device__ __forceinline__ ES es_zero() { return {0.0, -100000, 0}; }

__device__ __forceinline__ void es_add(ES& a, double x) {
  double ax = fabs(x);
  if (!(ax <= 1.7976931348623157e308)) {
    a.flags |= (ax != ax) ? 2 : 1;
    return;
  }
  if (ax == 0.0) return;
  int ex = ilogb(ax) + 1;  // ax < 2^ex
  if (ex > a.e) {
    a.s = scalbn(a.s, 2 * (a.e - ex));
    a.e = ex;
  }
  double q = scalbn(ax, -a.e);
  a.s = __dadd_rn(a.s, __dmul_rn(q, q));
}

__device__ __forceinline__ void es_merge(ES& a, const ES& b) {
  a.flags |= b.flags;
  if (b.s == 0.0) return;
  if (a.s == 0.0) {
    a.s = b.s;
    a.e = b.e;
    return;
  }
  if (b.e > a.e) {
    a.s = __dadd_rn(scalbn(a.s, 2 * (a.e - b.e)), b.s);
    a.e = b.e;
  } else {
    a.s = __dadd_rn(a.s, scalbn(b.s, 2 * (b.e - a.e)));
  }
}

__device__ __forceinline__ double es_norm(const ES& a) {
  if (a.flags & 1) return __longlong_as_double(0x7ff0000000000000LL);
  if (a.flags & 2) return __longlong_as_double(0x7ff8000000000000LL);
  if (a.s == 0.0) return 0.0;
  return scalbn(sqrt(a.s), a.e);
}

// ---------------------------------------------------------------------------
// Double-double accumulator (error-free TwoSum/TwoProd). Used where the
// reference uses Neumaier compensation (compensated_norm, condest.hpp:158-171).
struct DD {
  double hi, lo;
};

__device__ __forceinline__ DD dd_zero() { return {0.0, 0.0}; }

__device__ __forceinline__ void dd_add2(DD& a, double bh, double bl) {
  double s = __dadd_rn(a.hi, bh);
  double bb = __dsub_rn(s, a.hi);
  double err = __dadd_rn(__dsub_rn(a.hi, __dsub_rn(s, bb)), __dsub_rn(bh, bb));
  err = __dadd_rn(err, __dadd_rn(a.lo, bl));
  a.hi = __dadd_rn(s, err);
  a.lo = __dsub_rn(err, __dsub_rn(a.hi, s));
}

__device__ __forceinline__ void dd_add_sq(DD& a, double x) {
  double p = __dmul_rn(x, x);
  double pe = __fma_rn(x, x, -p);
  dd_add2(a, p, pe);
}

__device__ __forceinline__ void dd_merge(DD& a, const DD& b) { dd_add2(a, b.hi, b.lo); }

// ---------------------------------------------------------------------------
// Warp / block reductions with a fixed tree (bitwise reproducible).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ ES warp_es(ES a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ES b;
    b.s = __shfl_down_sync(0xffffffffu, a.s, o);
    b.e = __shfl_down_sync(0xffffffffu, a.e, o);
    b.flags = __shfl_down_sync(0xffffffffu, a.flags, o);
    es_merge(a, b);
  }
  return a;
}

__device__ __forceinline__ DD warp_dd(DD a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    DD b;
    b.hi = __shfl_down_sync(0xffffffffu, a.hi, o);
    b.lo = __shfl_down_sync(0xffffffffu, a.lo, o);
    dd_merge(a, b);
  }
  return a;
}

// Block-wide reductions for a 256-thread block. Result valid in thread 0.
// `scratch` must hold >= 8 entries of the reduced type; the call begins with a
// barrier so scratch can be reused back to back.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < (int)(blockDim.x >> 5) ? scratch[lane] : 0.0;
    v = warp_sum(v);
  }
  return v;
}

__device__ __forceinline__ ES block_es(ES a, double* ss, int* se, int* sf) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  a = warp_es(a);
  __syncthreads();
  if (lane == 0) {
    ss[w] = a.s;
    se[w] = a.e;
    sf[w] = a.flags;
  }
  __syncthreads();
  if (w == 0) {
    a = lane < (int)(blockDim.x >> 5) ? ES{ss[lane], se[lane], sf[lane]} : es_zero();
    a = warp_es(a);
  }
  return a;
}

__device__ __forceinline__ DD block_dd(DD a, double* sh, double* sl) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  a = warp_dd(a);
  __syncthreads();
  if (lane == 0) {
    sh[w] = a.hi;
    sl[w] = a.lo;
  }
  __syncthreads();
  if (w == 0) {
    a = lane < (int)(blockDim.x >> 5) ? DD{sh[lane], sl[lane]} : dd_zero();
    a = warp_dd(a);
  }
  return a;
}

// "Last block" election: every block publishes its partials, fences, and bumps
// a counter; the block that arrives last owns the final reduction. The counter
// is re-armed by that block, so the same kernel can be relaunched (graphs).
__device__ __forceinline__ bool elect_last_block(unsigned int* counter, unsigned int nblocks) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int prev = atomicAdd(counter, 1u);
    s_last = (prev == nblocks - 1);
    if (s_last) *counter = 0u;
  }
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}

// Streaming loads of matrix data (read once per sweep): evict-first so the
// gathered vectors keep their L2 residency.
__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ int ld_stream(const int* p) { return __ldcs(p); }
__device__ __forceinline__ int ld_stream(const uint16_t* p) {
  return (int)__ldcs(reinterpret_cast<const unsigned short*>(p));
}

// Base column of slice s (narrow format; 0 for wide).
template <bool NW>
__device__ __forceinline__ int slice_cbase(const SellView& A, int64_t s) {
  return NW ? A.cbase[s] : 0;
}

// Column of stored entry k of slice s, either format (setup kernels; the
// sweeps use the compile-time form in load_chunk).
__device__ __forceinline__ int sell_col(const SellView& A, int64_t s, int64_t k) {
  if (!A.narrow) return A.col[k];
  return A.cbase[s] + (int)A.col16[A.poff ? A.poff[s] + (k - A.sp[s]) : k];
}

// First column-array element of a row: its row base, or its place in the
// slice's dictionary pattern (narrow + pattern format).
__device__ __forceinline__ int64_t sell_colbase(const SellView& A, int64_t slice, int64_t row, int64_t rowbase) {
  return A.poff ? A.poff[slice] + 2 * (row & 31) : rowbase;
}

// Loads U consecutive stored entries (stored positions j0..j0+U-1, j0 and U
// even) of a sliced-ELL row with row base `base` (sell_rowbase): U/2 16-byte
// value loads and U/2 column-pair loads, all issued before any use. Positions
// at or beyond the warp-uniform (even) slice width w are predicated off and
// read as (column cb, value 0). Padding inside [len, w) is stored as (cb, 0.0),
// so the gathers that follow never need a bounds check. NW selects the narrow
// column format (cb = the slice's base column; 0 for wide).
// cbase0: the row's first element in the column array (sell_colbase; == base
// unless the operator uses a pattern dictionary, whose table is re-read by
// every slice with that pattern and so is loaded through the cached path).
template <int U, bool NW>
__device__ __forceinline__ void load_chunk(const SellView& A, int64_t base, int64_t cbase0, int cb, int j0,
                                           int w, int* c, double* v) {
  static_assert(U % 2 == 0, "chunks cover whole entry pairs");
#pragma unroll
  for (int m = 0; m < U / 2; ++m) {
    const int j = j0 + 2 * m;
    const bool ok = j < w;
    const int64_t k = sell_at(base, j);
    double2 vv = make_double2(0.0, 0.0);
    if (ok) vv = __ldcs(reinterpret_cast<const double2*>(A.val + k));
    v[2 * m] = vv.x;
    v[2 * m + 1] = vv.y;
    if (NW) {
      ushort2 cc = make_ushort2(0, 0);
      const ushort2* cp = reinterpret_cast<const ushort2*>(A.col16 + sell_at(cbase0, j));
      if (ok) cc = __ldg(cp);  // one load flavour: a branch here would serialise the chunk's loads
      c[2 * m] = cb + (int)cc.x;
      c[2 * m + 1] = cb + (int)cc.y;
    } else {
      int2 cc = make_int2(0, 0);
      if (ok) cc = __ldcs(reinterpret_cast<const int2*>(A.col + k));
      c[2 * m] = cc.x;
      c[2 * m + 1] = cc.y;
    }
  }
}

// Asynchronous global -> shared copies (cp.async, 8 bytes), grouped per thread.
__device__ __forceinline__ void cp_async_elem(double* smem, const double* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace ck
