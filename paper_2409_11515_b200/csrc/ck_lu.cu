// Band LU with row partial pivoting on the device and the four triangular
// sweeps of the InverseOracle (lu.hpp:55-227, condest.hpp:109-152).
//
// Factorisation: right-looking, 32-column panels (LAPACK gbtrf layout). A panel
// CTA factors its 32 columns (pivot = first largest |candidate|, the
// singularity tests of lu.hpp:112-129 with pivot_tol * column max); then every
// trailing column touched by the panel's interchanges receives, in pivot
// order, the interchange and the update -l(r,j) * u(j,k) of each panel step
// (one warp per column, the panel's multipliers staged in shared memory). Each
// entry therefore sees the same updates in the same order as the reference's
// left-looking elimination, with unfused multiply/subtract -- the factors agree
// with lu_factorize value for value when the pivot sequence agrees.
//
// Solves: one CTA sweeps 32-row blocks with the active rows of the right-hand
// side(s) in a shared-memory ring. Inside a block the 32x32 triangle is solved
// by one warp (shuffles); everything outside it is a GEMV over contiguous band
// columns spread over all warps. The L part interleaves row interchanges with
// eliminations; each block uses multipliers re-expressed in the block's local
// pivot order (convert_l_blocks), which turns the interleaved sequence into
// "permute window, unit-lower solve, update tail" without changing any value.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "ck_common.h"
#include "ck_device.cuh"
#include "ck_internal.h"
#include "ck_lu.h"
#include "ck_lu_sweeps.cuh"

namespace ck {


// ----------------------------------------------------------- band fill
__global__ void k_band_bounds(SellView A, int64_t nrows_pad, const int32_t* __restrict__ rperm,
                              const int32_t* __restrict__ cperm, int* klku) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nrows_pad) return;
  const int32_t row = rperm[p];
  if (row < 0) return;
  const int64_t base = sell_rowbase(A.sp[p >> 5], p);
  const int L = A.len[p];
  int lo = 0, up = 0;
  for (int j = 0; j < L; ++j) {
    const int32_t col = cperm[sell_col(A, p >> 5, sell_at(base, j))];
    lo = max(lo, row - col);
    up = max(up, col - row);
  }
  atomicMax(klku, lo);
  atomicMax(klku + 1, up);
}

__device__ __forceinline__ int64_t band_pos(const BandView& b, int64_t i, int64_t j) {
  return (b.kv + i - j) + j * b.ldab;
}

// Values of A into the band, and A's structure into the bitmap (explicit zeros
// of A are entries too: lu.hpp:89-94 touches every stored row of the column).
__global__ void k_band_fill(SellView A, int64_t nrows_pad, const int32_t* __restrict__ rperm,
                            const int32_t* __restrict__ cperm, BandView b, uint32_t* abit) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nrows_pad) return;
  const int32_t row = rperm[p];
  if (row < 0) return;
  const int64_t base = sell_rowbase(A.sp[p >> 5], p);
  const int L = A.len[p];
  for (int j = 0; j < L; ++j) {
    const int64_t k = sell_at(base, j);
    const int64_t q = band_pos(b, row, cperm[sell_col(A, p >> 5, k)]);
    b.ab[q] = A.val[k];
    atomicOr(abit + (q >> 5), 1u << (q & 31));
  }
}

__global__ void k_iota(int32_t* v, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) v[i] = (int32_t)i;
}

// ----------------------------------------------------------- factorisation
// Touch keys (BandView::key): the order in which the reference's left-looking
// elimination first touches each row of a working column (lu.hpp:88-110) --
// the original entries in ascending row order, then the fill in the order the
// pivot columns reach it (step ascending, and inside a step the order of that
// column's stored multipliers). Ties of the pivot search go to the first
// touched row (`mag > best_mag`, lu.hpp:115-124), and a column with no touched
// unpivoted row is structurally singular (lu.hpp:126).
__device__ __forceinline__ uint32_t& KEY(const BandView& b, int64_t i, int64_t j) {
  return b.key[(b.kv + i - j) + (j % b.kw) * b.ldab];
}

// Column views: col[i] is entry (i, j) of the band / of the key window.
__device__ __forceinline__ double* ab_col(const BandView& b, int64_t j) {
  return b.ab + (j * b.ldab + b.kv - j);
}
__device__ __forceinline__ uint32_t* key_col(const BandView& b, int64_t j) {
  return b.key + ((j % b.kw) * b.ldab + b.kv - j);
}

// Order of a touched row in its column: originals by original row, then fill.
__device__ __forceinline__ uint64_t order_key(uint32_t k, int32_t orig_row) {
  return k == kKeyOriginal ? (uint64_t)(uint32_t)orig_row : (1ull << 32) + k;
}

// Key slots of columns [c0, c1) enter the window: an entry of A or untouched.
__device__ __forceinline__ void init_key_slots(const BandView& b, int64_t c0, int64_t c1,
                                               int64_t part, int64_t nparts) {
  c1 = lmin(c1, b.n);
  if (c0 >= c1) return;
  const int64_t total = (c1 - c0) * b.ldab;
  const int64_t stride = nparts * blockDim.x;
  for (int64_t q = part * blockDim.x + threadIdx.x; q < total; q += stride) {
    const int64_t c = c0 + q / b.ldab, r = q % b.ldab;
    const int64_t pos = r + c * b.ldab;
    const bool orig = (b.abit[pos >> 5] >> (pos & 31)) & 1u;
    b.key[r + (c % b.kw) * b.ldab] = orig ? kKeyOriginal : kKeyUntouched;
  }
}

// Key slots of the columns the first panel can reach, [0, kv + 32) of each member
// (its own kv: the window of a narrower member of a batch is shorter).
__global__ void k_key_init(const BandView* __restrict__ bs) {
  const BandView& b = bs[blockIdx.y];
  init_key_slots(b, 0, b.kv + kLUBlock, blockIdx.x, gridDim.x);
}

// Fill stamp of step s in column k for a multiplier of rank `rank` (< kl + 1).
__device__ __forceinline__ uint32_t fill_key(const BandView& b, int64_t s, int64_t k, uint32_t rank) {
  return 1u + (uint32_t)(s - (k - b.kv)) * (uint32_t)(b.kl + 1) + rank;
}

// Panel: columns j0 .. j0+jb-1 by one CTA per factorisation (blockIdx.y
// selects the member of a batch; members shorter than j0 are done). Per column
// step: pivot search over rows j0..j+km (the column maximum of the rows above
// j0 -- final since the previous panel -- is taken for all 32 columns up front),
// interchange, multipliers, their ranks (a bitonic sort of packed order keys),
// and the update of the panel's remaining columns with one thread per row. The
// critical path of a step touches global memory only for the band itself: the
// original-row ids of the panel's rows, pivot_min and ju live on chip.
// Dynamic shared memory: s_sort[next_pow2(kl + 1)] then s_orig[32 + kl].
constexpr int kPanelThreads = 512;
constexpr int kRankBits = 14;  // row offsets inside a column: kl <= kLUMaxBand < 2^14

struct Cand {
  double mag, val, cmax;
  uint64_t key;
  int64_t row;
};

__device__ __forceinline__ void cand_take(Cand& a, const Cand& o) {
  if (o.mag > a.mag || (o.mag == a.mag && o.key < a.key)) {
    a.mag = o.mag;
    a.val = o.val;
    a.key = o.key;
    a.row = o.row;
  }
  a.cmax = fmax(a.cmax, o.cmax);
}

__device__ __forceinline__ void warp_best(Cand& c) {
  for (int o = 16; o > 0; o >>= 1) {
    Cand x;
    x.mag = __shfl_xor_sync(0xffffffffu, c.mag, o);
    x.val = __shfl_xor_sync(0xffffffffu, c.val, o);
    x.cmax = __shfl_xor_sync(0xffffffffu, c.cmax, o);
    x.key = __shfl_xor_sync(0xffffffffu, c.key, o);
    x.row = __shfl_xor_sync(0xffffffffu, c.row, o);
    cand_take(c, x);
  }
}

// Compare-exchange stages jj = 16 .. 1 of bitonic merge size kk2 on the elements
// e = lane-aligned positions, one element per thread in registers.
__device__ __forceinline__ uint64_t bitonic_warp(uint64_t x, int e, int kk2, int jj_top) {
  for (int jj = jj_top; jj > 0; jj >>= 1) {
    const uint64_t y = __shfl_xor_sync(0xffffffffu, x, jj);
    const bool lower = (e & jj) == 0;
    const bool up = (e & kk2) == 0;
    // the lower element keeps the min when ascending
    const bool take_min = (lower == up);
    x = take_min ? (y < x ? y : x) : (y > x ? y : x);
  }
  return x;
}

// Sorts s[0, ns) ascending (ns a power of two, kPanelThreads threads).
__device__ __forceinline__ void bitonic_sort(uint64_t* s, int ns) {
  const int tid = threadIdx.x;
  // blocks of 32 elements in registers (whole warps: ns < 32 pads warp 0 with
  // maxima, which sort to the end)
  if (ns < 32) {
    if (tid < 32) {
      uint64_t x = tid < ns ? s[tid] : ~0ull;
      for (int kk2 = 2; kk2 <= 32; kk2 <<= 1) x = bitonic_warp(x, tid, kk2, kk2 >> 1);
      if (tid < ns) s[tid] = x;
    }
    __syncthreads();
    return;
  }
  for (int e = tid; e < ns; e += kPanelThreads) {
    uint64_t x = s[e];
    for (int kk2 = 2; kk2 <= 32; kk2 <<= 1) x = bitonic_warp(x, e, kk2, kk2 >> 1);
    s[e] = x;
  }
  __syncthreads();
  for (int kk2 = 64; kk2 <= ns; kk2 <<= 1) {
    for (int jj = kk2 >> 1; jj >= 32; jj >>= 1) {
      for (int t = tid; t < (ns >> 1); t += kPanelThreads) {
        const int i1 = 2 * t - (t & (jj - 1));
        const int i2 = i1 + jj;
        const uint64_t x = s[i1], y = s[i2];
        if ((x > y) == ((i1 & kk2) == 0)) {
          s[i1] = y;
          s[i2] = x;
        }
      }
      __syncthreads();
    }
    for (int e = tid; e < ns; e += kPanelThreads) s[e] = bitonic_warp(s[e], e, kk2, 16);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kPanelThreads) k_gbtrf_panel(const BandView* __restrict__ bs, int64_t j0,
                                                               double pivot_tol, LUStatus* const* sts,
                                                               int sort_words) {
  extern __shared__ uint64_t s_sort[];
  constexpr int kWarps = kPanelThreads / 32;
  __shared__ Cand s_c[kWarps];
  __shared__ double s_cmax_u[kLUBlock];   // column max over rows < j0 (final)
  __shared__ double s_u[kLUBlock];        // pivot row of the current step, panel columns
  __shared__ int64_t s_kofs[kLUBlock];    // key_col offsets of the panel columns
  __shared__ int32_t s_ipiv[kLUBlock], s_rowperm[kLUBlock];
  __shared__ int s_wcnt[kWarps];
  __shared__ int64_t s_p;
  __shared__ double s_piv;
  const BandView b = bs[blockIdx.y];
  LUStatus* st = sts[blockIdx.y];
  if (j0 >= b.n) return;
  const int jb = (int)lmin(kLUBlock, b.n - j0);
  if (st->code != 0) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int32_t* s_orig = reinterpret_cast<int32_t*>(s_sort + sort_words);  // rows j0 ..
  const int nrow = (int)lmin(kLUBlock + b.kl, b.n - j0);
  CK_PROF_INIT;
  for (int r = tid; r < nrow; r += kPanelThreads) s_orig[r] = b.orig[j0 + r];
  if (tid < kLUBlock) s_ipiv[tid] = s_rowperm[tid] = -1;
  // column maxima of the rows above the panel, and the key-window offsets
  for (int c = warp; c < jb; c += kWarps) {
    const int64_t j = j0 + c;
    const double* aj = ab_col(b, j);
    double m = 0.0;
    for (int64_t i = lmax(0, j - b.kv) + lane; i < j0; i += 32) m = fmax(m, fabs(aj[i]));
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) {
      s_cmax_u[c] = m;
      s_kofs[c] = (j % b.kw) * b.ldab + b.kv - j;
    }
  }
  // running maximum over every step so far (dgbtf2's ju): rows of this panel may
  // carry fill from earlier panels out to the previous maximum
  int64_t ju = st->ju;
  double pivot_min = st->pivot_min;
  __syncthreads();
  for (int c = 0; c < jb; ++c) {
    const int64_t j = j0 + c;
    const int km = (int)lmin(b.kl, b.n - 1 - j);
    double* aj = ab_col(b, j);
    uint32_t* kj = b.key + s_kofs[c];
    // pivot search over the touched rows j..j+km: largest magnitude, first in
    // touched order on ties (lu.hpp:112-125; untouched rows hold 0)
    Cand cd{-1.0, 0.0, 0.0, ~0ull, -1};
    for (int64_t i = j0 + tid; i <= j + km; i += kPanelThreads) {
      const double v = aj[i];
      const double m = fabs(v);
      cd.cmax = fmax(cd.cmax, m);
      if (i >= j) {
        const uint32_t k = kj[i];
        if (k != kKeyUntouched) {
          const uint64_t o = order_key(k, s_orig[i - j0]);
          if (m > cd.mag || (m == cd.mag && o < cd.key)) {
            cd.mag = m;
            cd.val = v;
            cd.row = i;
            cd.key = o;
          }
        }
      }
    }
    warp_best(cd);
    if (lane == 0) s_c[warp] = cd;
    __syncthreads();
    CK_PROF(2);
    if (warp == 0) {
      cd = lane < kWarps ? s_c[lane] : Cand{-1.0, 0.0, 0.0, ~0ull, -1};
      warp_best(cd);
      if (lane == 0) {
        const double cmax = fmax(cd.cmax, s_cmax_u[c]);
        const int64_t p = cd.row;
        if (p < 0) {  // no touched unpivoted row (lu.hpp:126)
          st->code = CK_ERR_STRUCT_SINGULAR;
          st->column = j;
          st->pivot = 0.0;
          s_p = -1;
        } else if (cd.mag == 0.0 || cd.mag < pivot_tol * cmax) {  // lu.hpp:127-129
          st->code = CK_ERR_NUM_SINGULAR;
          st->column = j;
          st->pivot = cd.mag;
          s_p = -1;
        } else {
          pivot_min = fmin(pivot_min, cd.mag);
          s_ipiv[c] = (int32_t)p;
          const int32_t op = s_orig[p - j0];
          s_rowperm[c] = op;
          s_orig[p - j0] = s_orig[j - j0];
          s_orig[j - j0] = op;
          s_p = p;
          s_piv = cd.val;
        }
      }
    }
    __syncthreads();
    CK_PROF(3);
    const int64_t p = s_p;
    if (p < 0) break;
    ju = lmax(ju, lmin(j + b.ku + (p - j), b.n - 1));
    // interchange rows j and p inside the panel (columns j .. j0+jb-1); columns
    // beyond j + kv hold no entry in rows j..j+km (LAPACK's ju bound). The pivot
    // row's values are the step's u(j, k).
    const int64_t kend = lmin(j0 + jb, j + b.kv + 1);
    for (int64_t k = j + tid; k < kend; k += kPanelThreads) {
      double* ak = ab_col(b, k);
      double u = ak[j];
      if (p != j) {
        uint32_t* kk = b.key + s_kofs[k - j0];
        const double t = ak[p];
        ak[p] = u;
        ak[j] = t;
        u = t;
        const uint32_t tk = kk[j];
        kk[j] = kk[p];
        kk[p] = tk;
      }
      s_u[k - j0] = u;
    }
    // stored multipliers (touched, nonzero: lu.hpp:135-137) as packed order keys,
    // compacted in row order into s_sort[0, m); the key slots of the others
    // become kKeyUntouched, the stored ones receive their rank below
    __syncthreads();  // interchange done
    CK_PROF(6);
    int m = 0;
    for (int r0 = 0; r0 < km; r0 += kPanelThreads) {
      const int r = r0 + tid;
      uint64_t v = ~0ull;
      if (r < km) {
        const int64_t i = j + 1 + r;
        const uint32_t k = kj[i];
        if (k != kKeyUntouched && aj[i] != 0.0)
          v = (order_key(k, s_orig[i - j0]) << kRankBits) | (uint64_t)r;
        else
          kj[i] = kKeyUntouched;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, v != ~0ull);
      if (lane == 0) s_wcnt[warp] = __popc(bal);
      __syncthreads();
      int off = m;
      for (int w = 0; w < warp; ++w) off += s_wcnt[w];
      if (v != ~0ull) s_sort[off + __popc(bal & ((1u << lane) - 1u))] = v;
      for (int w = 0; w < kWarps; ++w) m += s_wcnt[w];
      __syncthreads();
    }
    CK_PROF(7);
    // position in order = rank among the stored multipliers (lcols[j] order); the
    // rows usually arrive in order already, otherwise a bitonic sort
    bool sorted = true;
    for (int q = tid; q + 1 < m; q += kPanelThreads) sorted = sorted && s_sort[q] < s_sort[q + 1];
    if (!__syncthreads_and(sorted)) {
      int nsort = 1;
      while (nsort < m) nsort <<= 1;
      for (int q = m + tid; q < nsort; q += kPanelThreads) s_sort[q] = ~0ull;
      __syncthreads();
      bitonic_sort(s_sort, nsort);
    }
    for (int q = tid; q < m; q += kPanelThreads)
      kj[j + 1 + (int64_t)(s_sort[q] & ((1u << kRankBits) - 1))] = (uint32_t)q;
    __syncthreads();
    CK_PROF(10);
    // update of the remaining panel columns by this step, one thread per row
    // (lu.hpp:97-110 order: skipped where u = 0; fill keyed on first touch --
    // the compare-and-swap needs no answer, so it stays off the critical path)
    const double piv = s_piv;
    const int ncol = (int)(kend - (j + 1));
    for (int r = tid; r < km; r += kPanelThreads) {
      const int64_t i = j + 1 + r;
      const double l = __ddiv_rn(aj[i], piv);
      aj[i] = l;
      const uint32_t rank = kj[i];
      if (rank == kKeyUntouched) continue;
      for (int c0 = 0; c0 < ncol; c0 += 8) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int cc = c + 1 + c0 + q;
          v[q] = (c0 + q < ncol && s_u[cc] != 0.0) ? ab_col(b, j0 + cc)[i] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int cc = c + 1 + c0 + q;
          if (c0 + q < ncol && s_u[cc] != 0.0) {
            ab_col(b, j0 + cc)[i] = __dsub_rn(v[q], __dmul_rn(l, s_u[cc]));
            atomicCAS(b.key + s_kofs[cc] + i, kKeyUntouched, fill_key(b, j, j0 + cc, rank));
          }
        }
      }
    }
    __syncthreads();
    CK_PROF(11);
  }
  for (int r = tid; r < nrow; r += kPanelThreads) b.orig[j0 + r] = s_orig[r];
  if (tid < jb) {
    b.ipiv[j0 + tid] = s_ipiv[tid];
    b.rowperm[j0 + tid] = s_rowperm[tid];
  }
  if (tid == 0) {
    st->ju = ju;
    st->pivot_min = pivot_min;
  }
}

// Trailing columns j0+jb .. ju: per column, the panel's interchanges and
// updates in pivot order. One warp per column. kSmem: the panel's multipliers
// and ranks staged in shared memory, s_l[c * (kl+1) + r] = l(j0+c+1+r, j0+c);
// otherwise read from the band (wide bands: 12 B x 32 x (kl+1) > 227 KB).
// Every CTA also brings the key slots of columns j0+kv+32 .. j0+kv+63 into
// the window for the next panel.
template <bool kSmem>
__global__ void __launch_bounds__(512) k_gbtrf_update(const BandView* __restrict__ bs, int64_t j0,
                                                      LUStatus* const* sts) {
  extern __shared__ double s_l[];
  const BandView b = bs[blockIdx.y];
  const LUStatus* st = sts[blockIdx.y];
  if (j0 >= b.n) return;
  if (st->code != 0) return;
  init_key_slots(b, j0 + b.kv + kLUBlock, j0 + b.kv + 2 * kLUBlock, blockIdx.x, gridDim.x);
  const int jb = (int)lmin(kLUBlock, b.n - j0);
  if (j0 + jb >= b.n) return;
  const int64_t ju = st->ju;
  const int64_t kfirst = j0 + jb;
  if (kfirst > ju) return;
  const int64_t ld = b.kl + 1;
  uint32_t* s_rk = reinterpret_cast<uint32_t*>(s_l + (kSmem ? (int64_t)jb * ld : 0));
  if (kSmem) {
    for (int64_t q = threadIdx.x; q < (int64_t)jb * ld; q += blockDim.x) {
      const int c = (int)(q / ld);
      const int64_t r = q % ld;
      const int64_t j = j0 + c, km = lmin(b.kl, b.n - 1 - j);
      s_l[q] = (r < km) ? AB(b, j + 1 + r, j) : 0.0;
      s_rk[q] = (r < km) ? KEY(b, j + 1 + r, j) : kKeyUntouched;
    }
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  for (int64_t k = kfirst + (int64_t)blockIdx.x * nw + warp; k <= ju; k += (int64_t)gridDim.x * nw) {
    double* ak = ab_col(b, k);
    uint32_t* kk = key_col(b, k);
    for (int c = 0; c < jb; ++c) {
      const int64_t j = j0 + c;
      if (k - j > b.kv) continue;  // row j (and p) hold no entry in column k
      const int64_t p = b.ipiv[j];
      const int km = (int)lmin(b.kl, b.n - 1 - j);
      if (p != j && lane == 0) {
        const double t = ak[j];
        ak[j] = ak[p];
        ak[p] = t;
        const uint32_t tk = kk[j];
        kk[j] = kk[p];
        kk[p] = tk;
      }
      __syncwarp();
      const double u = ak[j];
      if (u != 0.0) {
        const double* lc = kSmem ? s_l + c * ld : ab_col(b, j) + j + 1;
        const uint32_t* rc = kSmem ? s_rk + c * ld : key_col(b, j) + j + 1;
        const uint32_t base = fill_key(b, j, k, 0);
        double* a1 = ak + j + 1;
        uint32_t* k1 = kk + j + 1;
        for (int r = lane; r < km; r += 32) {
          const uint32_t rank = rc[r];
          if (rank == kKeyUntouched) continue;
          a1[r] = __dsub_rn(a1[r], __dmul_rn(lc[r], u));
          atomicCAS(k1 + r, kKeyUntouched, base + rank);
        }
      }
      __syncwarp();
    }
  }
}

// RN(1 / U(j, j)) per pivot for the solves' head triangles (ck_lu_sweeps.cuh).
__global__ void k_pivot_reciprocals(BandView b) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < b.n) b.rdiag[j] = __drcp_rn(b.ab[b.kv + j * b.ldab]);
}

// L blocks in local pivot order: for block blk (columns J..J+jb-1), column c
// holds the step-(J+c) multipliers with the later interchanges of the same
// block applied, at window rows (relative to J) 0 .. 32+kl-1.
__global__ void __launch_bounds__(256) k_convert_l_blocks(BandView b) {
  const int64_t blk = blockIdx.x;
  const int64_t J = blk * kLUBlock;
  const int jb = (int)lmin(kLUBlock, b.n - J);
  double* dst = b.lb + blk * kLUBlock * b.lb_ld;
  for (int64_t q = threadIdx.x; q < (int64_t)kLUBlock * b.lb_ld; q += blockDim.x) {
    const int c = (int)(q / b.lb_ld);
    const int64_t r = q % b.lb_ld;
    double v = 0.0;
    if (c < jb) {
      const int64_t j = J + c, row = J + r, km = lmin(b.kl, b.n - 1 - j);
      if (row > j && row <= j + km) v = AB(b, row, j);
    }
    dst[q] = v;
  }
  __syncthreads();
  if (threadIdx.x < jb) {
    const int c = threadIdx.x;
    double* col = dst + (int64_t)c * b.lb_ld;
    for (int c2 = c + 1; c2 < jb; ++c2) {
      const int64_t p = b.ipiv[J + c2];
      if (p != J + c2) {
        const int64_t ra = c2, rb = p - J;
        double t = col[ra];
        col[ra] = col[rb];
        col[rb] = t;
      }
    }
  }
  // composite interchange of the block: apply the swaps to an index list of the
  // touched window positions, then emit (dst, src) for every moved position
  if (threadIdx.x == 0) {
    int32_t pos[2 * kLUBlock], src[2 * kLUBlock];
    int m = 0;
    auto slot = [&](int32_t q) {
      for (int k = 0; k < m; ++k)
        if (pos[k] == q) return k;
      pos[m] = q;
      src[m] = q;
      return m++;
    };
    for (int c = 0; c < jb; ++c) {
      const int32_t p = (int32_t)(b.ipiv[J + c] - J);
      if (p == c) continue;
      const int ka = slot(c), kb = slot(p);
      const int32_t t = src[ka];
      src[ka] = src[kb];
      src[kb] = t;
    }
    int32_t* out = b.perm + blk * (1 + 4 * kLUBlock);
    int cnt = 0;
    for (int k = 0; k < m; ++k)
      if (src[k] != pos[k]) {
        out[1 + 2 * cnt] = pos[k];
        out[2 + 2 * cnt] = src[k];
        ++cnt;
      }
    out[0] = cnt;
  }
}

// ------------------------------------------------ dense blocks (ck_lu_dense.cuh)
// Composite block matrices of the dense sweeps, one CTA per 32-row block:
// inverses of the block's head triangles (substitution on the identity, one
// thread per column), their products with the band coefficients the block
// reaches, the interchange maps, and the growth factor || |Hinv| |H| ||_inf of
// both heads (atomicMax over the blocks; doubles >= 0 order like their bits).
__global__ void __launch_bounds__(256) k_dense_blocks(BandView b, double* clf, double* clt, double* cub,
                                                      double* cut, uint8_t* pinv, uint8_t* psrc,
                                                      unsigned long long* growth) {
  const int64_t blk = blockIdx.x, J = blk * kLUBlock, n = b.n;
  const int tid = threadIdx.x;
  const int kl = (int)b.kl, kv = (int)b.kv, wl = kLUBlock + kl, wu = kLUBlock + kv;
  __shared__ double Lh[32][33], Uh[32][33], Li[32][33], Ui[32][33];
  // heads: Lh(r, c) multipliers r > c (unit diagonal), Uh(r, c) r <= c; rows and
  // columns past n are the identity
  for (int q = tid; q < 1024; q += blockDim.x) {
    const int r = q >> 5, c = q & 31;
    double l = 0.0, u = r == c ? 1.0 : 0.0;
    if (J + r < n && J + c < n) {
      if (r > c) l = b.lb[(blk * kLUBlock + c) * b.lb_ld + r];
      if (r <= c && c - r <= kv) u = AB(b, J + r, J + c);
    }
    Lh[r][c] = l;
    Uh[r][c] = u;
    Li[r][c] = 0.0;
    Ui[r][c] = 0.0;
  }
  __syncthreads();
  if (tid < 32) {  // column c of Linv: forward substitution on e_c
    const int c = tid;
    Li[c][c] = 1.0;
    for (int i = c + 1; i < 32; ++i) {
      double s = 0.0;
      for (int k = c; k < i; ++k) s = __fma_rn(Lh[i][k], Li[k][c], s);
      Li[i][c] = -s;
    }
  } else if (tid < 64) {  // column c of Uinv: backward substitution on e_c
    const int c = tid - 32;
    Ui[c][c] = 1.0 / Uh[c][c];
    for (int i = c - 1; i >= 0; --i) {
      double s = 0.0;
      for (int k = i + 1; k <= c; ++k) s = __fma_rn(Uh[i][k], Ui[k][c], s);
      Ui[i][c] = -s / Uh[i][i];
    }
  }
  __syncthreads();
  if (tid < 64) {  // growth: row sums of |Hinv| |H|
    const int i = tid & 31;
    const bool low = tid < 32;
    double row = 0.0;
    for (int j = 0; j < 32; ++j) {
      double s = 0.0;
      for (int k = 0; k < 32; ++k) {
        const double hi = low ? Li[i][k] : Ui[i][k];
        const double h = low ? (k == j ? 1.0 : Lh[k][j]) : Uh[k][j];
        s += fabs(hi) * fabs(h);
      }
      row += s;
    }
    if (!(row == row)) row = INFINITY;
    atomicMax(growth, (unsigned long long)__double_as_longlong(row));
  }
  // interchange maps
  for (int q = tid; q < wl; q += blockDim.x) {
    pinv[blk * wl + q] = (uint8_t)q;
    psrc[blk * wl + q] = (uint8_t)q;
  }
  __syncthreads();
  if (tid == 0) {
    const int32_t* pp = b.perm + blk * (1 + 4 * kLUBlock);
    const int np = pp[0];
    for (int t = 0; t < np; ++t) {
      const int dst = pp[1 + 2 * t], src = pp[2 + 2 * t];
      psrc[blk * wl + dst] = (uint8_t)src;
      pinv[blk * wl + src] = (uint8_t)dst;
    }
  }
  double* F = clf + blk * 32 * wl;   // [c][r]
  double* T = clt + blk * wl * 32;   // [k][c]
  double* B = cub + blk * 32 * wu;   // [c][r]
  double* G = cut + blk * 32 * wu;   // [c][r]
  // L: rows r < 32 Linv, rows 32 + m: -(Tl Linv)(m, c), Tl(m, k) = lb[k][32 + m]
  for (int q = tid; q < 32 * wl; q += blockDim.x) {
    const int c = q / wl, r = q % wl;
    double v;
    if (r < 32) {
      v = Li[r][c];
    } else {
      const int m = r - 32;
      double s = 0.0;
      if (J + 32 + m < n)
        for (int k = c; k < 32; ++k)
          if (J + k < n) s = __fma_rn(b.lb[(blk * kLUBlock + k) * b.lb_ld + 32 + m], Li[k][c], s);
      v = -s;
    }
    F[q] = v;
    T[r * 32 + c] = v;
  }
  // U backward: rows m < kv: -(Tu Uinv)(m, c), Tu(m, k) = U(J - kv + m, J + k) for
  // m >= k; rows kv + r: Uinv(r, c)
  for (int q = tid; q < 32 * wu; q += blockDim.x) {
    const int c = q / wu, r = q % wu;
    double v;
    if (r >= kv) {
      v = Ui[r - kv][c];
    } else {
      const int64_t i = J - kv + r;
      double s = 0.0;
      if (i >= 0)
        for (int k = 0; k <= c && k <= r; ++k)
          if (J + k < n) s = __fma_rn(AB(b, i, J + k), Ui[k][c], s);
      v = -s;
    }
    B[q] = v;
  }
  // U^T forward: rows r < 32: Uinv^T(r, c) = Uinv(c, r); rows 32 + q2:
  // -(G Uinv^T)(q2, c), G(q2, k) = U(J + k, J + 32 + q2) inside the band
  for (int q = tid; q < 32 * wu; q += blockDim.x) {
    const int c = q / wu, r = q % wu;
    double v;
    if (r < 32) {
      v = Ui[c][r];
    } else {
      const int q2 = r - 32;
      const int64_t col = J + 32 + q2;
      double s = 0.0;
      if (col < n)
        for (int k = c; k < 32; ++k)
          if (J + k < n && 32 + q2 - k <= kv) s = __fma_rn(AB(b, J + k, col), Ui[c][k], s);
      v = -s;
    }
    G[q] = v;
  }
}

template <int R>
__global__ void __launch_bounds__(1024) k_lu_solve(BandView b, double* x0, double* x1, double* x2,
                                                   double* x3, int transpose, int ring_size) {
  extern __shared__ double smem[];
  double* xs[4] = {x0, x1, x2, x3};
  inv_solve<R>(b, xs, smem, ring_size, transpose != 0);
}

// ---------------------------------------------------------------- host side
int lu_ring_size(const BandView& b) {
  int64_t need = std::max<int64_t>(b.kv, b.kl) + 2 * kLUBlock + 1;
  int s = 64;
  while (s < need) s <<= 1;
  return s;
}

// Dynamic shared memory of a solve CTA: rings + dot scratch, then as much of
// a full TMA stage (32 runs of max(kl, kv) rows) as fits next to the static
// shared memory (Head, mbarrier, step scratch).
constexpr size_t kSolveDynMax = 227 * 1024 - 12 * 1024;

size_t lu_solve_smem(const BandView& b, int R) {
  const int64_t base = stage_offset(R, lu_ring_size(b));
  const int64_t full = (int64_t)kLUBlock * ((std::max(b.kl, b.kv) + 3) & ~(int64_t)1);
  return std::min(kSolveDynMax, sizeof(double) * (size_t)(base + full));
}

// Coefficient runs shorter than this are read straight from L2/HBM: for narrow
// bands the TMA stage's issue and completion latency outweighs the traffic it
// saves (config 1, runs of 64 and 128 rows: 1.78 vs 2.10 ms per inverse
// iteration unstaged); wide bands need it (config-5 member, runs of 255 and 510
// rows: 72.7 ms staged vs 83.0 with the 255-row runs unstaged, 103 with none
// staged; config 2 339 vs 465 ms). CK_LU_STAGE_MIN overrides (A/B).
int64_t lu_stage_min() {
  if (const char* e = std::getenv("CK_LU_STAGE_MIN")) return std::atoll(e);
  return kLUStageMinRows;
}

int64_t lu_stage_cap(const BandView& b, int R) {
  return (int64_t)(lu_solve_smem(b, R) / sizeof(double)) - stage_offset(R, lu_ring_size(b));
}

size_t inv_step_smem(const BandView& b, int R) { return lu_solve_smem(b, R); }

void lu_solve_launch(ck_lu_s* f, double* const* x, int R, bool transpose, cudaStream_t st) {
  BandView b = f->view();
  const int ring = lu_ring_size(b);
  const size_t smem = lu_solve_smem(b, R);
  b.stage_cap = lu_stage_cap(b, R);
  b.stage_min = lu_stage_min();
  if (b.stage_cap < 0) fail(CK_ERR_UNSUPPORTED, "band too wide for the on-chip solve window");
  double* xs[4] = {x[0], R > 1 ? x[1] : nullptr, R > 2 ? x[2] : nullptr, R > 3 ? x[3] : nullptr};
  switch (R) {
#define CK_SOLVE_CASE(RR)                                                                       \
  case RR:                                                                                      \
    CK_CUDA(allow_max_dynamic_smem(k_lu_solve<RR>));                                            \
    k_lu_solve<RR><<<1, 1024, smem, st>>>(b, xs[0], xs[1], xs[2], xs[3], transpose ? 1 : 0, ring); \
    break;
    CK_SOLVE_CASE(1)
    CK_SOLVE_CASE(2)
    CK_SOLVE_CASE(3)
    CK_SOLVE_CASE(4)
#undef CK_SOLVE_CASE
    default: fail(CK_ERR_INVALID_ARGUMENT, "1..4 right-hand sides");
  }
  CK_CUDA(cudaGetLastError());
}

// Widest band the solves take: the R = 1 solve ring (lu_ring_size, a power of
// two >= max(kv, kl) + 65 doubles) must fit the solve CTA's shared memory.
constexpr int64_t kLUMaxBand = 16384 - 2 * kLUBlock - 1;

// Band bounds, storage, fill and status of one factorisation (lu.hpp:55-100).
static void lu_prepare(ck_lu_s* f, ck_matrix_s* m) {
  if (m->nrows != m->ncols) fail(CK_ERR_DIMENSION, "lu_factorize: matrix must be square");
  f->device = m->device;
  // the factors outlive the matrix handle (LUFactors is a value in lu.hpp:42-47):
  // they get their own stream
  CK_CUDA(cudaStreamCreateWithFlags(&f->stream, cudaStreamNonBlocking));
  f->own_stream = true;
  CK_CUDA(cudaStreamSynchronize(m->stream));
  cudaStream_t st = f->stream;
  const int64_t n = m->nrows;
  f->n = n;
  DBuf<int> klku(2);
  CK_CUDA(cudaMemsetAsync(klku.p, 0, 2 * sizeof(int), st));
  const unsigned g = (unsigned)std::max<int64_t>(1, ceil_div(m->a.nrows_pad, 256));
  if (n > 0) k_band_bounds<<<g, 256, 0, st>>>(view(m->a), m->a.nrows_pad, m->a.perm.p, m->at.perm.p, klku.p);
  int h[2] = {0, 0};
  CK_CUDA(cudaMemcpyAsync(h, klku.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  CK_CUDA(cudaStreamSynchronize(st));
  f->kl = h[0];
  f->ku = h[1];
  const int64_t kv = f->kl + f->ku;
  // limits, checked before anything is allocated: the solve window (any band up
  // to 16319 rows above the diagonal of U) and device memory
  if (std::max(kv, f->kl) > kLUMaxBand)
    fail(CK_ERR_UNSUPPORTED, "lu_factorize: band too wide for the device solves (kl + ku = " +
                                 std::to_string(kv) + " > " + std::to_string(kLUMaxBand) + ")");
  const int64_t ldab = 2 * f->kl + f->ku + 1;
  const int64_t kw = kv + 2 * kLUBlock;
  const double band_b = (double)ldab * (double)n * 8.0;
  const double lb_b = (double)ceil_div(n, kLUBlock) * kLUBlock * (double)(kLUBlock + f->kl) * 8.0;
  const double aux_b = (double)ldab * (double)n / 8.0 + (double)kw * (double)ldab * 4.0 + 16.0 * n;
  size_t freeb = 0, totalb = 0;
  device_trim();  // cached pool blocks count as free
  CK_CUDA(cudaMemGetInfo(&freeb, &totalb));
  if ((band_b + lb_b + aux_b) * 1.05 > (double)freeb)
    fail(CK_ERR_OUT_OF_MEMORY, "band LU storage (" + std::to_string((band_b + lb_b + aux_b) / 1e9) +
                                   " GB for kl = " + std::to_string(f->kl) + ", ku = " +
                                   std::to_string(f->ku) + ") exceeds free device memory");
  f->ab.alloc(std::max<int64_t>(1, ldab * n));
  f->ipiv.alloc(std::max<int64_t>(1, n));
  f->rowperm.alloc(std::max<int64_t>(1, n));
  f->orig.alloc(std::max<int64_t>(1, n));
  f->abit.alloc(std::max<int64_t>(1, ceil_div(ldab * n, 32)));
  f->key.alloc(std::max<int64_t>(1, kw * ldab));
  f->status.alloc(1);
  CK_CUDA(cudaMemsetAsync(f->ab.p, 0, f->ab.bytes(), st));
  CK_CUDA(cudaMemsetAsync(f->abit.p, 0, f->abit.bytes(), st));
  LUStatus s0{0, 0, -1, 0.0, INFINITY, 0};
  CK_CUDA(cudaMemcpyAsync(f->status.p, &s0, sizeof(s0), cudaMemcpyHostToDevice, st));
  BandView b = f->view();
  if (n > 0) {
    k_band_fill<<<g, 256, 0, st>>>(view(m->a), m->a.nrows_pad, m->a.perm.p, m->at.perm.p, b, f->abit.p);
    k_iota<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(f->orig.p, n);
  }
  CK_CUDA(cudaGetLastError());
  CK_CUDA(cudaStreamSynchronize(st));
}

// Shared memory of the trailing update with the panel's multipliers and ranks staged.
static size_t update_smem(int64_t klmax) {
  return (sizeof(double) + sizeof(uint32_t)) * kLUBlock * (size_t)(klmax + 1);
}

// The right-looking panel loop (lu.hpp:100-177) of S prepared factorisations at
// once: two launches per 32-column panel for the whole batch (one CTA per member
// for the panel, a member row of CTAs for the trailing update), on stream st.
static void lu_panels(ck_lu_s* const* fs, int S, double pivot_tol, cudaStream_t st) {
  std::vector<BandView> hb((size_t)S);
  std::vector<LUStatus*> hs((size_t)S);
  int64_t nmax = 0, klmax = 0, colmax = 0, kvmax = 0;
  for (int g = 0; g < S; ++g) {
    hb[g] = fs[g]->view();
    hs[g] = fs[g]->status.p;
    nmax = std::max(nmax, fs[g]->n);
    klmax = std::max(klmax, fs[g]->kl);
    kvmax = std::max(kvmax, fs[g]->kl + fs[g]->ku);
    colmax = std::max(colmax, fs[g]->kl + fs[g]->ku + 1);
  }
  if (nmax == 0) return;
  DBuf<BandView> db(S);
  DBuf<LUStatus*> ds(S);
  CK_CUDA(cudaMemcpyAsync(db.p, hb.data(), sizeof(BandView) * S, cudaMemcpyHostToDevice, st));
  CK_CUDA(cudaMemcpyAsync(ds.p, hs.data(), sizeof(LUStatus*) * S, cudaMemcpyHostToDevice, st));
  // key slots of the first panel's reach (later ones: k_gbtrf_update)
  {
    const unsigned gx = (unsigned)std::min<int64_t>(148, std::max<int64_t>(1, ceil_div((kvmax + 2 * kLUBlock) * (2 * klmax + kvmax + 1), 4096)));
    k_key_init<<<dim3(gx, (unsigned)S), 256, 0, st>>>(db.p);
  }
  int sort_words = 1;
  while (sort_words < klmax + 1) sort_words <<= 1;
  const size_t psmem = sizeof(uint64_t) * (size_t)sort_words + sizeof(int32_t) * (size_t)(kLUBlock + klmax);
  CK_CUDA(allow_max_dynamic_smem(k_gbtrf_panel));
  size_t usmem = update_smem(klmax);
  bool stage = usmem <= 220 * 1024;
  if (const char* e = std::getenv("CK_LU_UPDATE_SMEM")) stage = stage && e[0] != '0';
  if (!stage) usmem = 0;
  CK_CUDA(allow_max_dynamic_smem(k_gbtrf_update<true>));
  const unsigned ublocks = (unsigned)std::min<int64_t>(148, std::max<int64_t>(1, ceil_div(colmax, 16)));
  for (int64_t j0 = 0; j0 < nmax; j0 += kLUBlock) {
    k_gbtrf_panel<<<dim3(1, (unsigned)S), kPanelThreads, psmem, st>>>(db.p, j0, pivot_tol, ds.p,
                                                                        sort_words);
    if (j0 + kLUBlock < nmax) {
      if (stage)
        k_gbtrf_update<true><<<dim3(ublocks, (unsigned)S), 512, usmem, st>>>(db.p, j0, ds.p);
      else
        k_gbtrf_update<false><<<dim3(ublocks, (unsigned)S), 512, 0, st>>>(db.p, j0, ds.p);
    }
  }
  CK_CUDA(cudaGetLastError());
  CK_CUDA(cudaStreamSynchronize(st));
}

// Status check (singular -> error) and the solve-side data of one factorisation.
static void lu_finish(ck_lu_s* f, int64_t* fail_col, double* fail_pivot) {
  cudaStream_t st = f->stream;
  const int64_t n = f->n;
  LUStatus s{};
  CK_CUDA(cudaMemcpyAsync(&s, f->status.p, sizeof(s), cudaMemcpyDeviceToHost, st));
  CK_CUDA(cudaStreamSynchronize(st));
  f->key.reset();
  f->abit.reset();
  f->orig.reset();
  if (s.code != 0) {
    if (fail_col) *fail_col = s.column;
    if (fail_pivot) *fail_pivot = s.pivot;
    f->ab.reset();
    fail(s.code == CK_ERR_STRUCT_SINGULAR ? CK_ERR_STRUCT_SINGULAR : CK_ERR_NUM_SINGULAR,
         (s.code == CK_ERR_STRUCT_SINGULAR
              ? std::string("structurally singular: no pivot candidate in column ")
              : std::string("numerically singular: best pivot ") + std::to_string(s.pivot) +
                    " below threshold in column ") +
             std::to_string(s.column));
  }
  f->pivot_min = n > 0 ? s.pivot_min : INFINITY;
  const int64_t nblk = ceil_div(n, kLUBlock);
  f->lb.alloc(nblk * kLUBlock * (kLUBlock + f->kl) + 2);  // +2: stage copies round up to 16 B
  f->bperm.alloc(std::max<int64_t>(1, nblk * (1 + 4 * kLUBlock)));
  f->work.alloc(2 * n + 3 * kNormParts + 16);
  f->rdiag.alloc(std::max<int64_t>(1, n));
  BandView b = f->view();
  if (n > 0) k_convert_l_blocks<<<(unsigned)nblk, 256, 0, st>>>(b);
  if (n > 0) k_pivot_reciprocals<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(b);
  CK_CUDA(cudaGetLastError());
  // narrow bands: the composite blocks of the dense sweeps (CK_LU_DENSE=0: A/B)
  f->dense_ok = false;
  const char* de = std::getenv("CK_LU_DENSE");
  if (n > 0 && std::max(f->kl, f->kl + f->ku) <= kDenseMaxBand && !(de && de[0] == '0')) {
    const int wl = kLUBlock + (int)f->kl, wu = kLUBlock + (int)(f->kl + f->ku);
    f->dense_cf.alloc(nblk * 32 * (2 * (int64_t)wl + 2 * (int64_t)wu));
    f->dense_perm.alloc(2 * nblk * wl);
    DBuf<unsigned long long> g(1);
    CK_CUDA(cudaMemsetAsync(g.p, 0, sizeof(unsigned long long), st));
    double* c = f->dense_cf.p;
    const int64_t sl = nblk * 32 * wl, su = nblk * 32 * wu;
    k_dense_blocks<<<(unsigned)nblk, 256, 0, st>>>(b, c, c + sl, c + 2 * sl, c + 2 * sl + su,
                                                   f->dense_perm.p, f->dense_perm.p + nblk * wl, g.p);
    CK_CUDA(cudaGetLastError());
    unsigned long long bits = 0;
    CK_CUDA(cudaMemcpyAsync(&bits, g.p, sizeof(bits), cudaMemcpyDeviceToHost, st));
    CK_CUDA(cudaStreamSynchronize(st));
    std::memcpy(&f->dense_growth, &bits, sizeof(double));
    f->dense_ok = f->dense_growth <= kDenseMaxGrowth || (de && de[0] == '2');  // 2: force (tests)
    if (!f->dense_ok) {
      f->dense_cf.reset();
      f->dense_perm.reset();
    }
  }
  CK_CUDA(cudaStreamSynchronize(st));
}

// Standalone dense-block solve (the witness check of a dense inverse session).
__global__ void __launch_bounds__(kDenseThreads, 1) k_dense_solve(DenseView d, double* x, int transpose,
                                                                  unsigned dyn_bytes) {
  __shared__ double smem[3 * kDenseThreads];
  extern __shared__ __align__(16) double dyn[];
  DenseRing R = dense_ring(d, dyn, dyn_bytes);
  dense_solve(d, x, smem, R, transpose != 0);
}

void lu_dense_solve_launch(ck_lu_s* f, double* x, bool transpose, cudaStream_t st) {
  if (!f->dense_ok) fail(CK_ERR_LOGIC, "dense blocks not built");
  const DenseView d = f->dense_view();
  const size_t dyn = dense_dyn_smem(d.wl, d.wu);
  CK_CUDA(cudaFuncSetAttribute(k_dense_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  k_dense_solve<<<1, kDenseThreads, dyn, st>>>(d, x, transpose ? 1 : 0, (unsigned)dyn);
  CK_CUDA(cudaGetLastError());
}

// ------------------------------------------------ LUFactors in the reference's shape
// lu.hpp:42-47 and 144-176: L strictly lower in pivot coordinates (unit
// diagonal implicit), U upper with the diagonal first in each row, both CSR
// with ascending columns, row_perm[k] = original row pivoted at step k. An
// entry is stored where the factor value is nonzero (the reference stores the
// touched rows with work != 0, lu.hpp:101,136; the two differ only when a
// multiplier underflows to zero).

__global__ void k_u_count(BandView b, int64_t* cnt) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= b.n) return;
  const int64_t hi = lmin(b.n - 1, k + b.kv);
  int64_t c = 0;
  for (int64_t j = k; j <= hi; ++j) c += AB(b, k, j) != 0.0;
  cnt[k] = c;
}

__global__ void k_u_fill(BandView b, const int64_t* __restrict__ rp, int32_t* ci, double* va) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= b.n) return;
  const int64_t hi = lmin(b.n - 1, k + b.kv);
  int64_t o = rp[k];
  for (int64_t j = k; j <= hi; ++j) {
    const double v = AB(b, k, j);
    if (v != 0.0) {
      ci[o] = (int32_t)j;
      va[o] = v;
      ++o;
    }
  }
}

__global__ void k_pinv(const int32_t* __restrict__ rowperm, int32_t* pinv, int64_t n) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < n) pinv[rowperm[k]] = (int32_t)k;
}

// Replays the interchanges (one CTA): after step j's interchange, position
// j+1+r holds original row ids[j+1+r], whose final (pivot) row is pinv[.].
__global__ void __launch_bounds__(1024) k_l_rows(BandView b, const int32_t* __restrict__ pinv,
                                                 int32_t* ids, int32_t* lrow) {
  for (int64_t i = threadIdx.x; i < b.n; i += blockDim.x) ids[i] = (int32_t)i;
  __syncthreads();
  for (int64_t j = 0; j < b.n; ++j) {
    if (threadIdx.x == 0) {
      const int64_t p = b.ipiv[j];
      const int32_t t = ids[j];
      ids[j] = ids[p];
      ids[p] = t;
    }
    __syncthreads();
    const int64_t km = lmin(b.kl, b.n - 1 - j);
    for (int64_t r = threadIdx.x; r < km; r += blockDim.x) lrow[j * b.kl + r] = pinv[ids[j + 1 + r]];
    __syncthreads();
  }
}

// Nonzero multipliers of each column (one warp per column).
__global__ void k_l_count(BandView b, int64_t* ccnt) {
  const int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= b.n) return;
  const int64_t km = lmin(b.kl, b.n - 1 - j);
  int64_t c = 0;
  for (int64_t r = lane; r < km; r += 32) c += AB(b, j + 1 + r, j) != 0.0;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) ccnt[j] = c;
}

// Compacts the nonzero multipliers in column-major order: (final row, entry).
__global__ void k_l_compact(BandView b, const int64_t* __restrict__ coff,
                            const int32_t* __restrict__ lrow, uint32_t* key, int64_t* idx,
                            int64_t* rcnt) {
  const int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= b.n) return;
  const int64_t km = lmin(b.kl, b.n - 1 - j);
  int64_t o = coff[j];
  for (int64_t r0 = 0; r0 < km; r0 += 32) {
    const int64_t r = r0 + lane;
    const bool nz = r < km && AB(b, j + 1 + r, j) != 0.0;
    const unsigned m = __ballot_sync(0xffffffffu, nz);
    if (nz) {
      const int64_t q = o + __popc(m & ((1u << lane) - 1u));
      const int32_t row = lrow[j * b.kl + r];
      key[q] = (uint32_t)row;
      idx[q] = j * b.kl + r;  // entry id: column j, multiplier r
      atomicAdd(reinterpret_cast<unsigned long long*>(rcnt + row), 1ull);
    }
    o += __popc(m);
  }
}

__global__ void k_l_gather(BandView b, const int64_t* __restrict__ idx, int64_t nnz, int32_t* ci,
                           double* va) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= nnz) return;
  const int64_t e = idx[q];
  const int64_t j = e / b.kl, r = e % b.kl;
  ci[q] = (int32_t)j;
  va[q] = AB(b, j + 1 + r, j);
}

static void exclusive_scan(const int64_t* in, int64_t* out, int64_t count, cudaStream_t st) {
  size_t tb = 0;
  CK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, count, st));
  DBuf<unsigned char> tmp((int64_t)tb + 1);
  CK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, count, st));
}

void lu_build_csr(ck_lu_s* f) {
  if (f->csr_built) return;
  cudaStream_t st = f->stream;
  const int64_t n = f->n;
  BandView b = f->view();
  const unsigned gr = (unsigned)std::max<int64_t>(1, ceil_div(n, 256));
  const unsigned gw = (unsigned)std::max<int64_t>(1, ceil_div(n * 32, 256));
  // U
  DBuf<int64_t> cnt(n + 1);
  CK_CUDA(cudaMemsetAsync(cnt.p, 0, cnt.bytes(), st));
  f->u_rp.alloc(n + 1);
  if (n > 0) k_u_count<<<gr, 256, 0, st>>>(b, cnt.p);
  exclusive_scan(cnt.p, f->u_rp.p, n + 1, st);
  int64_t nnz_u = 0;
  CK_CUDA(cudaMemcpyAsync(&nnz_u, f->u_rp.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK_CUDA(cudaStreamSynchronize(st));
  f->u_ci.alloc(std::max<int64_t>(1, nnz_u));
  f->u_va.alloc(std::max<int64_t>(1, nnz_u));
  if (n > 0) k_u_fill<<<gr, 256, 0, st>>>(b, f->u_rp.p, f->u_ci.p, f->u_va.p);
  // L
  DBuf<int64_t> ccnt(n + 1), coff(n + 1), rcnt(n + 1);
  CK_CUDA(cudaMemsetAsync(ccnt.p, 0, ccnt.bytes(), st));
  CK_CUDA(cudaMemsetAsync(rcnt.p, 0, rcnt.bytes(), st));
  if (n > 0) k_l_count<<<gw, 256, 0, st>>>(b, ccnt.p);
  exclusive_scan(ccnt.p, coff.p, n + 1, st);
  int64_t nnz_l = 0;
  CK_CUDA(cudaMemcpyAsync(&nnz_l, coff.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK_CUDA(cudaStreamSynchronize(st));
  f->l_rp.alloc(n + 1);
  f->l_ci.alloc(std::max<int64_t>(1, nnz_l));
  f->l_va.alloc(std::max<int64_t>(1, nnz_l));
  if (nnz_l > 0) {
    DBuf<int32_t> pinv(n), ids(n), lrow(std::max<int64_t>(1, n * f->kl));
    k_pinv<<<gr, 256, 0, st>>>(f->rowperm.p, pinv.p, n);
    k_l_rows<<<1, 1024, 0, st>>>(b, pinv.p, ids.p, lrow.p);
    DBuf<uint32_t> key(nnz_l), key2(nnz_l);
    DBuf<int64_t> idx(nnz_l), idx2(nnz_l);
    k_l_compact<<<gw, 256, 0, st>>>(b, coff.p, lrow.p, key.p, idx.p, rcnt.p);
    int bits = 1;
    while ((int64_t(1) << bits) < n) ++bits;
    size_t tb = 0;
    // stable: each row keeps the column-major (ascending column) order
    CK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, key2.p, idx.p, idx2.p, nnz_l, 0, bits, st));
    DBuf<unsigned char> tmp((int64_t)tb + 1);
    CK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.p, key2.p, idx.p, idx2.p, nnz_l, 0, bits, st));
    k_l_gather<<<(unsigned)ceil_div(nnz_l, 256), 256, 0, st>>>(b, idx2.p, nnz_l, f->l_ci.p, f->l_va.p);
  }
  exclusive_scan(rcnt.p, f->l_rp.p, n + 1, st);
  CK_CUDA(cudaGetLastError());
  CK_CUDA(cudaStreamSynchronize(st));
  f->nnz_l = nnz_l;
  f->nnz_u = nnz_u;
  f->csr_built = true;
}

void lu_factorize(ck_lu_s* f, ck_matrix_s* m, double pivot_tol, int64_t* fail_col,
                  double* fail_pivot) {
  lu_prepare(f, m);
  ck_lu_s* one[1] = {f};
  lu_panels(one, 1, pivot_tol, f->stream);
  lu_finish(f, fail_col, fail_pivot);
}

// Batch: every member prepared, one panel loop for all (the factorisation of a
// member is launch- and latency-bound alone), then each finished. codes[g] is
// CK_OK or the member's error status (its factors freed).
void lu_factorize_batch(ck_lu_s* const* fs, ck_matrix_s* const* ms, int S, double pivot_tol,
                        int32_t* codes, int64_t* fail_cols, double* fail_pivots) {
  for (int g = 0; g < S; ++g) lu_prepare(fs[g], ms[g]);
  lu_panels(fs, S, pivot_tol, fs[0]->stream);
  for (int g = 0; g < S; ++g) {
    codes[g] = CK_OK;
    try {
      lu_finish(fs[g], fail_cols ? fail_cols + g : nullptr, fail_pivots ? fail_pivots + g : nullptr);
    } catch (const Error& e) {
      codes[g] = e.code;
    }
  }
}

}  // namespace ck

#ifdef CK_SWEEP_PROF
// Profiling build only: read (and optionally reset) the phase cycles of the
// standalone solves (k_lu_solve, this translation unit's copy).
extern "C" int ck_debug_sweep_prof(unsigned long long* out32, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out32, ck::g_sweep_prof, sizeof(unsigned long long) * 32);
  if (reset) {
    unsigned long long z[32] = {};
    cudaMemcpyToSymbol(ck::g_sweep_prof, z, sizeof(z));
  }
  return 0;
}
#endif
