// Device-resident operator: upload, validation, A^T construction and the
// sliced-ELL layouts, plus the standalone operator kernels (matvec,
// transpose_matvec, residual norms, loss/grad) used for parity and by
// verify_solution.
//
// Reference: SparseMatrix (sparse.hpp:52-152), matvec (sparse.hpp:212-226),
// transpose_matvec (sparse.hpp:230-242), two_norm (sparse.hpp:175-186).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "ck_common.h"
#include "ck_device.cuh"
#include "ck_internal.h"

namespace ck {

// ------------------------------------------------------------ validation
// SparseMatrix::validate (sparse.hpp:129-145): offsets nondecreasing, columns
// in range and strictly increasing per row, finite values. Also gathers the
// maximum row length (SELL slice width bound).
__global__ void k_validate(int64_t nrows, int64_t ncols, const int64_t* __restrict__ rp,
                           const int32_t* __restrict__ ci, const double* __restrict__ va,
                           unsigned int* flags, int* maxlen) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  int64_t b = rp[i], e = rp[i + 1];
  unsigned int f = 0;
  if (e < b) {
    atomicOr(flags, 1u);
    return;
  }
  for (int64_t k = b; k < e; ++k) {
    int32_t c = ci[k];
    if (c < 0 || c >= ncols) f |= 2u;
    if (k > b && ci[k - 1] >= c) f |= 4u;
    double v = va[k];
    if (!(fabs(v) <= 1.7976931348623157e308)) f |= 8u;
  }
  if (f) atomicOr(flags, f);
  int len = (e - b) > 0x7fffffff ? 0x7fffffff : (int)(e - b);
  atomicMax(maxlen, len);
}

__global__ void k_row_len(int64_t n, const int64_t* __restrict__ rp, int32_t* len) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) len[i] = (int32_t)(rp[i + 1] - rp[i]);
}

__global__ void k_row_ids(int64_t n, const int64_t* __restrict__ rp, uint32_t* rowid) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int64_t k = rp[i]; k < rp[i + 1]; ++k) rowid[k] = (uint32_t)i;
}

__global__ void k_iota_u32(int64_t n, uint32_t* v) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) v[i] = (uint32_t)i;
}

__global__ void k_count_cols(int64_t nnz, const int32_t* __restrict__ ci, int32_t* cnt) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < nnz) atomicAdd(&cnt[ci[k]], 1);
}

__global__ void k_widen_counts(int64_t ncols, const int32_t* __restrict__ cnt, int64_t* out,
                               int* maxcnt) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < ncols) {
    out[j] = cnt[j];
    atomicMax(maxcnt, cnt[j]);
  } else if (j == ncols) {
    out[j] = 0;
  }
}

__global__ void k_gather_transpose(int64_t nnz, const uint32_t* __restrict__ idx,
                                   const uint32_t* __restrict__ rowid,
                                   const double* __restrict__ va, int32_t* at_ci, double* at_va) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  uint32_t e = idx[k];
  at_ci[k] = (int32_t)rowid[e];
  at_va[k] = va[e];
}

// Stable descending sort of row lengths inside each 256-row tile (the SELL
// "sigma" window): rank = #longer rows + #equal rows earlier in the tile.
__global__ void __launch_bounds__(kTile) k_tile_sort(int64_t n, const int32_t* __restrict__ len,
                                                     int32_t* perm, int32_t* inv,
                                                     uint16_t* len_out) {
  __shared__ int32_t s[kTile];
  int64_t i = blockIdx.x * (int64_t)kTile + threadIdx.x;
  int32_t L = i < n ? len[i] : -1;
  s[threadIdx.x] = L;
  __syncthreads();
  int rank = 0;
  for (int j = 0; j < kTile; ++j) {
    int32_t o = s[j];
    rank += (o > L) || (o == L && j < (int)threadIdx.x);
  }
  int64_t pos = blockIdx.x * (int64_t)kTile + rank;
  perm[pos] = i < n ? (int32_t)i : -1;
  if (i < n) inv[i] = (int32_t)pos;
  len_out[pos] = (uint16_t)(L > 0 ? L : 0);
}

// Slice entry counts: rows are sorted descending, so a slice's first row is its
// widest. The last element (index nslices) is left for the exclusive scan total.
__global__ void k_slice_entries(int64_t nslices, const uint16_t* __restrict__ len, int64_t* cnt) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s < nslices) cnt[s] = (((int64_t)len[s * kSlice] + 1) & ~int64_t(1)) * kSlice;  // even widths
  if (s == nslices) cnt[s] = 0;
}

__global__ void k_sell_fill(int64_t nrows_pad, const int32_t* __restrict__ perm,
                            const uint16_t* __restrict__ len, const int64_t* __restrict__ rp,
                            const int32_t* __restrict__ ci, const double* __restrict__ va,
                            const int32_t* __restrict__ colmap, const int64_t* __restrict__ sp,
                            int32_t* scol, double* sval) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= nrows_pad) return;
  int64_t slice = k >> 5;
  int lane = (int)(k & 31);
  int64_t base = sp[slice];
  int w = (int)((sp[slice + 1] - base) >> 5);
  int L = len[k];
  int32_t row = perm[k];
  int64_t src = row >= 0 ? rp[row] : 0;
  for (int j = 0; j < w; ++j) {
    int64_t d = sell_at(base + 2 * lane, j);
    if (j < L) {
      scol[d] = colmap[ci[src + j]];
      sval[d] = va[src + j];
    } else {
      scol[d] = 0;
      sval[d] = 0.0;
    }
  }
}

// Narrow column format (ck_common.h): per-slice base = smallest stored column
// of the slice's rows; flags bit0 when a slice's columns span >= 65536.
__global__ void k_slice_span(int64_t nslices, const int64_t* __restrict__ sp,
                             const uint16_t* __restrict__ len, const int32_t* __restrict__ col,
                             int32_t* cbase, unsigned int* flags) {
  const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= nslices) return;  // warp-uniform
  const int64_t base = sp[s] + 2 * lane;
  const int L = len[s * kSlice + lane];
  int lo = 0x7fffffff, hi = -1;
  for (int j = 0; j < L; ++j) {
    const int c = col[sell_at(base, j)];
    lo = min(lo, c);
    hi = max(hi, c);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (lane == 0) {
    const int b = hi < 0 ? 0 : lo;
    cbase[s] = b;
    if (hi >= 0 && (int64_t)hi - b > 65535) atomicOr(flags, 1u);
  }
}

__global__ void k_narrow_cols(int64_t nrows_pad, const int64_t* __restrict__ sp,
                              const uint16_t* __restrict__ len, const int32_t* __restrict__ cbase,
                              const int32_t* __restrict__ col, uint16_t* col16) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= nrows_pad) return;
  const int64_t slice = k >> 5, base = sell_rowbase(sp[slice], k);
  const int w = (int)((sp[slice + 1] - sp[slice]) >> 5), L = len[k];
  const int b = cbase[slice];
  for (int j = 0; j < w; ++j) {
    const int64_t d = sell_at(base, j);
    col16[d] = (uint16_t)(j < L ? col[d] - b : 0);
  }
}

// ------------------------------------------------------ pattern dictionary
// Slices with identical uint16 offset blocks share one copy (Sell::ptab). One
// warp per slice throughout.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// Order-independent 64-bit hash of (width, offsets): a sum of mixed (index, value) words.
__global__ void k_slice_hash(int64_t nslices, const int64_t* __restrict__ sp,
                             const uint16_t* __restrict__ col16, uint64_t* hash, int32_t* ids) {
  const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= nslices) return;
  const int64_t b = sp[s], n = sp[s + 1] - b;
  uint64_t h = 0;
  for (int64_t k = lane; k < n; k += 32) h += mix64(((uint64_t)k << 16) | col16[b + k]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if (lane == 0) {
    hash[s] = mix64(h ^ (uint64_t)n);
    ids[s] = (int32_t)s;
  }
}

// Sorted by hash: a run of equal keys is a candidate group; head[i] = 1 at its first slice.
__global__ void k_group_heads(int64_t n, const uint64_t* __restrict__ key, int32_t* head) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) head[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

// gid = inclusive scan of head: group g's representative is the slice at its head, its
// table size that slice's block.
__global__ void k_group_reps(int64_t n, const int32_t* __restrict__ head, const int32_t* __restrict__ gid,
                             const int32_t* __restrict__ sorted_slice, const int64_t* __restrict__ sp,
                             int32_t* rep, int64_t* gsize) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || !head[i]) return;
  const int32_t g = gid[i] - 1, s = sorted_slice[i];
  rep[g] = s;
  gsize[g] = sp[s + 1] - sp[s];
}

// Every slice takes its group's table offset and checks its block against the
// representative's, element by element (a hash collision clears *ok); the
// representative copies its block into the table.
__global__ void k_group_assign(int64_t n, const int32_t* __restrict__ gid, const int32_t* __restrict__ sorted_slice,
                               const int32_t* __restrict__ rep, const int64_t* __restrict__ goff,
                               const int64_t* __restrict__ sp, const uint16_t* __restrict__ col16,
                               int64_t* poff, uint16_t* ptab, unsigned int* bad) {
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const int32_t g = gid[i] - 1, s = sorted_slice[i], r = rep[g];
  const int64_t b = sp[s], len = sp[s + 1] - b, rb = sp[r], off = goff[g];
  if (lane == 0) poff[s] = off;
  if (s == r) {
    for (int64_t k = lane; k < len; k += 32) ptab[off + k] = col16[b + k];
  } else {
    bool same = sp[r + 1] - rb == len;
    if (same)
      for (int64_t k = lane; k < len; k += 32) same = same && col16[b + k] == col16[rb + k];
    if (!same) atomicOr(bad, 1u);
  }
}

// ------------------------------------------------------ standalone kernels
// One thread per permuted row; entries summed in stored order with unfused
// multiply/add, i.e. exactly matvec's arithmetic (sparse.hpp:221-223).
template <bool NW>
__global__ void __launch_bounds__(kTile) k_sell_spmv(SellView A, int64_t nrows_pad,
                                                     const double* __restrict__ x,
                                                     double* __restrict__ y) {
  constexpr int U = 8;
  int64_t row = blockIdx.x * (int64_t)kTile + threadIdx.x;
  if (row >= nrows_pad) return;
  const int64_t s0 = A.sp[row >> 5], s1 = A.sp[(row >> 5) + 1];
  const int64_t base = sell_rowbase(s0, row);
  const int w = (int)((s1 - s0) >> 5);
  const int L = A.len[row];
  const int cb = slice_cbase<NW>(A, row >> 5);
  double acc = 0.0;
  for (int j0 = 0; j0 < w; j0 += U) {
    int c[U];
    double v[U], xg[U];
    load_chunk<U, NW>(A, base, sell_colbase(A, row >> 5, row, base), cb, j0, w, c, v);
#pragma unroll
    for (int u = 0; u < U; ++u) xg[u] = __ldg(x + c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (j0 + u < L) acc = __dadd_rn(acc, __dmul_rn(v[u], xg[u]));
  }
  y[row] = acc;
}

__global__ void k_gather_perm(int64_t n_out, const int32_t* __restrict__ perm,
                              const double* __restrict__ in, double* out) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n_out) return;
  int32_t p = perm[k];
  out[k] = p >= 0 ? in[p] : 0.0;
}

__global__ void k_scatter_perm(int64_t n_in, const int32_t* __restrict__ perm,
                               const double* __restrict__ in, double* out) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n_in) return;
  int32_t p = perm[k];
  if (p >= 0) out[p] = in[k];
}

__global__ void k_sub(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                      double* out) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < n) out[k] = __dsub_rn(a[k], b[k]);
}

// grad_explicit combine, condest.hpp:103-105
__global__ void k_grad_combine(int64_t n, const double* __restrict__ v,
                               const double* __restrict__ atav, double inv_v2, double inv_av2,
                               double* g) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) g[i] = __dsub_rn(__dmul_rn(v[i], inv_v2), __dmul_rn(atav[i], inv_av2));
}

// Two-stage deterministic norm: per-block ES partials, then one block merges.
__global__ void __launch_bounds__(kTile) k_norm_partials(int64_t n, const double* __restrict__ v,
                                                         double* part) {
  __shared__ double ss[8];
  __shared__ int se[8], sf[8];
  ES a = es_zero();
  for (int64_t i = blockIdx.x * (int64_t)kTile + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kTile)
    es_add(a, v[i]);
  a = block_es(a, ss, se, sf);
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x] = a.s;
    part[3 * blockIdx.x + 1] = (double)a.e;
    part[3 * blockIdx.x + 2] = (double)a.flags;
  }
}

__global__ void __launch_bounds__(kTile) k_norm_final(int nparts, const double* __restrict__ part,
                                                      double* out) {
  __shared__ double ss[8];
  __shared__ int se[8], sf[8];
  ES a = es_zero();
  for (int i = threadIdx.x; i < nparts; i += kTile)
    es_merge(a, ES{part[3 * i], (int)part[3 * i + 1], (int)part[3 * i + 2]});
  a = block_es(a, ss, se, sf);
  if (threadIdx.x == 0) *out = es_norm(a);
}

// ------------------------------------------------------------ host side

static unsigned int grid_for(int64_t n, int threads = 256) {
  return (unsigned int)std::max<int64_t>(1, ceil_div(n, threads));
}

// y = op x over a SELL operator (whole padded row range), either column format.
static void sell_spmv(const Sell& op, const double* x, double* y, cudaStream_t st) {
  const unsigned g = (unsigned)(op.nrows_pad / kTile);
  if (op.narrow)
    k_sell_spmv<true><<<g, kTile, 0, st>>>(view(op), op.nrows_pad, x, y);
  else
    k_sell_spmv<false><<<g, kTile, 0, st>>>(view(op), op.nrows_pad, x, y);
  CK_CUDA(cudaGetLastError());
}

// Narrow column format unless CK_SELL_WIDE=1 (A/B switch) or a slice spans
// >= 65536 columns.
static bool narrow_allowed() {
  const char* e = std::getenv("CK_SELL_WIDE");
  return !(e && e[0] == '1');
}

double device_norm(const double* v, int64_t n, double* scratch, cudaStream_t st) {
  // scratch: >= 3*kNormParts + 1 doubles
  int parts = (int)std::min<int64_t>(kNormParts, std::max<int64_t>(1, ceil_div(n, kTile)));
  k_norm_partials<<<parts, kTile, 0, st>>>(n, v, scratch);
  k_norm_final<<<1, kTile, 0, st>>>(parts, scratch, scratch + 3 * kNormParts);
  double out = 0.0;
  CK_CUDA(cudaMemcpyAsync(&out, scratch + 3 * kNormParts, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK_CUDA(cudaStreamSynchronize(st));
  return out;
}

// Host -> device copy of a caller's array. Pinned (or registered) memory goes
// straight to cudaMemcpyAsync. Pageable memory -- what a numpy / std::vector
// caller passes -- is staged by the library itself: the runtime's own pageable
// path copies through one internal buffer on one thread (6-12 GB/s measured
// here); two 32 MB pinned chunks from the staging cache, filled by four host
// threads while the previous chunk is on the link, keep the copy near the host's
// memcpy rate. Returns with the source fully consumed.
static void h2d_upload(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  cudaPointerAttributes at{};
  const bool pinned = cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeHost;
  cudaGetLastError();
  constexpr size_t kChunk = size_t(32) << 20;
  if (pinned || bytes < 2 * kChunk || std::getenv("CK_NO_STAGED_UPLOAD")) {
    CK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    if (!pinned) CK_CUDA(cudaStreamSynchronize(st));
    return;
  }
  constexpr int kBufs = 2, kThreads = 4;
  PinnedBuf<unsigned char> buf[kBufs];
  cudaEvent_t done[kBufs];
  for (int b = 0; b < kBufs; ++b) {
    buf[b].resize((int64_t)kChunk);
    CK_CUDA(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
  }
  const unsigned char* sp = static_cast<const unsigned char*>(src);
  unsigned char* dp = static_cast<unsigned char*>(dst);
  int64_t i = 0;
  for (size_t off = 0; off < bytes; off += kChunk, ++i) {
    const int b = (int)(i % kBufs);
    const size_t len = std::min(kChunk, bytes - off);
    if (i >= kBufs) CK_CUDA(cudaEventSynchronize(done[b]));  // the chunk this buffer held has left
    const size_t part = (len + kThreads - 1) / kThreads;
    std::thread th[kThreads - 1];
    for (int t = 1; t < kThreads; ++t) {
      const size_t lo = std::min(len, t * part), hi = std::min(len, lo + part);
      th[t - 1] = std::thread([=, &buf] { if (hi > lo) std::memcpy(buf[b].p + lo, sp + off + lo, hi - lo); });
    }
    std::memcpy(buf[b].p, sp + off, std::min(len, part));
    for (auto& t : th) t.join();
    CK_CUDA(cudaMemcpyAsync(dp + off, buf[b].p, len, cudaMemcpyHostToDevice, st));
    CK_CUDA(cudaEventRecord(done[b], st));
  }
  CK_CUDA(cudaStreamSynchronize(st));
  for (int b = 0; b < kBufs; ++b) cudaEventDestroy(done[b]);
}

// Pattern dictionary of a narrow operator (Sell::ptab): adopted when the distinct
// slice patterns take at most 1/8 of the stored entries and 64 MB (stencil
// operators: a few hundred patterns; CK_SELL_PATTERN=0 keeps the per-entry offsets).
static void build_patterns(Sell& s, cudaStream_t st) {
  const char* e = std::getenv("CK_SELL_PATTERN");
  if (e && e[0] == '0') return;
  const int64_t ns = s.nrows_pad / kSlice;
  if (ns < 64 || s.entries < 4096) return;
  DBuf<uint64_t> key(ns), key_sorted(ns);
  DBuf<int32_t> ids(ns), sorted_slice(ns), head(ns), gid(ns);
  k_slice_hash<<<grid_for(ns * 32), 256, 0, st>>>(ns, s.slice_ptr.p, s.col16.p, key.p, ids.p);
  size_t tb = 0;
  CK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, key_sorted.p, ids.p, sorted_slice.p, ns, 0, 64, st));
  {
    DBuf<unsigned char> tmp((int64_t)std::max<size_t>(tb, 1));
    CK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.p, key_sorted.p, ids.p, sorted_slice.p, ns, 0, 64, st));
    k_group_heads<<<grid_for(ns), 256, 0, st>>>(ns, key_sorted.p, head.p);
    CK_CUDA(cudaStreamSynchronize(st));
  }
  CK_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, head.p, gid.p, ns, st));
  int32_t ngroups = 0;
  {
    DBuf<unsigned char> tmp((int64_t)std::max<size_t>(tb, 1));
    CK_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, head.p, gid.p, ns, st));
    CK_CUDA(cudaMemcpyAsync(&ngroups, gid.p + (ns - 1), sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK_CUDA(cudaStreamSynchronize(st));
  }
  if (ngroups <= 0 || (int64_t)ngroups * 8 > ns) return;  // too many distinct patterns to pay
  DBuf<int32_t> rep(ngroups);
  DBuf<int64_t> gsize(ngroups + 1), goff(ngroups + 1);
  CK_CUDA(cudaMemsetAsync(gsize.p, 0, sizeof(int64_t) * (ngroups + 1), st));
  k_group_reps<<<grid_for(ns), 256, 0, st>>>(ns, head.p, gid.p, sorted_slice.p, s.slice_ptr.p, rep.p, gsize.p);
  CK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, gsize.p, goff.p, ngroups + 1, st));
  int64_t total = 0;
  {
    DBuf<unsigned char> tmp((int64_t)std::max<size_t>(tb, 1));
    CK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, gsize.p, goff.p, ngroups + 1, st));
    CK_CUDA(cudaMemcpyAsync(&total, goff.p + ngroups, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK_CUDA(cudaStreamSynchronize(st));
  }
  if (total <= 0 || total * 8 > s.entries || total * 2 > (int64_t(64) << 20)) return;
  DBuf<uint16_t> ptab(total);
  DBuf<int64_t> poff(ns);
  DBuf<unsigned int> bad(1);
  CK_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(unsigned int), st));
  k_group_assign<<<grid_for(ns * 32), 256, 0, st>>>(ns, gid.p, sorted_slice.p, rep.p, goff.p, s.slice_ptr.p,
                                                    s.col16.p, poff.p, ptab.p, bad.p);
  CK_CUDA(cudaGetLastError());
  unsigned int h_bad = 0;
  CK_CUDA(cudaMemcpyAsync(&h_bad, bad.p, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
  CK_CUDA(cudaStreamSynchronize(st));
  if (h_bad) return;  // a hash collision: keep the per-entry offsets
  s.ptab = std::move(ptab);
  s.poff = std::move(poff);
  s.col16.reset();
  s.pattern = true;
}

void matrix_upload(ck_matrix_s* m, int64_t nrows, int64_t ncols, const int64_t* h_rp,
                   const int32_t* h_ci, const double* h_va) {
  if (nrows < 0 || ncols < 0) fail(CK_ERR_DIMENSION, "negative dimension");
  if (h_rp == nullptr) fail(CK_ERR_INVALID_ARGUMENT, "row_offsets is NULL");
  if (h_rp[0] != 0) fail(CK_ERR_DIMENSION, "inconsistent CSR arrays");
  int64_t nnz = h_rp[nrows];
  if (nnz < 0) fail(CK_ERR_DIMENSION, "inconsistent CSR arrays");
  if (nnz >= (int64_t(1) << 32) || nrows >= (int64_t(1) << 31) || ncols >= (int64_t(1) << 31))
    fail(CK_ERR_UNSUPPORTED, "matrix exceeds 2^31 rows/cols or 2^32 nonzeros");
  if (nnz > 0 && (h_ci == nullptr || h_va == nullptr))
    fail(CK_ERR_INVALID_ARGUMENT, "col_indices/values NULL");
  CK_CUDA(cudaGetDevice(&m->device));
  CK_CUDA(cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking));
  cudaStream_t st = m->stream;
  m->nrows = nrows;
  m->ncols = ncols;
  m->nnz = nnz;
  Trace tr("matrix_upload");

  DBuf<int64_t> rp(nrows + 1);
  DBuf<int32_t> ci(std::max<int64_t>(nnz, 1));
  DBuf<double> va(std::max<int64_t>(nnz, 1));
  h2d_upload(rp.p, h_rp, sizeof(int64_t) * (nrows + 1), st);
  if (nnz > 0) {
    h2d_upload(ci.p, h_ci, sizeof(int32_t) * nnz, st);
    h2d_upload(va.p, h_va, sizeof(double) * nnz, st);
  }
  tr.mark("alloc + H2D", st);
  DBuf<unsigned int> flags(1);
  DBuf<int> maxlen(2);
  CK_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(unsigned int), st));
  CK_CUDA(cudaMemsetAsync(maxlen.p, 0, 2 * sizeof(int), st));
  if (nrows > 0) k_validate<<<grid_for(nrows), 256, 0, st>>>(nrows, ncols, rp.p, ci.p, va.p, flags.p, maxlen.p);

  // A^T in CSR with each row's entries in increasing original-row order: a
  // stable radix sort of entry indices keyed by column keeps the CSR (row-major)
  // order inside every column -- exactly transpose_matvec's accumulation order.
  DBuf<int32_t> colcnt(std::max<int64_t>(ncols, 1) + 1);
  CK_CUDA(cudaMemsetAsync(colcnt.p, 0, sizeof(int32_t) * (std::max<int64_t>(ncols, 1) + 1), st));
  if (nnz > 0) k_count_cols<<<grid_for(nnz), 256, 0, st>>>(nnz, ci.p, colcnt.p);
  CK_CUDA(cudaGetLastError());

  unsigned int h_flags = 0;
  int h_maxlen[2] = {0, 0};
  CK_CUDA(cudaMemcpyAsync(&h_flags, flags.p, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
  CK_CUDA(cudaMemcpyAsync(h_maxlen, maxlen.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK_CUDA(cudaStreamSynchronize(st));
  if (h_flags & 1u) fail(CK_ERR_DIMENSION, "row offsets decrease");
  if (h_flags & 2u) fail(CK_ERR_DIMENSION, "column index out of range");
  if (h_flags & 4u) fail(CK_ERR_DIMENSION, "column indices not strictly increasing in a row");
  if (h_flags & 8u) fail(CK_ERR_DIMENSION, "non-finite entry");
  if (h_maxlen[0] > 65535) fail(CK_ERR_UNSUPPORTED, "row with more than 65535 entries");

  tr.mark("validate + column counts", st);
  DBuf<int64_t> at_rp(std::max<int64_t>(ncols, 1) + 1);
  {
    DBuf<int64_t> cnt64(std::max<int64_t>(ncols, 1) + 1);
    k_widen_counts<<<grid_for(ncols + 1), 256, 0, st>>>(ncols, colcnt.p, cnt64.p, maxlen.p + 1);
    size_t tb = 0;
    CK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt64.p, at_rp.p, ncols + 1, st));
    DBuf<unsigned char> tmp((int64_t)std::max<size_t>(tb, 1));
    CK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt64.p, at_rp.p, ncols + 1, st));
    CK_CUDA(cudaMemcpyAsync(h_maxlen + 1, maxlen.p + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK_CUDA(cudaStreamSynchronize(st));
    if (h_maxlen[1] > 65535) fail(CK_ERR_UNSUPPORTED, "column with more than 65535 entries");
  }
  DBuf<int32_t> at_ci(std::max<int64_t>(nnz, 1));
  DBuf<double> at_va(std::max<int64_t>(nnz, 1));
  if (nnz > 0) {
    DBuf<uint32_t> rowid(nnz), idx_in(nnz), idx_out(nnz);
    DBuf<uint32_t> key_out(nnz);
    k_row_ids<<<grid_for(nrows), 256, 0, st>>>(nrows, rp.p, rowid.p);
    k_iota_u32<<<grid_for(nnz), 256, 0, st>>>(nnz, idx_in.p);
    int end_bit = 1;
    while ((int64_t(1) << end_bit) < ncols) ++end_bit;
    size_t tb = 0;
    const uint32_t* keys_in = reinterpret_cast<const uint32_t*>(ci.p);
    CK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys_in, key_out.p, idx_in.p, idx_out.p,
                                            nnz, 0, end_bit, st));
    DBuf<unsigned char> tmp((int64_t)tb);
    CK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys_in, key_out.p, idx_in.p, idx_out.p,
                                            nnz, 0, end_bit, st));
    k_gather_transpose<<<grid_for(nnz), 256, 0, st>>>(nnz, idx_out.p, rowid.p, va.p, at_ci.p, at_va.p);
    CK_CUDA(cudaGetLastError());
    CK_CUDA(cudaStreamSynchronize(st));
  }

  // Row permutations (P for A's rows, Q for A's columns) and the two layouts.
  tr.mark("A^T (stable radix sort)", st);
  DBuf<int32_t> lenA(std::max<int64_t>(nrows, 1));
  if (nrows > 0) k_row_len<<<grid_for(nrows), 256, 0, st>>>(nrows, rp.p, lenA.p);
  DBuf<int32_t> lenAT(std::max<int64_t>(ncols, 1));
  if (ncols > 0) k_row_len<<<grid_for(ncols), 256, 0, st>>>(ncols, at_rp.p, lenAT.p);
  // Permutations first (each build needs the other's inverse as column map).
  {
    Sell& A = m->a;
    Sell& T = m->at;
    A.nrows = nrows;
    A.nrows_pad = std::max<int64_t>(kTile, round_up(nrows, kTile));
    T.nrows = ncols;
    T.nrows_pad = std::max<int64_t>(kTile, round_up(ncols, kTile));
    A.perm.alloc(A.nrows_pad);
    A.inv.alloc(std::max<int64_t>(nrows, 1));
    A.len.alloc(A.nrows_pad);
    T.perm.alloc(T.nrows_pad);
    T.inv.alloc(std::max<int64_t>(ncols, 1));
    T.len.alloc(T.nrows_pad);
    k_tile_sort<<<(unsigned)(A.nrows_pad / kTile), kTile, 0, st>>>(nrows, lenA.p, A.perm.p, A.inv.p, A.len.p);
    k_tile_sort<<<(unsigned)(T.nrows_pad / kTile), kTile, 0, st>>>(ncols, lenAT.p, T.perm.p, T.inv.p, T.len.p);
    CK_CUDA(cudaGetLastError());
  }
  auto finish = [&](Sell& s, const int64_t* srp, const int32_t* sci, const double* sva,
                    const int32_t* colmap) {
    int64_t nslices = s.nrows_pad / kSlice;
    s.slice_ptr.alloc(nslices + 1);
    DBuf<int64_t> cnt(nslices + 1);
    k_slice_entries<<<grid_for(nslices + 1), 256, 0, st>>>(nslices, s.len.p, cnt.p);
    size_t tb = 0;
    CK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, s.slice_ptr.p, nslices + 1, st));
    DBuf<unsigned char> tmp((int64_t)std::max<size_t>(tb, 1));
    CK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.p, s.slice_ptr.p, nslices + 1, st));
    CK_CUDA(cudaMemcpyAsync(&s.entries, s.slice_ptr.p + nslices, sizeof(int64_t),
                            cudaMemcpyDeviceToHost, st));
    CK_CUDA(cudaStreamSynchronize(st));
    s.col.alloc(std::max<int64_t>(s.entries, 1));
    s.val.alloc(std::max<int64_t>(s.entries, 1));
    k_sell_fill<<<grid_for(s.nrows_pad), 256, 0, st>>>(s.nrows_pad, s.perm.p, s.len.p, srp, sci,
                                                       sva, colmap, s.slice_ptr.p, s.col.p, s.val.p);
    CK_CUDA(cudaGetLastError());
    s.narrow = false;
    if (narrow_allowed()) {
      s.cbase.alloc(nslices);
      DBuf<unsigned int> wide(1);
      CK_CUDA(cudaMemsetAsync(wide.p, 0, sizeof(unsigned int), st));
      k_slice_span<<<grid_for(nslices * kSlice), 256, 0, st>>>(nslices, s.slice_ptr.p, s.len.p,
                                                                s.col.p, s.cbase.p, wide.p);
      unsigned int h_wide = 0;
      CK_CUDA(cudaMemcpyAsync(&h_wide, wide.p, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
      CK_CUDA(cudaStreamSynchronize(st));
      if (h_wide == 0) {
        s.col16.alloc(std::max<int64_t>(s.entries, 1));
        k_narrow_cols<<<grid_for(s.nrows_pad), 256, 0, st>>>(s.nrows_pad, s.slice_ptr.p, s.len.p,
                                                             s.cbase.p, s.col.p, s.col16.p);
        CK_CUDA(cudaGetLastError());
        CK_CUDA(cudaStreamSynchronize(st));
        s.col.reset();
        s.narrow = true;
        build_patterns(s, st);
      } else {
        s.cbase.reset();
      }
    }
    CK_CUDA(cudaStreamSynchronize(st));
  };
  tr.mark("tile sorts", st);
  finish(m->a, rp.p, ci.p, va.p, m->at.inv.p);   // A's columns -> Q positions
  tr.mark("SELL A", st);
  finish(m->at, at_rp.p, at_ci.p, at_va.p, m->a.inv.p);  // A^T's columns (A's rows) -> P positions
  tr.mark("SELL A^T", st);

  int64_t vec = std::max(m->a.nrows_pad, m->at.nrows_pad);
  m->s_in.alloc(vec);
  m->s_out.alloc(vec);
  m->s_perm_in.alloc(vec);
  m->s_perm_out.alloc(vec);
  m->s_red.alloc(3 * kNormParts + 8);
}

// y = A x (transpose=false) or y = A^T x (transpose=true), host buffers.
void matrix_apply_host(ck_matrix_s* m, bool transpose, const double* x, double* y) {
  cudaStream_t st = m->stream;
  const Sell& op = transpose ? m->at : m->a;     // rows of the applied operator
  const Sell& dom = transpose ? m->a : m->at;    // its column space (permutation source)
  int64_t nin = transpose ? m->nrows : m->ncols;
  int64_t nout = transpose ? m->ncols : m->nrows;
  if (nin > 0)
    CK_CUDA(cudaMemcpyAsync(m->s_in.p, x, sizeof(double) * nin, cudaMemcpyHostToDevice, st));
  k_gather_perm<<<grid_for(dom.nrows_pad), 256, 0, st>>>(dom.nrows_pad, dom.perm.p, m->s_in.p, m->s_perm_in.p);
  sell_spmv(op, m->s_perm_in.p, m->s_perm_out.p, st);
  k_scatter_perm<<<grid_for(op.nrows_pad), 256, 0, st>>>(op.nrows_pad, op.perm.p, m->s_perm_out.p, m->s_out.p);
  CK_CUDA(cudaGetLastError());
  if (nout > 0)
    CK_CUDA(cudaMemcpyAsync(y, m->s_out.p, sizeof(double) * nout, cudaMemcpyDeviceToHost, st));
  CK_CUDA(cudaStreamSynchronize(st));
}

// Device-pointer variant in permuted spaces: x_perm (column space of A, Q
// order, padded) -> y_perm (row space, P order, padded).
void matrix_apply_perm(ck_matrix_s* m, const double* x_perm, double* y_perm, cudaStream_t st) {
  sell_spmv(m->a, x_perm, y_perm, st);
}

void gather_perm(const int32_t* perm, int64_t n_out, const double* in, double* out, cudaStream_t st) {
  k_gather_perm<<<grid_for(n_out), 256, 0, st>>>(n_out, perm, in, out);
  CK_CUDA(cudaGetLastError());
}

void scatter_perm(const int32_t* perm, int64_t n_in, const double* in, double* out, cudaStream_t st) {
  k_scatter_perm<<<grid_for(n_in), 256, 0, st>>>(n_in, perm, in, out);
  CK_CUDA(cudaGetLastError());
}

void residual_norms(ck_matrix_s* m, const double* x, const double* b, double* rn, double* xn,
                    double* bn) {
  if (m->nrows != m->ncols) fail(CK_ERR_DIMENSION, "residual_norms: matrix must be square");
  cudaStream_t st = m->stream;
  int64_t n = m->nrows;
  // ||x||, ||b|| on the original-order vectors
  CK_CUDA(cudaMemcpyAsync(m->s_in.p, x, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  *xn = device_norm(m->s_in.p, n, m->s_red.p, st);
  CK_CUDA(cudaMemcpyAsync(m->s_out.p, b, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  *bn = device_norm(m->s_out.p, n, m->s_red.p, st);
  // r = A x - b in P order (the norm is permutation invariant)
  gather_perm(m->at.perm.p, m->at.nrows_pad, m->s_in.p, m->s_perm_in.p, st);
  matrix_apply_perm(m, m->s_perm_in.p, m->s_perm_out.p, st);
  gather_perm(m->a.perm.p, m->a.nrows_pad, m->s_out.p, m->s_in.p, st);
  k_sub<<<grid_for(m->a.nrows_pad), 256, 0, st>>>(m->a.nrows_pad, m->s_perm_out.p, m->s_in.p, m->s_perm_in.p);
  *rn = device_norm(m->s_perm_in.p, m->a.nrows_pad, m->s_red.p, st);
}

double loss_explicit_dev(ck_matrix_s* m, const double* x, bool* degenerate) {
  cudaStream_t st = m->stream;
  int64_t nc = m->ncols;
  CK_CUDA(cudaMemcpyAsync(m->s_in.p, x, sizeof(double) * nc, cudaMemcpyHostToDevice, st));
  double num = device_norm(m->s_in.p, nc, m->s_red.p, st);
  gather_perm(m->at.perm.p, m->at.nrows_pad, m->s_in.p, m->s_perm_in.p, st);
  matrix_apply_perm(m, m->s_perm_in.p, m->s_perm_out.p, st);
  double den = device_norm(m->s_perm_out.p, m->a.nrows_pad, m->s_red.p, st);
  *degenerate = den == 0.0;
  return std::log(num) - std::log(den);
}

void grad_explicit_dev(ck_matrix_s* m, const double* x, double* g, bool* degenerate) {
  cudaStream_t st = m->stream;
  int64_t nc = m->ncols;
  CK_CUDA(cudaMemcpyAsync(m->s_in.p, x, sizeof(double) * nc, cudaMemcpyHostToDevice, st));
  double vn = device_norm(m->s_in.p, nc, m->s_red.p, st);
  gather_perm(m->at.perm.p, m->at.nrows_pad, m->s_in.p, m->s_perm_in.p, st);
  matrix_apply_perm(m, m->s_perm_in.p, m->s_perm_out.p, st);  // av (P order)
  double avn = device_norm(m->s_perm_out.p, m->a.nrows_pad, m->s_red.p, st);
  *degenerate = avn == 0.0;
  if (*degenerate) return;
  // atav = A^T av (Q order)
  sell_spmv(m->at, m->s_perm_out.p, m->s_out.p, st);
  double inv_v2 = 1.0 / (vn * vn), inv_av2 = 1.0 / (avn * avn);
  k_grad_combine<<<grid_for(m->at.nrows_pad), 256, 0, st>>>(m->at.nrows_pad, m->s_perm_in.p, m->s_out.p, inv_v2, inv_av2, m->s_perm_out.p);
  scatter_perm(m->at.perm.p, m->at.nrows_pad, m->s_perm_out.p, m->s_in.p, st);
  CK_CUDA(cudaMemcpyAsync(g, m->s_in.p, sizeof(double) * nc, cudaMemcpyDeviceToHost, st));
  CK_CUDA(cudaStreamSynchronize(st));
}

}  // namespace ck
