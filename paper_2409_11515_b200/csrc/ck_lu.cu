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
#include <algorithm>
#include <cmath>
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

__global__ void k_band_fill(SellView A, int64_t nrows_pad, const int32_t* __restrict__ rperm,
                            const int32_t* __restrict__ cperm, BandView b) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nrows_pad) return;
  const int32_t row = rperm[p];
  if (row < 0) return;
  const int64_t base = sell_rowbase(A.sp[p >> 5], p);
  const int L = A.len[p];
  for (int j = 0; j < L; ++j) {
    const int64_t k = sell_at(base, j);
    AB(b, row, cperm[sell_col(A, p >> 5, k)]) = A.val[k];
  }
}

// ----------------------------------------------------------- factorisation
// Panel: columns j0 .. j0+jb-1 by one CTA per factorisation (blockIdx.y
// selects the member of a batch; members shorter than j0 are done).
__global__ void __launch_bounds__(256) k_gbtrf_panel(const BandView* __restrict__ bs, int64_t j0,
                                                     double pivot_tol, LUStatus* const* sts) {
  __shared__ double s_mag[256], s_cmax[256];
  __shared__ int64_t s_idx[256];
  __shared__ int64_t s_p;
  __shared__ double s_piv;
  const BandView b = bs[blockIdx.y];
  LUStatus* st = sts[blockIdx.y];
  if (j0 >= b.n) return;
  const int jb = (int)lmin(kLUBlock, b.n - j0);
  if (st->code != 0) return;
  const int tid = threadIdx.x;
  // running maximum over every step so far (dgbtf2's ju): rows of this panel may
  // carry fill from earlier panels out to the previous maximum
  int64_t ju = st->ju;
  for (int c = 0; c < jb; ++c) {
    const int64_t j = j0 + c;
    const int64_t km = lmin(b.kl, b.n - 1 - j);
    // pivot search over rows j..j+km; column maximum over every stored row of
    // column j (U part above the diagonal included), lu.hpp:112-125
    double best = -1.0, cmax = 0.0;
    int64_t bi = -1;
    const int64_t top = lmax(0, j - b.kv);
    for (int64_t i = top + tid; i <= j + km; i += blockDim.x) {
      const double m = fabs(AB(b, i, j));
      cmax = fmax(cmax, m);
      if (i >= j && m > best) {
        best = m;
        bi = i;
      }
    }
    s_mag[tid] = best;
    s_idx[tid] = bi;
    s_cmax[tid] = cmax;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
      if (tid < s) {
        const double om = s_mag[tid + s];
        const int64_t oi = s_idx[tid + s];
        if (om > s_mag[tid] || (om == s_mag[tid] && oi >= 0 && (s_idx[tid] < 0 || oi < s_idx[tid]))) {
          s_mag[tid] = om;
          s_idx[tid] = oi;
        }
        s_cmax[tid] = fmax(s_cmax[tid], s_cmax[tid + s]);
      }
      __syncthreads();
    }
    if (tid == 0) {
      const double bm = s_mag[0];
      const int64_t p = s_idx[0];
      if (bm == 0.0 || p < 0 || bm < pivot_tol * s_cmax[0]) {
        st->code = 5;
        st->column = j;
        st->pivot = bm < 0.0 ? 0.0 : bm;
        s_p = -1;
      } else {
        st->pivot_min = fmin(st->pivot_min, bm);
        b.ipiv[j] = (int32_t)p;
        s_p = p;
        s_piv = AB(b, p, j);
      }
    }
    __syncthreads();
    const int64_t p = s_p;
    if (p < 0) return;
    ju = lmax(ju, lmin(j + b.ku + (p - j), b.n - 1));
    // interchange rows j and p inside the panel (columns j .. j0+jb-1)
    // columns beyond j + kv hold no entry in rows j..j+km (LAPACK's ju bound)
    const int64_t kend = lmin(j0 + jb, j + b.kv + 1);
    if (p != j)
      for (int64_t k = j + tid; k < kend; k += blockDim.x) {
        double t = AB(b, j, k);
        AB(b, j, k) = AB(b, p, k);
        AB(b, p, k) = t;
      }
    __syncthreads();
    // multipliers l = a / pivot (lu.hpp:136)
    const double piv = s_piv;
    for (int64_t i = j + 1 + tid; i <= j + km; i += blockDim.x) AB(b, i, j) = __ddiv_rn(AB(b, i, j), piv);
    __syncthreads();
    // rank-1 update of the remaining panel columns (lu.hpp:102-109 order)
    const int64_t ncol = kend - (j + 1);
    for (int64_t q = tid; q < ncol * km; q += blockDim.x) {
      const int64_t k = j + 1 + q / km, i = j + 1 + q % km;
      const double u = AB(b, j, k);
      AB(b, i, k) = __dsub_rn(AB(b, i, k), __dmul_rn(AB(b, i, j), u));
    }
    __syncthreads();
  }
  if (tid == 0) st->ju = ju;
}

// Trailing columns j0+jb .. ju: per column, the panel's interchanges and
// updates in pivot order. One warp per column; multipliers of the panel in
// shared memory: s_l[c * (kl+1) + r] = l(j0+c+1+r, j0+c).
__global__ void __launch_bounds__(512) k_gbtrf_update(const BandView* __restrict__ bs, int64_t j0,
                                                      LUStatus* const* sts) {
  extern __shared__ double s_l[];
  const BandView b = bs[blockIdx.y];
  const LUStatus* st = sts[blockIdx.y];
  if (j0 >= b.n) return;
  const int jb = (int)lmin(kLUBlock, b.n - j0);
  if (j0 + jb >= b.n) return;
  if (st->code != 0) return;
  const int64_t ju = st->ju;
  const int64_t kfirst = j0 + jb;
  if (kfirst > ju) return;
  const int64_t ld = b.kl + 1;
  for (int64_t q = threadIdx.x; q < (int64_t)jb * ld; q += blockDim.x) {
    const int c = (int)(q / ld);
    const int64_t r = q % ld;
    const int64_t j = j0 + c, km = lmin(b.kl, b.n - 1 - j);
    s_l[q] = (r < km) ? AB(b, j + 1 + r, j) : 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  for (int64_t k = kfirst + (int64_t)blockIdx.x * nw + warp; k <= ju; k += (int64_t)gridDim.x * nw) {
    for (int c = 0; c < jb; ++c) {
      const int64_t j = j0 + c;
      if (k - j > b.kv) continue;  // row j (and p) hold no entry in column k
      const int64_t p = b.ipiv[j];
      const int64_t km = lmin(b.kl, b.n - 1 - j);
      if (p != j && lane == 0) {
        double t = AB(b, j, k);
        AB(b, j, k) = AB(b, p, k);
        AB(b, p, k) = t;
      }
      __syncwarp();
      const double u = AB(b, j, k);
      if (u != 0.0)
        for (int64_t r = lane; r < km; r += 32)
          AB(b, j + 1 + r, k) = __dsub_rn(AB(b, j + 1 + r, k), __dmul_rn(s_l[c * ld + r], u));
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
  const int64_t ldab = 2 * f->kl + f->ku + 1;
  const double bytes = (double)ldab * (double)n * 8.0;
  size_t freeb = 0, totalb = 0;
  CK_CUDA(cudaMemGetInfo(&freeb, &totalb));
  if (bytes * 1.2 > (double)freeb)
    fail(CK_ERR_OUT_OF_MEMORY, "band LU storage (" + std::to_string(bytes / 1e9) + " GB) exceeds free device memory");
  f->ab.alloc(std::max<int64_t>(1, ldab * n));
  f->ipiv.alloc(std::max<int64_t>(1, n));
  f->status.alloc(1);
  CK_CUDA(cudaMemsetAsync(f->ab.p, 0, f->ab.bytes(), st));
  LUStatus s0{0, 0, -1, 0.0, INFINITY, 0};
  CK_CUDA(cudaMemcpyAsync(f->status.p, &s0, sizeof(s0), cudaMemcpyHostToDevice, st));
  BandView b = f->view();
  if (n > 0) k_band_fill<<<g, 256, 0, st>>>(view(m->a), m->a.nrows_pad, m->a.perm.p, m->at.perm.p, b);
  CK_CUDA(cudaGetLastError());
  const size_t usmem = sizeof(double) * kLUBlock * (size_t)(f->kl + 1);
  if (usmem > 227 * 1024) fail(CK_ERR_UNSUPPORTED, "band too wide for the on-chip panel update");
  CK_CUDA(cudaStreamSynchronize(st));
}

// The right-looking panel loop (lu.hpp:100-177) of S prepared factorisations at
// once: two launches per 32-column panel for the whole batch (one CTA per member
// for the panel, a member row of CTAs for the trailing update), on stream st.
static void lu_panels(ck_lu_s* const* fs, int S, double pivot_tol, cudaStream_t st) {
  std::vector<BandView> hb((size_t)S);
  std::vector<LUStatus*> hs((size_t)S);
  int64_t nmax = 0, klmax = 0, colmax = 0;
  for (int g = 0; g < S; ++g) {
    hb[g] = fs[g]->view();
    hs[g] = fs[g]->status.p;
    nmax = std::max(nmax, fs[g]->n);
    klmax = std::max(klmax, fs[g]->kl);
    colmax = std::max(colmax, fs[g]->kl + fs[g]->ku + 1);
  }
  if (nmax == 0) return;
  DBuf<BandView> db(S);
  DBuf<LUStatus*> ds(S);
  CK_CUDA(cudaMemcpyAsync(db.p, hb.data(), sizeof(BandView) * S, cudaMemcpyHostToDevice, st));
  CK_CUDA(cudaMemcpyAsync(ds.p, hs.data(), sizeof(LUStatus*) * S, cudaMemcpyHostToDevice, st));
  const size_t usmem = sizeof(double) * kLUBlock * (size_t)(klmax + 1);
  CK_CUDA(allow_max_dynamic_smem(k_gbtrf_update));
  const unsigned ublocks = (unsigned)std::min<int64_t>(148, std::max<int64_t>(1, ceil_div(colmax, 16)));
  for (int64_t j0 = 0; j0 < nmax; j0 += kLUBlock) {
    k_gbtrf_panel<<<dim3(1, (unsigned)S), 256, 0, st>>>(db.p, j0, pivot_tol, ds.p);
    if (j0 + kLUBlock < nmax) k_gbtrf_update<<<dim3(ublocks, (unsigned)S), 512, usmem, st>>>(db.p, j0, ds.p);
  }
  CK_CUDA(cudaGetLastError());
  CK_CUDA(cudaStreamSynchronize(st));
}

// Status check (singular -> error) and the solve-side data of one factorisation.
static void lu_finish(ck_lu_s* f, ck_matrix_s* m, int64_t* fail_col, double* fail_pivot) {
  cudaStream_t st = f->stream;
  const int64_t n = f->n;
  LUStatus s{};
  CK_CUDA(cudaMemcpyAsync(&s, f->status.p, sizeof(s), cudaMemcpyDeviceToHost, st));
  CK_CUDA(cudaStreamSynchronize(st));
  if (s.code != 0) {
    if (fail_col) *fail_col = s.column;
    if (fail_pivot) *fail_pivot = s.pivot;
    f->ab.reset();
    if (s.code == 5 && s.pivot == 0.0 && s.column >= 0 && s.column < n) {
      // No nonzero candidate. The reference calls this structural when no
      // unpivoted row is touched at all (lu.hpp:126); the band form does not
      // track structure, so an empty column of A is the case classified here.
      int32_t pos = 0;
      uint16_t len = 1;
      CK_CUDA(cudaMemcpy(&pos, m->at.inv.p + s.column, sizeof(int32_t), cudaMemcpyDeviceToHost));
      CK_CUDA(cudaMemcpy(&len, m->at.len.p + pos, sizeof(uint16_t), cudaMemcpyDeviceToHost));
      if (len == 0) s.code = 4;
    }
    fail(s.code == 4 ? CK_ERR_STRUCT_SINGULAR : CK_ERR_NUM_SINGULAR,
         (s.code == 4 ? std::string("structurally singular: no pivot candidate in column ")
                      : std::string("numerically singular: best pivot below threshold in column ")) +
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
  CK_CUDA(cudaStreamSynchronize(st));
}

void lu_factorize(ck_lu_s* f, ck_matrix_s* m, double pivot_tol, int64_t* fail_col,
                  double* fail_pivot) {
  lu_prepare(f, m);
  ck_lu_s* one[1] = {f};
  lu_panels(one, 1, pivot_tol, f->stream);
  lu_finish(f, m, fail_col, fail_pivot);
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
      lu_finish(fs[g], ms[g], fail_cols ? fail_cols + g : nullptr, fail_pivots ? fail_pivots + g : nullptr);
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
