// Device band LU with row partial pivoting (the factorisation behind the
// InverseOracle, lu.hpp:55-227) -- shared by ck_lu.cu (factorisation, solves)
// and ck_inverse.cu (the Projected-Adam loop on A^-1).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "ck_common.h"
#include "ck_lu_dense.cuh"

namespace ck {

// LAPACK band layout (column major): entry (i, j) of the factored matrix at
// ab[(kv + i - j) + j * ldab] with kv = kl + ku and ldab = 2*kl + ku + 1, for
// max(0, j - kv) <= i <= min(n-1, j + kl). Rows kv+1.. of column j hold the
// multipliers of elimination step j (not permuted by later interchanges);
// ipiv[j] is the row interchanged with row j at step j.
struct BandView {
  int64_t n, kl, ku, kv, ldab;
  double* ab;
  int32_t* ipiv;
  // Per 32-column block of L, the multipliers re-expressed in the block's local
  // pivot order: lb[blk][c][r] for r in [0, nb + kl) rows of the window that
  // starts at row 32*blk (see ck_lu.cu, convert_l_blocks).
  double* lb;
  int64_t lb_ld;  // rows per column of lb (= 32 + kl)
  // per block: [count, (dst, src) x count] window positions of the block's
  // composite interchange (<= 64 moved positions), 1 + 128 int32 per block
  int32_t* perm;
  double* rdiag;  // RN(1 / U(j, j)) per pivot
  // doubles of dynamic shared memory the solve CTA has for its TMA stage
  // (set by the launcher, see lu_solve_smem)
  int64_t stage_cap;
  // runs shorter than this many rows are read directly instead of staged
  int64_t stage_min;
  // ---- factorisation only (ck_lu.cu) -------------------------------------
  // Touch keys: the reference's `touched` order of each working column
  // (lu.hpp:88-110), which decides pivot ties and structural singularity.
  // Entry (i, j) at key[(kv + i - j) + (j % kw) * ldab]: a window of kw
  // columns (kw = kv + 64 covers every column a panel step can reach).
  //   kKeyUntouched  never touched;   kKeyOriginal  an entry of A;
  //   1 + (s - (j - kv)) * (kl + 1) + rank   filled by step s, where rank is the
  //   row's position in the stored multipliers of column s (lcols[s] order).
  // Once column j is factored, its L rows hold their rank (kKeyUntouched when
  // the multiplier is not stored).
  uint32_t* key;
  int64_t kw;
  const uint32_t* abit;  // structure of A, one bit per band position (ab's indexing)
  int32_t* orig;         // orig[i]: original row now at position i
  int32_t* rowperm;      // rowperm[j]: original row pivoted at step j (LUFactors::row_perm)
};

constexpr uint32_t kKeyUntouched = 0xFFFFFFFFu;
constexpr uint32_t kKeyOriginal = 0xFFFFFFFEu;

struct LUStatus {
  int32_t code;  // 0 ok, 4 structurally singular, 5 numerically singular (ck_status values)
  int32_t _pad;
  int64_t column;
  double pivot;
  double pivot_min;
  int64_t ju;  // last column touched by the current panel's interchanges
};

constexpr int kLUBlock = 32;  // panel width / solve block
constexpr int64_t kLUStageMinRows = 129;  // runs of <= 128 rows unstaged; lu_stage_min (ck_lu.cu)
int64_t lu_stage_min();
// bands at least this wide (kl + ku rows above the diagonal of U) sweep on a
// cluster of CTAs per system (ck_lu_sweeps.cuh, Clu)
constexpr int64_t kLUClusterMinRows = 256;

// Raise a kernel's dynamic shared-memory ceiling to everything the SM has
// left beside its static shared memory. Always the same value, so concurrent
// host threads (factorisations of an ensemble) never race a smaller ceiling
// in under each other's launches.
template <class K>
inline cudaError_t allow_max_dynamic_smem(K* kernel) {
  cudaFuncAttributes fa{};
  cudaError_t e = cudaFuncGetAttributes(&fa, kernel);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(227 * 1024 - fa.sharedSizeBytes));
}

// Dynamic shared memory of a solve CTA, in doubles: R rings of ring_size,
// R*32 dot scratch, then the TMA stage (16-byte aligned, stage_cap doubles).
__host__ __device__ __forceinline__ int64_t stage_offset(int R, int ring_size) {
  return (int64_t)R * ring_size + (int64_t)R * kLUBlock;
}

}  // namespace ck

struct ck_lu_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int64_t n = 0, kl = 0, ku = 0;
  double pivot_min = 0.0;
  ck::DBuf<double> ab, lb, rdiag;
  ck::DBuf<int32_t> ipiv, bperm, rowperm;
  // factorisation-time state (freed by lu_finish)
  ck::DBuf<uint32_t> key, abit;
  ck::DBuf<int32_t> orig;
  ck::DBuf<ck::LUStatus> status;
  ck::DBuf<double> work;  // solve scratch
  // dense-block sweeps of narrow bands (ck_lu_dense.cuh), built by lu_finish
  bool dense_ok = false;
  double dense_growth = 0.0;  // max over blocks of || |Hinv| |H| ||_inf
  ck::DBuf<double> dense_cf;  // clf | clt | cub | cut
  ck::DBuf<uint8_t> dense_perm;  // pinv | psrc
  ck::DenseView dense_view() const {
    const int nb = (int)((n + ck::kLUBlock - 1) / ck::kLUBlock);
    const int wl = ck::kLUBlock + (int)kl, wu = ck::kLUBlock + (int)(kl + ku);
    const double* c = dense_cf.p;
    const int64_t sl = (int64_t)nb * 32 * wl, su = (int64_t)nb * 32 * wu;
    return ck::DenseView{n, nb, (int)kl, (int)(kl + ku), wl, wu, c, c + sl, c + 2 * sl, c + 2 * sl + su,
                         dense_perm.p, dense_perm.p + (int64_t)nb * wl};
  }
  // CSR factors in the reference's LUFactors shape (built on request: lu_build_csr)
  bool csr_built = false;
  int64_t nnz_l = 0, nnz_u = 0;
  ck::DBuf<int64_t> l_rp, u_rp;
  ck::DBuf<int32_t> l_ci, u_ci;
  ck::DBuf<double> l_va, u_va;
  ck_lu_s() = default;
  ck_lu_s(const ck_lu_s&) = delete;
  ck_lu_s& operator=(const ck_lu_s&) = delete;
  ~ck_lu_s() {
    if (own_stream && stream) {
      cudaStreamSynchronize(stream);
      cudaStreamDestroy(stream);
    }
  }
  ck::BandView view() {
    return ck::BandView{n, kl, ku, kl + ku, 2 * kl + ku + 1, ab.p, ipiv.p, lb.p,
                        ck::kLUBlock + kl, bperm.p, rdiag.p, 0, 0,
                        key.p, kl + ku + 64, abit.p, orig.p, rowperm.p};
  }
};
