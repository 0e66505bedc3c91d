// Session state of the device-resident Projected-Adam loop (shared between
// ck_adam.cu, which owns the kernels, and ck_api.cu, which owns the ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <random>
#include <vector>

#include "ck_common.h"
#include "ck_lu.h"

namespace ck {

enum Phase : int32_t { PH_PRO = 0, PH_GRAD = 1, PH_APPLY = 2, PH_WAIT = 3, PH_DONE = 4 };

struct ColState {
  int32_t phase, cur, nxt, best;
  int32_t pend, mat, converged, budget;
  uint64_t t, since, t_loss, n_loss;
  double b1p, b2p, mc, vc;
  double rad, ndiv, inv_x2, inv_y2;
  double loss_min, loss, xnorm, ynorm;
  double obs_xd, obs_dn;
};

struct Header {
  int32_t needA, needT, nwait, ndone;
  uint32_t cntA, cntT;
  int32_t observe, ncols;
};

struct Params {
  double alpha, beta1, beta2, eps, rel_tol;
  uint64_t max_iter, patience;
};

struct LoopArgs {
  SellView A, AT;
  int64_t nr, nc, nr_pad, nc_pad;
  int tiles_A, tpu_A, units_A;
  int tiles_T, tpu_T, units_T;
  double2* PX;  // [3][nc_pad][R] (x, delta) pairs; three rotating iterate buffers
  double2* MV;  // [nc_pad][R]    (m, v) Adam moments
  double* y;    // [nr_pad][R]    A x~
  double* partA;
  double* partT;
  ColState* st;  // [S][R]
  Header* hdr;   // [S]
  Params prm;
  // block-diagonal batches (config 5): S members, units own tile ranges
  int S;
  const int32_t* unit_seg;
  const int32_t* unit_t0;
  const int32_t* unit_t1;
  const int32_t* seg_u0;  // [S + 1]
};

// Arguments of the inverse-operator step (ck_inverse.cu).
// Per-member arguments of the inverse step (one CTA per member; a batch of
// S members keeps S of these in device memory).
struct InvArgs {
  BandView b;
  int64_t n;
  int ring_size;
  double2* PX;      // member's [n][R] slice of buffer 0; buffer k at PX + k * pstride
  int64_t pstride;  // double2 elements per PX buffer (whole session)
  double2* MV;      // [n][R]
  double* y;        // [R][n] work vector (solve in place)
  ColState* st;     // R columns
  Header* hdr;
  Params prm;
};

}  // namespace ck

struct ck_session_s {
  using ColState = ck::ColState;
  using Header = ck::Header;
  using Params = ck::Params;
  using LoopArgs = ck::LoopArgs;
  template <class T>
  using DBuf = ck::DBuf<T>;
  ck_matrix_s* A = nullptr;
  int R = 1;
  Params prm{};
  LoopArgs args{};
  int kind = 0;              // 0: ExplicitOracle (ck_matrix), 1: InverseOracle (ck_lu)
  ck_lu_s* lu = nullptr;      // kind 1: the factors of member 0
  std::vector<ck_lu_s*> lus;  // kind 1: factors per member
  DBuf<ck::InvArgs> dargs;    // kind 1: per-member step arguments
  size_t inv_smem = 0;        // kind 1: dynamic shared memory of the step CTA
  cudaStream_t stream = nullptr;
  int device = 0;
  int64_t n = 0;            // operator dimension (columns of A)
  int64_t npad = 0;         // length of the internal vectors
  int64_t thalf = 0;        // tmp holds two halves of thalf doubles
  int S = 1;                // members (block-diagonal batch); R columns each
  std::vector<int64_t> seg_n, seg_off, seg_pad;
  DBuf<int32_t> units;
  const int32_t* perm = nullptr;  // internal position -> original index (nullptr: identity)
  DBuf<double2> PX, MV;
  DBuf<double> y, partA, partT, tmp, obs;
  DBuf<ColState> st;
  DBuf<Header> hdr;
  std::vector<std::mt19937_64> gens;
  ColState* h_st = nullptr;
  Header* h_hdr = nullptr;
  cudaGraphExec_t gexec = nullptr;
  int gsteps = 0;
  std::vector<double> hx;
  bool observe_on = false;

  ~ck_session_s() {
    if (gexec) cudaGraphExecDestroy(gexec);
    if (h_st) cudaFreeHost(h_st);
    if (h_hdr) cudaFreeHost(h_hdr);
  }
};

