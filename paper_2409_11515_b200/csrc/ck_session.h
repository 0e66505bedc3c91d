// Session state of the device-resident Projected-Adam loop (shared between
// ck_adam.cu, which owns the kernels, and ck_api.cu, which owns the ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <random>
#include <vector>

#include "ck_common.h"
#include "ck_lu.h"

struct ck_session_s;

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
  double2* PX;  // [nbuf][nc_pad][R] (x, delta) pairs; nbuf = R + 2 rotating iterate buffers
  int nbuf;
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
  const int32_t* seg_t0;  // [S + 1] first tile of each member
  // every entry's column lies in the tile before, of, or after its row (A and
  // A^T, banded members): the sweeps gather from a sliding shared-memory window
  int win;
  // row-block partition (ck_dist.cu): the last CTA publishes this rank's
  // merged partials in rank_part instead of running the control step
  int dist;
  double* rank_part;
  int tile_base;  // S == 1: first own tile (a partition rank's local block)
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
  // cluster split of the sweeps (cl > 1, ck_lu_sweeps.cuh Clu): offsets in
  // doubles into the dynamic shared memory of the leader's tail sums [R][cl_ts]
  // and dot partials [cl][R][32]
  int cl;
  int64_t cl_tsum_off, cl_ts, cl_dpart_off;
  // narrow bands: composite blocks of the dense sweeps (ck_lu_dense.cuh)
  DenseView dv;
};

// Row-block partition rank (ck_dist.cu): this rank owns global rows/columns
// [g0, g0 + n_loc), the fused kernels run over its own tiles and exchange
// halos and per-rank partials with the other ranks every half step.
struct DistPart {
  int rank = 0, nranks = 1;
  bool nccl = false;
  void* comm = nullptr;             // ncclComm_t (nccl backend)
  ck_session_s* const* group = nullptr;  // in-process backend: every rank's session
  int64_t n_global = 0;
  std::vector<int64_t> ext_global;  // extended column position -> global index (-1: padding)
  std::vector<int64_t> xs_off, xr_off, ys_off, yr_off;  // [nranks + 1] per-peer offsets
  DBuf<int32_t> xs_pos, xr_pos, ys_pos, yr_pos;         // permuted positions
  DBuf<double2> xs_buf, xr_buf;                         // [count][R]
  DBuf<double> ys_buf, yr_buf;                          // [count][R]
  DBuf<double> part, gather;  // [R*(kPA+1)] this rank, [nranks][R*(kPA+1)] gathered
  DBuf<double> chk;           // witness-norm exchange
  double chk_local = 0.0;     // ||(A x_min) on this rank's rows||
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
  int inv_cl = 1;             // kind 1: CTAs per system (cluster split of the sweeps)
  bool inv_dense = false;     // kind 1: dense-block sweeps (narrow bands, one column per system)
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
  ck::PinnedBuf<double> hx;  // start-vector staging (original order)
  bool observe_on = false;
  ck::DistPart* dist = nullptr;  // owned by the ck_dist group

  ~ck_session_s() {
    if (gexec) cudaGraphExecDestroy(gexec);
    if (h_st) cudaFreeHost(h_st);
    if (h_hdr) cudaFreeHost(h_hdr);
  }
};

// Session internals shared by ck_adam.cu (single device, batches, inverse)
// and ck_dist.cu (row-block partitions).
namespace ck {
void launch_apply_only(ck_session_s* s, cudaStream_t st);
void launch_transpose_only(ck_session_s* s, cudaStream_t st);
void launch_step(ck_session_s* s, cudaStream_t st);
void pull_state(ck_session_s* s);
void push_state(ck_session_s* s);
int64_t total_done(const ck_session_s* s);
bool any_wait(const ck_session_s* s);
double2* col_buf(ck_session_s* s, int b, int c);
void to_host(ck_session_s* s, int g, const double* src, double* host, cudaStream_t st);
void load_start(ck_session_s* s, int g, int c, int b, const double* x);
void service_restarts(ck_session_s* s);
void build_graph(ck_session_s* s, int steps);
void session_init_common(ck_session_s* s, const ck_adam_cfg* cfg, const uint64_t* seeds,
                         int64_t ywords, double bytes_per_step);
void session_setup_explicit(ck_session_s* s, ck_matrix_s* A, const ck_adam_cfg* cfg, int R,
                            const int64_t* seg_n, int S);
void session_result(ck_session_s* s, int k, ck_norm_result* res, double* witness);
void session_run(ck_session_s* s, uint64_t max_steps, int32_t* finished);
void session_time(ck_session_s* s, uint64_t steps, int32_t mode, double* ms_total,
                  double* ms_apply, double* ms_transpose);
void session_set_tiles(ck_session_s* s, int t0, int t1);
void launch_dist_combine(ck_session_s* s, bool apply, const double* gathered, int nranks, int64_t n,
                         const int32_t* pos, const void* buf, cudaStream_t st);
int partial_words(int R);
void dist_step(ck_session_s* s, cudaStream_t st);
double dist_op_norm(ck_session_s* s, const double* xbest_internal, cudaStream_t st);
}  // namespace ck

struct ck_dist_s;
namespace ck {
void dist_nccl_id(void* out128);
ck_dist_s* dist_new();
void dist_free(ck_dist_s* D);
void dist_create(ck_dist_s* D, const ck_dist_part* parts, int np, int rank0, int nranks,
                 const void* nccl_id, const ck_adam_cfg* cfg, const uint64_t* seeds, int R);
void dist_run(ck_dist_s* D, uint64_t max_steps, int32_t* finished);
double dist_time(ck_dist_s* D, uint64_t steps);
const ck_matrix_s* dist_part_matrix(const ck_dist_s* D, int part);
void dist_result(ck_dist_s* D, int col, int part, ck_norm_result* res, double* witness);
}  // namespace ck
