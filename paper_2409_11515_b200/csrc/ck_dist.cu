// Row-block partition of one operator across ranks:
// rank p owns global rows/columns [g0, g0 + n_loc) of A and the matching
// entries of every iterate vector.
//
// Each rank uploads an *extended* local operator C_p whose index spaces are,
// in increasing global order, [left halo | own block | right halo], the own
// block padded to whole 256-row tiles:
//   * rows: the own rows of A (complete), plus the halo rows -- rows of A
//     outside the block with entries in own columns, restricted to those
//     columns (so the own columns of C_p^T are complete columns of A);
//   * columns: own columns plus the halo columns the own rows reference.
// The fused kernels (ck_adam.cu) run unchanged over the own tiles: y' = A x~
// for own rows gathers x~ at halo columns, z = A^T y' for own columns gathers
// y' at halo rows, and every row keeps the reference's summation order, so the
// sparse products are bit-identical to one device. Per half step:
//   k_apply (own tiles) -> one exchange {partials to every rank, y' halo}
//   -> combine + control (every rank) -> k_transpose (own tiles)
//   -> one exchange {partials, (x, delta) halo of the buffers the radial step
//   makes live} -> combine + radial step.
// Only the reductions change association (per-rank partials merged in rank
// order, the same on every rank), so results match one device to rounding.
//
// Two backends: NCCL (one rank per process and GPU; the whole step, NCCL calls
// included, is captured in the session's CUDA graph) and in-process (several
// ranks' sessions on one device, driven in lockstep with device copies in
// place of the collectives -- the multi-rank path exercised on one GPU).
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "ck_common.h"
#include "ck_internal.h"
#include "ck_session.h"

namespace ck {

// ------------------------------------------------------------------ NCCL
// Loaded at run time: the libnccl.so.2 already in the process (torch's) or
// the system one.
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    auto sym = [&](auto& f, const char* name) { f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name)); };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.AllGather, "ncclAllGather");
    sym(a.Send, "ncclSend");
    sym(a.Recv, "ncclRecv");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.GetErrorString, "ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllGather && a.Send && a.Recv &&
           a.GroupStart && a.GroupEnd && a.GetErrorString;
    return a;
  }();
  if (!api.ok) fail(CK_ERR_UNSUPPORTED, "libnccl.so.2 not loadable");
  return api;
}

#define CK_NCCL(x)                                                                        \
  do {                                                                                    \
    ncclResult_t r_ = (x);                                                                \
    if (r_ != ncclSuccess) fail(CK_ERR_CUDA, std::string("NCCL: ") + nccl().GetErrorString(r_)); \
  } while (0)

// ------------------------------------------------------------- halo kernels
// Two small kernels frame every exchange. The pack kernel gathers the outgoing
// halo into the send buffer and files this rank's reduction partials in its
// own slot of the gather buffer; the combine kernel (k_combine_apply /
// k_combine_transpose, ck_adam.cu) merges every rank's partials into the
// control step and scatters the received halo. Block 0 carries the scalar
// work, so a rank without halo (one rank) still launches one block.
__global__ void k_pack_y(int64_t n, int R, const int32_t* __restrict__ pos, const double* __restrict__ y,
                         double* buf, const double* __restrict__ part, double* slot, int words) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < words) slot[k] = part[k];
  if (k >= n * R) return;
  buf[k] = y[(int64_t)pos[k / R] * R + k % R];
}

// (x, delta) of the buffer the transpose control step is about to make live
// (control_tail_transpose: a gradient column moves on to nxt; every other
// column keeps cur).
__global__ void k_pack_x_next(int64_t n, int R, const int32_t* __restrict__ pos,
                              const double2* __restrict__ px, int64_t nc_pad,
                              const ColState* __restrict__ st, double2* buf,
                              const double* __restrict__ part, double* slot, int words) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < words) slot[k] = part[k];
  if (k >= n * R) return;
  const int r = (int)(k % R);
  const ColState& c = st[r];
  const int b = c.phase == PH_GRAD ? c.nxt : c.cur;
  buf[k] = px[((int64_t)b * nc_pad + pos[k / R]) * R + r];
}

static unsigned blocks_for(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + 255) / 256); }

// ------------------------------------------------------------ communication
// ss: the sessions this process drives (NCCL: exactly one). One exchange per
// half step carries both the per-rank reduction partials (an allgather, as
// point-to-point messages) and the halo of y' (x_side = false) or of the
// (x, delta) pairs (x_side = true): a single NCCL group, so every half step
// pays one communication latency.
static void pack_halo(ck_session_s* const* ss, int np, bool x_side, cudaStream_t st) {
  const int R = ss[0]->R;
  const int w = partial_words(R);
  for (int p = 0; p < np; ++p) {
    ck_session_s* s = ss[p];
    DistPart& d = *s->dist;
    const int64_t n = x_side ? d.xs_off.back() : d.ys_off.back();
    double* slot = d.gather.p + (size_t)d.rank * w;
    const unsigned blocks = blocks_for(std::max<int64_t>(n * R, w));
    if (x_side)
      k_pack_x_next<<<blocks, 256, 0, st>>>(n, R, d.xs_pos.p, s->PX.p, s->npad, s->st.p, d.xs_buf.p,
                                            d.part.p, slot, w);
    else
      k_pack_y<<<blocks, 256, 0, st>>>(n, R, d.ys_pos.p, s->y.p, d.ys_buf.p, d.part.p, slot, w);
  }
}

// Control step of every rank (all ranks merge the same gathered partials in
// rank order) fused with the scatter of the received halo.
static void combine(ck_session_s* const* ss, int np, bool x_side, cudaStream_t st) {
  for (int q = 0; q < np; ++q) {
    ck_session_s* s = ss[q];
    DistPart& d = *s->dist;
    const int64_t n = x_side ? d.xr_off.back() : d.yr_off.back();
    launch_dist_combine(s, !x_side, d.gather.p, d.nranks, n, x_side ? d.xr_pos.p : d.yr_pos.p,
                        x_side ? (const void*)d.xr_buf.p : (const void*)d.yr_buf.p, st);
  }
}

static void transfer(ck_session_s* const* ss, int np, bool x_side, cudaStream_t st) {
  const int R = ss[0]->R;
  const size_t w = (size_t)partial_words(R);
  const size_t esz = x_side ? sizeof(double2) : sizeof(double);  // per entry and column
  const DistPart& d0 = *ss[0]->dist;
  if (d0.nccl) {
    const DistPart& d = d0;
    const char* sb = x_side ? (const char*)d.xs_buf.p : (const char*)d.ys_buf.p;
    char* rb = x_side ? (char*)d.xr_buf.p : (char*)d.yr_buf.p;
    const auto& so = x_side ? d.xs_off : d.ys_off;
    const auto& ro = x_side ? d.xr_off : d.yr_off;
    const size_t words = esz / sizeof(double) * R;  // doubles per entry
    CK_NCCL(nccl().GroupStart());
    for (int q = 0; q < d.nranks; ++q) {
      if (q == d.rank) continue;
      CK_NCCL(nccl().Send(d.part.p, w, ncclDouble, q, (ncclComm_t)d.comm, st));
      CK_NCCL(nccl().Recv(d.gather.p + (size_t)q * w, w, ncclDouble, q, (ncclComm_t)d.comm, st));
      const int64_t ns = so[q + 1] - so[q], nr = ro[q + 1] - ro[q];
      if (ns) CK_NCCL(nccl().Send(sb + so[q] * esz * R, ns * words, ncclDouble, q, (ncclComm_t)d.comm, st));
      if (nr) CK_NCCL(nccl().Recv(rb + ro[q] * esz * R, nr * words, ncclDouble, q, (ncclComm_t)d.comm, st));
    }
    CK_NCCL(nccl().GroupEnd());
    return;
  }
  for (int q = 0; q < np; ++q)  // partials (a rank's own slot was filed by its pack kernel)
    for (int p = 0; p < np; ++p)
      if (p != q)
        CK_CUDA(cudaMemcpyAsync(ss[q]->dist->gather.p + (size_t)p * w, ss[p]->dist->part.p,
                                w * sizeof(double), cudaMemcpyDeviceToDevice, st));
  for (int p = 0; p < np; ++p)  // halos
    for (int q = 0; q < np; ++q) {
      const DistPart& a = *ss[p]->dist;  // sender
      DistPart& b = *ss[q]->dist;        // receiver
      const auto& so = x_side ? a.xs_off : a.ys_off;
      const auto& ro = x_side ? b.xr_off : b.yr_off;
      const int64_t ns = so[q + 1] - so[q];
      if (ns == 0) continue;
      if (ro[p + 1] - ro[p] != ns) fail(CK_ERR_LOGIC, "halo lists of two ranks disagree");
      const char* src = (x_side ? (const char*)a.xs_buf.p : (const char*)a.ys_buf.p) + so[q] * esz * R;
      char* dst = (x_side ? (char*)b.xr_buf.p : (char*)b.yr_buf.p) + ro[p] * esz * R;
      CK_CUDA(cudaMemcpyAsync(dst, src, ns * esz * R, cudaMemcpyDeviceToDevice, st));
    }
}

// One Projected-Adam iteration of every rank in ss.
static void run_step(ck_session_s* const* ss, int np, cudaStream_t st) {
  // four launches and one exchange per half step: sweep, pack, [exchange], combine
  for (int p = 0; p < np; ++p) launch_apply_only(ss[p], st);
  pack_halo(ss, np, false, st);
  transfer(ss, np, false, st);  // apply partials + y' halo
  combine(ss, np, false, st);
  for (int p = 0; p < np; ++p) launch_transpose_only(ss[p], st);
  pack_halo(ss, np, true, st);  // the buffers the control step below makes live
  transfer(ss, np, true, st);   // transpose partials + (x, delta) halo
  combine(ss, np, true, st);
  CK_CUDA(cudaGetLastError());
}

void dist_step(ck_session_s* s, cudaStream_t st) {
  if (!s->dist->nccl) fail(CK_ERR_LOGIC, "in-process partitions step as a group");
  run_step(&s, 1, st);
}

// ||(C_p x)|| over this rank's own rows, x = the internal (column-order)
// witness candidate; recorded for the cross-rank check in ck_dist_result.
double dist_op_norm(ck_session_s* s, const double* x, cudaStream_t st) {
  DistPart& d = *s->dist;
  matrix_apply_perm(s->A, x, s->tmp.p, st);
  const LoopArgs& a = s->args;
  const int64_t r0 = (int64_t)a.tile_base * kTile, r1 = (int64_t)a.tiles_A * kTile;
  d.chk_local = device_norm(s->tmp.p + r0, r1 - r0, s->A->s_red.p, st);
  return d.chk_local;
}

}  // namespace ck

using namespace ck;

// A partition group: the ranks this process drives.
struct ck_dist_s {
  int device = 0;
  bool nccl = false;
  void* comm = nullptr;
  cudaStream_t stream = nullptr;  // in-process backend: one stream for every rank
  int nranks = 1;
  std::vector<ck_matrix_s*> mats;
  std::vector<ck_session_s*> sess;
  std::vector<DistPart*> parts;
  ~ck_dist_s() {
    cudaSetDevice(device);
    cudaDeviceSynchronize();
    for (auto* s : sess) delete s;
    for (auto* p : parts) delete p;
    for (auto* m : mats) {
      cudaStream_t st = m->stream;
      delete m;
      if (st) cudaStreamDestroy(st);
    }
    if (comm) ck::nccl().CommDestroy((ncclComm_t)comm);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace ck {

ck_dist_s* dist_new() { return new ck_dist_s(); }

const ck_matrix_s* dist_part_matrix(const ck_dist_s* D, int part) {
  if (part < 0 || part >= (int)D->mats.size()) fail(CK_ERR_INVALID_ARGUMENT, "part out of range");
  return D->mats[(size_t)part];
}
void dist_free(ck_dist_s* D) { delete D; }

void dist_nccl_id(void* out128) {
  ncclUniqueId id;
  CK_NCCL(nccl().GetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, sizeof(id));
}

static DBuf<int32_t> upload_positions(const int32_t* ext_pos, int64_t n, const std::vector<int32_t>& inv) {
  DBuf<int32_t> d(std::max<int64_t>(1, n));
  std::vector<int32_t> h((size_t)n);
  for (int64_t k = 0; k < n; ++k) {
    const int32_t e = ext_pos[k];
    if (e < 0 || (size_t)e >= inv.size()) fail(CK_ERR_INVALID_ARGUMENT, "halo position out of range");
    h[k] = inv[(size_t)e];
  }
  if (n) CK_CUDA(cudaMemcpy(d.p, h.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  return d;
}

void dist_create(ck_dist_s* D, const ck_dist_part* parts, int np, int rank0, int nranks,
                 const void* nccl_id, const ck_adam_cfg* cfg, const uint64_t* seeds, int R) {
  if (R < 1 || R > kMaxCols) fail(CK_ERR_INVALID_ARGUMENT, "session columns must be 1..4");
  if (np < 1 || nranks < 1 || rank0 < 0 || rank0 + np > nranks)
    fail(CK_ERR_INVALID_ARGUMENT, "bad rank layout");
  D->nccl = nccl_id != nullptr;
  if (D->nccl && np != 1) fail(CK_ERR_INVALID_ARGUMENT, "NCCL backend: one rank per process");
  if (!D->nccl && np != nranks) fail(CK_ERR_INVALID_ARGUMENT, "in-process backend: all ranks here");
  D->nranks = nranks;
  CK_CUDA(cudaGetDevice(&D->device));
  if (D->nccl) {
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    ncclComm_t c = nullptr;
    CK_NCCL(nccl().CommInitRank(&c, nranks, id, rank0));
    D->comm = c;
  } else {
    CK_CUDA(cudaStreamCreateWithFlags(&D->stream, cudaStreamNonBlocking));
  }
  for (int p = 0; p < np; ++p) {
    const ck_dist_part& in = parts[p];
    if (in.tile0 < 0 || in.tile1 <= in.tile0) fail(CK_ERR_INVALID_ARGUMENT, "empty own tile range");
    if (in.tile1 * (int64_t)kTile > std::min(in.ext_rows, in.ext_cols) + (int64_t)kTile)
      fail(CK_ERR_INVALID_ARGUMENT, "own tiles exceed the extended operator");
    auto* M = new ck_matrix_s();
    D->mats.push_back(M);
    matrix_upload(M, in.ext_rows, in.ext_cols, in.rp, in.ci, in.va);
    auto* s = new ck_session_s();
    D->sess.push_back(s);
    session_setup_explicit(s, M, cfg, R, nullptr, 1);
    session_set_tiles(s, (int)in.tile0, (int)in.tile1);
    auto* d = new DistPart();
    D->parts.push_back(d);
    d->rank = rank0 + p;
    d->nranks = nranks;
    d->nccl = D->nccl;
    d->comm = D->comm;
    d->n_global = in.n_global;
    d->ext_global.assign(in.ext_global, in.ext_global + in.ext_cols);
    auto offs = [&](const int64_t* o) { return std::vector<int64_t>(o, o + nranks + 1); };
    d->xs_off = offs(in.xs_off);
    d->xr_off = offs(in.xr_off);
    d->ys_off = offs(in.ys_off);
    d->yr_off = offs(in.yr_off);
    std::vector<int32_t> inv_a((size_t)in.ext_rows), inv_t((size_t)in.ext_cols);
    if (in.ext_rows)
      CK_CUDA(cudaMemcpy(inv_a.data(), M->a.inv.p, sizeof(int32_t) * in.ext_rows, cudaMemcpyDeviceToHost));
    if (in.ext_cols)
      CK_CUDA(cudaMemcpy(inv_t.data(), M->at.inv.p, sizeof(int32_t) * in.ext_cols, cudaMemcpyDeviceToHost));
    d->xs_pos = upload_positions(in.xs_idx, d->xs_off.back(), inv_t);
    d->xr_pos = upload_positions(in.xr_idx, d->xr_off.back(), inv_t);
    d->ys_pos = upload_positions(in.ys_idx, d->ys_off.back(), inv_a);
    d->yr_pos = upload_positions(in.yr_idx, d->yr_off.back(), inv_a);
    d->xs_buf.alloc(std::max<int64_t>(1, d->xs_off.back() * R));
    d->xr_buf.alloc(std::max<int64_t>(1, d->xr_off.back() * R));
    d->ys_buf.alloc(std::max<int64_t>(1, d->ys_off.back() * R));
    d->yr_buf.alloc(std::max<int64_t>(1, d->yr_off.back() * R));
    d->part.alloc(partial_words(R));
    d->gather.alloc((int64_t)nranks * partial_words(R));
    d->chk.alloc(nranks);
    s->args.dist = 1;
    s->args.rank_part = d->part.p;
    s->dist = d;
  }
  for (int p = 0; p < np; ++p) D->parts[p]->group = D->sess.data();
  for (int p = 0; p < np; ++p) {
    ck_session_s* s = D->sess[p];
    if (!D->nccl) s->stream = D->stream;
    const int64_t yw = std::max(s->args.nr_pad, s->args.nc_pad) * R;
    const double own = (double)(s->args.tiles_A - s->args.tile_base) * kTile;
    const double bytes_per_step = 24.0 * (double)D->mats[p]->nnz + 100.0 * own * R;
    session_init_common(s, cfg, seeds, yw, bytes_per_step);
  }
}

void dist_run(ck_dist_s* D, uint64_t max_steps, int32_t* finished) {
  CK_CUDA(cudaSetDevice(D->device));
  if (D->nccl) {
    session_run(D->sess[0], max_steps, finished);
    return;
  }
  ck_session_s* const* ss = D->sess.data();
  const int np = (int)D->sess.size();
  ck_session_s* s0 = ss[0];
  uint64_t done = 0;
  *finished = 0;
  for (;;) {
    pull_state(s0);
    if (total_done(s0) == (int64_t)s0->R) {
      *finished = 1;
      return;
    }
    if (any_wait(s0))
      for (int p = 0; p < np; ++p) {
        pull_state(ss[p]);
        service_restarts(ss[p]);
      }
    if (max_steps && done >= max_steps) return;
    const uint64_t n = max_steps ? std::min<uint64_t>(max_steps - done, 16) : 16;
    for (uint64_t k = 0; k < n; ++k) run_step(ss, np, D->stream);
    done += n;
  }
}

double dist_time(ck_dist_s* D, uint64_t steps) {
  CK_CUDA(cudaSetDevice(D->device));
  if (D->nccl) {
    double ms = 0.0, a = 0.0, t = 0.0;
    session_time(D->sess[0], steps, 1, &ms, &a, &t);
    return ms;
  }
  // in-process ranks: the steps are replayed from a CUDA graph, so the figure is
  // device time (sweeps, pack / combine kernels, the copies standing in for the
  // exchange), not the host's launch rate
  ck_session_s* const* ss = D->sess.data();
  const int np = (int)D->sess.size();
  const uint64_t chunk = std::min<uint64_t>(steps, 10);
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  CK_CUDA(cudaStreamSynchronize(D->stream));
  CK_CUDA(cudaStreamBeginCapture(D->stream, cudaStreamCaptureModeThreadLocal));
  for (uint64_t k = 0; k < chunk; ++k) run_step(ss, np, D->stream);
  CK_CUDA(cudaStreamEndCapture(D->stream, &g));
  CK_CUDA(cudaGraphInstantiate(&ge, g, 0));
  CK_CUDA(cudaGraphDestroy(g));
  cudaEvent_t e0, e1;
  CK_CUDA(cudaEventCreate(&e0));
  CK_CUDA(cudaEventCreate(&e1));
  CK_CUDA(cudaGraphLaunch(ge, D->stream));  // warm
  CK_CUDA(cudaStreamSynchronize(D->stream));
  CK_CUDA(cudaEventRecord(e0, D->stream));
  uint64_t k = 0;
  for (; k + chunk <= steps; k += chunk) CK_CUDA(cudaGraphLaunch(ge, D->stream));
  for (; k < steps; ++k) run_step(ss, np, D->stream);
  CK_CUDA(cudaEventRecord(e1, D->stream));
  CK_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  CK_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaGraphExecDestroy(ge);
  return ms;
}

// Result of restart column `col` on local rank index `part` (witness: that
// rank's extended-order vector, ext_cols doubles); the witness norm is checked
// across all ranks.
void dist_result(ck_dist_s* D, int col, int part, ck_norm_result* res, double* witness) {
  CK_CUDA(cudaSetDevice(D->device));
  const int np = (int)D->sess.size();
  if (part < 0 || part >= np) fail(CK_ERR_INVALID_ARGUMENT, "rank index out of range");
  double total2 = 0.0;
  if (D->nccl) {
    ck_session_s* s = D->sess[0];
    DistPart& d = *s->dist;
    session_result(s, col, res, witness);
    if (res->value == 0.0) return;
    CK_CUDA(cudaMemcpyAsync(d.chk.p + d.rank, &d.chk_local, sizeof(double), cudaMemcpyHostToDevice, s->stream));
    CK_NCCL(nccl().AllGather(d.chk.p + d.rank, d.chk.p, 1, ncclDouble, (ncclComm_t)d.comm, s->stream));
    std::vector<double> h((size_t)d.nranks);
    CK_CUDA(cudaMemcpyAsync(h.data(), d.chk.p, sizeof(double) * d.nranks, cudaMemcpyDeviceToHost, s->stream));
    CK_CUDA(cudaStreamSynchronize(s->stream));
    for (double v : h) total2 += v * v;
  } else {
    for (int p = 0; p < np; ++p) {
      ck_norm_result r{};
      session_result(D->sess[p], col, &r, p == part ? witness : nullptr);
      if (p == part) *res = r;
      total2 += D->parts[p]->chk_local * D->parts[p]->chk_local;
    }
    if (res->value == 0.0) return;
  }
  const double chk = std::sqrt(total2);
  if (!(std::fabs(chk - res->value) <= 1e-12 * std::max(res->value, chk)))
    fail(CK_ERR_LOGIC, "norm estimate does not match ||Op witness||");
}

}  // namespace ck
