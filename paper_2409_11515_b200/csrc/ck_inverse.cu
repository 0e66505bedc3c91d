// Projected Adam on Op = A^{-1} (InverseOracle, condest.hpp:109-152) through the
// device band LU (ck_lu.cu). One CTA owns the whole iteration -- the solves are
// a single dependency chain each -- and one launch is one loop trip:
//
//   x~ = x - (delta - r x)          ||x~|| (double-double)
//   y' = U^{-1} L^{-1} P x~         ||y'|| (scaled sum of squares)   -> control
//   z  = P^T L^{-T} U^{-T} y'       (grad_inverse, :112-123)
//   Adam / projection on (x, delta), (m, v); r = x.delta             -> control
//
// State layout and control are those of the explicit path (ck_adam.cu), so the
// host session, restarts, best tracking and observer mode are shared.
// Two step kernels: k_inv_step (substitution sweeps, ck_lu_sweeps.cuh; any band,
// 1..4 columns, optional cluster split) and k_inv_step_dense (narrow bands, one
// column: dense-block sweeps, ck_lu_dense.cuh).
#include <cmath>
#include <cooperative_groups.h>
#include <cstdlib>
#include <algorithm>

#include "ck_common.h"
#include "ck_device.cuh"
#include "ck_internal.h"
#include "ck_control.cuh"
#include "ck_lu.h"
#include "ck_lu_sweeps.cuh"
#include "ck_session.h"

namespace ck {

__device__ __forceinline__ double xtilde_inv(double2 p, double rad) {
  return __dsub_rn(p.x, __dsub_rn(p.y, __dmul_rn(rad, p.x)));
}

// One CTA per member: blockIdx.x selects the member's arguments. half: 0 the
// whole step, 1 the apply half only, 2 the transpose half only (observer).
// CLU: one cluster per member (launched with cluster dims a.cl); rank 0 runs the
// step, the other ranks only help with the sweeps (helper_solve).
template <int R, bool CLU>
__global__ void __launch_bounds__(1024) k_inv_step(const InvArgs* __restrict__ args, int half) {
  const unsigned crank = CLU ? cooperative_groups::this_cluster().block_rank() : 0u;
  const unsigned csize = CLU ? cooperative_groups::this_cluster().num_blocks() : 1u;
  const InvArgs& a = args[blockIdx.x / csize];
  extern __shared__ double smem[];
  Clu C{(int)csize, (int)crank, smem + a.cl_tsum_off, a.cl_ts, smem + a.cl_dpart_off, smem};
  if (CLU && crank > 0) {
    bool any = false;
    for (int r = 0; r < R; ++r) {
      const int ph = a.st[r].phase;
      any |= ph == PH_PRO || ph == PH_APPLY;
    }
    if (any && half != 2) helper_solve<R>(a.b, smem, a.ring_size, false, C);
    clu_sync();  // the leader's control step is done
    bool anyg = false;
    for (int r = 0; r < R; ++r) anyg |= __ldcg(&a.st[r].phase) == PH_GRAD;
    if (anyg && half != 1) helper_solve<R>(a.b, smem, a.ring_size, true, C);
    clu_sync();
    return;
  }
  __shared__ double s_h[32], s_l[32];
  __shared__ int s_e[32], s_f[32];
  __shared__ double s_res[R][4];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t n = a.n;
  double* ys[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) ys[r] = a.y + (int64_t)(r < R ? r : 0) * n;

  // ---------------- apply half: y' = A^{-1} x~ and the control step
  bool act[R], pro[R];
  double rad[R];
  const double2* xc[R];
  bool any = false;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int ph = a.st[r].phase;
    act[r] = ph == PH_PRO || ph == PH_APPLY;
    pro[r] = ph == PH_PRO;
    rad[r] = pro[r] ? 0.0 : a.st[r].rad;
    xc[r] = a.PX + a.st[r].cur * a.pstride + r;  // element i at xc[r][i * R]
    any |= act[r];
  }
  if (any && half != 2) {
    DD dd[R];
    ES dn[R];
    double xd[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      dd[r] = dd_zero();
      dn[r] = es_zero();
      xd[r] = 0.0;
    }
    for (int64_t i = tid; i < n; i += nt) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double2 p = xc[r][i * R];
        const double xt = xtilde_inv(p, rad[r]);
        ys[r][i] = xt;
        if (act[r]) {
          dd_add_sq(dd[r], xt);
          if (!pro[r]) {
            const double dp = __dsub_rn(p.y, __dmul_rn(rad[r], p.x));
            xd[r] = __fma_rn(p.x, dp, xd[r]);
            es_add(dn[r], dp);
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      DD d = block_dd(dd[r], s_h, s_l);
      double x2 = block_sum(xd[r], s_h);
      ES e2 = block_es(dn[r], s_h, s_e, s_f);
      if (tid == 0) {
        s_res[r][0] = sqrt(__dadd_rn(d.hi, d.lo));
        s_res[r][2] = x2;
        s_res[r][3] = es_norm(e2);
      }
    }
    __syncthreads();
    inv_solve<R, CLU>(a.b, ys, smem, a.ring_size, false, C);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
      ES e = es_zero();
      for (int64_t i = tid; i < n; i += nt) es_add(e, ys[r][i]);
      e = block_es(e, s_h, s_e, s_f);
      if (tid == 0) s_res[r][1] = es_norm(e);
    }
    if (tid == 0) {
      for (int r = 0; r < R; ++r) {
        ColState* s = a.st + r;
        const int ph = s->phase;
        if (ph == PH_PRO || ph == PH_APPLY) {
          if (ph == PH_APPLY) {
            s->obs_xd = s_res[r][2];
            s->obs_dn = s_res[r][3];
          }
          control_apply(s, &a.prm, s_res[r][0], s_res[r][1], -1);
        }
      }
    }
    __syncthreads();
  }
  if (CLU) {
    __threadfence();
    clu_sync();  // the helpers read the control state next
  }

  // ---------------- transpose half: z = A^{-T} y', Adam, r = x.delta
  bool grad[R], mat[R];
  double ndiv[R], ix2[R], iy2[R], mc[R], vc[R];
  double2* xn_out[R];
  bool anyg = false;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const ColState& s = a.st[r];
    grad[r] = s.phase == PH_GRAD;
    mat[r] = s.mat != 0;
    rad[r] = s.rad;
    ndiv[r] = s.ndiv;
    ix2[r] = s.inv_x2;
    iy2[r] = s.inv_y2;
    mc[r] = s.mc;
    vc[r] = s.vc;
    xc[r] = a.PX + s.cur * a.pstride + r;
    xn_out[r] = a.PX + (mat[r] ? s.nxt : s.cur) * a.pstride + r;
    anyg |= grad[r];
  }
  if (anyg && half != 1) {
    inv_solve<R, CLU>(a.b, ys, smem, a.ring_size, true, C);
    __syncthreads();
    const Params& p = a.prm;
    const double om1 = 1.0 - p.beta1, om2 = 1.0 - p.beta2;
    double dot[R];
#pragma unroll
    for (int r = 0; r < R; ++r) dot[r] = 0.0;
    for (int64_t j = tid; j < n; j += nt) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (!grad[r]) continue;
        const int64_t e = j * R + r;
        const double2 px = xc[r][j * R];
        const double xn = mat[r] ? __ddiv_rn(xtilde_inv(px, rad[r]), ndiv[r]) : px.x;
        const double zz = __ddiv_rn(ys[r][j], ndiv[r]);
        const double g = __dsub_rn(__dmul_rn(xn, ix2[r]), __dmul_rn(zz, iy2[r]));
        const double2 mv = a.MV[e];
        const double mm = __dadd_rn(__dmul_rn(p.beta1, mv.x), __dmul_rn(om1, g));
        const double vv = __dadd_rn(__dmul_rn(p.beta2, mv.y), __dmul_rn(__dmul_rn(om2, g), g));
        const double d = __ddiv_rn(__dmul_rn(p.alpha, __dmul_rn(mm, mc[r])),
                                   __dadd_rn(__dsqrt_rn(__dmul_rn(vv, vc[r])), p.eps));
        a.MV[e] = make_double2(mm, vv);
        xn_out[r][j * R] = make_double2(xn, d);
        dot[r] = __fma_rn(xn, d, dot[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double s = block_sum(dot[r], s_h);
      if (tid == 0) s_res[r][0] = s;
    }
    __syncthreads();
    if (tid == 0) {
      for (int r = 0; r < R; ++r) {
        ColState* s = a.st + r;
        if (s->phase == PH_GRAD) {
          s->rad = s_res[r][0];
          if (s->mat) {
            s->cur = s->nxt;
            s->pend = 0;
          }
          s->phase = PH_APPLY;
        }
      }
    }
  }
  if (tid == 0) {
    int nwait = 0, ndone = 0;
    for (int r = 0; r < R; ++r) {
      nwait += a.st[r].phase == PH_WAIT;
      ndone += a.st[r].phase == PH_DONE;
    }
    a.hdr->nwait = nwait;
    a.hdr->ndone = ndone;
    a.hdr->needA = 1;
  }
  if (CLU) clu_sync();  // no rank leaves while another may still touch its shared memory
}

// The same loop trip on the dense-block sweeps (narrow bands, ck_lu_dense.cuh):
// one column per system, kDenseThreads threads.
__global__ void __launch_bounds__(kDenseThreads, 1) k_inv_step_dense(const InvArgs* __restrict__ args, int half,
                                                                     unsigned dyn_bytes) {
  const InvArgs& a = args[blockIdx.x];
  __shared__ double smem[3 * kDenseThreads];
  extern __shared__ __align__(16) double dyn[];
  DenseRing ring = dense_ring(a.dv, dyn, dyn_bytes);
  __shared__ double s_h[32], s_l[32];
  __shared__ int s_e[32], s_f[32];
  __shared__ double s_res[4];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t n = a.n;
  double* ys = a.y;
  ColState* s = a.st;

  // ---------------- apply half: y' = A^{-1} x~ and the control step
  const int ph = s->phase;
  if ((ph == PH_PRO || ph == PH_APPLY) && half != 2) {
    const bool pro = ph == PH_PRO;
    const double rad = pro ? 0.0 : s->rad;
    const double2* xc = a.PX + s->cur * a.pstride;
    DD dd = dd_zero();
    ES dn = es_zero();
    double xd = 0.0;
    for (int64_t i = tid; i < n; i += nt) {
      const double2 p = xc[i];
      const double xt = xtilde_inv(p, rad);
      ys[i] = xt;
      dd_add_sq(dd, xt);
      if (!pro) {
        const double dp = __dsub_rn(p.y, __dmul_rn(rad, p.x));
        xd = __fma_rn(p.x, dp, xd);
        es_add(dn, dp);
      }
    }
    dd = block_dd(dd, s_h, s_l);
    const double x2 = block_sum(xd, s_h);
    const ES e2 = block_es(dn, s_h, s_e, s_f);
    if (tid == 0) {
      s_res[0] = sqrt(__dadd_rn(dd.hi, dd.lo));
      s_res[2] = x2;
      s_res[3] = es_norm(e2);
    }
    __syncthreads();
    dense_solve(a.dv, ys, smem, ring, false);
    ES e = es_zero();
    for (int64_t i = tid; i < n; i += nt) es_add(e, ys[i]);
    e = block_es(e, s_h, s_e, s_f);
    if (tid == 0) {
      s_res[1] = es_norm(e);
      if (ph == PH_APPLY) {
        s->obs_xd = s_res[2];
        s->obs_dn = s_res[3];
      }
      control_apply(s, &a.prm, s_res[0], s_res[1], -1);
    }
    __syncthreads();
  }

  // ---------------- transpose half: z = A^{-T} y', Adam, r = x.delta
  if (s->phase == PH_GRAD && half != 1) {
    const bool mat = s->mat != 0;
    const double rad = s->rad, ndiv = s->ndiv, ix2 = s->inv_x2, iy2 = s->inv_y2, mc = s->mc, vc = s->vc;
    const double2* xc = a.PX + s->cur * a.pstride;
    double2* xn_out = a.PX + (mat ? s->nxt : s->cur) * a.pstride;
    __syncthreads();  // every thread has read the control state
    dense_solve(a.dv, ys, smem, ring, true);
    const Params& p = a.prm;
    const double om1 = 1.0 - p.beta1, om2 = 1.0 - p.beta2;
    double dot = 0.0;
    for (int64_t j = tid; j < n; j += nt) {
      const double2 px = xc[j];
      const double xn = mat ? __ddiv_rn(xtilde_inv(px, rad), ndiv) : px.x;
      const double zz = __ddiv_rn(ys[j], ndiv);
      const double g = __dsub_rn(__dmul_rn(xn, ix2), __dmul_rn(zz, iy2));
      const double2 mv = a.MV[j];
      const double mm = __dadd_rn(__dmul_rn(p.beta1, mv.x), __dmul_rn(om1, g));
      const double vv = __dadd_rn(__dmul_rn(p.beta2, mv.y), __dmul_rn(__dmul_rn(om2, g), g));
      const double d = __ddiv_rn(__dmul_rn(p.alpha, __dmul_rn(mm, mc)),
                                 __dadd_rn(__dsqrt_rn(__dmul_rn(vv, vc)), p.eps));
      a.MV[j] = make_double2(mm, vv);
      xn_out[j] = make_double2(xn, d);
      dot = __fma_rn(xn, d, dot);
    }
    const double sdot = block_sum(dot, s_h);
    if (tid == 0) {
      s->rad = sdot;
      if (s->mat) {
        s->cur = s->nxt;
        s->pend = 0;
      }
      s->phase = PH_APPLY;
    }
  }
  if (tid == 0) {
    a.hdr->nwait = s->phase == PH_WAIT;
    a.hdr->ndone = s->phase == PH_DONE;
    a.hdr->needA = 1;
  }
}

// dyn: dynamic shared memory of the block ring (dense_dyn_smem of the widest member)
void launch_inv_step_dense(const InvArgs* args, int S, int half, size_t dyn, cudaStream_t st) {
  k_inv_step_dense<<<S, kDenseThreads, dyn, st>>>(args, half, (unsigned)dyn);
}

void prepare_inv_step_dense(size_t dyn) {
  CK_CUDA(cudaFuncSetAttribute(k_inv_step_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
}

void prepare_inv_step(size_t smem, int R) {
  switch (R) {
    case 1:
      CK_CUDA(allow_max_dynamic_smem(k_inv_step<1, false>));
      CK_CUDA(allow_max_dynamic_smem(k_inv_step<1, true>));
      break;
    case 2:
      CK_CUDA(allow_max_dynamic_smem(k_inv_step<2, false>));
      CK_CUDA(allow_max_dynamic_smem(k_inv_step<2, true>));
      break;
    case 3:
      CK_CUDA(allow_max_dynamic_smem(k_inv_step<3, false>));
      CK_CUDA(allow_max_dynamic_smem(k_inv_step<3, true>));
      break;
    default:
      CK_CUDA(allow_max_dynamic_smem(k_inv_step<4, false>));
      CK_CUDA(allow_max_dynamic_smem(k_inv_step<4, true>));
      break;
  }
}

template <int R>
static void launch_cluster(const InvArgs* args, int S, int cl, size_t smem, int half, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(S * cl));
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK_CUDA(cudaLaunchKernelEx(&cfg, k_inv_step<R, true>, args, half));
}

// S members, one CTA (cl == 1) or one cluster of cl CTAs each, smem bytes of
// dynamic shared memory per CTA.
void launch_inv_step(const InvArgs* args, int S, int R, size_t smem, int half, cudaStream_t st, int cl) {
  if (cl > 1) {
    switch (R) {
      case 1: launch_cluster<1>(args, S, cl, smem, half, st); break;
      case 2: launch_cluster<2>(args, S, cl, smem, half, st); break;
      case 3: launch_cluster<3>(args, S, cl, smem, half, st); break;
      case 4: launch_cluster<4>(args, S, cl, smem, half, st); break;
      default: fail(CK_ERR_INVALID_ARGUMENT, "1..4 columns");
    }
    return;
  }
  switch (R) {
#define CK_INV_CASE(RR)                                                                        \
  case RR:                                                                                     \
    k_inv_step<RR, false><<<S, 1024, smem, st>>>(args, half);                                  \
    break;
    CK_INV_CASE(1)
    CK_INV_CASE(2)
    CK_INV_CASE(3)
    CK_INV_CASE(4)
#undef CK_INV_CASE
    default: fail(CK_ERR_INVALID_ARGUMENT, "1..4 columns");
  }
}

// Cluster size for the sweeps of S systems of band b (measured,
// scripts/check_cluster.py): 8 CTAs per system from kl + ku >= 256 (config-5
// member 74 -> 54 ms per inverse iteration), 12 from kl + ku >= 1024 (config 2
// 358 -> 124 ms; 134 with 8, 125 with 16), when the clusters fit the chip;
// else 1. CK_LU_CLUSTER=1 disables, =2..16 forces a size.
static bool cluster_fits(int cl, int S, int R, size_t smem) {
  prepare_inv_step(smem, R);
  if (cl > 8) {  // non-portable cluster sizes need the opt-in
    switch (R) {
      case 1: cudaFuncSetAttribute(k_inv_step<1, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); break;
      case 2: cudaFuncSetAttribute(k_inv_step<2, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); break;
      case 3: cudaFuncSetAttribute(k_inv_step<3, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); break;
      default: cudaFuncSetAttribute(k_inv_step<4, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); break;
    }
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(S * cl));
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  cudaError_t e = cudaErrorInvalidValue;
  switch (R) {
    case 1: e = cudaOccupancyMaxActiveClusters(&nclusters, k_inv_step<1, true>, &cfg); break;
    case 2: e = cudaOccupancyMaxActiveClusters(&nclusters, k_inv_step<2, true>, &cfg); break;
    case 3: e = cudaOccupancyMaxActiveClusters(&nclusters, k_inv_step<3, true>, &cfg); break;
    default: e = cudaOccupancyMaxActiveClusters(&nclusters, k_inv_step<4, true>, &cfg); break;
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return nclusters >= 1;
}

bool inv_cluster_fits(int cl, int S, int R, size_t smem) { return cluster_fits(cl, S, R, smem); }

}  // namespace ck

#ifdef CK_SWEEP_PROF
// Profiling build only: phase cycles of the sweeps inside the inverse step
// (this translation unit's copy of the counters; the leader CTA's thread 0).
extern "C" int ck_debug_sweep_prof_inv(unsigned long long* out32, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out32, ck::g_sweep_prof, sizeof(unsigned long long) * 32);
  if (reset) {
    unsigned long long z[32] = {};
    cudaMemcpyToSymbol(ck::g_sweep_prof, z, sizeof(z));
  }
  return 0;
}
#endif
