// Device-resident Projected Adam (condest.hpp:184-297) for the explicit
// operator (ExplicitOracle, condest.hpp:125-135).
//
// One loop trip ("step") is two kernels over HBM-resident state:
//
//   k_apply<R>      x~ = x - (delta - r x)          (tangent step, :231-240)
//                   y' = A x~                        (sliced-ELL SpMV; the loss at
//                                                     x_{t+1} = x~/||x~||, :249-251)
//                   reduce ||x~|| (double-double; the compensated norm, :241)
//                   and ||y'|| (one-pass scaled sum of squares, two_norm)
//                   -> last CTA: loss, patience, best-tracking, next-iteration
//                      scalars (:221-224, :257-275)
//   k_transpose<R>  x_{t+1} = x~/||x~|| materialised into a free buffer,
//                   z = A^T y' / ||x~||              (grad, :96-107)
//                   g, m, v, delta (Adam, :225-229); reduce r = x.delta (:231)
//                   -> last CTA: radial scalar for the next k_apply.
//
// A x_{t+1} is computed once per iteration and serves both the loss of
// iteration t and the gradient of iteration t+1 (the reference evaluates it
// twice on bitwise-identical input). The best iterate is tracked by rotating
// R + 2 iterate buffers instead of copying x_min (:264-267). R independent runs
// (restarts, :301-312) share one sweep over the matrix as columns of a
// multi-vector; each column's arithmetic is independent of R. The columns
// rotate their buffers in lockstep (shared_cur / pick_shared_nxt), so a row's R
// (x, delta) pairs are contiguous. Banded ensembles (config 5) sweep from a
// sliding shared-memory window of x~ / y' (WIN).
//
// Layout: (x, delta) and (m, v) are stored as double2 pairs, so the SpMV gather
// of x~ is one 16-byte load and the Adam update moves 16-byte vectors.
//
// Per-column control state lives on the device; the host only services
// degenerate-direction restarts (which need the reference's mt19937_64 stream,
// :199-219) at chunk boundaries.
#include <cmath>
#include <cstring>
#include <exception>
#include <memory>
#include <random>
#include <thread>
#include <vector>

#include "ck_common.h"
#include "ck_control.cuh"
#include "ck_device.cuh"
#include "ck_internal.h"
#include "ck_session.h"

namespace ck {

constexpr int kPA = 9;  // per-column partials of k_apply
constexpr int kPT = 1;  // per-column partials of k_transpose

// Resident CTAs per SM the fused kernels are compiled for (register budget),
// hence their one-wave grid sizes. Fixed constants: the reduction tree -- and
// every result bit -- is the same on every device.
template <int R>
struct Occ {
  // measured optima (config 4 and config 5, scripts/ab_restarts.py): R = 1 and
  // R = 3 want the full 4 CTAs; R = 2 apply 3; R = 4 apply is latency-bound at
  // 2 (more CTAs spill); every transpose runs 4 CTAs
  static constexpr int apply = R == 1 || R == 3 ? 4 : R == 2 ? 3 : 2;
  static constexpr int transpose = 4;
};

// Entries per matrix chunk of the R-column kernels (their values and columns
// are loaded before any use); measured per R.
template <int R>
struct Tune {
  static constexpr int apply_u = R == 1 ? 8 : 4;
  static constexpr int transpose_u = R <= 2 ? 8 : 4;
};

// The window kernels (banded ensembles) hold no gathered operands in
// registers, so their chunks are wider (config 5, scripts/ab_win.sh).
template <int R>
struct WinTune {
  static constexpr int apply_u = 8;
  static constexpr int apply_occ = R == 1 ? 4 : R == 4 ? 2 : 3;
  static constexpr int transpose_u = R == 4 ? 8 : Tune<R>::transpose_u;
  static constexpr int transpose_occ = R == 4 ? 3 : Occ<R>::transpose;
};

// Window ring of the banded-ensemble sweeps: element (ring position q in
// [0, 4 * kTile), column r). Column pairs form planes of 16-byte slots, so the
// gather of a row's pair is one 16-byte read whose 8 lanes per wavefront spread
// over all 8 slots of the bank row (a [q][R] layout with R = 4 reaches 4).
template <int R>
__device__ __forceinline__ int win_idx(int q, int r) {
  if constexpr (R % 2 == 0)
    return ((r >> 1) * 4 * kTile + q) * 2 + (r & 1);
  else
    return q * R + r;
}

// Work assignment of CTA `unit`. One operator (S == 1): the tiles are dealt
// round-robin over the grid, so at any moment the resident CTAs sweep one
// contiguous window of the matrix and the stencil neighbours of the gathered
// vectors stay in L2. A block-diagonal batch (S > 1, config 5): each unit owns
// a contiguous tile range inside one member.
__device__ __forceinline__ void unit_range(const LoopArgs& a, int unit, int tiles, int& seg,
                                           int& t0, int& tend, int& stride, int& u0, int& u1) {
  if (a.S == 1) {
    seg = 0;
    t0 = a.tile_base + unit;
    tend = tiles;
    stride = gridDim.x;
    u0 = 0;
    u1 = gridDim.x;
  } else {
    seg = a.unit_seg[unit];
    t0 = a.unit_t0[unit];
    tend = a.unit_t1[unit];
    stride = 1;
    u0 = a.seg_u0[seg];
    u1 = a.seg_u0[seg + 1];
  }
}

// x~ from a stored (x, delta) pair: x - (delta - r x)  (:232, :240)
__device__ __forceinline__ double xtilde(double2 p, double rad) {
  return __dsub_rn(p.x, __dsub_rn(p.y, __dmul_rn(rad, p.x)));
}

// Lockstep buffer rotation. Every active column of an operator reads its
// (x, delta) pairs from the same iterate buffer (cur) and writes the next pairs
// to the same buffer (nxt), so a row's R pairs are one contiguous R*16-byte
// load. A column's best iterate stays behind in whatever buffer it was written
// to (ColState::best, per column); with R + 2 buffers there is always one that
// is neither cur nor any column's best.
template <int R>
__device__ __forceinline__ int shared_cur(const ColState* sts) {
  int cur = 0;
  for (int r = 0; r < R; ++r) {
    const int ph = sts[r].phase;
    if (ph == PH_PRO || ph == PH_APPLY || ph == PH_GRAD) cur = sts[r].cur;
  }
  return cur;
}

template <int R>
__device__ __forceinline__ int pick_shared_nxt(const ColState* sts, int cur, int nbuf) {
  unsigned used = 1u << cur;
  for (int r = 0; r < R; ++r) used |= 1u << sts[r].best;
  for (int b = 0; b < nbuf; ++b)
    if (!((used >> b) & 1u)) return b;
  CK_DASSERT(false);  // unreachable with nbuf = R + 2
  return (cur + 1) % nbuf;
}

// 256-bit accesses of two adjacent double2 (32-byte aligned).
__device__ __forceinline__ void ld256(const double2* ptr, double2& a, double2& b) {
  asm("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y) : "l"(ptr));
}
__device__ __forceinline__ void st256(double2* ptr, double2 a, double2 b) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(ptr), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y)
               : "memory");
}

// Control step after the apply sweep (condest.hpp:251-275 via control_apply)
// from the global scalars res[r] = {||x~||, ||y'||, x.delta, ||delta||}; one
// thread. Shared by the fused kernel and the partition combine kernel.
template <int R, bool OBS>
__device__ __forceinline__ void control_tail_apply(ColState* sts, Header* hdr, const Params& prm,
                                                   const double (*res)[4], int nbuf) {
  int needT = 0, nwait = 0, ndone = 0;
  const int nxt = pick_shared_nxt<R>(sts, shared_cur<R>(sts), nbuf);
  for (int r = 0; r < R; ++r) {
    ColState* s = sts + r;
    const int ph = s->phase;
    if (ph == PH_PRO || ph == PH_APPLY) {
      if (OBS && ph == PH_APPLY) {
        s->obs_xd = res[r][2];
        s->obs_dn = res[r][3];
      }
      control_apply(s, &prm, res[r][0], res[r][1], nxt);
    }
    needT |= s->phase == PH_GRAD;
    nwait += s->phase == PH_WAIT;
    ndone += s->phase == PH_DONE;
  }
  hdr->needT = needT;
  hdr->needA = 0;
  hdr->nwait = nwait;
  hdr->ndone = ndone;
}

// After the transpose sweep: publish r = x.delta (condest.hpp:231) and move
// every gradient column on to its apply half (and to the buffer the sweep just
// wrote); one thread.
template <int R>
__device__ __forceinline__ void control_tail_transpose(ColState* sts, Header* hdr, const double* rad) {
  int needA = 0;
  for (int r = 0; r < R; ++r) {
    ColState* s = sts + r;
    if (s->phase == PH_GRAD) {
      s->rad = rad[r];
      s->cur = s->nxt;
      s->pend = 0;
      s->phase = PH_APPLY;
    }
    needA |= s->phase == PH_APPLY;
  }
  hdr->needA = needA;
  hdr->needT = 0;
}

template <int R, bool OBS, bool NW, bool WIN = false, int U = Tune<R>::apply_u, int OCC = Occ<R>::apply>
__global__ void __launch_bounds__(kTile, OCC) k_apply(const __grid_constant__ LoopArgs a) {
  int seg, tile0, tend, stride, u0, u1;
  unit_range(a, blockIdx.x, a.tiles_A, seg, tile0, tend, stride, u0, u1);
  Header* hdr = a.hdr + seg;
  if (!hdr->needA) return;
  ColState* sts = a.st + (int64_t)seg * R;
  __shared__ double s_h[8], s_l[8];
  __shared__ int s_e[8], s_f[8];
  __shared__ double s_res[R][4];

  bool act[R], pro[R];
  double rad[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int ph = sts[r].phase;
    act[r] = ph == PH_PRO || ph == PH_APPLY;
    pro[r] = ph == PH_PRO;
    // prologue: delta is zero, so x~ = x exactly (x - (0 - 0 x) = x)
    rad[r] = pro[r] ? 0.0 : sts[r].rad;
  }
  // every active column reads the same buffer: row i's pairs at xb[i * R + r]
  const double2* xb = a.PX + (int64_t)shared_cur<R>(sts) * a.nc_pad * R;
  // WIN (banded members, a unit's tiles are consecutive): x~ of the tiles t-1,
  // t, t+1 that tile t's entries reference sits in a four-tile shared-memory
  // ring, each element computed once and staged one tile ahead; the gathers
  // are shared-memory reads.
  __shared__ __align__(16) double s_win[WIN ? 4 * kTile * R : 2];
  int m0 = 0, m1 = 0;
  auto win_load = [&](int q, double2* pr) {  // row q * kTile + tid of the live buffer
    const bool in = q >= m0 && q < m1;
    const double2* row = xb + ((int64_t)q * kTile + threadIdx.x) * R;
    if constexpr (R % 2 == 0) {  // a column pair's (x, delta) pairs: one 256-bit load
#pragma unroll
      for (int r = 0; r < R; r += 2) {
        pr[r] = pr[r + 1] = make_double2(0.0, 0.0);
        if (in) ld256(row + r, pr[r], pr[r + 1]);
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) pr[r] = in ? row[r] : make_double2(0.0, 0.0);
    }
  };
  auto win_store = [&](int q, const double2* pr) {
#pragma unroll
    for (int r = 0; r < R; ++r)
      s_win[win_idx<R>((q & 3) * kTile + threadIdx.x, r)] = act[r] ? xtilde(pr[r], rad[r]) : 0.0;
  };
  if (WIN) {
    m0 = a.seg_t0[seg];
    m1 = a.seg_t0[seg + 1];
    double2 pr[R];
    for (int q = tile0 - 1; q <= tile0 + 1; ++q) {
      win_load(q, pr);
      win_store(q, pr);
    }
    __syncthreads();
  }
  DD dd[R];
  ES es[R], dn[R];
  double xd[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    dd[r] = dd_zero();
    es[r] = es_zero();
    dn[r] = es_zero();
    xd[r] = 0.0;
  }
  int64_t i = (int64_t)tile0 * kTile + threadIdx.x;
  const int64_t istep = (int64_t)stride * kTile;
  int64_t sp0 = 0, sp1 = 0, po = 0;
  int L = 0, cb = 0;
  if (tile0 < tend && i < a.nr_pad) {
    sp0 = a.A.sp[i >> 5];
    sp1 = a.A.sp[(i >> 5) + 1];
    L = a.A.len[i];
    cb = slice_cbase<NW>(a.A, i >> 5);
    po = sell_colbase(a.A, i >> 5, i, sell_rowbase(sp0, i));
  }
  for (int tile = tile0; tile < tend; tile += stride, i += istep) {
    const int64_t base = sell_rowbase(sp0, i);
    const int64_t cbase0 = NW ? po : base;
    const int w = (int)((sp1 - sp0) >> 5);  // slice width: uniform across the warp
    const int Lc = L, cbc = cb;
    const int64_t inext = i + istep;
    if (tile + stride < tend && inext < a.nr_pad) {
      sp0 = a.A.sp[inext >> 5];
      sp1 = a.A.sp[(inext >> 5) + 1];
      L = a.A.len[inext];
      cb = slice_cbase<NW>(a.A, inext >> 5);
      po = sell_colbase(a.A, inext >> 5, inext, sell_rowbase(sp0, inext));
    }
    double2 ahead[R];
    if (WIN && tile + 1 < tend) win_load(tile + 2, ahead);  // needed by the next tile
    if (WIN) {  // own column-space element: ||x~||^2 from the staged x~
      if (i < a.nc) {
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (act[r]) dd_add_sq(dd[r], s_win[win_idx<R>((tile & 3) * kTile + threadIdx.x, r)]);
      }
    } else if (i < a.nc) {  // own column-space element: ||x~||^2 (and observer stats)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (!act[r]) continue;
        const double2 p = __ldg(xb + i * R + r);
        if (OBS && !pro[r]) {
          const double dp = __dsub_rn(p.y, __dmul_rn(rad[r], p.x));
          xd[r] = __fma_rn(p.x, dp, xd[r]);
          es_add(dn[r], dp);
        }
        dd_add_sq(dd[r], xtilde(p, rad[r]));
      }
    }
    if (i < a.nr_pad) {
      double acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = 0.0;
      for (int j0 = 0; j0 < w; j0 += U) {
        int c[U];
        double v[U];
        load_chunk<U, NW>(a.A, base, cbase0, cbc, j0, w, c, v);
        if (WIN) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int qw = c[u] & (4 * kTile - 1);
            CK_DASSERT(!(j0 + u < Lc) || ((c[u] >> 8) >= max(tile - 1, m0) && (c[u] >> 8) <= tile + 1 &&
                                          (c[u] >> 8) < m1));
            if (j0 + u < Lc) {
              double xv[R];
              if constexpr (R % 2 == 0) {  // a row's column pair is one 16-byte read
#pragma unroll
                for (int r = 0; r < R; r += 2) {
                  const double2 t = *reinterpret_cast<const double2*>(s_win + win_idx<R>(qw, r));
                  xv[r] = t.x;
                  xv[r + 1] = t.y;
                }
              } else {
#pragma unroll
                for (int r = 0; r < R; ++r) xv[r] = s_win[win_idx<R>(qw, r)];
              }
#pragma unroll
              for (int r = 0; r < R; ++r)
                if (act[r]) acc[r] = __dadd_rn(acc[r], __dmul_rn(v[u], xv[r]));
            }
          }
        } else {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (!act[r]) continue;
            double2 g[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              CK_DASSERT(c[u] >= 0 && c[u] < a.nc_pad);
              g[u] = __ldg(xb + (int64_t)c[u] * R + r);
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
              if (j0 + u < Lc) acc[r] = __dadd_rn(acc[r], __dmul_rn(v[u], xtilde(g[u], rad[r])));
          }
        }
      }
      if constexpr (R % 2 == 0) {
#pragma unroll
        for (int r = 0; r < R; r += 2) {
          if (act[r] && act[r + 1]) {  // a pair of columns: one 16-byte store
            *reinterpret_cast<double2*>(a.y + i * R + r) = make_double2(acc[r], acc[r + 1]);
          } else {
            if (act[r]) a.y[i * R + r] = acc[r];
            if (act[r + 1]) a.y[i * R + r + 1] = acc[r + 1];
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (act[r]) a.y[i * R + r] = acc[r];
      }
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (act[r]) es_add(es[r], acc[r]);
    }
    if (WIN) {
      // slot (tile + 2) & 3 held tile - 2, last read before the previous barrier
      if (tile + 1 < tend) win_store(tile + 2, ahead);
      __syncthreads();
    }
  }
  // Per-CTA partials.
#pragma unroll
  for (int r = 0; r < R; ++r) {
    DD d = block_dd(dd[r], s_h, s_l);
    ES e = block_es(es[r], s_h, s_e, s_f);
    double x2 = 0.0;
    ES e2 = es_zero();
    if (OBS) {
      x2 = block_sum(xd[r], s_h);
      e2 = block_es(dn[r], s_h, s_e, s_f);
    }
    if (threadIdx.x == 0) {
      double* p = a.partA + ((int64_t)blockIdx.x * R + r) * kPA;
      p[0] = d.hi;
      p[1] = d.lo;
      p[2] = e.s;
      p[3] = (double)e.e;
      p[4] = (double)e.flags;
      p[5] = x2;
      p[6] = e2.s;
      p[7] = (double)e2.e;
      p[8] = (double)e2.flags;
    }
  }
  if (!elect_last_block(&hdr->cntA, (unsigned)(u1 - u0))) return;

  // Last CTA (of this member): fixed-order merge of its partials, then control
  // (or, for a partition rank, publish the merged partials).
#pragma unroll
  for (int r = 0; r < R; ++r) {
    DD d = dd_zero();
    ES e = es_zero(), e2 = es_zero();
    double x2 = 0.0;
    for (int u = u0 + threadIdx.x; u < u1; u += kTile) {
      const double* p = a.partA + ((int64_t)u * R + r) * kPA;
      dd_merge(d, DD{__ldcg(p), __ldcg(p + 1)});
      es_merge(e, ES{__ldcg(p + 2), (int)__ldcg(p + 3), (int)__ldcg(p + 4)});
      if (OBS) {
        x2 = __dadd_rn(x2, __ldcg(p + 5));
        es_merge(e2, ES{__ldcg(p + 6), (int)__ldcg(p + 7), (int)__ldcg(p + 8)});
      }
    }
    d = block_dd(d, s_h, s_l);
    e = block_es(e, s_h, s_e, s_f);
    if (OBS) {
      x2 = block_sum(x2, s_h);
      e2 = block_es(e2, s_h, s_e, s_f);
    }
    if (threadIdx.x == 0) {
      if (a.dist) {
        double* q = a.rank_part + r * kPA;
        q[0] = d.hi;
        q[1] = d.lo;
        q[2] = e.s;
        q[3] = (double)e.e;
        q[4] = (double)e.flags;
        q[5] = x2;
        q[6] = e2.s;
        q[7] = (double)e2.e;
        q[8] = (double)e2.flags;
      } else {
        s_res[r][0] = sqrt(__dadd_rn(d.hi, d.lo));
        s_res[r][1] = es_norm(e);
        s_res[r][2] = x2;
        s_res[r][3] = es_norm(e2);
      }
    }
  }
  if (threadIdx.x == 0 && !a.dist) control_tail_apply<R, OBS>(sts, hdr, a.prm, s_res, a.nbuf);
}

template <int R, bool NW, bool WIN = false, int U = Tune<R>::transpose_u, int OCC = Occ<R>::transpose>
__global__ void __launch_bounds__(kTile, OCC) k_transpose(const __grid_constant__ LoopArgs a) {
  int seg, tile0, tend, stride, u0, u1;
  unit_range(a, blockIdx.x, a.tiles_T, seg, tile0, tend, stride, u0, u1);
  Header* hdr = a.hdr + seg;
  if (!hdr->needT) return;
  ColState* sts = a.st + (int64_t)seg * R;
  __shared__ double s_h[8];
  __shared__ double s_res[R];
  const Params& p = a.prm;
  bool act[R], mat[R];
  double rad[R], ndiv[R], ix2[R], iy2[R], mc[R], vc[R];
  int nxt = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const ColState& s = sts[r];
    act[r] = s.phase == PH_GRAD;
    mat[r] = s.mat != 0;
    rad[r] = s.rad;
    ndiv[r] = s.ndiv;
    ix2[r] = s.inv_x2;
    iy2[r] = s.inv_y2;
    mc[r] = s.mc;
    vc[r] = s.vc;
    if (act[r]) nxt = s.nxt;
  }
  CK_DASSERT(nxt >= 0 && nxt < a.nbuf && nxt != shared_cur<R>(sts));
  // gradient columns read buffer cur and write buffer nxt in lockstep (a
  // prologue column, mat = 0, carries its x over unchanged)
  const double2* xb = a.PX + (int64_t)shared_cur<R>(sts) * a.nc_pad * R;
  double2* xo = a.PX + (int64_t)nxt * a.nc_pad * R;
  const double om1 = 1.0 - p.beta1, om2 = 1.0 - p.beta2;
  double dot[R];
#pragma unroll
  for (int r = 0; r < R; ++r) dot[r] = 0.0;
  // WIN: y' of the row tiles t-1, t, t+1 in a four-tile shared-memory ring (see k_apply)
  __shared__ __align__(16) double s_win[WIN ? 4 * kTile * R : 2];
  int m0 = 0, m1 = 0;
  auto win_load = [&](int q, double* yr) {
    const bool in = q >= m0 && q < m1;
#pragma unroll
    for (int r = 0; r < R; ++r) yr[r] = in ? a.y[((int64_t)q * kTile + threadIdx.x) * R + r] : 0.0;
  };
  auto win_store = [&](int q, const double* yr) {
#pragma unroll
    for (int r = 0; r < R; ++r) s_win[win_idx<R>((q & 3) * kTile + threadIdx.x, r)] = yr[r];
  };
  if (WIN) {
    m0 = a.seg_t0[seg];
    m1 = a.seg_t0[seg + 1];
    double yr[R];
    for (int q = tile0 - 1; q <= tile0 + 1; ++q) {
      win_load(q, yr);
      win_store(q, yr);
    }
    __syncthreads();
  }
  const int64_t jstep = (int64_t)stride * kTile;
  int64_t j = (int64_t)tile0 * kTile + threadIdx.x;
  int64_t sp0 = 0, sp1 = 0, po = 0;
  int L = 0, cb = 0;
  if (tile0 < tend) {
    sp0 = a.AT.sp[j >> 5];
    sp1 = a.AT.sp[(j >> 5) + 1];
    L = a.AT.len[j];
    cb = slice_cbase<NW>(a.AT, j >> 5);
    po = sell_colbase(a.AT, j >> 5, j, sell_rowbase(sp0, j));
  }
  for (int tile = tile0; tile < tend; tile += stride, j += jstep) {
    const int64_t base = sell_rowbase(sp0, j);
    const int64_t cbase0 = NW ? po : base;
    const int w = (int)((sp1 - sp0) >> 5);
    const int Lc = L, cbc = cb;
    if (tile + stride < tend) {
      const int64_t jn = j + jstep;
      sp0 = a.AT.sp[jn >> 5];
      sp1 = a.AT.sp[(jn >> 5) + 1];
      L = a.AT.len[jn];
      cb = slice_cbase<NW>(a.AT, jn >> 5);
      po = sell_colbase(a.AT, jn >> 5, jn, sell_rowbase(sp0, jn));
    }
    double ahead[R];
    if (WIN && tile + 1 < tend) win_load(tile + 2, ahead);
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    for (int j0 = 0; j0 < w; j0 += U) {
      int c[U];
      double v[U];
      load_chunk<U, NW>(a.AT, base, cbase0, cbc, j0, w, c, v);
      if (WIN) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int qw = c[u] & (4 * kTile - 1);
          CK_DASSERT(!(j0 + u < Lc) || ((c[u] >> 8) >= max(tile - 1, m0) && (c[u] >> 8) <= tile + 1 &&
                                        (c[u] >> 8) < m1));
          if (j0 + u < Lc) {
            double yv[R];
            if constexpr (R % 2 == 0) {
#pragma unroll
              for (int r = 0; r < R; r += 2) {
                const double2 t = *reinterpret_cast<const double2*>(s_win + win_idx<R>(qw, r));
                yv[r] = t.x;
                yv[r + 1] = t.y;
              }
            } else {
#pragma unroll
              for (int r = 0; r < R; ++r) yv[r] = s_win[win_idx<R>(qw, r)];
            }
#pragma unroll
            for (int r = 0; r < R; ++r)
              if (act[r]) acc[r] = __dadd_rn(acc[r], __dmul_rn(v[u], yv[r]));
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (!act[r]) continue;
          double yg[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            CK_DASSERT(c[u] >= 0 && c[u] < max(a.nr_pad, a.nc_pad));
            yg[u] = __ldg(a.y + (int64_t)c[u] * R + r);
          }
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (j0 + u < Lc) acc[r] = __dadd_rn(acc[r], __dmul_rn(v[u], yg[u]));
        }
      }
    }
    if (j < a.nc) {
      // one column's Adam step (condest.hpp:225-229, 240-247) from its pairs
      auto column = [&](int r, double2 px, double2 mv, double2& px_out, double2& mv_out) {
        const double xn = mat[r] ? __ddiv_rn(xtilde(px, rad[r]), ndiv[r]) : px.x;  // :240-247
        const double z = __ddiv_rn(acc[r], ndiv[r]);                               // A^T A x_{t+1}
        const double g = __dsub_rn(__dmul_rn(xn, ix2[r]), __dmul_rn(z, iy2[r]));  // :105
        const double mm = __dadd_rn(__dmul_rn(p.beta1, mv.x), __dmul_rn(om1, g));             // :226
        const double vv = __dadd_rn(__dmul_rn(p.beta2, mv.y), __dmul_rn(__dmul_rn(om2, g), g));  // :227
        const double d = __ddiv_rn(__dmul_rn(p.alpha, __dmul_rn(mm, mc[r])),
                                   __dadd_rn(__dsqrt_rn(__dmul_rn(vv, vc[r])), p.eps));  // :228
        mv_out = make_double2(mm, vv);
        px_out = make_double2(xn, d);
        dot[r] = __fma_rn(xn, d, dot[r]);
      };
      auto single = [&](int r) {
        const int64_t e = j * R + r;
        double2 xo0, mo0;
        column(r, xb[e], a.MV[e], xo0, mo0);
        a.MV[e] = mo0;
        xo[e] = xo0;
      };
      if constexpr (R % 2 == 0) {
#pragma unroll
        for (int r = 0; r < R; r += 2) {
          if (act[r] && act[r + 1]) {
            // a column pair's (x, delta) and (m, v) are 32 contiguous bytes each:
            // 256-bit accesses halve the partially used lines of the 16-byte ones
            const int64_t e = j * R + r;
            double2 px0, px1, mv0, mv1, xo0, xo1, mo0, mo1;
            ld256(xb + e, px0, px1);
            ld256(a.MV + e, mv0, mv1);
            column(r, px0, mv0, xo0, mo0);
            column(r + 1, px1, mv1, xo1, mo1);
            st256(a.MV + e, mo0, mo1);
            st256(xo + e, xo0, xo1);
          } else {
            if (act[r]) single(r);
            if (act[r + 1]) single(r + 1);
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (act[r]) single(r);
      }
    }
    if (WIN) {
      if (tile + 1 < tend) win_store(tile + 2, ahead);
      __syncthreads();
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const double s = block_sum(dot[r], s_h);
    if (threadIdx.x == 0) a.partT[(int64_t)blockIdx.x * R + r] = s;
  }
  if (!elect_last_block(&hdr->cntT, (unsigned)(u1 - u0))) return;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double s = 0.0;
    for (int u = u0 + threadIdx.x; u < u1; u += kTile)
      s = __dadd_rn(s, __ldcg(a.partT + (int64_t)u * R + r));
    s = block_sum(s, s_h);
    if (threadIdx.x == 0) {
      if (a.dist)
        a.rank_part[R * kPA + r] = s;  // after the apply partials
      else
        s_res[r] = s;
    }
  }
  if (threadIdx.x == 0 && !a.dist) control_tail_transpose<R>(sts, hdr, s_res);
}

// ------------------------------------------------ row-block partition combine
// Every rank merges the gathered per-rank partials in rank order (identical
// on all ranks, so every rank takes the same control decisions), then runs the
// control step of the single-device kernels. One thread; g holds per rank the
// R*kPA apply partials followed by the R transpose partials.
template <int R>
__device__ __forceinline__ void dist_control_apply(const LoopArgs& a, const double* __restrict__ g, int nranks) {
  if (!a.hdr->needA) return;
  double res[R][4];
  for (int r = 0; r < R; ++r) {
    DD d = dd_zero();
    ES e = es_zero();
    for (int q = 0; q < nranks; ++q) {
      const double* p = g + (int64_t)q * R * (kPA + 1) + r * kPA;
      dd_merge(d, DD{p[0], p[1]});
      es_merge(e, ES{p[2], (int)p[3], (int)p[4]});
    }
    res[r][0] = sqrt(__dadd_rn(d.hi, d.lo));
    res[r][1] = es_norm(e);
    res[r][2] = res[r][3] = 0.0;
  }
  control_tail_apply<R, false>(a.st, a.hdr, a.prm, res, a.nbuf);
}

template <int R>
__device__ __forceinline__ void dist_control_transpose(const LoopArgs& a, const double* __restrict__ g,
                                                       int nranks) {
  if (!a.hdr->needT) return;
  double rad[R];
  for (int r = 0; r < R; ++r) {
    double s = 0.0;
    for (int q = 0; q < nranks; ++q) s = __dadd_rn(s, g[(int64_t)q * R * (kPA + 1) + R * kPA + r]);
    rad[r] = s;
  }
  control_tail_transpose<R>(a.st, a.hdr, rad);
}

// Combine kernels of a partition rank (ck_dist.cu): thread 0 merges every
// rank's partials and runs the control step; all threads scatter the received
// halo (n entries x R columns at permuted positions pos).
template <int R>
__global__ void k_combine_apply(LoopArgs a, const double* __restrict__ g, int nranks, int64_t n,
                                const int32_t* __restrict__ pos, const double* __restrict__ buf) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k == 0) dist_control_apply<R>(a, g, nranks);
  if (k >= n * R) return;
  a.y[(int64_t)pos[k / R] * R + k % R] = buf[k];
}

// The (x, delta) halo lands in the buffer the control step makes live. The
// control thread runs concurrently with the scatter threads: a column read
// before the step is a gradient column (-> nxt), read after it an apply column
// whose cur is that same buffer (cur is written before phase, nxt not at all).
template <int R>
__global__ void k_combine_transpose(LoopArgs a, const double* __restrict__ g, int nranks, int64_t n,
                                    const int32_t* __restrict__ pos, const double2* __restrict__ buf) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int r = (int)(k % R);
  int b = 0;
  double2 v = make_double2(0.0, 0.0);
  if (k < n * R) {
    const volatile ColState* c = a.st + r;
    const int ph = c->phase;
    const int nx = c->nxt;
    b = ph == PH_GRAD ? nx : c->cur;
    v = buf[k];
  }
  if (k == 0) dist_control_transpose<R>(a, g, nranks);
  if (k < n * R) a.PX[((int64_t)b * a.nc_pad + pos[k / R]) * R + r] = v;
}

// x_{t+1} = x~ / N from (x, delta) pairs, into a plain vector (epilogue / observer).
__global__ void k_materialise(int64_t nc, int R, const double2* __restrict__ px, double rad,
                              double ndiv, double* out) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < nc) out[j] = __ddiv_rn(xtilde(px[j * R], rad), ndiv);
}

__global__ void k_extract_x(int64_t n, int R, const double2* __restrict__ px, double* out) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < n) out[j] = px[j * R].x;
}

__global__ void k_store_x(int64_t n, int R, const double* __restrict__ x, double2* px) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < n) px[j * R] = make_double2(x[j], 0.0);
}

// One column's pairs from one buffer to another (stride R).
__global__ void k_copy_col(int64_t n, int R, const double2* __restrict__ src, double2* dst) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < n) dst[j * R] = src[j * R];
}

__global__ void k_zero_moments(int64_t n, int R, int col, double2* mv) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < n) mv[j * R + col] = make_double2(0.0, 0.0);
}

// Largest distance, in 256-row tiles, between a stored entry's row and column
// positions (the window kernels need <= 1).
__global__ void k_tile_reach(SellView A, int64_t nrows_pad, int* out) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nrows_pad) return;
  const int64_t base = sell_rowbase(A.sp[p >> 5], p);
  const int L = A.len[p];
  int reach = 0;
  for (int j = 0; j < L; ++j) {
    const int col = sell_col(A, p >> 5, sell_at(base, j));
    reach = max(reach, abs((col >> 8) - (int)(p >> 8)));
  }
  if (reach > 0) atomicMax(out, reach);
}

// ---------------------------------------------------------------- host side

static unsigned grid256(int64_t n) { return (unsigned)std::max<int64_t>(1, ceil_div(n, 256)); }

static int tile_reach(const Sell& m, cudaStream_t st);
// Every entry of A and A^T within one tile of its row: the window sweeps apply.
bool matrix_window_ok(ck_matrix_s* m) {
  return tile_reach(m->a, m->stream) <= 1 && tile_reach(m->at, m->stream) <= 1;
}

static int tile_reach(const Sell& m, cudaStream_t st) {
  static_assert(kTile == 256, "k_tile_reach shifts by 8");
  DBuf<int> d(1);
  CK_CUDA(cudaMemsetAsync(d.p, 0, sizeof(int), st));
  k_tile_reach<<<grid256(m.nrows_pad), 256, 0, st>>>(view(m), m.nrows_pad, d.p);
  int h = 0;
  CK_CUDA(cudaMemcpyAsync(&h, d.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK_CUDA(cudaStreamSynchronize(st));
  return h;
}

template <int R>
static void launch_apply_r(const ck_session_s* s, cudaStream_t st) {
  const bool nw = s->A->a.narrow;
  if (s->observe_on) {
    if (nw)
      k_apply<R, true, true><<<s->args.units_A, kTile, 0, st>>>(s->args);
    else
      k_apply<R, true, false><<<s->args.units_A, kTile, 0, st>>>(s->args);
  } else if (s->args.win) {
    if (nw)
      k_apply<R, false, true, true, WinTune<R>::apply_u, WinTune<R>::apply_occ><<<s->args.units_A, kTile, 0, st>>>(s->args);
    else
      k_apply<R, false, false, true, WinTune<R>::apply_u, WinTune<R>::apply_occ><<<s->args.units_A, kTile, 0, st>>>(s->args);
  } else {
    if (nw)
      k_apply<R, false, true><<<s->args.units_A, kTile, 0, st>>>(s->args);
    else
      k_apply<R, false, false><<<s->args.units_A, kTile, 0, st>>>(s->args);
  }
}

template <int R>
static void launch_transpose_r(const ck_session_s* s, cudaStream_t st) {
  if (s->args.win) {
    if (s->A->at.narrow)
      k_transpose<R, true, true, WinTune<R>::transpose_u, WinTune<R>::transpose_occ>
          <<<s->args.units_T, kTile, 0, st>>>(s->args);
    else
      k_transpose<R, false, true, WinTune<R>::transpose_u, WinTune<R>::transpose_occ>
          <<<s->args.units_T, kTile, 0, st>>>(s->args);
    return;
  }
  if (s->A->at.narrow)
    k_transpose<R, true><<<s->args.units_T, kTile, 0, st>>>(s->args);
  else
    k_transpose<R, false><<<s->args.units_T, kTile, 0, st>>>(s->args);
}

void launch_inv_step(const InvArgs* args, int S, int R, size_t smem, int half, cudaStream_t st, int cl);
void launch_inv_step_dense(const InvArgs* args, int S, int half, size_t dyn, cudaStream_t st);
void prepare_inv_step_dense(size_t dyn);
void lu_dense_solve_launch(ck_lu_s* f, double* x, bool transpose, cudaStream_t st);
bool inv_cluster_fits(int cl, int S, int R, size_t smem);
void prepare_inv_step(size_t smem, int R);
size_t inv_step_smem(const BandView& b, int R);
int lu_ring_size(const BandView& b);
int64_t lu_stage_cap(const BandView& b, int R);
void lu_solve_launch(ck_lu_s* f, double* const* x, int R, bool transpose, cudaStream_t st);

static void launch_inv_half(ck_session_s* s, int half, cudaStream_t st) {
  if (s->inv_dense) {
    launch_inv_step_dense(s->dargs.p, s->S, half, s->inv_smem, st);
    return;
  }
  launch_inv_step(s->dargs.p, s->S, s->R, s->inv_smem, half, st, s->inv_cl);
}

void launch_apply_only(ck_session_s* s, cudaStream_t st) {
  if (s->kind == 1) {
    launch_inv_half(s, 1, st);
    return;
  }
  switch (s->R) {
    case 1: launch_apply_r<1>(s, st); break;
    case 2: launch_apply_r<2>(s, st); break;
    case 3: launch_apply_r<3>(s, st); break;
    default: launch_apply_r<4>(s, st); break;
  }
}

void launch_transpose_only(ck_session_s* s, cudaStream_t st) {
  if (s->kind == 1) {
    launch_inv_half(s, 2, st);
    return;
  }
  switch (s->R) {
    case 1: launch_transpose_r<1>(s, st); break;
    case 2: launch_transpose_r<2>(s, st); break;
    case 3: launch_transpose_r<3>(s, st); break;
    default: launch_transpose_r<4>(s, st); break;
  }
}

void launch_step(ck_session_s* s, cudaStream_t st) {
  if (s->dist) {
    dist_step(s, st);
    return;
  }
  if (s->kind == 1) {
    launch_inv_half(s, 0, st);
    return;
  }
  launch_apply_only(s, st);
  launch_transpose_only(s, st);
}

static int occ_apply(int R) {
  return R == 1 ? Occ<1>::apply : R == 2 ? Occ<2>::apply : R == 3 ? Occ<3>::apply : Occ<4>::apply;
}
static int occ_transpose(int R) {
  return R == 1   ? Occ<1>::transpose
         : R == 2 ? Occ<2>::transpose
         : R == 3 ? Occ<3>::transpose
                  : Occ<4>::transpose;
}

// Partition ranks: own tiles [t0, t1) of the extended local operator.
void session_set_tiles(ck_session_s* s, int t0, int t1) {
  LoopArgs& a = s->args;
  a.tile_base = t0;
  a.tiles_A = a.tiles_T = t1;
  a.units_A = std::max(1, std::min(t1 - t0, 148 * occ_apply(s->R)));
  a.units_T = std::max(1, std::min(t1 - t0, 148 * occ_transpose(s->R)));
}

void launch_dist_combine(ck_session_s* s, bool apply, const double* gathered, int nranks, int64_t n,
                         const int32_t* pos, const void* buf, cudaStream_t st) {
  const LoopArgs& a = s->args;
  const unsigned blocks = (unsigned)std::max<int64_t>(1, ceil_div(n * s->R, 256));
#define CK_DC(RR)                                                                                  \
  case RR:                                                                                         \
    if (apply)                                                                                     \
      k_combine_apply<RR><<<blocks, 256, 0, st>>>(a, gathered, nranks, n, pos, (const double*)buf); \
    else                                                                                           \
      k_combine_transpose<RR><<<blocks, 256, 0, st>>>(a, gathered, nranks, n, pos,                 \
                                                      (const double2*)buf);                        \
    break;
  switch (s->R) {
    CK_DC(1)
    CK_DC(2)
    CK_DC(3)
    CK_DC(4)
  }
#undef CK_DC
}

int partial_words(int R) { return R * (kPA + 1); }

void pull_state(ck_session_s* s) {
  cudaStream_t st = s->stream;
  CK_CUDA(cudaMemcpyAsync(s->h_st, s->st.p, sizeof(ColState) * s->S * s->R,
                          cudaMemcpyDeviceToHost, st));
  CK_CUDA(cudaMemcpyAsync(s->h_hdr, s->hdr.p, sizeof(Header) * s->S, cudaMemcpyDeviceToHost, st));
  CK_CUDA(cudaStreamSynchronize(st));
}

void push_state(ck_session_s* s) {
  cudaStream_t st = s->stream;
  CK_CUDA(cudaMemcpyAsync(s->st.p, s->h_st, sizeof(ColState) * s->S * s->R,
                          cudaMemcpyHostToDevice, st));
  CK_CUDA(cudaMemcpyAsync(s->hdr.p, s->h_hdr, sizeof(Header) * s->S, cudaMemcpyHostToDevice, st));
  CK_CUDA(cudaStreamSynchronize(st));
}

int64_t total_done(const ck_session_s* s) {
  int64_t d = 0;
  for (int g = 0; g < s->S; ++g) d += s->h_hdr[g].ndone;
  return d;
}

bool any_wait(const ck_session_s* s) {
  for (int g = 0; g < s->S; ++g)
    if (s->h_hdr[g].nwait > 0) return true;
  return false;
}

// (x, delta) pairs of buffer b, column c: element i at col_buf(...)[i * R]
double2* col_buf(ck_session_s* s, int b, int c) {
  return s->PX.p + (int64_t)b * s->npad * s->R + c;
}

// host vector of member g (original order, seg_n[g] doubles) -> internal plain
// vector `dst` over the member's internal range [seg_off[g], seg_off[g]+seg_pad[g])
static void to_internal(ck_session_s* s, int g, const double* host, double* dst,
                        cudaStream_t st) {
  const int64_t off = s->seg_off[g], pad = s->seg_pad[g];
  CK_CUDA(cudaMemsetAsync(s->tmp.p + off, 0, sizeof(double) * pad, st));
  if (s->perm) {
    CK_CUDA(cudaMemcpyAsync(s->tmp.p + off, host, sizeof(double) * s->seg_n[g],
                            cudaMemcpyHostToDevice, st));
    gather_perm(s->perm + off, pad, s->tmp.p, dst + off, st);
  } else {
    CK_CUDA(cudaMemcpyAsync(dst + off, host, sizeof(double) * s->seg_n[g], cudaMemcpyHostToDevice,
                            st));
  }
}

// internal plain vector -> host vector of member g (original order)
void to_host(ck_session_s* s, int g, const double* src, double* host, cudaStream_t st) {
  const int64_t off = s->seg_off[g], pad = s->seg_pad[g];
  const double* out = src + off;
  if (s->perm) {
    double* scratch = s->tmp.p;
    scatter_perm(s->perm + off, pad, src + off, scratch, st);
    out = scratch + off;
  }
  const int64_t n = s->seg_n[g];
  if (s->hx.n < n) {
    CK_CUDA(cudaMemcpyAsync(host, out, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CK_CUDA(cudaStreamSynchronize(st));
    return;
  }
  // through the pinned staging buffer (full-rate D2H), then a threaded copy
  CK_CUDA(cudaMemcpyAsync(s->hx.p, out, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  CK_CUDA(cudaStreamSynchronize(st));
  const int64_t nt = n < (int64_t(1) << 20) ? 1 : 8, chunk = ceil_div(n, nt);
  std::vector<std::thread> pool;
  for (int64_t t = 1; t < nt; ++t) {
    const int64_t lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo < hi) pool.emplace_back([=] { std::memcpy(host + lo, s->hx.p + lo, sizeof(double) * (hi - lo)); });
  }
  std::memcpy(host, s->hx.p, sizeof(double) * std::min(n, chunk));
  for (auto& th : pool) th.join();
}

// Upload a fresh start vector for member g, column c into buffer b: (x,
// delta = 0) pairs in the internal (permuted) space, m = v = 0.
void load_start(ck_session_s* s, int g, int c, int b, const double* x) {
  cudaStream_t st = s->stream;
  const int64_t off = s->seg_off[g], pad = s->seg_pad[g];
  double* plain = s->tmp.p + s->thalf;
  CK_CUDA(cudaMemsetAsync(plain + off, 0, sizeof(double) * pad, st));
  to_internal(s, g, x, plain, st);
  k_store_x<<<grid256(pad), 256, 0, st>>>(pad, s->R, plain + off, col_buf(s, b, c) + off * s->R);
  k_zero_moments<<<grid256(pad), 256, 0, st>>>(pad, s->R, c, s->MV.p + off * s->R);
  CK_CUDA(cudaGetLastError());
}

// restart(), condest.hpp:201-207: the next vector of the column's own stream,
// m = v = 0, bias powers reset; x_min and the patience counters are kept.
// Next start vector of column k (member g) into `out` (the member's
// original-order vector): random_unit_vector from the column's own stream; a
// partition rank draws the global vector and keeps its extended slice.
static void draw_start(ck_session_s* s, int k, int g, double* out,
                       const std::function<double*()>& dst = {}) {
  if (!s->dist) {
    random_unit_vector_host(&s->gens[k], s->seg_n[g], out, dst);
    return;
  }
  const DistPart& d = *s->dist;
  std::vector<double> full((size_t)d.n_global);
  random_unit_vector_host(&s->gens[k], d.n_global, full.data());
  double* to = dst ? dst() : out;
  for (size_t e = 0; e < d.ext_global.size(); ++e)
    to[e] = d.ext_global[e] >= 0 ? full[(size_t)d.ext_global[e]] : 0.0;
}

void service_restarts(ck_session_s* s) {
  bool any = false;
  for (int g = 0; g < s->S; ++g) {
    for (int c = 0; c < s->R; ++c) {
      const int k = g * s->R + c;
      ColState& cs = s->h_st[k];
      if (cs.phase != PH_WAIT) continue;
      draw_start(s, k, g, s->hx.data());
      int b;
      if (s->kind == 1) {  // inverse loop: every column rotates its own three buffers
        b = cs.cur != cs.best ? cs.cur : (cs.best + 1) % 3;
      } else {
        // explicit sweeps: the operator's columns share their live buffer. Join
        // the running columns there; if this column's x_min sits in that buffer,
        // move it to another one first (only this column's slots are touched).
        b = cs.cur;
        for (int c2 = 0; c2 < s->R; ++c2) {
          const int ph = s->h_st[g * s->R + c2].phase;
          if (c2 != c && (ph == PH_PRO || ph == PH_APPLY || ph == PH_GRAD)) b = s->h_st[g * s->R + c2].cur;
        }
        if (b == cs.best) {
          const int f = (b + 1) % s->args.nbuf;
          const int64_t off = s->seg_off[g], pad = s->seg_pad[g];
          k_copy_col<<<grid256(pad), 256, 0, s->stream>>>(pad, s->R, col_buf(s, cs.best, c) + off * s->R,
                                                         col_buf(s, f, c) + off * s->R);
          CK_CUDA(cudaGetLastError());
          cs.best = f;
        }
      }
      load_start(s, g, c, b, s->hx.data());
      cs.cur = b;
      cs.b1p = 1.0;
      cs.b2p = 1.0;
      cs.mat = 0;
      cs.pend = 0;
      cs.rad = 0.0;
      cs.phase = PH_PRO;
      s->h_hdr[g].needA = 1;
      s->h_hdr[g].nwait = 0;
      any = true;
    }
  }
  if (any) {
    CK_CUDA(cudaStreamSynchronize(s->stream));
    push_state(s);
  }
}

void build_graph(ck_session_s* s, int steps) {
  if (s->dist && !s->dist->nccl) return;  // in-process partitions: the group drives every step
  cudaStream_t st = s->stream;
  cudaGraph_t g;
  CK_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  for (int k = 0; k < steps; ++k) launch_step(s, st);
  CK_CUDA(cudaStreamEndCapture(st, &g));
  CK_CUDA(cudaGraphInstantiate(&s->gexec, g, 0));
  CK_CUDA(cudaGraphDestroy(g));
  s->gsteps = steps;
}

// Common part of session creation: state buffers, x0 per (member, column), graphs.
void session_init_common(ck_session_s* s, const ck_adam_cfg* cfg, const uint64_t* seeds,
                                int64_t ywords, double bytes_per_step) {
  cudaStream_t st = s->stream;
  const int R = s->R, S = s->S;
  Trace tr("session_init");
  s->thalf = std::max(s->npad, ywords / R);
  s->tmp.alloc(2 * s->thalf);
  CK_CUDA(cudaMemsetAsync(s->PX.p, 0, s->PX.bytes(), st));
  CK_CUDA(cudaMemsetAsync(s->MV.p, 0, s->MV.bytes(), st));
  CK_CUDA(cudaMemsetAsync(s->y.p, 0, s->y.bytes(), st));
  CK_CUDA(cudaMallocHost(reinterpret_cast<void**>(&s->h_st), sizeof(ColState) * S * R));
  CK_CUDA(cudaMallocHost(reinterpret_cast<void**>(&s->h_hdr), sizeof(Header) * S));
  int64_t nmax = 0;
  for (int g = 0; g < S; ++g) nmax = std::max(nmax, s->seg_n[g]);
  // The n-sized pinned staging buffer (start vectors, restarts, witness D2H)
  // takes ~0.1 s to pin at config-4 size: it is allocated on a helper thread
  // while the first start vector is drawn into pageable scratch (uninitialised,
  // so the RNG's worker threads fault its pages in parallel); the normalisation
  // pass then writes into the pinned buffer, which uploads at full rate.
  // The first start vector, when ck_start_vector_prefetch drew it during the
  // matrix upload: hx adopts its pinned buffer (then the resize below is a no-op).
  std::mt19937_64 g0;
  const bool x0_ready = !s->dist && S == 1 && s->seg_n[0] == nmax &&
                        take_start_prefetch(seeds[0], nmax, &g0, &s->hx);
  std::exception_ptr pin_err;
  std::thread pin([s, nmax, &pin_err] {
    try {
      CK_CUDA(cudaSetDevice(s->device));
      s->hx.resize(nmax);
    } catch (...) {
      pin_err = std::current_exception();
    }
  });
  struct Joiner {
    std::thread& t;
    ~Joiner() {
      if (t.joinable()) t.join();
    }
  } pin_join{pin};
  auto pinned = [&]() -> double* {
    if (pin.joinable()) pin.join();
    if (pin_err) std::rethrow_exception(pin_err);
    return s->hx.data();
  };
  std::unique_ptr<double[]> scratch(new double[(size_t)std::max<int64_t>(nmax, 1)]);
  s->gens.clear();
  s->gens.reserve((size_t)S * R);
  for (int g = 0; g < S; ++g) {
    for (int c = 0; c < R; ++c) {
      s->gens.emplace_back(seeds[g * R + c]);
      if (g == 0 && c == 0) tr.mark("buffers", st);
      if (g == 0 && c == 0 && x0_ready)
        s->gens.back() = g0;  // drawn during the matrix upload, already in hx
      else
        draw_start(s, g * R + c, g, scratch.get(), pinned);  // x0, rng.hpp:68-77
      if (g == 0 && c == 0) tr.mark("x0 host RNG", st);
      load_start(s, g, c, 0, pinned());
      CK_CUDA(cudaStreamSynchronize(st));  // hx is reused for the next upload
      if (g == 0 && c == 0) tr.mark("x0 upload", st);
      ColState cs{};
      cs.phase = cfg->max_iter == 0 ? PH_DONE : PH_PRO;
      cs.cur = 0;
      cs.best = 0;  // x_min = x (condest.hpp:194)
      cs.nxt = 1;
      cs.budget = 16;
      cs.b1p = cs.b2p = 1.0;
      cs.loss_min = INFINITY;
      cs.loss = NAN;
      s->h_st[g * R + c] = cs;
    }
    Header h{};
    h.needA = cfg->max_iter == 0 ? 0 : 1;
    h.ncols = R;
    h.ndone = cfg->max_iter == 0 ? R : 0;
    s->h_hdr[g] = h;
  }
  pinned();
  tr.mark("remaining columns", st);
  push_state(s);
  // chunk length: about 4 ms of device work per host round trip, 16..256 steps (a finished
  // column's kernels return at once, so a chunk that overshoots the end costs launches only)
  // bytes_per_step < 0: a fixed chunk of -bytes_per_step steps (latency-bound
  // loops, where streamed bytes say nothing about the step time)
  const int steps = bytes_per_step < 0
                        ? (int)-bytes_per_step
                        : (int)std::min(256.0, std::max(16.0, 4e-3 * 6.0e12 / std::max(bytes_per_step, 1.0)));
  build_graph(s, steps);
  tr.mark("graph capture", st);
}

// Explicit-operator session over S >= 1 square-or-rectangular members packed
// block-diagonally in A (member g occupies rows/cols [off_g, off_g + n_g) with
// off_g = sum of round_up(n_h, 256), h < g). S == 1 is a single operator.
void session_setup_explicit(ck_session_s* s, ck_matrix_s* A, const ck_adam_cfg* cfg, int R,
                            const int64_t* seg_n, int S) {
  if (R < 1 || R > kMaxCols) fail(CK_ERR_INVALID_ARGUMENT, "session columns must be 1..4");
  if (A->ncols == 0) fail(CK_ERR_INVALID_ARGUMENT, "projected_adam: zero-dimensional operator");
  if (S < 1) fail(CK_ERR_INVALID_ARGUMENT, "at least one member");
  s->kind = 0;
  s->A = A;
  s->R = R;
  s->S = S;
  s->stream = A->stream;
  s->device = A->device;
  s->n = A->ncols;
  s->npad = A->at.nrows_pad;
  s->perm = A->at.perm.p;
  s->prm = Params{cfg->alpha, cfg->beta1, cfg->beta2, cfg->eps_stab, cfg->rel_tol, cfg->max_iter,
                  cfg->patience};
  s->seg_n.assign(S, 0);
  s->seg_off.assign(S, 0);
  s->seg_pad.assign(S, 0);
  if (S == 1) {
    s->seg_n[0] = A->ncols;
    s->seg_pad[0] = s->npad;
  } else {
    if (A->nrows != A->ncols) fail(CK_ERR_DIMENSION, "batched members must be square");
    int64_t off = 0;
    for (int g = 0; g < S; ++g) {
      if (seg_n[g] <= 0) fail(CK_ERR_INVALID_ARGUMENT, "empty batch member");
      s->seg_n[g] = seg_n[g];
      s->seg_off[g] = off;
      s->seg_pad[g] = round_up(seg_n[g], kTile);
      off += s->seg_pad[g];
    }
    if (off != A->nrows) fail(CK_ERR_DIMENSION, "member sizes do not tile the packed matrix");
  }
  LoopArgs& a = s->args;
  a.A = view(A->a);
  a.AT = view(A->at);
  a.nr = A->nrows;
  a.nc = A->ncols;
  a.nr_pad = A->a.nrows_pad;
  a.nc_pad = A->at.nrows_pad;
  a.tiles_A = (int)(std::max(a.nr_pad, a.nc_pad) / kTile);
  a.tiles_T = (int)(a.nc_pad / kTile);
  a.S = S;
  a.tpu_A = a.tpu_T = 0;
  if (S == 1) {
    a.units_A = (int)std::min<int64_t>(a.tiles_A, 148 * occ_apply(R));
    a.units_T = (int)std::min<int64_t>(a.tiles_T, 148 * occ_transpose(R));
    a.unit_seg = a.unit_t0 = a.unit_t1 = a.seg_u0 = a.seg_t0 = nullptr;
    a.win = 0;
  } else {
    // members are tile-aligned; each unit takes up to 32 consecutive tiles of one member
    std::vector<int32_t> useg, ut0, ut1, su0(S + 1, 0), st0(S + 1, 0);
    for (int g = 0; g < S; ++g) {
      const int t0 = (int)(s->seg_off[g] / kTile), nt = (int)(s->seg_pad[g] / kTile);
      su0[g] = (int)useg.size();
      st0[g] = t0;
      st0[g + 1] = t0 + nt;
      for (int t = 0; t < nt; t += 32) {
        useg.push_back(g);
        ut0.push_back(t0 + t);
        ut1.push_back(t0 + std::min(nt, t + 32));
      }
    }
    su0[S] = (int)useg.size();
    a.units_A = a.units_T = (int)useg.size();
    s->units.alloc(3 * (int64_t)useg.size() + 2 * (S + 1));
    int32_t* d = s->units.p;
    CK_CUDA(cudaMemcpy(d, useg.data(), sizeof(int32_t) * useg.size(), cudaMemcpyHostToDevice));
    CK_CUDA(cudaMemcpy(d + useg.size(), ut0.data(), sizeof(int32_t) * useg.size(), cudaMemcpyHostToDevice));
    CK_CUDA(cudaMemcpy(d + 2 * useg.size(), ut1.data(), sizeof(int32_t) * useg.size(), cudaMemcpyHostToDevice));
    CK_CUDA(cudaMemcpy(d + 3 * useg.size(), su0.data(), sizeof(int32_t) * (S + 1), cudaMemcpyHostToDevice));
    a.unit_seg = d;
    a.unit_t0 = d + useg.size();
    a.unit_t1 = d + 2 * useg.size();
    CK_CUDA(cudaMemcpy(d + 3 * useg.size() + S + 1, st0.data(), sizeof(int32_t) * (S + 1), cudaMemcpyHostToDevice));
    a.seg_u0 = d + 3 * useg.size();
    a.seg_t0 = a.seg_u0 + S + 1;
    // banded members: gather from the sliding shared-memory window (CK_NO_WINDOW=1: A/B)
    a.win = !std::getenv("CK_NO_WINDOW") && tile_reach(A->a, s->stream) <= 1 &&
            tile_reach(A->at, s->stream) <= 1;
  }
  s->partA.alloc((int64_t)a.units_A * R * kPA);
  s->partT.alloc((int64_t)a.units_T * R * kPT);
  const int64_t yw = std::max(a.nr_pad, a.nc_pad) * R;
  a.prm = s->prm;
  a.nbuf = R + 2;  // lockstep rotation: cur, nxt and one best per column
  s->PX.alloc((int64_t)a.nbuf * R * s->npad);
  s->MV.alloc(s->npad * R);
  s->y.alloc(yw);
  s->st.alloc((int64_t)S * R);
  s->hdr.alloc(S);
  a.PX = s->PX.p;
  a.MV = s->MV.p;
  a.y = s->y.p;
  a.partA = s->partA.p;
  a.partT = s->partT.p;
  a.st = s->st.p;
  a.hdr = s->hdr.p;
  a.dist = 0;
  a.rank_part = nullptr;
  a.tile_base = 0;
}

static void session_create_explicit(ck_session_s* s, ck_matrix_s* A, const ck_adam_cfg* cfg,
                                    const uint64_t* seeds, int R, const int64_t* seg_n, int S) {
  session_setup_explicit(s, A, cfg, R, seg_n, S);
  const int64_t yw = std::max(s->args.nr_pad, s->args.nc_pad) * R;
  const double bytes_per_step = 24.0 * (double)A->nnz + 100.0 * (double)A->ncols * R;
  session_init_common(s, cfg, seeds, yw, bytes_per_step);
}

void session_create(ck_session_s* s, ck_matrix_s* A, const ck_adam_cfg* cfg,
                    const uint64_t* seeds, int R) {
  session_create_explicit(s, A, cfg, seeds, R, nullptr, 1);
}

void session_create_batch(ck_session_s* s, ck_matrix_s* A, const int64_t* seg_n, int S,
                          const ck_adam_cfg* cfg, const uint64_t* seeds, int R) {
  session_create_explicit(s, A, cfg, seeds, R, seg_n, S);
}

// InverseOracle session over S >= 1 independent factorisations (member g's
// vectors at [off_g, off_g + n_g) of the internal vectors, off_g = sum of
// round_up(n_h, 32)); one CTA per member advances its R columns.
void session_create_inverse_batch(ck_session_s* s, ck_lu_s* const* lus, int S,
                                  const ck_adam_cfg* cfg, const uint64_t* seeds, int R) {
  if (R < 1 || R > kMaxCols) fail(CK_ERR_INVALID_ARGUMENT, "session columns must be 1..4");
  if (S < 1) fail(CK_ERR_INVALID_ARGUMENT, "at least one member");
  for (int g = 0; g < S; ++g) {
    if (lus[g]->n == 0) fail(CK_ERR_INVALID_ARGUMENT, "projected_adam: zero-dimensional operator");
    if (lus[g]->device != lus[0]->device) fail(CK_ERR_INVALID_ARGUMENT, "members on different devices");
  }
  s->kind = 1;
  s->lus.assign(lus, lus + S);
  s->lu = lus[0];
  s->A = nullptr;
  s->R = R;
  s->S = S;
  s->stream = lus[0]->stream;
  s->device = lus[0]->device;
  s->perm = nullptr;
  s->seg_n.assign(S, 0);
  s->seg_off.assign(S, 0);
  s->seg_pad.assign(S, 0);
  int64_t off = 0;
  size_t smem = 0;
  for (int g = 0; g < S; ++g) {
    const int64_t n = lus[g]->n;
    s->seg_n[g] = n;
    s->seg_off[g] = off;
    s->seg_pad[g] = S == 1 ? n : ceil_div(n, 32) * 32;
    off += s->seg_pad[g];
    smem = std::max(smem, inv_step_smem(lus[g]->view(), R));
  }
  s->npad = off;
  s->n = S == 1 ? s->seg_n[0] : off;
  s->prm = Params{cfg->alpha, cfg->beta1, cfg->beta2, cfg->eps_stab, cfg->rel_tol, cfg->max_iter,
                  cfg->patience};
  s->inv_smem = smem;
  prepare_inv_step(smem, R);
  // widest band of the batch decides the cluster split of the sweeps
  BandView wide = lus[0]->view();
  for (int g = 1; g < S; ++g)
    if (lus[g]->kl + lus[g]->ku > wide.kv) wide = lus[g]->view();
  const int64_t ts = (std::max(wide.kl, wide.kv) + 2) & ~(int64_t)1;
  // dynamic shared memory of a cluster CTA (doubles): the leader's rings, dot
  // scratch, two tail-sum slots and the dot partials (no stage); a helper's
  // two head slots, dot rows and coefficient share
  auto clu_smem = [&](int cl) {
    int64_t ring_max = 0;
    for (int g = 0; g < S; ++g) ring_max = std::max<int64_t>(ring_max, lu_ring_size(lus[g]->view()));
    const int64_t leader = stage_offset(R, (int)ring_max) + 2 * (int64_t)R * ts + 2 * (int64_t)cl * R * kLUBlock;
    const int64_t sh = (std::max(wide.kl, wide.kv) + cl - 2) / (cl - 1) + 2;
    const int64_t helper = (int64_t)2 * R * kLUBlock + (int64_t)(R + 2 * kLUBlock) * sh;  // two cf slots
    return (size_t)(8 * std::max(leader, helper) + 256);
  };
  // cluster size (scripts/check_cluster.py): 12 CTAs from kl + ku >= 1024 (config 2),
  // 8 from >= 256 (config-5 member), when the clusters fit; CK_LU_CLUSTER forces
  // narrow bands, one column per system: the dense-block sweeps (ck_lu_dense.cuh)
  bool dense = R == 1;
  for (int g = 0; g < S; ++g) dense = dense && lus[g]->dense_ok;
  s->inv_dense = dense;
  int cl = 1;
  auto try_cl = [&](int c) {
    if (cl == 1 && c > 1 && inv_cluster_fits(c, S, R, clu_smem(c))) cl = c;
  };
  if (dense) {
    // no cluster split: the sweeps are bound by the block chain, not by bandwidth
  } else if (const char* e = std::getenv("CK_LU_CLUSTER")) {
    try_cl(std::max(1, std::min(16, std::atoi(e))));
  } else if (R == 1) {  // measured with one column per system; 4 columns ran slower split (214 vs 134 ms)
    if (wide.kv >= 4 * kLUClusterMinRows && S * 12 <= 148) try_cl(12);
    if (wide.kv >= kLUClusterMinRows && S * 8 <= 148) try_cl(8);
  }
  if (cl > 1) {
    smem = clu_smem(cl);
    s->inv_smem = smem;
    prepare_inv_step(smem, R);
  }
  if (dense) {  // the block ring of the widest member
    size_t dyn = 0;
    for (int g = 0; g < S; ++g)
      dyn = std::max(dyn, dense_dyn_smem(kLUBlock + (int)lus[g]->kl, kLUBlock + (int)(lus[g]->kl + lus[g]->ku)));
    s->inv_smem = dyn;
    prepare_inv_step_dense(dyn);
  }
  const int64_t dyn = (int64_t)(smem / sizeof(double));
  const int64_t dpart_off = cl > 1 ? dyn - 32 - 2 * (int64_t)cl * R * kLUBlock : dyn;  // two slots
  const int64_t tsum_off = cl > 1 ? dpart_off - (int64_t)2 * R * ts : dyn;  // two slots (block parity)
  s->inv_cl = cl;
  const int64_t yw = s->npad * R;
  s->PX.alloc(3 * R * s->npad);
  s->MV.alloc(s->npad * R);
  s->y.alloc(yw);
  s->st.alloc((int64_t)S * R);
  s->hdr.alloc(S);
  std::vector<InvArgs> h((size_t)S);
  for (int g = 0; g < S; ++g) {
    InvArgs& a = h[g];
    const BandView b = lus[g]->view();
    const int64_t o = s->seg_off[g];
    a.b = b;
    a.n = s->seg_n[g];
    a.ring_size = lu_ring_size(b);
    a.b.stage_cap = tsum_off - stage_offset(R, a.ring_size);
    if (a.b.stage_cap < 0) fail(CK_ERR_UNSUPPORTED, "band too wide for the on-chip solve window");
    a.cl = cl;
    a.cl_tsum_off = tsum_off;
    a.cl_ts = ts;
    a.cl_dpart_off = dpart_off;
    a.b.stage_min = lu_stage_min();
    a.dv = dense ? lus[g]->dense_view() : DenseView{};
    a.PX = s->PX.p + o * R;
    a.pstride = s->npad * R;
    a.MV = s->MV.p + o * R;
    a.y = s->y.p + o * R;
    a.st = s->st.p + (int64_t)g * R;
    a.hdr = s->hdr.p + g;
    a.prm = s->prm;
  }
  s->dargs.alloc(S);
  CK_CUDA(cudaMemcpy(s->dargs.p, h.data(), sizeof(InvArgs) * S, cudaMemcpyHostToDevice));
  // the sweeps are a latency chain (~0.1-0.5 ms per step): 32 steps per graph
  // chunk keep the host round trips (restart service, termination) negligible
  session_init_common(s, cfg, seeds, yw, -32.0);
}

void session_create_inverse(ck_session_s* s, ck_lu_s* lu, const ck_adam_cfg* cfg,
                            const uint64_t* seeds, int R) {
  session_create_inverse_batch(s, &lu, 1, cfg, seeds, R);
}

void session_run(ck_session_s* s, uint64_t max_steps, int32_t* finished) {
  cudaStream_t st = s->stream;
  uint64_t done = 0;
  *finished = 0;
  for (;;) {
    pull_state(s);
    if (total_done(s) == (int64_t)s->S * s->R) {
      *finished = 1;
      return;
    }
    if (any_wait(s)) service_restarts(s);
    if (max_steps && done >= max_steps) return;
    if (s->observe_on || (max_steps && max_steps - done < (uint64_t)s->gsteps)) {
      const uint64_t n = max_steps ? std::min<uint64_t>(max_steps - done, s->gsteps) : s->gsteps;
      for (uint64_t k = 0; k < n; ++k) launch_step(s, st);
      CK_CUDA(cudaGetLastError());
      done += n;
    } else {
      CK_CUDA(cudaGraphLaunch(s->gexec, st));
      done += (uint64_t)s->gsteps;
    }
  }
}

void session_time(ck_session_s* s, uint64_t steps, int32_t mode, double* ms_total,
                  double* ms_apply, double* ms_transpose) {
  cudaStream_t st = s->stream;
  pull_state(s);
  if (any_wait(s)) service_restarts(s);
  if (mode == 1 || s->kind == 1) {  // whole steps (graph chunks), no per-kernel split
    cudaEvent_t e0, e1;
    CK_CUDA(cudaEventCreate(&e0));
    CK_CUDA(cudaEventCreate(&e1));
    CK_CUDA(cudaStreamSynchronize(st));
    CK_CUDA(cudaEventRecord(e0, st));
    uint64_t k = 0;
    for (; k + (uint64_t)s->gsteps <= steps; k += (uint64_t)s->gsteps)
      CK_CUDA(cudaGraphLaunch(s->gexec, st));
    for (; k < steps; ++k) launch_step(s, st);
    CK_CUDA(cudaEventRecord(e1, st));
    CK_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *ms_total = ms;
    *ms_apply = s->kind == 1 ? ms : -1.0;
    *ms_transpose = s->kind == 1 ? 0.0 : -1.0;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return;
  }
  std::vector<cudaEvent_t> ev(2 * steps + 1);
  for (auto& e : ev) CK_CUDA(cudaEventCreate(&e));
  CK_CUDA(cudaStreamSynchronize(st));
  for (uint64_t k = 0; k < steps; ++k) {
    CK_CUDA(cudaEventRecord(ev[2 * k], st));
    launch_apply_only(s, st);
    CK_CUDA(cudaEventRecord(ev[2 * k + 1], st));
    launch_transpose_only(s, st);
  }
  CK_CUDA(cudaEventRecord(ev[2 * steps], st));
  CK_CUDA(cudaEventSynchronize(ev[2 * steps]));
  CK_CUDA(cudaGetLastError());
  double ta = 0.0, tt = 0.0;
  for (uint64_t k = 0; k < steps; ++k) {
    float x = 0.f, y = 0.f;
    CK_CUDA(cudaEventElapsedTime(&x, ev[2 * k], ev[2 * k + 1]));
    CK_CUDA(cudaEventElapsedTime(&y, ev[2 * k + 1], ev[2 * k + 2]));
    ta += x;
    tt += y;
  }
  float tot = 0.f;
  CK_CUDA(cudaEventElapsedTime(&tot, ev[0], ev[2 * steps]));
  for (auto& e : ev) cudaEventDestroy(e);
  *ms_total = tot;
  *ms_apply = ta;
  *ms_transpose = tt;
}


// ||Op v|| for an internal plain vector v (witness re-check, condest.hpp:284-289);
// v is zero outside the member's range, so the whole-operator norm is the member's.
static double op_norm(ck_session_s* s, int g, const double* v, cudaStream_t st) {
  if (s->kind == 0) {
    matrix_apply_perm(s->A, v, s->tmp.p, st);
    return device_norm(s->tmp.p, s->A->a.nrows_pad, s->A->s_red.p, st);
  }
  ck_lu_s* lu = s->lus[g];
  const int64_t n = s->seg_n[g];
  double* w = lu->work.p;
  CK_CUDA(cudaMemcpyAsync(w, v + s->seg_off[g], sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  double* xs[1] = {w};
  if (s->inv_dense)
    lu_dense_solve_launch(lu, w, false, st);  // the solver the loop evaluated its losses with
  else
    lu_solve_launch(lu, xs, 1, false, st);
  return device_norm(w, n, w + n, st);
}

// Final NormEstimate of column k = g * R + c (member g, restart column c),
// condest.hpp:278-296.
void session_result(ck_session_s* s, int k, ck_norm_result* res, double* witness) {
  if (k < 0 || k >= s->S * s->R) fail(CK_ERR_INVALID_ARGUMENT, "column out of range");
  const int g = k / s->R, c = k % s->R;
  cudaStream_t st = s->stream;
  Trace tr("session_result");
  pull_state(s);
  ColState& cs = s->h_st[k];
  const int64_t ncp = s->npad, off = s->seg_off[g], pad = s->seg_pad[g];
  double* xbest = s->tmp.p + s->thalf;  // plain copy of x_min (internal order)
  CK_CUDA(cudaMemsetAsync(xbest, 0, sizeof(double) * ncp, st));
  if (cs.pend) {  // x_{t+1} became the best but was never materialised
    k_materialise<<<grid256(pad), 256, 0, st>>>(s->S == 1 ? s->n : pad, s->R,
                                               col_buf(s, cs.cur, c) + off * s->R, cs.rad, cs.ndiv,
                                               xbest + off);
  } else {
    k_extract_x<<<grid256(pad), 256, 0, st>>>(pad, s->R, col_buf(s, cs.best, c) + off * s->R,
                                             xbest + off);
  }
  CK_CUDA(cudaGetLastError());
  res->iterations = cs.t;
  res->converged = cs.converged;
  res->_pad = 0;
  if (std::isfinite(cs.loss_min)) {
    res->value = std::exp(-cs.loss_min);
    if (s->dist) {
      dist_op_norm(s, xbest, st);  // this rank's part; ck_dist checks the combined norm
    } else {
      const double chk = op_norm(s, g, xbest, st);
      if (!(std::fabs(chk - res->value) <= 1e-12 * std::max(res->value, chk)))
        fail(CK_ERR_LOGIC, "norm estimate does not match ||Op witness||");
    }
  } else {
    res->value = 0.0;
    res->converged = 0;
  }
  tr.mark("witness check", st);
  if (witness) to_host(s, g, xbest, witness, st);
  tr.mark("witness D2H", st);
}

// x of buffer b / column c as a plain internal vector in `out` (npad doubles).
static void extract_x(ck_session_s* s, int b, int c, double* out, cudaStream_t st) {
  k_extract_x<<<grid256(s->npad), 256, 0, st>>>(s->npad, s->R, col_buf(s, b, c), out);
  CK_CUDA(cudaGetLastError());
}

// Observer mode (AdamObserver, condest.hpp:234-238, 268-271) for column 0:
// advances until column 0 evaluates a loss (or finishes) and reports the
// iteration's scalars and, optionally, x_{t+1} and x_min.
void session_step_observed(ck_session_s* s, ck_step_info* info, double* x, double* x_min) {
  cudaStream_t st = s->stream;
  s->observe_on = true;  // k_apply<R, true> from here on (no graphs in this mode)
  pull_state(s);
  const uint64_t n0 = s->h_st[0].n_loss;
  std::memset(info, 0, sizeof(*info));
  const int64_t ncp = s->npad;
  // scratch: y work vector is free between steps only for the explicit kind;
  // use dedicated buffers
  if (s->obs.n < 2 * ncp) s->obs.alloc(2 * ncp);
  double* xnext = s->obs.p;
  double* xm = s->obs.p + ncp;
  for (;;) {
    if (s->h_st[0].phase == PH_DONE) {
      info->phase = 2;
      info->t = s->h_st[0].t;
      info->loss_min = s->h_st[0].loss_min;
      return;
    }
    if (any_wait(s)) service_restarts(s);
    launch_apply_only(s, st);
    CK_CUDA(cudaGetLastError());
    pull_state(s);
    const bool reported = s->h_st[0].n_loss != n0;
    ColState cs = s->h_st[0];
    if (reported) {
      // x_{t+1} from the pre-step pair buffer, before the transpose half moves on
      CK_CUDA(cudaMemsetAsync(xnext, 0, sizeof(double) * ncp, st));
      k_materialise<<<grid256(ncp), 256, 0, st>>>(s->n, s->R, col_buf(s, cs.cur, 0), cs.rad, cs.ndiv,
                                                  xnext);
      if (!cs.pend) extract_x(s, cs.best, 0, xm, st);
    }
    launch_transpose_only(s, st);
    CK_CUDA(cudaGetLastError());
    pull_state(s);
    if (!reported) continue;
    info->t = cs.t_loss;
    info->loss = cs.loss;
    info->loss_min = cs.loss_min;
    info->x_dot_delta = cs.obs_xd;
    info->delta_norm = cs.obs_dn;
    info->phase = 0;
    if (x) to_host(s, 0, xnext, x, st);
    if (x_min) to_host(s, 0, cs.pend ? xnext : xm, x_min, st);
    return;
  }
}

}  // namespace ck
