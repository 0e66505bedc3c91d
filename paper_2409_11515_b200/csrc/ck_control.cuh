// Per-column control step of the Projected-Adam loop (condest.hpp:210-276),
// run by one thread after an operator application's reductions; shared by the
// explicit (ck_adam.cu) and inverse (ck_inverse.cu) loops.
#pragma once
#include <cmath>

#include "ck_session.h"

namespace ck {

__device__ __forceinline__ int pick_free(int cur, int best) {
  for (int b = 0; b < 3; ++b)
    if (b != cur && b != best) return b;
  return 0;
}

// DegenerateDirection handling, condest.hpp:213-219/242-256: spend one unit of
// the 16-restart budget or stop; the host supplies the re-randomised start.
__device__ __forceinline__ void on_degenerate(ColState& s, const Params& p) {
  if (s.budget == 0) {
    s.phase = PH_DONE;
    s.converged = 0;
    return;
  }
  s.budget -= 1;
  s.phase = (s.t >= p.max_iter) ? PH_DONE : PH_WAIT;
}

__device__ __forceinline__ void begin_iteration(ColState& s, const Params& p) {
  s.b1p = __dmul_rn(s.b1p, p.beta1);
  s.b2p = __dmul_rn(s.b2p, p.beta2);
  s.mc = 1.0 / (1.0 - s.b1p);
  s.vc = 1.0 / (1.0 - s.b2p);
}

// Control step after k_apply's reductions (thread 0 of the last CTA).
// nxt_shared >= 0: the iterate buffer every active column of the operator moves
// to in this step (explicit sweeps: the columns rotate their (x, delta) buffers
// in lockstep, so one wide load gathers all of them); < 0: the column picks its
// own free buffer (inverse loop, three buffers per column).
static __device__ __noinline__ void control_apply(ColState* sp, const Params* pp, double N, double yn,
                                                  int nxt_shared) {
  ColState& s = *sp;
  const Params& p = *pp;
  s.xnorm = N;
  s.ynorm = yn;
  if (s.phase == PH_PRO) {
    // First iteration after a (re)start: the gradient at x needs ||A x|| != 0.
    s.t += 1;
    if (yn == 0.0) {
      on_degenerate(s, p);
      return;
    }
    begin_iteration(s, p);
    s.inv_x2 = 1.0 / (N * N);
    s.inv_y2 = 1.0 / (yn * yn);
    s.ndiv = 1.0;
    s.mat = 0;
    if (nxt_shared >= 0) s.nxt = nxt_shared;
    s.phase = PH_GRAD;
    return;
  }
  // PH_APPLY: finish iteration t at x_{t+1} = x~/N.
  if (N == 0.0 || !isfinite(N)) {
    on_degenerate(s, p);
    return;
  }
  double den = yn / N;  // ||A x_{t+1}||
  if (den == 0.0) {
    on_degenerate(s, p);
    return;
  }
  double loss = -log(den);  // log||x_{t+1}|| - log||A x_{t+1}||, ||x_{t+1}|| = 1
  s.loss = loss;
  s.t_loss = s.t;
  s.n_loss += 1;
  bool improved = !isfinite(s.loss_min) || s.loss_min - loss > p.rel_tol * fabs(s.loss_min);
  s.since = improved ? 0 : s.since + 1;
  s.nxt = nxt_shared >= 0 ? nxt_shared : pick_free(s.cur, s.best);
  s.ndiv = N;
  if (loss < s.loss_min) {
    s.loss_min = loss;
    s.best = s.nxt;  // x_{t+1} lands there (k_transpose or the epilogue)
    s.pend = 1;
  }
  if (s.since >= p.patience) {
    s.phase = PH_DONE;
    s.converged = 1;
    return;
  }
  if (s.t >= p.max_iter) {
    s.phase = PH_DONE;
    return;
  }
  s.t += 1;
  begin_iteration(s, p);
  s.inv_x2 = 1.0;
  s.inv_y2 = 1.0 / (den * den);
  s.mat = 1;
  s.phase = PH_GRAD;
}

}  // namespace ck
