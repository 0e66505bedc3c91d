// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Exposes the UNMODIFIED reference library (header-only condkit, compiled in
// place from /root/reference/proj/include by oracle/Makefile) through the same
// C signatures as condkit_oracle.h, with the prefix `ckref_` instead of `cko_`.
// Nothing here restates an algorithm: every function converts arguments and
// calls the reference symbol named in its comment. The resulting
// oracle/_ref/libcondkit_ref.so is git-ignored and travels to the GPU box with
// the gpurun snapshot; it pins the plain-C restatement (condkit_oracle.c) and
// serves as bench.py's `--impl reference` CPU arm.
#include <condkit/condest.hpp>
#include <condkit/error_bounds.hpp>
#include <condkit/lu.hpp>
#include <condkit/rng.hpp>
#include <condkit/sparse.hpp>
#include <condkit/bench.hpp>
#include <condkit/matrix_market.hpp>
#include <fstream>

#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include <chrono>

#include "condkit_oracle.h"

using ckref_adam_cfg = cko_adam_cfg;
using ckref_norm_result = cko_norm_result;
using ckref_bounds_report = cko_bounds_report;
using ckref_verify_options = cko_verify_options;

using namespace condkit;

namespace {

SparseMatrix to_sparse(int64_t nr, int64_t nc, const int64_t* rp, const int32_t* ci,
                       const double* va) {
  std::vector<std::size_t> off(rp, rp + nr + 1);
  std::vector<std::size_t> cols(ci, ci + rp[nr]);
  std::vector<double> vals(va, va + rp[nr]);
  return SparseMatrix(static_cast<std::size_t>(nr), static_cast<std::size_t>(nc), std::move(off),
                      std::move(cols), std::move(vals));
}

AdamConfig to_cfg(const ckref_adam_cfg* c) {
  AdamConfig a;
  a.alpha = c->alpha;
  a.beta1 = c->beta1;
  a.beta2 = c->beta2;
  a.eps_stab = c->eps_stab;
  a.max_iter = c->max_iter;
  a.seed = c->seed;
  a.rel_tol = c->rel_tol;
  a.patience = c->patience;
  return a;
}

void put(const NormEstimate& e, ckref_norm_result* r, double* witness) {
  r->value = e.value;
  r->iterations = e.iterations;
  r->converged = e.converged ? 1 : 0;
  if (witness) std::memcpy(witness, e.witness.data(), e.witness.size() * sizeof(double));
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const DimensionMismatch&) {
    return 1;
  } catch (const StructurallySingular&) {
    return 4;
  } catch (const NumericallySingular&) {
    return 5;
  } catch (const ZeroRHS&) {
    return 6;
  } catch (const ZeroSolution&) {
    return 7;
  } catch (const std::invalid_argument&) {
    return 2;
  } catch (const std::logic_error&) {
    return 3;
  } catch (const DegenerateDirection&) {
    return 100;
  }
}

}  // namespace

struct ckref_lu {
  LUFactors f;
};

extern "C" {

uint64_t ckref_mix_seed(uint64_t base, uint64_t stream) { return mix_seed(base, stream); }

void ckref_mt_draws(uint64_t seed, int64_t count, uint64_t* out) {
  std::mt19937_64 g(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = g();
}

void ckref_random_unit_vectors(uint64_t seed, int64_t n, int64_t count, double* out) {
  std::mt19937_64 g(seed);
  for (int64_t c = 0; c < count; ++c) {
    DenseVector x = random_unit_vector(static_cast<std::size_t>(n), g);
    std::memcpy(out + c * n, x.data(), static_cast<std::size_t>(n) * sizeof(double));
  }
}

void ckref_uniform_in(uint64_t seed, int64_t count, double lo, double hi, double* out) {
  std::mt19937_64 g(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = uniform_in(g, lo, hi);
}

double ckref_two_norm(int64_t n, const double* v) { return two_norm(DenseVector(v, v + n)); }

double ckref_dot(int64_t n, const double* a, const double* b) {
  return dot(DenseVector(a, a + n), DenseVector(b, b + n));
}

double ckref_compensated_norm(int64_t n, const double* v) {
  return detail::compensated_norm(DenseVector(v, v + n));
}

void ckref_matvec(int64_t nr, int64_t nc, const int64_t* rp, const int32_t* ci, const double* va,
                  const double* x, double* y) {
  DenseVector r = matvec(to_sparse(nr, nc, rp, ci, va), DenseVector(x, x + nc));
  std::memcpy(y, r.data(), r.size() * sizeof(double));
}

void ckref_transpose_matvec(int64_t nr, int64_t nc, const int64_t* rp, const int32_t* ci,
                            const double* va, const double* x, double* y) {
  DenseVector r = transpose_matvec(to_sparse(nr, nc, rp, ci, va), DenseVector(x, x + nr));
  std::memcpy(y, r.data(), r.size() * sizeof(double));
}

// generate_illconditioned (bench.hpp:35-127) with the default spec at (n, seed):
// the two-plateau matrix of acceptance criterion 5. rp == nullptr: nnz only.
int64_t ckref_generate_illconditioned(int64_t n, uint64_t seed, int64_t* rp, int32_t* ci,
                                      double* va) {
  GeneratorSpec g;
  g.n = (std::size_t)n;
  g.seed = seed;
  SparseMatrix a = generate_illconditioned(g);
  if (rp) {
    for (std::size_t i = 0; i <= a.nrows(); ++i) rp[i] = (int64_t)a.row_offsets()[i];
    for (std::size_t k = 0; k < a.nnz(); ++k) {
      ci[k] = (int32_t)a.col_indices()[k];
      va[k] = a.values()[k];
    }
  }
  return (int64_t)a.nnz();
}

// read_matrix_market (matrix_market.hpp:118-209) of a file: rp == nullptr
// returns nnz (and the shape); -1 on a parse error.
int64_t ckref_read_matrix_market(const char* path, int64_t* nr, int64_t* nc, int64_t* rp, int32_t* ci,
                                 double* va) {
  try {
    std::ifstream in(path);
    SparseMatrix a = read_matrix_market(in);
    *nr = (int64_t)a.nrows();
    *nc = (int64_t)a.ncols();
    if (rp) {
      for (std::size_t i = 0; i <= a.nrows(); ++i) rp[i] = (int64_t)a.row_offsets()[i];
      for (std::size_t k = 0; k < a.nnz(); ++k) {
        ci[k] = (int32_t)a.col_indices()[k];
        va[k] = a.values()[k];
      }
    }
    return (int64_t)a.nnz();
  } catch (...) {
    return -1;
  }
}

void ckref_column_norms(int64_t nr, int64_t nc, const int64_t* rp, const int32_t* ci,
                        const double* va, double* out) {
  DenseVector r = column_norms(to_sparse(nr, nc, rp, ci, va));
  std::memcpy(out, r.data(), r.size() * sizeof(double));
}

// row_scale's factors: two_norm of each row (sparse.hpp:295-311)
void ckref_row_norms(int64_t nr, const int64_t* rp, const double* va, double* out) {
  for (int64_t i = 0; i < nr; ++i) out[i] = two_norm(DenseVector(va + rp[i], va + rp[i + 1]));
}

int ckref_loss_explicit(int64_t nr, int64_t nc, const int64_t* rp, const int32_t* ci,
                        const double* va, const double* x, double* loss) {
  SparseMatrix a = to_sparse(nr, nc, rp, ci, va);
  return guard([&] { *loss = loss_explicit(a, DenseVector(x, x + nc)); });
}

int ckref_grad_explicit(int64_t nr, int64_t nc, const int64_t* rp, const int32_t* ci,
                        const double* va, const double* x, double* g) {
  SparseMatrix a = to_sparse(nr, nc, rp, ci, va);
  return guard([&] {
    DenseVector r = grad_explicit(a, DenseVector(x, x + nc));
    std::memcpy(g, r.data(), r.size() * sizeof(double));
  });
}

int ckref_projected_adam_explicit(int64_t nr, int64_t nc, const int64_t* rp, const int32_t* ci,
                                  const double* va, const ckref_adam_cfg* cfg,
                                  ckref_norm_result* res, double* witness, double* loss_trace) {
  SparseMatrix a = to_sparse(nr, nc, rp, ci, va);
  ExplicitOracle ox(a);
  AdamConfig c = to_cfg(cfg);
  if (loss_trace)
    for (uint64_t i = 0; i < cfg->max_iter; ++i) loss_trace[i] = std::nan("");
  AdamObserver obs;
  if (loss_trace)
    obs = [&](const AdamState& st, const AdamStepInfo& info) { loss_trace[st.t - 1] = info.loss; };
  return guard([&] { put(projected_adam(ox, c, obs), res, witness); });
}

int ckref_estimate_norm_explicit(int64_t nr, int64_t nc, const int64_t* rp, const int32_t* ci,
                                 const double* va, const ckref_adam_cfg* cfg, uint64_t restarts,
                                 ckref_norm_result* res, double* witness) {
  SparseMatrix a = to_sparse(nr, nc, rp, ci, va);
  ExplicitOracle ox(a);
  return guard([&] { put(estimate_norm(ox, to_cfg(cfg), restarts), res, witness); });
}

int ckref_lu_factorize(int64_t n, const int64_t* rp, const int32_t* ci, const double* va,
                       double pivot_tol, ckref_lu** out, int64_t* fail_col, double* fail_pivot) {
  SparseMatrix a = to_sparse(n, n, rp, ci, va);
  try {
    auto* h = new ckref_lu{lu_factorize(a, pivot_tol)};
    *out = h;
    return 0;
  } catch (const StructurallySingular& e) {
    if (fail_col) *fail_col = static_cast<int64_t>(e.column);
    if (fail_pivot) *fail_pivot = 0.0;
    return 4;
  } catch (const NumericallySingular& e) {
    if (fail_col) *fail_col = static_cast<int64_t>(e.column);
    if (fail_pivot) *fail_pivot = e.pivot;
    return 5;
  } catch (const DimensionMismatch&) {
    return 1;
  }
}

void ckref_lu_free(ckref_lu* f) { delete f; }

void ckref_lu_info(const ckref_lu* f, int64_t* n, int64_t* nnz_l, int64_t* nnz_u, double* pmin) {
  *n = static_cast<int64_t>(f->f.row_perm.size());
  *nnz_l = static_cast<int64_t>(f->f.l.nnz());
  *nnz_u = static_cast<int64_t>(f->f.u.nnz());
  *pmin = f->f.pivot_min;
}

void ckref_lu_export(const ckref_lu* f, int64_t* l_rp, int32_t* l_ci, double* l_va,
                     int64_t* u_rp, int32_t* u_ci, double* u_va, int64_t* row_perm) {
  auto dump = [](const SparseMatrix& m, int64_t* rp, int32_t* ci, double* va) {
    for (std::size_t i = 0; i < m.row_offsets().size(); ++i)
      rp[i] = static_cast<int64_t>(m.row_offsets()[i]);
    for (std::size_t k = 0; k < m.nnz(); ++k) {
      ci[k] = static_cast<int32_t>(m.col_indices()[k]);
      va[k] = m.values()[k];
    }
  };
  dump(f->f.l, l_rp, l_ci, l_va);
  dump(f->f.u, u_rp, u_ci, u_va);
  for (std::size_t k = 0; k < f->f.row_perm.size(); ++k)
    row_perm[k] = static_cast<int64_t>(f->f.row_perm[k]);
}

int ckref_lu_solve(const ckref_lu* f, const double* b, double* x) {
  std::size_t n = f->f.row_perm.size();
  return guard([&] {
    DenseVector r = lu_solve(f->f, DenseVector(b, b + n));
    std::memcpy(x, r.data(), n * sizeof(double));
  });
}

int ckref_lu_transpose_solve(const ckref_lu* f, const double* b, double* x) {
  std::size_t n = f->f.row_perm.size();
  return guard([&] {
    DenseVector r = lu_transpose_solve(f->f, DenseVector(b, b + n));
    std::memcpy(x, r.data(), n * sizeof(double));
  });
}

int ckref_loss_inverse(const ckref_lu* f, const double* x, double* loss) {
  InverseOracle o(f->f);
  std::size_t n = f->f.row_perm.size();
  return guard([&] { *loss = o.loss(DenseVector(x, x + n)); });
}

int ckref_grad_inverse(const ckref_lu* f, const double* x, double* g) {
  std::size_t n = f->f.row_perm.size();
  return guard([&] {
    DenseVector r = grad_inverse(f->f, DenseVector(x, x + n));
    std::memcpy(g, r.data(), n * sizeof(double));
  });
}

int ckref_projected_adam_inverse(const ckref_lu* f, const ckref_adam_cfg* cfg,
                                 ckref_norm_result* res, double* witness, double* loss_trace) {
  InverseOracle o(f->f);
  if (loss_trace)
    for (uint64_t i = 0; i < cfg->max_iter; ++i) loss_trace[i] = std::nan("");
  AdamObserver obs;
  if (loss_trace)
    obs = [&](const AdamState& st, const AdamStepInfo& info) { loss_trace[st.t - 1] = info.loss; };
  return guard([&] { put(projected_adam(o, to_cfg(cfg), obs), res, witness); });
}

int ckref_estimate_norm_inverse(const ckref_lu* f, const ckref_adam_cfg* cfg, uint64_t restarts,
                                ckref_norm_result* res, double* witness) {
  InverseOracle o(f->f);
  return guard([&] { put(estimate_norm(o, to_cfg(cfg), restarts), res, witness); });
}

int ckref_cond2(int64_t n, const int64_t* rp, const int32_t* ci, const double* va,
                const ckref_adam_cfg* cfg, uint64_t restarts, double pivot_tol, double* kappa,
                ckref_norm_result* fwd, ckref_norm_result* inv, int32_t* has_factors) {
  SparseMatrix a = to_sparse(n, n, rp, ci, va);
  return guard([&] {
    Cond2Result r = cond2(a, to_cfg(cfg), restarts, pivot_tol);
    *kappa = r.kappa;
    put(r.operator_norm, fwd, nullptr);
    put(r.inverse_norm, inv, nullptr);
    *has_factors = r.factors.has_value() ? 1 : 0;
  });
}

int ckref_loose_bounds(double rn, double bn, double kappa, double* lo, double* hi) {
  return guard([&] {
    Bounds b = loose_bounds(rn, bn, kappa);
    *lo = b.lower;
    *hi = b.upper;
  });
}

int ckref_tight_bounds(double rn, double an, double xn, double kappa, double* lo, double* hi) {
  return guard([&] {
    Bounds b = tight_bounds(rn, an, xn, kappa);
    *lo = b.lower;
    *hi = b.upper;
  });
}

int ckref_propagate_bound(double e, double* out) {
  return guard([&] { *out = propagate_bound(e); });
}

int ckref_singularity_bound(double kappa, double eps, double* out) {
  return guard([&] { *out = singularity_bound(kappa, eps); });
}

int ckref_verify_solution(int64_t n, const int64_t* rp, const int32_t* ci, const double* va,
                          const double* xhat, const double* b, const ckref_verify_options* opt,
                          ckref_bounds_report* rep) {
  SparseMatrix a = to_sparse(n, n, rp, ci, va);
  VerifyOptions o;
  o.threshold = opt->threshold;
  if (opt->has_kappa) o.kappa = opt->kappa;
  if (opt->has_a_norm) o.a_norm = opt->a_norm;
  o.eps_mach = opt->eps_mach;
  o.adam = to_cfg(&opt->adam);
  o.restarts = opt->restarts;
  o.pivot_tol = opt->pivot_tol;
  return guard([&] {
    BoundsReport r = verify_solution(a, DenseVector(xhat, xhat + n), DenseVector(b, b + n), o);
    rep->residual_norm = r.residual_norm;
    rep->b_norm = r.b_norm;
    rep->a_norm = r.a_norm;
    rep->xhat_norm = r.xhat_norm;
    rep->kappa = r.kappa;
    rep->kappa_supplied = r.kappa_supplied ? 1 : 0;
    rep->verdict = static_cast<int32_t>(r.verdict);
    rep->loose_lower = r.loose_lower;
    rep->loose_upper = r.loose_upper;
    rep->tight_lower = r.tight_lower;
    rep->tight_upper = r.tight_upper;
    rep->true_error_cap = r.true_error_cap;
    rep->singularity_cap = r.singularity_cap;
    rep->threshold = r.threshold;
    rep->eps_mach = r.eps_mach;
  });
}

// Throughput mode for bench.py's reference arm: `nthreads` independent
// projected_adam runs (seeds cfg.seed, mix_seed(seed,1), ...) on std::threads,
// each limited to cfg->max_iter iterations (SPEC.md:320 permits concurrent
// restarts). Returns the wall seconds and total iterations.
int ckref_throughput_explicit(int64_t nr, int64_t nc, const int64_t* rp, const int32_t* ci,
                              const double* va, const ckref_adam_cfg* cfg, int32_t nthreads,
                              double* seconds, uint64_t* total_iterations) {
  SparseMatrix a = to_sparse(nr, nc, rp, ci, va);
  ExplicitOracle ox(a);
  std::vector<uint64_t> iters(static_cast<std::size_t>(nthreads), 0);
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int32_t k = 0; k < nthreads; ++k) {
    pool.emplace_back([&, k] {
      AdamConfig c = to_cfg(cfg);
      c.seed = k == 0 ? cfg->seed : mix_seed(cfg->seed, static_cast<uint64_t>(k));
      try {
        iters[static_cast<std::size_t>(k)] = projected_adam(ox, c).iterations;
      } catch (...) {
      }
    });
  }
  for (auto& t : pool) t.join();
  *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  uint64_t tot = 0;
  for (auto v : iters) tot += v;
  *total_iterations = tot;
  return 0;
}

// Steady-state iteration rate of the reference projected_adam (condest.hpp:210-276)
// for bench.py's CPU arm: `nthreads` independent runs (seeds cfg.seed,
// mix_seed(seed, k)) on std::threads, each limited to `iters` iterations; the
// rate of each run is measured between its first and last observer callback
// (so setup -- x0 draw, matrix conversion -- is excluded). Returns the summed
// iterations/s, the iterations timed and the wall seconds of the timed spans.
int ckref_time_iterations(int64_t nr, int64_t nc, const int64_t* rp, const int32_t* ci,
                          const double* va, const ckref_adam_cfg* cfg, int32_t nthreads,
                          uint64_t iters, double* rate, uint64_t* timed_iters, double* span) {
  SparseMatrix a = to_sparse(nr, nc, rp, ci, va);
  ExplicitOracle ox(a);
  std::vector<double> rates(static_cast<std::size_t>(nthreads), 0.0), spans(rates.size(), 0.0);
  std::vector<uint64_t> counts(rates.size(), 0);
  std::vector<std::thread> pool;
  for (int32_t k = 0; k < nthreads; ++k) {
    pool.emplace_back([&, k] {
      AdamConfig c = to_cfg(cfg);
      c.seed = k == 0 ? cfg->seed : mix_seed(cfg->seed, static_cast<uint64_t>(k));
      c.max_iter = iters;
      c.patience = iters + 1;
      using clk = std::chrono::steady_clock;
      clk::time_point first{}, last{};
      uint64_t seen = 0;
      AdamObserver obs = [&](const AdamState&, const AdamStepInfo&) {
        last = clk::now();
        if (seen == 0) first = last;
        ++seen;
      };
      try {
        projected_adam(ox, c, obs);
      } catch (...) {
      }
      if (seen >= 2) {
        double sec = std::chrono::duration<double>(last - first).count();
        rates[static_cast<std::size_t>(k)] = static_cast<double>(seen - 1) / sec;
        spans[static_cast<std::size_t>(k)] = sec;
        counts[static_cast<std::size_t>(k)] = seen - 1;
      }
    });
  }
  for (auto& t : pool) t.join();
  double r = 0.0, sp = 0.0;
  uint64_t n = 0;
  for (std::size_t k = 0; k < rates.size(); ++k) {
    r += rates[k];
    sp = std::max(sp, spans[k]);
    n += counts[k];
  }
  *rate = r;
  *timed_iters = n;
  *span = sp;
  return 0;
}

}  // extern "C"
