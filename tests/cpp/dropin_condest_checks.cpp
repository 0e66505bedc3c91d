// TEST: the reference's own condest / lu / error-bound call sites, compiled
// against the B200 headers of proj/include/condkit (they shadow the
// reference's condest.hpp, lu.hpp and error_bounds.hpp) and run on the device.
// The cases restate the reference unit tests' known answers and invariants
// (tests/test_condest.cpp, test_lu.cpp, test_error_bounds.cpp in the
// reference); each prints "ok <name>" or "FAIL <name>: why", and the exit
// status is the number of failures.
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "condkit/condest.hpp"
#include "condkit/error_bounds.hpp"
#include "condkit/lu.hpp"
#include "condkit/sparse.hpp"

using namespace condkit;

static int g_fail = 0;

static void check(const std::string& name, const std::function<std::string()>& body) {
  std::string why;
  try {
    why = body();
  } catch (const std::exception& e) {
    why = std::string("unexpected exception: ") + e.what();
  }
  if (why.empty()) {
    std::printf("ok %s\n", name.c_str());
  } else {
    std::printf("FAIL %s: %s\n", name.c_str(), why.c_str());
    ++g_fail;
  }
}

static SparseMatrix diag(const std::vector<double>& d) {
  std::vector<Triplet> t;
  for (std::size_t i = 0; i < d.size(); ++i) t.push_back({i, i, d[i]});
  return SparseMatrix::from_triplets(d.size(), d.size(), t);
}

static SparseMatrix grid(std::size_t g) {  // 5-point stencil, perturbed diagonal
  std::vector<Triplet> t;
  for (std::size_t r = 0; r < g; ++r)
    for (std::size_t c = 0; c < g; ++c) {
      const std::size_t i = r * g + c;
      t.push_back({i, i, 4.0 + 0.01 * static_cast<double>(i % 7)});
      if (r > 0) t.push_back({i, i - g, -1.0});
      if (r + 1 < g) t.push_back({i, i + g, -1.0});
      if (c > 0) t.push_back({i, i - 1, -1.0});
      if (c + 1 < g) t.push_back({i, i + 1, -1.0});
    }
  return SparseMatrix::from_triplets(g * g, g * g, t);
}

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static std::string near(double got, double want, double rel, const char* what) {
  if (std::abs(got - want) <= rel * std::abs(want)) return "";
  char buf[200];
  std::snprintf(buf, sizeof buf, "%s = %.17g, expected %.17g (rel %.1e)", what, got, want, rel);
  return buf;
}

struct ThirdPartyOracle : GradientOracle {  // an oracle with no device operator
  std::size_t dimension() const override { return 2; }
  double loss(const DenseVector&) const override { return 0.0; }
  DenseVector grad(const DenseVector& x) const override { return x; }
  DenseVector apply(const DenseVector& x) const override { return x; }
};

int main() {
  // test_condest.cpp:58-76: closed-form loss and gradient of diag(2, 1) at (s, s)
  check("loss_grad_closed_form", [] {
    SparseMatrix a = diag({2.0, 1.0});
    const double s = 1.0 / std::sqrt(2.0);
    ExplicitOracle o(a);
    std::string w = near(o.loss({s, s}), -0.5 * std::log(2.5), 1e-15, "loss");
    if (!w.empty()) return w;
    DenseVector g = o.grad({s, s});
    w = near(g[0], s * (1.0 - 4.0 / 2.5), 1e-14, "g0");
    if (!w.empty()) return w;
    return near(g[1], s * (1.0 - 1.0 / 2.5), 1e-14, "g1");
  });
  // test_condest.cpp:77-84: the zero operator maps every direction to zero
  check("degenerate_direction", [] {
    SparseMatrix z = SparseMatrix::from_triplets(2, 2, {{0, 0, 0.0}});
    if (!throws<DegenerateDirection>([&] { loss_explicit(z, {1.0, 0.0}); }))
      return std::string("loss_explicit did not throw DegenerateDirection");
    return std::string();
  });
  // test_condest.cpp:140-160: identity and diag(3, 1, 1e-3), both oracles
  check("identity_norm", [] {
    NormEstimate e = norm2(SparseMatrix::identity(5));
    if (!e.converged || e.iterations >= 2000) return std::string("identity run did not converge");
    return near(e.value, 1.0, 1e-12, "||I||");
  });
  check("diagonal_norms_both_oracles", [] {
    SparseMatrix a = diag({3.0, 1.0, 1e-3});
    std::string w = near(norm2(a).value, 3.0, 1e-9, "||A||");
    if (!w.empty()) return w;
    LUFactors f = lu_factorize(a);
    return near(inv_norm2(f).value, 1e3, 1e-9, "||A^-1||");
  });
  // test_condest.cpp:182-220: observer invariants of the trajectory
  for (int inverse = 0; inverse < 2; ++inverse) {
    check(inverse ? "observer_invariants_inverse" : "observer_invariants_explicit", [inverse] {
      SparseMatrix a = grid(6);
      LUFactors f = lu_factorize(a);
      ExplicitOracle ox(a);
      InverseOracle oi(f);
      const GradientOracle& o = inverse ? static_cast<const GradientOracle&>(oi) : ox;
      AdamConfig cfg;
      cfg.max_iter = 150;
      cfg.seed = 7;
      std::size_t last_t = 0, calls = 0;
      double last_min = std::numeric_limits<double>::infinity();
      std::string why;
      NormEstimate e = projected_adam(o, cfg, [&](const AdamState& st, const AdamStepInfo& info) {
        ++calls;
        double nx = 0.0;
        for (double v : st.x) nx += v * v;
        if (why.empty() && std::abs(std::sqrt(nx) - 1.0) > 1e-14) why = "||x|| != 1";
        if (why.empty() && std::abs(info.x_dot_delta) > 1e-13 * info.delta_norm + 1e-300)
          why = "x . delta not tangent";
        if (why.empty() && st.loss_min > last_min) why = "loss_min increased";
        if (why.empty() && st.t != last_t + 1) why = "t did not increment by one";
        last_min = st.loss_min;
        last_t = st.t;
      });
      if (!why.empty()) return why;
      if (calls != e.iterations) return std::string("observer calls != iterations");
      NormEstimate plain = projected_adam(o, cfg);
      if (plain.value != e.value || plain.iterations != e.iterations || plain.witness != e.witness)
        return std::string("observed run differs from the graph run");
      return std::string();
    });
  }
  // test_condest.cpp:222-272: bitwise determinism and restart seeding
  check("bitwise_reruns_and_restarts", [] {
    SparseMatrix a = grid(8);
    AdamConfig cfg;
    cfg.seed = 11;
    NormEstimate e1 = norm2(a, cfg), e2 = norm2(a, cfg);
    if (e1.value != e2.value || e1.witness != e2.witness || e1.iterations != e2.iterations)
      return std::string("reruns differ");
    ExplicitOracle o(a);
    NormEstimate best = estimate_norm(o, cfg, 3);
    double want = e1.value;
    for (std::uint64_t r = 1; r < 3; ++r) {
      AdamConfig c = cfg;
      c.seed = mix_seed(cfg.seed, r);
      want = std::max(want, projected_adam(o, c).value);
    }
    return near(best.value, want, 0.0, "estimate_norm vs best single run");
  });
  check("argument_validation", [] {
    SparseMatrix a = grid(3);
    ExplicitOracle o(a);
    if (!throws<std::invalid_argument>([&] { estimate_norm(o, AdamConfig{}, 0); }))
      return std::string("restarts = 0 accepted");
    ThirdPartyOracle t;
    if (!throws<std::invalid_argument>([&] { projected_adam(t); }))
      return std::string("an oracle without a device operator was accepted");
    SparseMatrix rect = SparseMatrix::from_triplets(2, 3, {{0, 0, 1.0}, {1, 2, 1.0}});
    if (!throws<DimensionMismatch>([&] { cond2(rect); })) return std::string("rectangular cond2");
    return std::string();
  });
  // test_condest.cpp:274-301: cond2 against known answers
  check("cond2_known_answers", [] {
    std::string w = near(cond2(SparseMatrix::identity(4)).kappa, 1.0, 1e-9, "kappa(I)");
    if (!w.empty()) return w;
    Cond2Result r = cond2(diag({10.0, 2.0, 1.0}));
    w = near(r.kappa, 10.0, 1e-9, "kappa(diag(10,2,1))");
    if (!w.empty()) return w;
    if (!r.factors || r.factors->row_perm.size() != 3) return std::string("factors missing");
    return std::string();
  });
  // test_condest.cpp:303-326: singular -> kappa = +inf; lu_factorize throws
  check("singular_matrices", [] {
    SparseMatrix s = SparseMatrix::from_triplets(3, 3, {{0, 0, 2.0}, {0, 1, 1.0}, {1, 2, 1.0},
                                                        {2, 2, 1.0}});
    Cond2Result r = cond2(s);
    if (!std::isinf(r.kappa) || r.factors) return std::string("kappa finite for a singular matrix");
    try {
      lu_factorize(s);
      return std::string("lu_factorize did not throw");
    } catch (const StructurallySingular& e) {
      if (e.column != 1) return std::string("wrong structurally singular column");
    }
    SparseMatrix t = SparseMatrix::from_triplets(2, 2, {{0, 0, 1.0}, {0, 1, 1.0}, {1, 0, 1.0},
                                                        {1, 1, 1.0}});
    if (!throws<NumericallySingular>([&] { lu_factorize(t); }))
      return std::string("rank-1 matrix factored");
    return std::string();
  });
  // test_lu.cpp:28-151: factor shape, reconstruction, solves
  check("lu_shape_and_solves", [] {
    SparseMatrix a = grid(5);
    LUFactors f = lu_factorize(a, 1e-12);
    const std::size_t n = a.nrows();
    // P A = L U with the unit diagonal implicit, |L| <= 1, U's diagonal first per row
    for (std::size_t i = 0; i < n; ++i) {
      auto uc = f.u.row_cols(i);
      if (uc.empty() || uc[0] != i) return std::string("U row without leading diagonal");
      for (double v : f.l.row_vals(i))
        if (std::abs(v) > 1.0) return std::string("|L| > 1");
    }
    for (std::size_t i = 0; i < n; ++i)
      for (std::size_t j = 0; j < n; ++j) {
        double lu = 0.0;
        for (std::size_t k = 0; k <= std::min(i, j); ++k)
          lu += (k == i ? 1.0 : f.l.coeff(i, k)) * f.u.coeff(k, j);
        if (std::abs(lu - a.coeff(f.row_perm[i], j)) > 1e-13 * 5.0) return std::string("P A != L U");
      }
    DenseVector b(n);
    for (std::size_t i = 0; i < n; ++i) b[i] = std::sin(1.0 + static_cast<double>(i));
    DenseVector x = lu_solve(f, b), ax = matvec(a, x);
    DenseVector y = lu_transpose_solve(f, b), aty = transpose_matvec(a, y);
    for (std::size_t i = 0; i < n; ++i)
      if (std::abs(ax[i] - b[i]) > 1e-13 || std::abs(aty[i] - b[i]) > 1e-13)
        return std::string("solve residual > 1e-13");
    LUFactors host;  // assembled on the host (solvers.hpp ilu0 style): no device solves
    host.row_perm = {0};
    if (!throws<std::invalid_argument>([&] { lu_solve(host, {1.0}); }))
      return std::string("host-assembled factors accepted");
    return std::string();
  });
  // error_bounds: frozen singularity_bound values (test_error_bounds.cpp:102-111) and
  // verify_solution cases (:222-325)
  check("bounds_and_verify", [] {
    const double want[] = {2.2204460492503136e-16, 2.220446049496832e-10,
                           2.220448514443379e-06, 2.2206925956553440e-04};
    const double kap[] = {1.0, 1e6, 1e10, 1e12};
    for (int k = 0; k < 4; ++k)
      if (singularity_bound(kap[k]) != want[k]) return std::string("singularity_bound value");
    if (singularity_bound(0x1p52) != 2.0) return std::string("pole value");
    SparseMatrix a = grid(6);
    const std::size_t n = a.nrows();
    DenseVector xs(n), xh(n);
    for (std::size_t i = 0; i < n; ++i) {
      xs[i] = std::cos(0.3 * static_cast<double>(i));
      xh[i] = xs[i] * (1.0 + 1e-9);
    }
    DenseVector b = matvec(a, xs);
    BoundsReport rep = verify_solution(a, xh, b);
    if (rep.verdict != Verdict::accepted || rep.kappa_supplied) return std::string("verdict");
    if (rep.to_kv().size() != 15) return std::string("kv record size");
    VerifyOptions opt;
    opt.kappa = 10.0;
    opt.a_norm = 6.0;
    BoundsReport sup = verify_solution(a, xh, b, opt);
    if (!sup.kappa_supplied || sup.kappa != 10.0 || sup.a_norm != 6.0) return std::string("supplied");
    if (!throws<ZeroRHS>([&] { verify_solution(a, xh, DenseVector(n, 0.0)); }))
      return std::string("ZeroRHS");
    if (!throws<ZeroSolution>([&] { verify_solution(a, DenseVector(n, 0.0), b); }))
      return std::string("ZeroSolution");
    return std::string();
  });
  std::printf("failures %d\n", g_fail);
  return g_fail;
}
