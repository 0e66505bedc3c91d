#pragma once

// condkit/condest.hpp -- B200 build of the reference's spectral-norm and
// condition-number estimator interface (reference: proj/include/condkit/
// condest.hpp). Same declarations: DegenerateDirection (:35-37), AdamConfig
// (:39-48), AdamState (:51-56), AdamStepInfo (:61-65), AdamObserver (:67),
// NormEstimate (:69-74), GradientOracle (:78-85), loss_explicit /
// grad_explicit / grad_inverse (:88-123), ExplicitOracle / InverseOracle
// (:125-152), projected_adam (:184), estimate_norm (:301), norm2 / inv_norm2
// (:315-322), Cond2Result / cond2 (:324-365).
//
// The oracles are device operators: ExplicitOracle uploads A once (A and Aᵀ in
// the device layouts) and InverseOracle uses the device factors of
// lu_factorize. projected_adam / estimate_norm on them run the device-resident
// Projected-Adam loop (CUDA graphs, no per-iteration host traffic); an
// observer switches to the synchronous observed mode, which hands it x,
// x_min, t and loss_min each iteration (m and v stay on the device, so the
// observer's AdamState carries them empty). The host-vector methods
// (loss / grad / apply) are the slow per-call path for cross-checks.
// Oracles other than these two have no device operator and are rejected with
// std::invalid_argument: this build has no host fallback.

#include <cmath>
#include <cstdint>
#include <functional>
#include <limits>
#include <memory>
#include <optional>
#include <random>
#include <stdexcept>
#include <utility>
#include <vector>

#include "condkit/b200_device.hpp"
#include "condkit/lu.hpp"
#include "condkit/rng.hpp"
#include "condkit/sparse.hpp"

namespace condkit {

/// The operator maps the direction to zero; the device loop re-randomizes
/// internally, the host-vector oracle methods throw it.
struct DegenerateDirection : std::runtime_error {
  DegenerateDirection() : std::runtime_error("operator maps direction to zero") {}
};

struct AdamConfig {
  double alpha = 0.05;
  double beta1 = 0.9;
  double beta2 = 0.999;
  double eps_stab = 1e-8;
  std::size_t max_iter = 2000;
  std::uint64_t seed = 1;
  double rel_tol = 1e-12;
  std::size_t patience = 100;
};

struct AdamState {
  DenseVector x, m, v;
  std::size_t t = 0;
  double loss_min = std::numeric_limits<double>::infinity();
  DenseVector x_min;
};

struct AdamStepInfo {
  double x_dot_delta = 0.0;
  double delta_norm = 0.0;
  double loss = 0.0;
};

using AdamObserver = std::function<void(const AdamState&, const AdamStepInfo&)>;

struct NormEstimate {
  double value = 0.0;
  DenseVector witness;
  std::size_t iterations = 0;
  bool converged = false;
};

class GradientOracle {
 public:
  virtual ~GradientOracle() = default;
  virtual std::size_t dimension() const = 0;
  virtual double loss(const DenseVector& x) const = 0;
  virtual DenseVector grad(const DenseVector& x) const = 0;
  virtual DenseVector apply(const DenseVector& x) const = 0;
};

namespace b200 {

inline ck_adam_cfg to_c(const AdamConfig& c) {
  return ck_adam_cfg{c.alpha, c.beta1, c.beta2, c.eps_stab, static_cast<std::uint64_t>(c.max_iter),
                     c.seed, c.rel_tol, static_cast<std::uint64_t>(c.patience)};
}

inline NormEstimate from_c(const ck_norm_result& r, DenseVector witness) {
  NormEstimate e;
  e.value = r.value;
  e.witness = std::move(witness);
  e.iterations = static_cast<std::size_t>(r.iterations);
  e.converged = r.converged != 0;
  return e;
}

// The device reports a zero-norm image (condest.hpp:91,100,115,144) as an
// invalid argument naming DegenerateDirection.
inline void check_oracle(ck_status s) {
  if (s == CK_ERR_INVALID_ARGUMENT &&
      std::string(ck_last_error()).find("DegenerateDirection") != std::string::npos)
    throw DegenerateDirection();
  check(s);
}

}  // namespace b200

/// L(v) = log||v|| - log||Av|| on the device (one upload of A per call).
inline double loss_explicit(const SparseMatrix& a, const DenseVector& v) {
  if (v.size() != a.ncols()) throw DimensionMismatch("loss_explicit: vector length != ncols");
  b200::DeviceMatrix d(a);
  double l = 0.0;
  b200::check_oracle(ck_loss_explicit(d.handle(), v.data(), &l));
  return l;
}

/// grad L(v) = v/||v||^2 - AᵀA·v/||Av||^2 on the device (one upload per call).
inline DenseVector grad_explicit(const SparseMatrix& a, const DenseVector& v) {
  if (v.size() != a.ncols()) throw DimensionMismatch("grad_explicit: vector length != ncols");
  b200::DeviceMatrix d(a);
  DenseVector g(v.size());
  b200::check_oracle(ck_grad_explicit(d.handle(), v.data(), g.data()));
  return g;
}

/// grad L(x) for Op = A⁻¹ through the device factors.
inline DenseVector grad_inverse(const LUFactors& f, const DenseVector& x) {
  const b200::DeviceLU& d = b200::device_factors(f, "grad_inverse");
  if (x.size() != f.row_perm.size()) throw DimensionMismatch("grad_inverse: vector length != n");
  DenseVector g(x.size());
  b200::check_oracle(ck_grad_inverse(d.handle(), x.data(), g.data()));
  return g;
}

/// Op = A, uploaded to the device on first use and kept there for the
/// oracle's lifetime. Holds A by reference like the reference's oracle.
class ExplicitOracle : public GradientOracle {
 public:
  explicit ExplicitOracle(const SparseMatrix& a) : a_(a) {}
  std::size_t dimension() const override { return a_.ncols(); }
  double loss(const DenseVector& x) const override {
    check_len(x, "loss");
    double l = 0.0;
    b200::check_oracle(ck_loss_explicit(device().handle(), x.data(), &l));
    return l;
  }
  DenseVector grad(const DenseVector& x) const override {
    check_len(x, "grad");
    DenseVector g(x.size());
    b200::check_oracle(ck_grad_explicit(device().handle(), x.data(), g.data()));
    return g;
  }
  DenseVector apply(const DenseVector& x) const override {
    check_len(x, "apply");
    DenseVector y(a_.nrows());
    b200::check(ck_spmv(device().handle(), x.data(), y.data()));
    return y;
  }
  const SparseMatrix& matrix() const { return a_; }
  const b200::DeviceMatrix& device() const {
    if (!dev_) dev_ = b200::DeviceMatrix(a_);
    return dev_;
  }

 private:
  void check_len(const DenseVector& x, const char* who) const {
    if (x.size() != a_.ncols())
      throw DimensionMismatch(std::string("ExplicitOracle::") + who + ": vector length != ncols");
  }
  const SparseMatrix& a_;
  mutable b200::DeviceMatrix dev_;
};

/// Op = A⁻¹ through the device factors; the factors must outlive the oracle.
class InverseOracle : public GradientOracle {
 public:
  explicit InverseOracle(const LUFactors& f) : f_(f) {}
  std::size_t dimension() const override { return f_.row_perm.size(); }
  double loss(const DenseVector& x) const override {
    check_len(x, "loss");
    double l = 0.0;
    b200::check_oracle(ck_loss_inverse(handle(), x.data(), &l));
    return l;
  }
  DenseVector grad(const DenseVector& x) const override { return grad_inverse(f_, x); }
  DenseVector apply(const DenseVector& x) const override { return lu_solve(f_, x); }
  const LUFactors& factors() const { return f_; }
  ck_lu handle() const { return b200::device_factors(f_, "InverseOracle").handle(); }

 private:
  void check_len(const DenseVector& x, const char* who) const {
    if (x.size() != dimension())
      throw DimensionMismatch(std::string("InverseOracle::") + who + ": vector length != n");
  }
  const LUFactors& f_;
};

namespace b200 {

// The device operator behind an oracle: 1 = explicit (matrix), 2 = inverse.
struct OracleRef {
  int kind = 0;
  ck_matrix a = nullptr;
  ck_lu f = nullptr;
};

inline OracleRef device_oracle(const GradientOracle& o, const char* who) {
  if (auto* e = dynamic_cast<const ExplicitOracle*>(&o)) return {1, e->device().handle(), nullptr};
  if (auto* i = dynamic_cast<const InverseOracle*>(&o)) return {2, nullptr, i->handle()};
  throw std::invalid_argument(std::string(who) +
                              ": the B200 build runs ExplicitOracle and InverseOracle "
                              "(device operators); other oracles have no device path");
}

// Observed mode: one device loop trip per call, the observer sees each one.
inline NormEstimate observed_run(const OracleRef& d, std::size_t n, const AdamConfig& cfg,
                                 const AdamObserver& observer) {
  const ck_adam_cfg c = to_c(cfg);
  const std::uint64_t seed = cfg.seed;
  ck_session s = nullptr;
  check(d.kind == 1 ? ck_session_create(d.a, &c, &seed, 1, &s)
                    : ck_session_create_inverse(d.f, &c, &seed, 1, &s));
  std::unique_ptr<ck_session_s, void (*)(ck_session)> guard(s, [](ck_session p) {
    ck_session_free(p);
  });
  AdamState st;
  st.x.resize(n);
  st.x_min.resize(n);
  for (;;) {
    ck_step_info info{};
    check(ck_session_step_observed(s, &info, st.x.data(), st.x_min.data()));
    if (info.phase == 2) break;
    st.t = static_cast<std::size_t>(info.t);
    st.loss_min = info.loss_min;
    AdamStepInfo si;
    si.x_dot_delta = info.x_dot_delta;
    si.delta_norm = info.delta_norm;
    si.loss = info.loss;
    observer(st, si);
  }
  ck_norm_result r{};
  DenseVector w(n);
  check(ck_session_result(s, 0, &r, w.data()));
  return from_c(r, std::move(w));
}

}  // namespace b200

/// Minimizes the oracle loss over the unit sphere (condest.hpp:175-297) with
/// the device-resident loop: same start vector (mt19937_64(cfg.seed)), same
/// update, projection, renormalisation, patience, best tracking and
/// degenerate-direction restarts; the witness re-check raises
/// std::logic_error as in the reference.
inline NormEstimate projected_adam(const GradientOracle& oracle, const AdamConfig& cfg = {},
                                   const AdamObserver& observer = {}) {
  const std::size_t n = oracle.dimension();
  if (n == 0) throw std::invalid_argument("projected_adam: zero-dimensional operator");
  const b200::OracleRef d = b200::device_oracle(oracle, "projected_adam");
  if (observer) return b200::observed_run(d, n, cfg, observer);
  const ck_adam_cfg c = b200::to_c(cfg);
  ck_norm_result r{};
  DenseVector w(n);
  b200::check(d.kind == 1 ? ck_projected_adam(d.a, &c, &r, w.data())
                          : ck_inv_projected_adam(d.f, &c, &r, w.data()));
  return b200::from_c(r, std::move(w));
}

/// Best of `restarts` runs seeded cfg.seed, mix_seed(cfg.seed, r)
/// (condest.hpp:299-312); the restarts run concurrently on the device.
inline NormEstimate estimate_norm(const GradientOracle& oracle, const AdamConfig& cfg = {},
                                  std::size_t restarts = 3) {
  if (restarts == 0) throw std::invalid_argument("estimate_norm: restarts must be >= 1");
  const std::size_t n = oracle.dimension();
  const b200::OracleRef d = b200::device_oracle(oracle, "estimate_norm");
  const ck_adam_cfg c = b200::to_c(cfg);
  ck_norm_result r{};
  DenseVector w(n);
  b200::check(d.kind == 1 ? ck_estimate_norm(d.a, &c, restarts, &r, w.data())
                          : ck_inv_estimate_norm(d.f, &c, restarts, &r, w.data()));
  return b200::from_c(r, std::move(w));
}

inline NormEstimate norm2(const SparseMatrix& a, const AdamConfig& cfg = {}) {
  return projected_adam(ExplicitOracle(a), cfg);
}

inline NormEstimate inv_norm2(const LUFactors& f, const AdamConfig& cfg = {}) {
  return projected_adam(InverseOracle(f), cfg);
}

struct Cond2Result {
  double kappa = 0.0;          // +infinity when the factorization breaks down
  NormEstimate operator_norm;  // ||A||_2
  NormEstimate inverse_norm;   // ||A⁻¹||_2
  std::optional<LUFactors> factors;
};

namespace b200 {

// cond2 over an uploaded operator (shared with verify_solution).
inline Cond2Result cond2_on(const ExplicitOracle& forward, const AdamConfig& cfg,
                            std::size_t restarts, double pivot_tol) {
  Cond2Result result;
  result.operator_norm = estimate_norm(forward, cfg, restarts);
  try {
    LUFactors f = factorize(forward.device(), pivot_tol);
    AdamConfig cfg_inv = cfg;
    cfg_inv.seed = mix_seed(cfg.seed, 0x1234);
    result.inverse_norm = estimate_norm(InverseOracle(f), cfg_inv, restarts);
    result.kappa = result.operator_norm.value * result.inverse_norm.value;
    result.factors = std::move(f);
  } catch (const StructurallySingular&) {
    result.inverse_norm.value = std::numeric_limits<double>::infinity();
    result.kappa = std::numeric_limits<double>::infinity();
  } catch (const NumericallySingular&) {
    result.inverse_norm.value = std::numeric_limits<double>::infinity();
    result.kappa = std::numeric_limits<double>::infinity();
  }
  return result;
}

}  // namespace b200

/// kappa2(A) = ||A||_2 ||A⁻¹||_2 (condest.hpp:331-365): A uploaded once for
/// the forward estimate and the factorisation, the inverse restarts seeded
/// mix_seed(cfg.seed, 0x1234), a factorisation breakdown reported as kappa = +inf.
inline Cond2Result cond2(const SparseMatrix& a, const AdamConfig& cfg = {},
                         std::size_t restarts = 3, double pivot_tol = 1e-14) {
  if (a.nrows() != a.ncols()) throw DimensionMismatch("cond2: matrix must be square");
  return b200::cond2_on(ExplicitOracle(a), cfg, restarts, pivot_tol);
}

}  // namespace condkit
