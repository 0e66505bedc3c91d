// condkit_b200.hpp -- standalone C++ API over the C ABI of condkit_b200.h
// (no reference headers needed). Link with libcondkit_b200.so.
//
// The drop-in for code written against the reference is proj/include/condkit/
// (condest.hpp, lu.hpp, error_bounds.hpp in namespace condkit, shadowing the
// reference's headers of the same names); this header is the same device
// functionality under namespace condkit_b200 for callers without them.
//
// Call sites keep their types: every function is a template over any CSR type
// with the accessors of condkit::SparseMatrix (nrows(), ncols(),
// row_offsets(), col_indices(), values(); sparse.hpp:105-111), so
//
//     condkit::SparseMatrix a = ...;                 // the reference's own type
//     auto r = condkit_b200::cond2(a);               // was condkit::cond2(a)
//
// runs on the B200. Results come back in the reference's shapes (NormEstimate,
// Cond2Result, BoundsReport) and failures raise the same exception kinds
// (DimensionMismatch, StructurallySingular, NumericallySingular, ZeroRHS,
// ZeroSolution, std::invalid_argument, std::logic_error).
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "condkit_b200.h"

namespace condkit_b200 {

using DenseVector = std::vector<double>;

struct DimensionMismatch : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StructurallySingular : std::runtime_error {
  StructurallySingular(const std::string& w, std::size_t c) : std::runtime_error(w), column(c) {}
  std::size_t column;
};
struct NumericallySingular : std::runtime_error {
  NumericallySingular(const std::string& w, std::size_t c, double p)
      : std::runtime_error(w), column(c), pivot(p) {}
  std::size_t column;
  double pivot;
};
struct ZeroRHS : std::invalid_argument {
  ZeroRHS() : std::invalid_argument("right-hand side has zero norm") {}
};
struct ZeroSolution : std::invalid_argument {
  ZeroSolution() : std::invalid_argument("candidate solution has zero norm") {}
};
struct ZeroColumn : std::runtime_error {
  explicit ZeroColumn(std::size_t j)
      : std::runtime_error("column " + std::to_string(j) + " has zero norm"), column(j) {}
  std::size_t column;
};
struct ZeroRow : std::runtime_error {
  explicit ZeroRow(std::size_t i)
      : std::runtime_error("row " + std::to_string(i) + " has zero norm"), row(i) {}
  std::size_t row;
};
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// AdamConfig (condest.hpp:39-48)
struct AdamConfig {
  double alpha = 0.05, beta1 = 0.9, beta2 = 0.999, eps_stab = 1e-8;
  std::size_t max_iter = 2000;
  std::uint64_t seed = 1;
  double rel_tol = 1e-12;
  std::size_t patience = 100;
};

// NormEstimate (condest.hpp:69-74)
struct NormEstimate {
  double value = 0.0;
  DenseVector witness;
  std::size_t iterations = 0;
  bool converged = false;
};

namespace detail {

inline void check(ck_status s, int64_t col = -1, double piv = 0.0) {
  if (s == CK_OK) return;
  std::string m = ck_last_error();
  switch (s) {
    case CK_ERR_DIMENSION: throw DimensionMismatch(m);
    case CK_ERR_INVALID_ARGUMENT: throw std::invalid_argument(m);
    case CK_ERR_LOGIC: throw std::logic_error(m);
    case CK_ERR_STRUCT_SINGULAR: throw StructurallySingular(m, static_cast<std::size_t>(col));
    case CK_ERR_NUM_SINGULAR: throw NumericallySingular(m, static_cast<std::size_t>(col), piv);
    case CK_ERR_ZERO_RHS: throw ZeroRHS();
    case CK_ERR_ZERO_SOLUTION: throw ZeroSolution();
    case CK_ERR_ZERO_COLUMN: throw ZeroColumn(static_cast<std::size_t>(col));
    case CK_ERR_ZERO_ROW: throw ZeroRow(static_cast<std::size_t>(col));
    default: throw DeviceError(m);
  }
}

inline ck_adam_cfg to_c(const AdamConfig& c) {
  return ck_adam_cfg{c.alpha, c.beta1, c.beta2, c.eps_stab, c.max_iter, c.seed, c.rel_tol,
                     c.patience};
}

inline NormEstimate from_c(const ck_norm_result& r, DenseVector w) {
  return NormEstimate{r.value, std::move(w), static_cast<std::size_t>(r.iterations),
                      r.converged != 0};
}

}  // namespace detail

// Device-resident operator (A and A^T), uploaded once from any CSR type.
class DeviceMatrix {
 public:
  template <class Csr>
  explicit DeviceMatrix(const Csr& a) : nrows_(a.nrows()), ncols_(a.ncols()) {
    const auto& ro = a.row_offsets();
    const auto& ci = a.col_indices();
    std::vector<int64_t> rp(ro.begin(), ro.end());
    std::vector<int32_t> c(ci.size());
    for (std::size_t k = 0; k < ci.size(); ++k) {
      if (ci[k] >= static_cast<std::size_t>(INT32_MAX)) throw DeviceError("column index >= 2^31");
      c[k] = static_cast<int32_t>(ci[k]);
    }
    ck_matrix h = nullptr;
    detail::check(ck_matrix_upload(static_cast<int64_t>(nrows_), static_cast<int64_t>(ncols_),
                                   rp.data(), c.data(), a.values().data(), &h));
    h_.reset(h);
  }
  ck_matrix handle() const { return h_.get(); }
  std::size_t nrows() const { return nrows_; }
  std::size_t ncols() const { return ncols_; }

 private:
  struct Free {
    void operator()(ck_matrix m) const { ck_matrix_free(m); }
  };
  std::unique_ptr<ck_matrix_s, Free> h_;
  std::size_t nrows_, ncols_;
};

// LUFactors (lu.hpp:42-47), device resident.
class LUFactors {
 public:
  explicit LUFactors(ck_lu h) : h_(h, Free{}) {
    int64_t n, kl, ku, bytes;
    detail::check(ck_lu_get_info(h, &n, &kl, &ku, &pivot_min, &bytes));
    n_ = static_cast<std::size_t>(n);
  }
  ck_lu handle() const { return h_.get(); }
  std::size_t size() const { return n_; }
  double pivot_min = 0.0;

 private:
  struct Free {
    void operator()(ck_lu f) const { ck_lu_free(f); }
  };
  std::shared_ptr<ck_lu_s> h_{nullptr, Free{}};
  std::size_t n_ = 0;
};

// matvec / transpose_matvec (sparse.hpp:212-242)
inline DenseVector matvec(const DeviceMatrix& a, const DenseVector& x) {
  if (x.size() != a.ncols()) throw DimensionMismatch("matvec: vector length != ncols");
  DenseVector y(a.nrows());
  detail::check(ck_spmv(a.handle(), x.data(), y.data()));
  return y;
}
inline DenseVector transpose_matvec(const DeviceMatrix& a, const DenseVector& x) {
  if (x.size() != a.nrows()) throw DimensionMismatch("transpose_matvec: vector length != nrows");
  DenseVector y(a.ncols());
  detail::check(ck_spmv_t(a.handle(), x.data(), y.data()));
  return y;
}

// projected_adam(ExplicitOracle(a), cfg) / norm2 (condest.hpp:184-297, 315-317)
inline NormEstimate norm2(const DeviceMatrix& a, const AdamConfig& cfg = {}) {
  ck_adam_cfg c = detail::to_c(cfg);
  ck_norm_result r{};
  DenseVector w(a.ncols());
  detail::check(ck_projected_adam(a.handle(), &c, &r, w.data()));
  return detail::from_c(r, std::move(w));
}

// estimate_norm(ExplicitOracle(a), cfg, restarts) (condest.hpp:301-312)
inline NormEstimate estimate_norm(const DeviceMatrix& a, const AdamConfig& cfg = {},
                                  std::size_t restarts = 3) {
  ck_adam_cfg c = detail::to_c(cfg);
  ck_norm_result r{};
  DenseVector w(a.ncols());
  detail::check(ck_estimate_norm(a.handle(), &c, restarts, &r, w.data()));
  return detail::from_c(r, std::move(w));
}

// lu_factorize (lu.hpp:55-177)
inline LUFactors lu_factorize(const DeviceMatrix& a, double pivot_tol = 1e-12) {
  ck_lu f = nullptr;
  int64_t col = -1;
  double piv = 0.0;
  detail::check(ck_lu_factorize(a.handle(), pivot_tol, &f, &col, &piv), col, piv);
  return LUFactors(f);
}

inline DenseVector lu_solve(const LUFactors& f, const DenseVector& b) {
  if (b.size() != f.size()) throw DimensionMismatch("lu_solve: rhs length != n");
  DenseVector x(f.size());
  detail::check(ck_lu_solve(f.handle(), b.data(), x.data()));
  return x;
}
inline DenseVector lu_transpose_solve(const LUFactors& f, const DenseVector& b) {
  if (b.size() != f.size()) throw DimensionMismatch("lu_transpose_solve: rhs length != n");
  DenseVector x(f.size());
  detail::check(ck_lu_transpose_solve(f.handle(), b.data(), x.data()));
  return x;
}

// inv_norm2 (condest.hpp:320-322) and estimate_norm over InverseOracle
inline NormEstimate inv_norm2(const LUFactors& f, const AdamConfig& cfg = {}) {
  ck_adam_cfg c = detail::to_c(cfg);
  ck_norm_result r{};
  DenseVector w(f.size());
  detail::check(ck_inv_projected_adam(f.handle(), &c, &r, w.data()));
  return detail::from_c(r, std::move(w));
}
inline NormEstimate estimate_inverse_norm(const LUFactors& f, const AdamConfig& cfg = {},
                                          std::size_t restarts = 3) {
  ck_adam_cfg c = detail::to_c(cfg);
  ck_norm_result r{};
  DenseVector w(f.size());
  detail::check(ck_inv_estimate_norm(f.handle(), &c, restarts, &r, w.data()));
  return detail::from_c(r, std::move(w));
}

// Cond2Result / cond2 (condest.hpp:324-365)
struct Cond2Result {
  double kappa = 0.0;
  NormEstimate operator_norm;
  NormEstimate inverse_norm;
  std::optional<LUFactors> factors;
};

inline Cond2Result cond2(const DeviceMatrix& a, const AdamConfig& cfg = {},
                         std::size_t restarts = 3, double pivot_tol = 1e-14) {
  if (a.nrows() != a.ncols()) throw DimensionMismatch("cond2: matrix must be square");
  Cond2Result res;
  res.operator_norm = estimate_norm(a, cfg, restarts);
  try {
    LUFactors f = lu_factorize(a, pivot_tol);
    AdamConfig ci = cfg;
    ci.seed = ck_mix_seed(cfg.seed, 0x1234);
    res.inverse_norm = estimate_inverse_norm(f, ci, restarts);
    res.kappa = res.operator_norm.value * res.inverse_norm.value;
    res.factors = std::move(f);
  } catch (const StructurallySingular&) {
    res.inverse_norm.value = std::numeric_limits<double>::infinity();
    res.kappa = std::numeric_limits<double>::infinity();
  } catch (const NumericallySingular&) {
    res.inverse_norm.value = std::numeric_limits<double>::infinity();
    res.kappa = std::numeric_limits<double>::infinity();
  }
  return res;
}

// error_bounds.hpp:59-217
struct Bounds {
  double lower = 0.0, upper = 0.0;
};
inline Bounds loose_bounds(double rn, double bn, double kappa) {
  Bounds b;
  detail::check(ck_loose_bounds(rn, bn, kappa, &b.lower, &b.upper));
  return b;
}
inline Bounds tight_bounds(double rn, double an, double xn, double kappa) {
  Bounds b;
  detail::check(ck_tight_bounds(rn, an, xn, kappa, &b.lower, &b.upper));
  return b;
}
inline double propagate_bound(double e) {
  double o = 0.0;
  detail::check(ck_propagate_bound(e, &o));
  return o;
}
inline constexpr double kEpsMach = 0x1p-53;
inline double singularity_bound(double kappa, double eps = kEpsMach) {
  double o = 0.0;
  detail::check(ck_singularity_bound(kappa, eps, &o));
  return o;
}

enum class Verdict { accepted, rejected, numerically_singular };

struct BoundsReport {
  double residual_norm = 0.0, b_norm = 0.0, a_norm = 0.0, xhat_norm = 0.0, kappa = 0.0;
  bool kappa_supplied = false;
  double loose_lower = 0.0, loose_upper = 0.0, tight_lower = 0.0, tight_upper = 0.0;
  double true_error_cap = 0.0, singularity_cap = 0.0, threshold = 0.0, eps_mach = kEpsMach;
  Verdict verdict = Verdict::rejected;
};

struct VerifyOptions {
  double threshold = 1e-7;
  std::optional<double> kappa, a_norm;
  double eps_mach = kEpsMach;
  AdamConfig adam;
  std::size_t restarts = 3;
  double pivot_tol = 1e-14;
};

inline BoundsReport verify_solution(const DeviceMatrix& a, const DenseVector& xhat,
                                    const DenseVector& b, const VerifyOptions& opt = {}) {
  if (a.nrows() != a.ncols()) throw DimensionMismatch("verify_solution: matrix must be square");
  if (xhat.size() != a.ncols()) throw DimensionMismatch("verify_solution: solution length");
  if (b.size() != a.nrows()) throw DimensionMismatch("verify_solution: rhs length");
  if (!(opt.threshold > 0.0)) throw std::invalid_argument("threshold must be > 0");
  BoundsReport rep;
  rep.threshold = opt.threshold;
  rep.eps_mach = opt.eps_mach;
  detail::check(ck_residual_norms(a.handle(), xhat.data(), b.data(), &rep.residual_norm,
                                  &rep.xhat_norm, &rep.b_norm));
  if (rep.xhat_norm == 0.0) throw ZeroSolution();
  if (rep.b_norm == 0.0) throw ZeroRHS();
  if (opt.kappa) {
    if (!(*opt.kappa >= 1.0)) throw std::invalid_argument("kappa must be >= 1");
    rep.kappa = *opt.kappa;
    rep.kappa_supplied = true;
    rep.a_norm = opt.a_norm ? *opt.a_norm : estimate_norm(a, opt.adam, opt.restarts).value;
  } else {
    Cond2Result c = cond2(a, opt.adam, opt.restarts, opt.pivot_tol);
    rep.kappa = std::max(1.0, c.kappa);
    rep.a_norm = opt.a_norm ? *opt.a_norm : c.operator_norm.value;
  }
  if (!(rep.a_norm > 0.0)) throw std::invalid_argument("operator norm must be > 0");
  Bounds lb = loose_bounds(rep.residual_norm, rep.b_norm, rep.kappa);
  rep.loose_lower = lb.lower;
  rep.loose_upper = lb.upper;
  Bounds tb = tight_bounds(rep.residual_norm, rep.a_norm, rep.xhat_norm, rep.kappa);
  rep.tight_lower = tb.lower;
  rep.tight_upper = tb.upper;
  rep.true_error_cap = propagate_bound(rep.tight_upper);
  rep.singularity_cap = singularity_bound(rep.kappa, rep.eps_mach);
  if (rep.kappa >= 1.0 / rep.eps_mach)
    rep.verdict = Verdict::numerically_singular;
  else
    rep.verdict = rep.tight_upper <= rep.threshold ? Verdict::accepted : Verdict::rejected;
  return rep;
}

// column_norms / column_scale / unscale_solution (sparse.hpp:244-293) with the
// norms on the device. column_scale returns the scaled values in the CSR
// order of `a` (the structure is unchanged) and the column norms D.
template <class Csr, class = decltype(std::declval<const Csr&>().row_offsets())>
DenseVector column_norms(const Csr& a) {
  DeviceMatrix d(a);
  DenseVector out(a.ncols());
  detail::check(ck_column_norms(d.handle(), out.data()));
  return out;
}
template <class Csr, class = decltype(std::declval<const Csr&>().row_offsets())>
std::pair<DenseVector, DenseVector> column_scale_values(const Csr& a) {
  DeviceMatrix d(a);
  const auto& ci = a.col_indices();
  std::vector<int32_t> c(ci.begin(), ci.end());
  DenseVector vals(a.values().size()), norms(a.ncols());
  int64_t zero = -1;
  detail::check(ck_column_scale(d.handle(), c.data(), a.values().data(), vals.data(), norms.data(),
                                &zero),
                zero);
  return {std::move(vals), std::move(norms)};
}
inline DenseVector unscale_solution(const DenseVector& y, const DenseVector& d) {
  if (y.size() != d.size()) throw DimensionMismatch("unscale_solution: length mismatch");
  DenseVector x(y.size());
  detail::check(ck_unscale_solution(static_cast<int64_t>(y.size()), y.data(), d.data(), x.data()));
  return x;
}

// Convenience overloads taking the CSR type directly (one upload per call).
template <class Csr, class = decltype(std::declval<const Csr&>().row_offsets())>
NormEstimate norm2(const Csr& a, const AdamConfig& cfg = {}) {
  return norm2(DeviceMatrix(a), cfg);
}
template <class Csr, class = decltype(std::declval<const Csr&>().row_offsets())>
NormEstimate estimate_norm(const Csr& a, const AdamConfig& cfg = {}, std::size_t restarts = 3) {
  return estimate_norm(DeviceMatrix(a), cfg, restarts);
}
template <class Csr, class = decltype(std::declval<const Csr&>().row_offsets())>
Cond2Result cond2(const Csr& a, const AdamConfig& cfg = {}, std::size_t restarts = 3,
                  double pivot_tol = 1e-14) {
  return cond2(DeviceMatrix(a), cfg, restarts, pivot_tol);
}
template <class Csr, class = decltype(std::declval<const Csr&>().row_offsets())>
BoundsReport verify_solution(const Csr& a, const DenseVector& xhat, const DenseVector& b,
                             const VerifyOptions& opt = {}) {
  return verify_solution(DeviceMatrix(a), xhat, b, opt);
}

}  // namespace condkit_b200
