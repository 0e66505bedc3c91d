#pragma once

// condkit/lu.hpp -- B200 build of the reference's sparse LU interface
// (reference: proj/include/condkit/lu.hpp). Same types and signatures:
// StructurallySingular / NumericallySingular (lu.hpp:24-40), LUFactors
// (:42-47), lu_factorize (:55), lu_solve (:180), lu_transpose_solve (:207).
//
// The factorisation runs on the device (band LU with row partial pivoting and
// the reference's pivot rule, ties included, ck_lu_factorize); the factors
// come back in the reference's shape -- L strictly lower in pivot coordinates,
// U upper with the diagonal first per row, row_perm -- and stay on the device
// as well (LUFactors::device), where every solve runs.

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "condkit/b200_device.hpp"
#include "condkit/sparse.hpp"

namespace condkit {

struct StructurallySingular : std::runtime_error {
  explicit StructurallySingular(std::size_t col)
      : std::runtime_error("structurally singular: no pivot candidate in column " +
                           std::to_string(col)),
        column(col) {}
  std::size_t column;
};

struct NumericallySingular : std::runtime_error {
  NumericallySingular(std::size_t col, double pivot)
      : std::runtime_error("numerically singular: best pivot " + std::to_string(pivot) +
                           " in column " + std::to_string(col) + " below threshold"),
        column(col),
        pivot(pivot) {}
  std::size_t column;
  double pivot;
};

struct LUFactors {
  SparseMatrix l;                     // strictly lower triangle, unit diagonal implicit
  SparseMatrix u;                     // upper triangle including the diagonal
  std::vector<std::size_t> row_perm;  // row_perm[k] = original row pivoted at step k
  double pivot_min = std::numeric_limits<double>::infinity();
  // B200: the same factors resident on the device (null for factors assembled
  // on the host, e.g. solvers.hpp's ilu0, which the device solves do not take)
  std::shared_ptr<b200::DeviceLU> device;
};

namespace b200 {

inline const DeviceLU& device_factors(const LUFactors& f, const char* who) {
  if (!f.device)
    throw std::invalid_argument(std::string(who) +
                                ": factors not produced by lu_factorize (B200 build: the solves "
                                "run on the device factors)");
  return *f.device;
}

// Factor a device-resident matrix; singular -> the reference's exceptions.
inline LUFactors factorize(const DeviceMatrix& a, double pivot_tol) {
  ck_lu h = nullptr;
  std::int64_t col = -1;
  double piv = 0.0;
  const ck_status s = ck_lu_factorize(a.handle(), pivot_tol, &h, &col, &piv);
  if (s == CK_ERR_STRUCT_SINGULAR) throw StructurallySingular(static_cast<std::size_t>(col));
  if (s == CK_ERR_NUM_SINGULAR) throw NumericallySingular(static_cast<std::size_t>(col), piv);
  check(s);
  LUFactors f;
  f.device = std::make_shared<DeviceLU>(h);
  std::int64_t n = 0, kl = 0, ku = 0, bytes = 0, nl = 0, nu = 0;
  check(ck_lu_get_info(h, &n, &kl, &ku, &f.pivot_min, &bytes));
  check(ck_lu_csr_info(h, &nl, &nu));
  const auto N = static_cast<std::size_t>(n);
  std::vector<std::int64_t> lrp(N + 1), urp(N + 1), perm(N);
  std::vector<std::int32_t> lci(static_cast<std::size_t>(nl)), uci(static_cast<std::size_t>(nu));
  std::vector<double> lva(static_cast<std::size_t>(nl)), uva(static_cast<std::size_t>(nu));
  check(ck_lu_export_csr(h, lrp.data(), lci.data(), lva.data(), urp.data(), uci.data(),
                         uva.data(), perm.data()));
  auto csr = [N](const std::vector<std::int64_t>& rp, const std::vector<std::int32_t>& ci,
                 std::vector<double> va) {
    return SparseMatrix(N, N, std::vector<std::size_t>(rp.begin(), rp.end()),
                        std::vector<std::size_t>(ci.begin(), ci.end()), std::move(va));
  };
  f.l = csr(lrp, lci, std::move(lva));
  f.u = csr(urp, uci, std::move(uva));
  f.row_perm.assign(perm.begin(), perm.end());
  return f;
}

}  // namespace b200

/// Factorizes a square matrix as P·A = L·U on the B200: in each column the
/// largest-magnitude candidate among the unpivoted rows, the first one the
/// elimination touched on ties. Throws StructurallySingular when a column has
/// no candidate and NumericallySingular when the best candidate magnitude is
/// below pivot_tol times the column's largest magnitude (lu.hpp:49-54).
inline LUFactors lu_factorize(const SparseMatrix& a, double pivot_tol = 1e-12) {
  if (a.nrows() != a.ncols()) throw DimensionMismatch("lu_factorize: matrix must be square");
  return b200::factorize(b200::DeviceMatrix(a), pivot_tol);
}

/// Solves A·x = b through the factors (lu.hpp:179-202), on the device.
inline DenseVector lu_solve(const LUFactors& f, const DenseVector& b) {
  const b200::DeviceLU& d = b200::device_factors(f, "lu_solve");
  if (b.size() != f.row_perm.size()) throw DimensionMismatch("lu_solve: rhs length != n");
  DenseVector x(b.size());
  b200::check(ck_lu_solve(d.handle(), b.data(), x.data()));
  return x;
}

/// Solves Aᵀ·x = b through the same factors (lu.hpp:204-227), on the device.
inline DenseVector lu_transpose_solve(const LUFactors& f, const DenseVector& b) {
  const b200::DeviceLU& d = b200::device_factors(f, "lu_transpose_solve");
  if (b.size() != f.row_perm.size())
    throw DimensionMismatch("lu_transpose_solve: rhs length != n");
  DenseVector x(b.size());
  b200::check(ck_lu_transpose_solve(d.handle(), b.data(), x.data()));
  return x;
}

}  // namespace condkit
