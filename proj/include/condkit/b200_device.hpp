#pragma once

// condkit/b200_device.hpp -- plumbing shared by the B200 builds of
// condkit/lu.hpp, condkit/condest.hpp and condkit/error_bounds.hpp (this
// directory). Not a reference header: the reference has no device code.
//
// The B200 headers keep the reference's estimator / error-bound interface
// (same names, types, defaults and exception types) and run every numeric step
// in libcondkit_b200.so through its C ABI (include/condkit_b200.h). Put this
// directory in front of the reference's include directory:
//
//     -I<repo>/proj/include -I<repo>/include -I<reference>/proj/include
//     -L<repo>/paper_2409_11515_b200 -lcondkit_b200
//
// condkit/sparse.hpp, rng.hpp, format.hpp, matrix_market.hpp, solvers.hpp and
// bench.hpp stay the reference's; their includes of condest.hpp / lu.hpp /
// error_bounds.hpp resolve to the B200 builds.

#include <cstddef>
#include <cstdint>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "condkit/sparse.hpp"
#include "condkit_b200.h"

namespace condkit {
namespace b200 {

/// A failure with no reference counterpart: CUDA runtime error, no sm_100
/// device, out of device memory, or an input beyond this build's limits.
struct DeviceError : std::runtime_error {
  DeviceError(ck_status s, const std::string& what) : std::runtime_error(what), status(s) {}
  ck_status status;
};

/// Maps the statuses every entry point can return onto the reference's
/// exception types (sparse.hpp:25-27, condest.hpp:187,288,303); the callers
/// handle the statuses specific to them (singularity, zero norms) first.
[[noreturn]] inline void raise(ck_status s) {
  const std::string m = ck_last_error();
  switch (s) {
    case CK_ERR_DIMENSION: throw DimensionMismatch(m);
    case CK_ERR_INVALID_ARGUMENT: throw std::invalid_argument(m);
    case CK_ERR_LOGIC: throw std::logic_error(m);
    case CK_ERR_ZERO_COLUMN: throw ZeroColumn(0);
    case CK_ERR_ZERO_ROW: throw ZeroRow(0);
    default: throw DeviceError(s, m);
  }
}

inline void check(ck_status s) {
  if (s != CK_OK) raise(s);
}

/// A SparseMatrix resident on the B200 (A and its transpose in the device
/// layouts, ck_matrix_upload). Shared by copies; freed with the last one.
class DeviceMatrix {
 public:
  DeviceMatrix() = default;
  explicit DeviceMatrix(const SparseMatrix& a) : nrows_(a.nrows()), ncols_(a.ncols()) {
    const auto& ro = a.row_offsets();
    const auto& ci = a.col_indices();
    std::vector<std::int64_t> rp(ro.begin(), ro.end());
    std::vector<std::int32_t> cols(ci.size());
    for (std::size_t k = 0; k < ci.size(); ++k) {
      if (ci[k] > static_cast<std::size_t>(std::numeric_limits<std::int32_t>::max()))
        throw DeviceError(CK_ERR_UNSUPPORTED, "column index beyond 2^31 - 1");
      cols[k] = static_cast<std::int32_t>(ci[k]);
    }
    ck_matrix h = nullptr;
    check(ck_matrix_upload(static_cast<std::int64_t>(nrows_), static_cast<std::int64_t>(ncols_),
                           rp.data(), cols.data(), a.values().data(), &h));
    h_ = std::shared_ptr<ck_matrix_s>(h, [](ck_matrix m) { ck_matrix_free(m); });
  }
  ck_matrix handle() const { return h_.get(); }
  explicit operator bool() const { return h_ != nullptr; }
  std::size_t nrows() const { return nrows_; }
  std::size_t ncols() const { return ncols_; }

 private:
  std::shared_ptr<ck_matrix_s> h_;
  std::size_t nrows_ = 0, ncols_ = 0;
};

/// Band LU factors on the B200 (ck_lu_factorize). Shared by copies of LUFactors.
class DeviceLU {
 public:
  explicit DeviceLU(ck_lu f) : h_(f, [](ck_lu p) { ck_lu_free(p); }) {}
  ck_lu handle() const { return h_.get(); }

 private:
  std::shared_ptr<ck_lu_s> h_;
};

}  // namespace b200
}  // namespace condkit
