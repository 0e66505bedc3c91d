// Drop-in demo (TEST): the reference's call sites compiled against
// include/condkit_b200.hpp. With -DWITH_REFERENCE_TYPES the matrix is the
// reference's own condkit::SparseMatrix (headers from /root/reference); without
// it a minimal CSR struct with the same accessors stands in (GPU box).
#include <cstdio>
#include <vector>

#include "condkit_b200.hpp"

#ifdef WITH_REFERENCE_TYPES
#include <condkit/sparse.hpp>
using Matrix = condkit::SparseMatrix;
static Matrix make(std::size_t g) {
  std::vector<condkit::Triplet> t;
  for (std::size_t r = 0; r < g; ++r)
    for (std::size_t c = 0; c < g; ++c) {
      std::size_t i = r * g + c;
      t.push_back({i, i, 4.0 + 0.01 * static_cast<double>(i % 7)});
      if (r > 0) t.push_back({i, i - g, -1.0});
      if (r + 1 < g) t.push_back({i, i + g, -1.0});
      if (c > 0) t.push_back({i, i - 1, -1.0});
      if (c + 1 < g) t.push_back({i, i + 1, -1.0});
    }
  return Matrix::from_triplets(g * g, g * g, t);
}
#else
struct Matrix {
  std::size_t n = 0;
  std::vector<std::size_t> rp, ci;
  std::vector<double> va;
  std::size_t nrows() const { return n; }
  std::size_t ncols() const { return n; }
  const std::vector<std::size_t>& row_offsets() const { return rp; }
  const std::vector<std::size_t>& col_indices() const { return ci; }
  const std::vector<double>& values() const { return va; }
};
static Matrix make(std::size_t g) {
  Matrix m;
  m.n = g * g;
  m.rp.push_back(0);
  for (std::size_t r = 0; r < g; ++r)
    for (std::size_t c = 0; c < g; ++c) {
      std::size_t i = r * g + c;
      auto add = [&](std::size_t j, double v) {
        m.ci.push_back(j);
        m.va.push_back(v);
      };
      if (r > 0) add(i - g, -1.0);
      if (c > 0) add(i - 1, -1.0);
      add(i, 4.0 + 0.01 * static_cast<double>(i % 7));
      if (c + 1 < g) add(i + 1, -1.0);
      if (r + 1 < g) add(i + g, -1.0);
      m.rp.push_back(m.ci.size());
    }
  return m;
}
#endif

int main() {
  Matrix a = make(12);
  condkit_b200::AdamConfig cfg;
  auto r = condkit_b200::cond2(a, cfg);
  std::vector<double> x(a.ncols(), 1.0), b;
  condkit_b200::DeviceMatrix d(a);
  b = condkit_b200::matvec(d, x);
  x[0] += 1e-9;
  auto rep = condkit_b200::verify_solution(d, x, b);
  std::printf("kappa %.17g sigma_max %.17g inv %.17g iters %zu %zu bound %.17g verdict %d\n",
              r.kappa, r.operator_norm.value, r.inverse_norm.value, r.operator_norm.iterations,
              r.inverse_norm.iterations, rep.loose_upper, static_cast<int>(rep.verdict));
  return 0;
}
