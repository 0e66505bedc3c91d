// Synthetic operators for the five BASELINE.json configurations (host code,
// multithreaded). These are inputs, not part of the estimator: the reference
// ships no generator for configs 2-5, so the operators are
// stated here and in DESIGN.md section 3.
//
//  kind 1  row-scaled 5-point Dirichlet Laplacian (acceptance.cpp:240-254
//          layout; row i scaled by 10^U(-3,3), U drawn row-major from
//          mt19937_64(seed) with uniform_in, rng.hpp:36-38).
//  kind 2  staggered-grid (MAC) variable-viscosity Stokes, unknowns
//          (vx, vy, P) per cell interleaved, viscosity 10^U(18,24) Pa s per
//          cell nondimensionalised by 1e21, pressure block unscaled, one
//          pressure DOF pinned.
//  kind 3  coupled hydro-mechanical staggered operator, 6 unknowns per cell
//          (solid vx, vy, total P; fluid vx, vy, fluid P), stress-scale
//          entries 10^U(7,8), velocity-scale entries ~1e-9, permeability
//          10^U(-22,-14) (fluid viscosity 1e-3).
//  kind 5  random banded matrix: 7..15 entries per row with |i-j| < bw, a
//          nonzero diagonal, values N(0,1) times a per-column 10^U(-8,8).
//
// Every random quantity except kind 1's row scales comes from a counter-based
// hash of (seed, stream, index), so the output does not depend on threading.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "ck_common.h"

namespace ck {
namespace {

inline uint64_t splitmix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

inline double hash_u01(uint64_t seed, uint64_t stream, uint64_t idx) {
  uint64_t h = splitmix(splitmix(seed ^ (stream * 0xD1B54A32D192ED03ull)) + idx);
  return static_cast<double>(h >> 11) * 0x1.0p-53;
}

inline double hash_normal(uint64_t seed, uint64_t stream, uint64_t idx) {
  double u1 = 1.0 - hash_u01(seed, stream, 2 * idx);
  double u2 = hash_u01(seed, stream, 2 * idx + 1);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793 * u2);
}

struct Ent {
  int64_t col;
  double val;
};

template <class F>
void par_for(int64_t n, F&& f) {
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  int64_t nt = n < 4096 ? 1 : std::min<int64_t>(hw, 128);
  if (nt <= 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> pool;
  int64_t chunk = ceil_div(n, nt);
  for (int64_t t = 0; t < nt; ++t) {
    int64_t b = t * chunk, e = std::min(n, b + chunk);
    if (b >= e) break;
    pool.emplace_back([&f, b, e] { f(b, e); });
  }
  for (auto& th : pool) th.join();
}

// Sort a row's entries by column and merge duplicates (summed in generation
// order, like SparseMatrix::from_triplets, sparse.hpp:67-96).
inline int finish_row(Ent* e, int k) {
  std::stable_sort(e, e + k, [](const Ent& a, const Ent& b) { return a.col < b.col; });
  int w = 0;
  for (int r = 0; r < k; ++r) {
    if (w > 0 && e[w - 1].col == e[r].col) {
      e[w - 1].val += e[r].val;
    } else {
      e[w++] = e[r];
    }
  }
  return w;
}

// Two passes (count, fill) over rows produced by `gen(row, buf) -> count`.
template <class G>
void emit(int64_t nrows, G&& gen, int64_t* rp, int32_t* ci, double* va) {
  std::vector<int32_t> cnt((size_t)nrows);
  par_for(nrows, [&](int64_t b, int64_t e) {
    Ent buf[64];
    for (int64_t i = b; i < e; ++i) cnt[(size_t)i] = finish_row(buf, gen(i, buf));
  });
  rp[0] = 0;
  for (int64_t i = 0; i < nrows; ++i) rp[i + 1] = rp[i] + cnt[(size_t)i];
  if (!ci) return;
  par_for(nrows, [&](int64_t b, int64_t e) {
    Ent buf[64];
    for (int64_t i = b; i < e; ++i) {
      int k = finish_row(buf, gen(i, buf));
      int64_t o = rp[i];
      for (int q = 0; q < k; ++q) {
        ci[o + q] = (int32_t)buf[q].col;
        va[o + q] = buf[q].val;
      }
    }
  });
}

// ----------------------------------------------------------- kind 1
void gen_laplacian(int64_t g, uint64_t seed, int64_t* rp, int32_t* ci, double* va) {
  const int64_t n = g * g;
  std::vector<double> scale((size_t)n);
  std::mt19937_64 gen(seed);
  for (int64_t i = 0; i < n; ++i) {
    double u = -3.0 + (3.0 - -3.0) * (static_cast<double>(gen() >> 11) * 0x1.0p-53);
    scale[(size_t)i] = std::pow(10.0, u);
  }
  emit(n, [&](int64_t row, Ent* e) {
    int64_t r = row / g, c = row % g;
    double s = scale[(size_t)row];
    int k = 0;
    e[k++] = {row, 4.0 * s};
    if (r > 0) e[k++] = {row - g, -1.0 * s};
    if (r + 1 < g) e[k++] = {row + g, -1.0 * s};
    if (c > 0) e[k++] = {row - 1, -1.0 * s};
    if (c + 1 < g) e[k++] = {row + 1, -1.0 * s};
    return k;
  }, rp, ci, va);
}

// ----------------------------------------------------------- kind 2
struct StokesGrid {
  int64_t g;
  std::vector<double> eta;  // cell viscosity, nondimensional
  double cell(int64_t i, int64_t j) const { return eta[(size_t)(i * g + j)]; }
  // viscosity at the grid node (i, j) = bottom-left corner of cell (i, j)
  double node(int64_t i, int64_t j) const {
    double s = 0.0;
    int n = 0;
    for (int64_t a = i - 1; a <= i; ++a)
      for (int64_t b = j - 1; b <= j; ++b)
        if (a >= 0 && a < g && b >= 0 && b < g) {
          s += cell(a, b);
          ++n;
        }
    return s / n;
  }
};

void gen_stokes(int64_t g, uint64_t seed, int64_t* rp, int32_t* ci, double* va) {
  StokesGrid G{g, std::vector<double>((size_t)(g * g))};
  par_for(g * g, [&](int64_t b, int64_t e) {
    for (int64_t c = b; c < e; ++c)
      G.eta[(size_t)c] = std::pow(10.0, 18.0 + 6.0 * hash_u01(seed, 1, (uint64_t)c)) / 1e21;
  });
  const double g2 = (double)g * (double)g, gh = (double)g;
  auto VX = [g](int64_t i, int64_t j) { return 3 * (i * g + j); };
  auto VY = [g](int64_t i, int64_t j) { return 3 * (i * g + j) + 1; };
  auto P = [g](int64_t i, int64_t j) { return 3 * (i * g + j) + 2; };
  emit(3 * g * g, [&](int64_t row, Ent* e) {
    int64_t cellid = row / 3, t = row % 3, i = cellid / g, j = cellid % g;
    int k = 0;
    if (t == 0) {  // x-momentum at the left face of cell (i, j)
      if (j == 0) {
        e[k++] = {row, -4.0 * G.cell(i, 0) * g2};
        return k;
      }
      double eL = G.cell(i, j - 1), eR = G.cell(i, j);
      double eS = i >= 1 ? G.node(i, j) : 0.0, eN = i + 1 < g ? G.node(i + 1, j) : 0.0;
      if (j + 1 < g) e[k++] = {VX(i, j + 1), 2.0 * eR * g2};
      e[k++] = {VX(i, j - 1), 2.0 * eL * g2};
      if (i + 1 < g) e[k++] = {VX(i + 1, j), eN * g2};
      if (i >= 1) e[k++] = {VX(i - 1, j), eS * g2};
      e[k++] = {VX(i, j), -(2.0 * eR + 2.0 * eL + eN + eS) * g2};
      if (i + 1 < g) {
        e[k++] = {VY(i + 1, j), eN * g2};
        e[k++] = {VY(i + 1, j - 1), -eN * g2};
      }
      if (i >= 1) {
        e[k++] = {VY(i, j), -eS * g2};
        e[k++] = {VY(i, j - 1), eS * g2};
      }
      e[k++] = {P(i, j), -gh};
      e[k++] = {P(i, j - 1), gh};
      return k;
    }
    if (t == 1) {  // y-momentum at the bottom face of cell (i, j)
      if (i == 0) {
        e[k++] = {row, -4.0 * G.cell(0, j) * g2};
        return k;
      }
      double eB = G.cell(i - 1, j), eT = G.cell(i, j);
      double eW = j >= 1 ? G.node(i, j) : 0.0, eE = j + 1 < g ? G.node(i, j + 1) : 0.0;
      if (i + 1 < g) e[k++] = {VY(i + 1, j), 2.0 * eT * g2};
      e[k++] = {VY(i - 1, j), 2.0 * eB * g2};
      if (j + 1 < g) e[k++] = {VY(i, j + 1), eE * g2};
      if (j >= 1) e[k++] = {VY(i, j - 1), eW * g2};
      e[k++] = {VY(i, j), -(2.0 * eT + 2.0 * eB + eE + eW) * g2};
      if (j + 1 < g) {
        e[k++] = {VX(i, j + 1), eE * g2};
        e[k++] = {VX(i - 1, j + 1), -eE * g2};
      }
      if (j >= 1) {
        e[k++] = {VX(i, j), -eW * g2};
        e[k++] = {VX(i - 1, j), eW * g2};
      }
      e[k++] = {P(i, j), -gh};
      e[k++] = {P(i - 1, j), gh};
      return k;
    }
    // continuity: div v = 0 (one pressure DOF pinned in cell 0)
    if (j + 1 < g) e[k++] = {VX(i, j + 1), gh};
    e[k++] = {VX(i, j), -gh};
    if (i + 1 < g) e[k++] = {VY(i + 1, j), gh};
    e[k++] = {VY(i, j), -gh};
    if (cellid == 0) e[k++] = {P(0, 0), gh};
    return k;
  }, rp, ci, va);
}

// ----------------------------------------------------------- kind 3
void gen_hydromech(int64_t g, uint64_t seed, int64_t* rp, int32_t* ci, double* va) {
  const int64_t nc = g * g;
  std::vector<double> cv((size_t)nc), perm((size_t)nc), beta((size_t)nc), wsm((size_t)nc);
  par_for(nc, [&](int64_t b, int64_t e) {
    for (int64_t c = b; c < e; ++c) {
      cv[(size_t)c] = std::pow(10.0, 7.0 + hash_u01(seed, 11, (uint64_t)c));          // stress scale
      perm[(size_t)c] = std::pow(10.0, -22.0 + 8.0 * hash_u01(seed, 12, (uint64_t)c)) / 1e-3;  // k/eta_f
      beta[(size_t)c] = std::pow(10.0, -11.0 + hash_u01(seed, 13, (uint64_t)c));      // compressibility
      wsm[(size_t)c] = 1e-9 * std::pow(10.0, hash_u01(seed, 14, (uint64_t)c));         // velocity scale
    }
  });
  const double alpha = 0.9, phi = 0.1;
  auto C = [&](const std::vector<double>& a, int64_t i, int64_t j) {
    return a[(size_t)(std::min(std::max<int64_t>(i, 0), g - 1) * g +
                      std::min(std::max<int64_t>(j, 0), g - 1))];
  };
  auto node = [&](int64_t i, int64_t j) {
    double s = 0.0;
    int n = 0;
    for (int64_t a = i - 1; a <= i; ++a)
      for (int64_t b = j - 1; b <= j; ++b)
        if (a >= 0 && a < g && b >= 0 && b < g) {
          s += cv[(size_t)(a * g + b)];
          ++n;
        }
    return s / n;
  };
  auto U = [g](int64_t i, int64_t j, int f) { return 6 * (i * g + j) + f; };
  auto in = [g](int64_t i, int64_t j) { return i >= 0 && i < g && j >= 0 && j < g; };
  emit(6 * nc, [&](int64_t row, Ent* e) {
    const int64_t cell = row / 6, i = cell / g, j = cell % g;
    const int f = (int)(row % 6);
    int k = 0;
    auto add = [&](int64_t a, int64_t b, int fld, double v) {
      if (in(a, b)) e[k++] = {U(a, b, fld), v};
    };
    const double w = wsm[(size_t)cell];
    if (f == 0 || f == 1) {  // solid momentum (x: faces j >= 1; y: faces i >= 1)
      const bool xdir = f == 0;
      if ((xdir && j == 0) || (!xdir && i == 0)) {
        e[k++] = {row, -4.0 * cv[(size_t)cell]};
        return k;
      }
      // own velocity: viscous 5-point with face/node viscosities
      const int sv = xdir ? 0 : 1, so = xdir ? 1 : 0;      // solid velocity fields
      const int fv = xdir ? 3 : 4, fo = xdir ? 4 : 3;      // fluid velocity fields
      int64_t di = xdir ? 0 : 1, dj = xdir ? 1 : 0;        // along the component
      double eA = C(cv, i, j), eB = C(cv, i - di, j - dj);  // cells after / before the face
      double eP = node(i + dj, j + di), eM = node(i, j);    // nodes across
      double diag = 0.0;
      if (in(i + di, j + dj)) { add(i + di, j + dj, sv, 2.0 * eA); diag += 2.0 * eA; }
      add(i - di, j - dj, sv, 2.0 * eB);
      diag += 2.0 * eB;
      if (in(i + dj, j + di)) { add(i + dj, j + di, sv, eP); diag += eP; }
      if (in(i - dj, j - di)) { add(i - dj, j - di, sv, eM); diag += eM; }
      e[k++] = {row, -diag};
      // cross viscous terms in the other solid component
      add(i + dj, j + di, so, eP);
      add(i + dj - di, j + di - dj, so, -eP);
      add(i, j, so, -eM);
      add(i - di, j - dj, so, eM);
      // total and fluid pressure gradients (effective stress, Biot alpha)
      add(i, j, 2, -1.0);
      add(i - di, j - dj, 2, 1.0);
      add(i, j, 5, alpha);
      add(i - di, j - dj, 5, -alpha);
      // fluid-velocity coupling (inertia / interphase terms), velocity scale
      add(i, j, fv, -4.0 * w);
      add(i + di, j + dj, fv, w);
      add(i - di, j - dj, fv, w);
      add(i + dj, j + di, fv, w);
      add(i - dj, j - di, fv, w);
      add(i + dj, j + di, fo, w);
      add(i + dj - di, j + di - dj, fo, -w);
      add(i, j, fo, -w);
      add(i - di, j - dj, fo, w);
      return k;
    }
    if (f == 3 || f == 4) {  // Darcy: phi (vf - vs) + (k/eta_f) grad Pf = 0
      const bool xdir = f == 3;
      if ((xdir && j == 0) || (!xdir && i == 0)) {
        e[k++] = {row, phi};
        return k;
      }
      const int sv = xdir ? 0 : 1, fo = xdir ? 4 : 3;
      int64_t di = xdir ? 0 : 1, dj = xdir ? 1 : 0;
      double kf = 0.5 * (C(perm, i, j) + C(perm, i - di, j - dj));
      e[k++] = {row, phi + 4.0 * w};
      add(i + di, j + dj, f, -w);
      add(i - di, j - dj, f, -w);
      add(i + dj, j + di, f, -w);
      add(i - dj, j - di, f, -w);
      add(i, j, sv, -phi);
      add(i + di, j + dj, sv, w);
      add(i - di, j - dj, sv, w);
      add(i + dj, j + di, sv, w);
      add(i - dj, j - di, sv, w);
      add(i, j, 5, kf);
      add(i - di, j - dj, 5, -kf);
      add(i, j, 2, 1e-9 * kf);
      add(i - di, j - dj, 2, -1e-9 * kf);
      add(i + dj, j + di, fo, w);
      add(i + dj - di, j + di - dj, fo, -w);
      add(i, j, fo, -w);
      add(i - di, j - dj, fo, w);
      return k;
    }
    // mass rows: f == 2 total pressure (solid), f == 5 fluid pressure
    const bool solid = f == 2;
    const double b = beta[(size_t)cell];
    const double sv = solid ? 1.0 : -phi, fvv = solid ? 1e-9 : phi;
    add(i, j + 1, 0, sv);
    add(i, j, 0, -sv);
    add(i + 1, j, 1, sv);
    add(i, j, 1, -sv);
    add(i, j + 1, 3, fvv);
    add(i, j, 3, -fvv);
    add(i + 1, j, 4, fvv);
    add(i, j, 4, -fvv);
    const int own = solid ? 2 : 5, other = solid ? 5 : 2;
    e[k++] = {row, b + 4.0 * w};
    add(i + 1, j, own, -w);
    add(i - 1, j, own, -w);
    add(i, j + 1, own, -w);
    add(i, j - 1, own, -w);
    add(i, j, other, -(solid ? alpha : 1.0) * b);
    add(i + 1, j, other, 0.5 * w);
    add(i - 1, j, other, 0.5 * w);
    add(i, j + 1, other, 0.5 * w);
    add(i, j - 1, other, 0.5 * w);
    return k;
  }, rp, ci, va);
}

// ----------------------------------------------------------- kind 5
void gen_banded(int64_t n, int64_t bw, uint64_t seed, int64_t* rp, int32_t* ci, double* va) {
  std::vector<double> cs((size_t)n);
  par_for(n, [&](int64_t b, int64_t e) {
    for (int64_t j = b; j < e; ++j)
      cs[(size_t)j] = std::pow(10.0, -8.0 + 16.0 * hash_u01(seed, 21, (uint64_t)j));
  });
  emit(n, [&](int64_t row, Ent* e) {
    int want = 7 + (int)(splitmix(seed ^ splitmix((uint64_t)row + 0x5151)) % 9);
    int k = 0;
    e[k++] = {row, (0.5 + hash_u01(seed, 22, (uint64_t)row)) * cs[(size_t)row]};
    uint64_t draw = 0;
    while (k < want && draw < 4096) {
      uint64_t h = splitmix(splitmix(seed ^ 0xB5A7ull) + (uint64_t)row * 4096 + draw);
      int64_t off = (int64_t)(h % (uint64_t)(2 * bw - 1)) - (bw - 1);
      int64_t col = row + off;
      double z = hash_normal(seed, 23, (uint64_t)row * 4096 + draw);
      ++draw;
      if (off == 0 || col < 0 || col >= n) continue;
      bool dup = false;
      for (int q = 0; q < k; ++q) dup |= e[q].col == col;
      if (dup) continue;
      e[k++] = {col, z * cs[(size_t)col]};
    }
    return k;
  }, rp, ci, va);
}

}  // namespace
}  // namespace ck

extern "C" ck_status ck_generate(int32_t kind, int64_t grid, int64_t param, uint64_t seed,
                                 int64_t* nrows, int64_t* nnz, int64_t* rp, int32_t* ci,
                                 double* va);

ck_status ck_generate(int32_t kind, int64_t grid, int64_t param, uint64_t seed, int64_t* nrows,
                      int64_t* nnz, int64_t* rp, int32_t* ci, double* va) {
  using namespace ck;
  if (grid <= 0 || !nrows || !nnz) return CK_ERR_INVALID_ARGUMENT;
  int64_t n = 0;
  switch (kind) {
    case 1: n = grid * grid; break;
    case 2: n = 3 * grid * grid; break;
    case 3: n = 6 * grid * grid; break;
    case 5: n = grid; break;
    default: return CK_ERR_INVALID_ARGUMENT;
  }
  if (kind == 5 && (param < 8 || param > 65536)) return CK_ERR_INVALID_ARGUMENT;
  if (n >= (int64_t(1) << 31)) return CK_ERR_UNSUPPORTED;
  try {
    std::vector<int64_t> tmp;
    int64_t* r = rp;
    if (!r) {
      tmp.resize((size_t)n + 1);
      r = tmp.data();
    }
    double* v = rp ? va : nullptr;
    int32_t* c = rp ? ci : nullptr;
    switch (kind) {
      case 1: gen_laplacian(grid, seed, r, c, v); break;
      case 2: gen_stokes(grid, seed, r, c, v); break;
      case 3: gen_hydromech(grid, seed, r, c, v); break;
      case 5: gen_banded(grid, param, seed, r, c, v); break;
    }
    *nrows = n;
    *nnz = r[n];
    return CK_OK;
  } catch (...) {
    return CK_ERR_OUT_OF_MEMORY;
  }
}
