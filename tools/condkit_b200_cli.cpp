// condkit_b200_cli: the reference CLI's estimator subcommands (cond, norm,
// verify; condkit_cli.cpp:141-326) on the B200 backend, plus `convert` to a
// binary CSR container so that large operators skip text parsing.
//
// Output protocol as the reference's: effective configuration as
// "# key = value" rows, then data as "key = value" rows with 17 significant
// digits; prose and errors on stderr. Exit codes: 0 ok / accepted, 2 usage or
// input error, 3 numerically singular, 4 verification rejected.
//
// Matrix files: Matrix Market (coordinate or array; real or integer; general
// or symmetric -- symmetric storage mirrored, duplicates summed, 1-based), or
// .csrb (binary CSR, written by `convert`):
//   "CKCSR001" | int64 nrows, ncols, nnz | int64 row_offsets[nrows+1] |
//   int32 col_indices[nnz] | float64 values[nnz]
// Vector files: one value per line, '#' comments.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <limits>
#include <map>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "condkit_b200.hpp"

namespace {

constexpr int kExitOk = 0;
constexpr int kExitUsage = 2;
constexpr int kExitSingular = 3;
constexpr int kExitRejected = 4;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------- CSR
struct Csr {
  std::size_t nr = 0, nc = 0;
  std::vector<std::size_t> rp;
  std::vector<std::size_t> ci;
  std::vector<double> va;
  std::size_t nrows() const { return nr; }
  std::size_t ncols() const { return nc; }
  std::size_t nnz() const { return va.size(); }
  const std::vector<std::size_t>& row_offsets() const { return rp; }
  const std::vector<std::size_t>& col_indices() const { return ci; }
  const std::vector<double>& values() const { return va; }
};

std::string slurp(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw UsageError("cannot open file: " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

bool ends_with(const std::string& s, const std::string& suf) {
  return s.size() >= suf.size() && s.compare(s.size() - suf.size(), suf.size(), suf) == 0;
}

// Line cursor over a text buffer.
struct Lines {
  const std::string& s;
  std::size_t pos = 0, lineno = 0;
  bool next(const char*& b, const char*& e) {
    if (pos >= s.size()) return false;
    const std::size_t nl = s.find('\n', pos);
    const std::size_t end = nl == std::string::npos ? s.size() : nl;
    b = s.data() + pos;
    e = s.data() + end;
    if (e > b && e[-1] == '\r') --e;
    pos = end + 1;
    ++lineno;
    return true;
  }
};

bool blank(const char* b, const char* e) {
  for (; b < e; ++b)
    if (!std::isspace(static_cast<unsigned char>(*b))) return false;
  return true;
}

std::vector<std::string_view> tokens(const char* b, const char* e) {
  std::vector<std::string_view> t;
  while (b < e) {
    while (b < e && std::isspace(static_cast<unsigned char>(*b))) ++b;
    const char* s = b;
    while (b < e && !std::isspace(static_cast<unsigned char>(*b))) ++b;
    if (b > s) t.emplace_back(s, (std::size_t)(b - s));
  }
  return t;
}

[[noreturn]] void parse_fail(std::size_t line, const std::string& why) {
  throw UsageError("parse error at line " + std::to_string(line) + ": " + why);
}

double to_double(std::string_view t, std::size_t line) {
  const char* b = t.data();
  const char* e = b + t.size();
  if (b != e && *b == '+') ++b;
  double v = 0.0;
  auto r = std::from_chars(b, e, v);
  if (r.ec != std::errc() || r.ptr != e) parse_fail(line, "bad number '" + std::string(t) + "'");
  return v;
}

std::size_t to_index(std::string_view t, std::size_t line) {
  std::size_t v = 0;
  auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  if (r.ec != std::errc() || r.ptr != t.data() + t.size())
    parse_fail(line, "bad index '" + std::string(t) + "'");
  return v;
}

struct Trip {
  std::size_t i, j;
  double v;
};

// from_triplets semantics: row-major order, duplicates summed in input order.
Csr from_triplets(std::size_t nr, std::size_t nc, std::vector<Trip>& t) {
  std::stable_sort(t.begin(), t.end(), [](const Trip& a, const Trip& b) {
    return a.i != b.i ? a.i < b.i : a.j < b.j;
  });
  Csr a;
  a.nr = nr;
  a.nc = nc;
  a.rp.assign(nr + 1, 0);
  for (std::size_t k = 0; k < t.size();) {
    std::size_t k2 = k + 1;
    double v = t[k].v;
    while (k2 < t.size() && t[k2].i == t[k].i && t[k2].j == t[k].j) v += t[k2++].v;
    a.ci.push_back(t[k].j);
    a.va.push_back(v);
    ++a.rp[t[k].i + 1];
    k = k2;
  }
  for (std::size_t i = 0; i < nr; ++i) a.rp[i + 1] += a.rp[i];
  return a;
}

Csr read_matrix_market(const std::string& text) {
  Lines L{text};
  const char *b, *e;
  if (!L.next(b, e)) parse_fail(1, "empty input");
  auto h = tokens(b, e);
  auto low = [](std::string_view s) {
    std::string o(s);
    for (char& c : o) c = (char)std::tolower((unsigned char)c);
    return o;
  };
  if (h.size() != 5 || low(h[0]) != "%%matrixmarket" || low(h[1]) != "matrix")
    parse_fail(1, "not a MatrixMarket matrix header");
  const std::string fmt = low(h[2]), field = low(h[3]), sym = low(h[4]);
  if (fmt != "coordinate" && fmt != "array") throw UsageError("unsupported format: " + fmt);
  if (field != "real" && field != "integer") throw UsageError("unsupported format: " + field);
  if (sym != "general" && sym != "symmetric") throw UsageError("unsupported format: " + sym);
  std::vector<std::string_view> t;
  for (;;) {
    if (!L.next(b, e)) parse_fail(L.lineno + 1, "missing size line");
    if ((e > b && *b == '%') || blank(b, e)) continue;
    t = tokens(b, e);
    break;
  }
  if (fmt == "coordinate" ? t.size() != 3 : t.size() != 2)
    parse_fail(L.lineno, fmt == "coordinate" ? "size line must be 'nrows ncols nnz'"
                                             : "size line must be 'nrows ncols'");
  const std::size_t nr = to_index(t[0], L.lineno), nc = to_index(t[1], L.lineno);
  const bool symmetric = sym == "symmetric";
  if (symmetric && nr != nc) parse_fail(L.lineno, "symmetric matrix must be square");
  std::vector<Trip> ent;
  auto push = [&](std::size_t i, std::size_t j, double v, std::size_t at) {
    if (i == 0 || j == 0 || i > nr || j > nc) parse_fail(at, "index outside the matrix");
    ent.push_back({i - 1, j - 1, v});
    if (symmetric && i != j) ent.push_back({j - 1, i - 1, v});
  };
  if (fmt == "coordinate") {
    const std::size_t nnz = to_index(t[2], L.lineno);
    ent.reserve(symmetric ? 2 * nnz : nnz);
    std::size_t seen = 0;
    while (seen < nnz) {
      if (!L.next(b, e)) parse_fail(L.lineno + 1, "fewer entries than the size line declares");
      if (blank(b, e) || *b == '%') continue;
      auto q = tokens(b, e);
      if (q.size() != 3) parse_fail(L.lineno, "entry must be 'row col value'");
      push(to_index(q[0], L.lineno), to_index(q[1], L.lineno), to_double(q[2], L.lineno), L.lineno);
      ++seen;
    }
  } else {
    const std::size_t count = symmetric ? nr * (nr + 1) / 2 : nr * nc;
    std::size_t seen = 0, i = 0, j = 0;
    while (seen < count) {
      if (!L.next(b, e)) parse_fail(L.lineno + 1, "fewer values than the size line declares");
      if (blank(b, e) || *b == '%') continue;
      for (auto tok : tokens(b, e)) {
        if (seen == count) parse_fail(L.lineno, "more values than the size line declares");
        const double v = to_double(tok, L.lineno);
        if (v != 0.0) push(i + 1, j + 1, v, L.lineno);
        ++seen;
        if (++i == nr) {
          ++j;
          i = symmetric ? j : 0;
        }
      }
    }
  }
  return from_triplets(nr, nc, ent);
}

constexpr char kMagic[8] = {'C', 'K', 'C', 'S', 'R', '0', '0', '1'};

Csr read_csrb(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw UsageError("cannot open file: " + path);
  char m[8];
  int64_t h[3];
  in.read(m, 8);
  in.read(reinterpret_cast<char*>(h), sizeof(h));
  if (!in || std::memcmp(m, kMagic, 8) != 0) throw UsageError("not a .csrb file: " + path);
  if (h[0] < 0 || h[1] < 0 || h[2] < 0) throw UsageError("corrupt .csrb header: " + path);
  std::vector<int64_t> rp((size_t)h[0] + 1);
  std::vector<int32_t> ci((size_t)h[2]);
  Csr a;
  a.nr = (size_t)h[0];
  a.nc = (size_t)h[1];
  a.va.resize((size_t)h[2]);
  in.read(reinterpret_cast<char*>(rp.data()), (std::streamsize)(8 * rp.size()));
  in.read(reinterpret_cast<char*>(ci.data()), (std::streamsize)(4 * ci.size()));
  in.read(reinterpret_cast<char*>(a.va.data()), (std::streamsize)(8 * a.va.size()));
  if (!in) throw UsageError("truncated .csrb file: " + path);
  a.rp.assign(rp.begin(), rp.end());
  a.ci.assign(ci.begin(), ci.end());
  return a;
}

void write_csrb(const Csr& a, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw UsageError("cannot open output file: " + path);
  const int64_t h[3] = {(int64_t)a.nr, (int64_t)a.nc, (int64_t)a.nnz()};
  out.write(kMagic, 8);
  out.write(reinterpret_cast<const char*>(h), sizeof(h));
  std::vector<int64_t> rp(a.rp.begin(), a.rp.end());
  std::vector<int32_t> ci(a.ci.size());
  for (std::size_t k = 0; k < ci.size(); ++k) {
    if (a.ci[k] >= (std::size_t)INT32_MAX) throw UsageError("column index >= 2^31");
    ci[k] = (int32_t)a.ci[k];
  }
  out.write(reinterpret_cast<const char*>(rp.data()), (std::streamsize)(8 * rp.size()));
  out.write(reinterpret_cast<const char*>(ci.data()), (std::streamsize)(4 * ci.size()));
  out.write(reinterpret_cast<const char*>(a.va.data()), (std::streamsize)(8 * a.va.size()));
  if (!out) throw std::runtime_error("write failed: " + path);
}

Csr load_matrix(const std::string& path) {
  if (ends_with(path, ".csrb")) return read_csrb(path);
  return read_matrix_market(slurp(path));
}

std::vector<double> load_vector(const std::string& path) {
  const std::string text = slurp(path);
  Lines L{text};
  const char *b, *e;
  std::vector<double> v;
  while (L.next(b, e)) {
    if (blank(b, e) || *b == '#') continue;
    auto t = tokens(b, e);
    if (t.size() != 1) parse_fail(L.lineno, "expected one value per line");
    v.push_back(to_double(t[0], L.lineno));
  }
  return v;
}

// ---------------------------------------------------------------- output
std::string sig17(double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::general, 17);
  return std::string(buf, r.ptr);
}
void kv(const std::string& k, const std::string& v) { std::cout << k << " = " << v << "\n"; }
void kv(const std::string& k, double v) { kv(k, sig17(v)); }
void kv(const std::string& k, std::size_t v) { kv(k, std::to_string(v)); }
void kv(const std::string& k, bool v) { kv(k, std::string(v ? "true" : "false")); }
void header(const std::string& k, const std::string& v) { std::cout << "# " << k << " = " << v << "\n"; }
void header(const std::string& k, double v) { header(k, sig17(v)); }
void header(const std::string& k, std::size_t v) { header(k, std::to_string(v)); }

// ------------------------------------------------------------------ flags
struct Args {
  std::map<std::string, std::string> kv;
  std::string get(const std::string& k, const std::string& dflt = "") const {
    auto it = kv.find(k);
    return it == kv.end() ? dflt : it->second;
  }
  bool has(const std::string& k) const { return kv.count(k) != 0; }
  double num(const std::string& k, double d) const { return has(k) ? std::stod(get(k)) : d; }
  std::size_t idx(const std::string& k, std::size_t d) const {
    return has(k) ? (std::size_t)std::stoull(get(k)) : d;
  }
  std::string need(const std::string& k) const {
    if (!has(k)) throw UsageError("missing --" + k);
    return get(k);
  }
};

// Shared estimator flags (condkit_cli.cpp:81-121 defaults).
struct AdamFlags {
  double alpha = 0.05, rel_tol = 1e-12, pivot_tol = 1e-14;
  std::size_t max_iter = 2000, patience = 100, restarts = 3;
  std::uint64_t seed = 1;
  explicit AdamFlags(const Args& a)
      : alpha(a.num("alpha", 0.05)), rel_tol(a.num("rel-tol", 1e-12)), pivot_tol(a.num("pivot-tol", 1e-14)),
        max_iter(a.idx("max-iter", 2000)), patience(a.idx("patience", 100)), restarts(a.idx("restarts", 3)),
        seed(a.has("seed") ? std::stoull(a.get("seed")) : 1) {}
  condkit_b200::AdamConfig config() const {
    condkit_b200::AdamConfig c;
    c.alpha = alpha;
    c.max_iter = max_iter;
    c.rel_tol = rel_tol;
    c.patience = patience;
    c.seed = seed;
    return c;
  }
  void echo() const {
    header("alpha", alpha);
    header("max_iter", max_iter);
    header("rel_tol", rel_tol);
    header("patience", patience);
    header("seed", std::to_string(seed));
    header("restarts", restarts);
    header("pivot_tol", pivot_tol);
  }
};

double device_norm_of_product(const condkit_b200::DeviceMatrix& d, const std::vector<double>& x) {
  // ||A x|| on the device (residual norm with b = 0)
  std::vector<double> zero(d.nrows(), 0.0);
  double rn = 0.0, xn = 0.0, bn = 0.0;
  condkit_b200::detail::check(ck_residual_norms(d.handle(), x.data(), zero.data(), &rn, &xn, &bn));
  return rn;
}

double two_norm(const std::vector<double>& v) {  // sparse.hpp:175-186, for the report line
  double amax = 0.0;
  for (double x : v) amax = std::max(amax, std::abs(x));
  if (amax == 0.0) return 0.0;
  if (!std::isfinite(amax)) return amax;
  double s = 0.0;
  for (double x : v) {
    const double q = x / amax;
    s += q * q;
  }
  return amax * std::sqrt(s);
}

// -------------------------------------------------------------- commands
int run_cond(const Args& a) {
  const std::string path = a.need("matrix"), scale = a.get("scale", "none");
  const AdamFlags f(a);
  header("subcommand", "cond");
  header("matrix", path);
  header("scale", scale);
  f.echo();
  Csr m = load_matrix(path);
  if (scale == "column") {
    auto [vals, norms] = condkit_b200::column_scale_values(m);
    m.va = std::move(vals);
  } else if (scale == "row") {
    condkit_b200::DeviceMatrix d0(m);
    std::vector<int64_t> rp(m.rp.begin(), m.rp.end());
    std::vector<double> vals(m.nnz()), norms(m.nr);
    int64_t zero = -1;
    condkit_b200::detail::check(
        ck_row_scale(d0.handle(), rp.data(), m.va.data(), vals.data(), nullptr, nullptr, norms.data(), &zero),
        zero);
    m.va = std::move(vals);
  } else if (scale != "none") {
    throw UsageError("--scale must be none, column or row");
  }
  condkit_b200::DeviceMatrix d(m);
  condkit_b200::Cond2Result r = condkit_b200::cond2(d, f.config(), f.restarts, f.pivot_tol);
  kv("n", m.nr);
  kv("nnz", m.nnz());
  kv("kappa2", r.kappa);
  kv("operator_norm", r.operator_norm.value);
  kv("operator_norm_iterations", r.operator_norm.iterations);
  kv("operator_norm_converged", r.operator_norm.converged);
  double op_check = std::numeric_limits<double>::quiet_NaN();
  if (!r.operator_norm.witness.empty()) op_check = device_norm_of_product(d, r.operator_norm.witness);
  kv("operator_norm_recomputed", op_check);
  kv("inverse_norm", r.inverse_norm.value);
  kv("inverse_norm_iterations", r.inverse_norm.iterations);
  kv("inverse_norm_converged", r.inverse_norm.converged);
  double inv_check = std::numeric_limits<double>::quiet_NaN();
  if (r.factors && !r.inverse_norm.witness.empty())
    inv_check = two_norm(condkit_b200::lu_solve(*r.factors, r.inverse_norm.witness));
  kv("inverse_norm_recomputed", inv_check);
  kv("singularity_cap", condkit_b200::singularity_bound(std::max(1.0, r.kappa)));
  const bool singular = r.kappa >= 1.0 / condkit_b200::kEpsMach;
  kv("verdict", std::string(singular ? "numerically_singular" : "regular"));
  return singular ? kExitSingular : kExitOk;
}

int run_norm(const Args& a) {
  const std::string path = a.need("matrix");
  const AdamFlags f(a);
  header("subcommand", "norm");
  header("matrix", path);
  f.echo();
  Csr m = load_matrix(path);
  condkit_b200::DeviceMatrix d(m);
  condkit_b200::NormEstimate est = condkit_b200::estimate_norm(d, f.config(), f.restarts);
  kv("n", m.nr);
  kv("nnz", m.nnz());
  kv("operator_norm", est.value);
  kv("iterations", est.iterations);
  kv("converged", est.converged);
  double check = std::numeric_limits<double>::quiet_NaN();
  if (!est.witness.empty()) check = device_norm_of_product(d, est.witness);
  kv("operator_norm_recomputed", check);
  return kExitOk;
}

const char* verdict_name(condkit_b200::Verdict v) {
  switch (v) {
    case condkit_b200::Verdict::accepted: return "accepted";
    case condkit_b200::Verdict::rejected: return "rejected";
    default: return "numerically_singular";
  }
}

int run_verify(const Args& a) {
  const std::string path = a.need("matrix"), rhs = a.need("rhs"), sol = a.need("solution");
  const AdamFlags f(a);
  condkit_b200::VerifyOptions o;
  o.threshold = a.num("threshold", 1e-7);
  if (a.has("kappa")) o.kappa = a.num("kappa", 0.0);
  if (a.has("a-norm")) o.a_norm = a.num("a-norm", 0.0);
  o.adam = f.config();
  o.restarts = f.restarts;
  o.pivot_tol = f.pivot_tol;
  header("subcommand", "verify");
  header("matrix", path);
  header("rhs", rhs);
  header("solution", sol);
  header("threshold", o.threshold);
  if (o.kappa) header("kappa", *o.kappa);
  if (o.a_norm) header("a_norm", *o.a_norm);
  f.echo();
  Csr m = load_matrix(path);
  const std::vector<double> b = load_vector(rhs), x = load_vector(sol);
  condkit_b200::DeviceMatrix d(m);
  condkit_b200::BoundsReport r = condkit_b200::verify_solution(d, x, b, o);
  kv("residual_norm", r.residual_norm);
  kv("b_norm", r.b_norm);
  kv("a_norm", r.a_norm);
  kv("xhat_norm", r.xhat_norm);
  kv("kappa", r.kappa);
  kv("kappa_source", std::string(r.kappa_supplied ? "supplied" : "estimated"));
  kv("loose_lower", r.loose_lower);
  kv("loose_upper", r.loose_upper);
  kv("tight_lower", r.tight_lower);
  kv("tight_upper", r.tight_upper);
  kv("true_error_cap", r.true_error_cap);
  kv("singularity_cap", r.singularity_cap);
  kv("threshold", r.threshold);
  kv("eps_mach", r.eps_mach);
  kv("verdict", std::string(verdict_name(r.verdict)));
  switch (r.verdict) {
    case condkit_b200::Verdict::accepted: return kExitOk;
    case condkit_b200::Verdict::numerically_singular: return kExitSingular;
    default: return kExitRejected;
  }
}

int run_convert(const Args& a) {
  const std::string in = a.need("matrix"), out = a.need("out");
  Csr m = load_matrix(in);
  write_csrb(m, out);
  header("subcommand", "convert");
  kv("n", m.nr);
  kv("ncols", m.nc);
  kv("nnz", m.nnz());
  kv("output", out);
  return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: condkit_b200_cli {cond|norm|verify|convert} --matrix FILE [--key value ...]\n";
    return kExitUsage;
  }
  const std::string cmd = argv[1];
  Args args;
  for (int k = 2; k < argc; ++k) {
    std::string key = argv[k];
    if (key.rfind("--", 0) != 0 || k + 1 >= argc) {
      std::cerr << "error: expected --key value, got '" << key << "'\n";
      return kExitUsage;
    }
    args.kv[key.substr(2)] = argv[++k];
  }
  try {
    if (cmd == "cond") return run_cond(args);
    if (cmd == "norm") return run_norm(args);
    if (cmd == "verify") return run_verify(args);
    if (cmd == "convert") return run_convert(args);
    std::cerr << "error: unknown subcommand '" << cmd << "'\n";
    return kExitUsage;
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  }
}
