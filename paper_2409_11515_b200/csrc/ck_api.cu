// C ABI (include/condkit_b200.h): argument checking, exception -> status
// mapping, the host RNG mirror, the scalar error-bound formulas and the
// estimate_norm orchestration over device sessions.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <mutex>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "ck_common.h"
#include "ck_internal.h"
#include "ck_lu.h"
#include "ck_session.h"

namespace ck {
void session_create(ck_session_s* s, ck_matrix_s* A, const ck_adam_cfg* cfg,
                    const uint64_t* seeds, int R);
void session_run(ck_session_s* s, uint64_t max_steps, int32_t* finished);
void session_time(ck_session_s* s, uint64_t steps, int32_t mode, double* ms_total,
                  double* ms_apply, double* ms_transpose);
void session_result(ck_session_s* s, int c, ck_norm_result* res, double* witness);
void session_step_observed(ck_session_s* s, ck_step_info* info, double* x, double* x_min);

static thread_local std::string g_last_error;

void fail(ck_status c, const std::string& msg) { throw Error(c, msg); }

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  // the error is reported through the status / exception: clear the runtime's
  // per-thread "last error" so it does not resurface in an unrelated later call
  cudaGetLastError();
  std::string m = std::string(what) + " failed: " + cudaGetErrorString(e) + " (" + file + ":" +
                  std::to_string(line) + ")";
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) throw Error(CK_ERR_NO_DEVICE, m);
  if (e == cudaErrorMemoryAllocation) throw Error(CK_ERR_OUT_OF_MEMORY, m);
  throw Error(CK_ERR_CUDA, m);
}

template <class F>
static ck_status guarded(const char* name, F&& f) {
  NvtxRange range(name);  // one NVTX range per C-ABI call (nsys / ncu --nvtx)
  try {
    f();
    return CK_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return CK_ERR_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return CK_ERR_LOGIC;
  }
}

// sparse.hpp:175-186, sequential so the result is bit-identical.
static double two_norm_seq(const double* v, int64_t n) {
  double amax = 0.0;
  for (int64_t i = 0; i < n; ++i) amax = std::max(amax, std::abs(v[i]));
  if (amax == 0.0) return 0.0;
  if (!std::isfinite(amax)) return amax;
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double q = v[i] / amax;
    s += q * q;
  }
  return amax * std::sqrt(s);
}

// Host cores random_unit_vector_host leaves free on the calling thread's behalf.
static thread_local int tl_rng_reserve_cores = 0;

template <class F>
static void parallel_for(int64_t n, F&& f) {
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  int64_t nt = n < (int64_t(1) << 18) ? 1 : std::min<int64_t>(hw, 64);
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

// std::mt19937_64 (the reference's engine, rng.hpp:23-33) in bulk. The state
// leaves the engine through its standard text form, words are produced 312 at
// a time by a branch-free twist and a temper loop the compiler vectorises, and
// the state goes back, so the engine continues exactly as if it had been
// called `count` times. A one-time self-check against the engine's own
// operator() gates it (any mismatch -> per-call draws).
struct Mt64Bulk {
  static constexpr int N = 312, M = 156;
  static constexpr uint64_t kA = 0xB5026F5AA96619E9ull, kUp = ~uint64_t(0) << 31,
                            kLo = ~kUp;
  uint64_t x[N];
  uint64_t p = N;
  bool ok = false;

  explicit Mt64Bulk(const std::mt19937_64& g) {
    std::stringstream ss;
    ss << g;
    for (auto& w : x) ss >> w;
    ss >> p;
    ok = !ss.fail() && p <= (uint64_t)N;
  }
  void store(std::mt19937_64& g) const {
    std::stringstream ss;
    for (auto w : x) ss << w << ' ';
    ss << p;
    ss >> g;
  }
  static uint64_t mix(uint64_t a, uint64_t b, uint64_t c) {
    const uint64_t y = (a & kUp) | (b & kLo);
    return c ^ (y >> 1) ^ ((0 - (y & 1)) & kA);
  }
  void twist() {
    for (int i = 0; i < N - M; ++i) x[i] = mix(x[i], x[i + 1], x[i + M]);
    for (int i = N - M; i < N - 1; ++i) x[i] = mix(x[i], x[i + 1], x[i + M - N]);
    x[N - 1] = mix(x[N - 1], x[0], x[M - 1]);
    p = 0;
  }
  static uint64_t temper(uint64_t z) {
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71D67FFFEDA60000ull;
    z ^= (z << 37) & 0xFFF7EEE000000000ull;
    return z ^ (z >> 43);
  }
  // the next `count` state words, untempered (temper() of each is the output)
  void fill_raw(uint64_t* __restrict out, int64_t count) {
    while (count > 0) {
      if (p == (uint64_t)N) twist();
      const int64_t k = std::min<int64_t>(N - (int64_t)p, count);
      std::memcpy(out, x + p, sizeof(uint64_t) * (size_t)k);
      p += (uint64_t)k;
      out += k;
      count -= k;
    }
  }
  static bool verified() {
    static const bool v = [] {
      std::mt19937_64 g(12345), h(12345);
      for (int i = 0; i < 100; ++i) g();
      for (int i = 0; i < 100; ++i) h();
      Mt64Bulk b(g);
      if (!b.ok) return false;
      std::vector<uint64_t> w(1000);
      b.fill_raw(w.data(), 1000);
      b.store(g);
      for (auto v : w)
        if (temper(v) != h()) return false;
      return g() == h() && g == h;
    }();
    return v;
  }
};

// random_unit_vector (rng.hpp:68-77) with standard_normal (rng.hpp:61-65) and
// uniform01 (rng.hpp:31-33). The engine draws stay sequential (they define the
// stream) and run on the calling thread block by block, while a helper thread
// applies the Box-Muller transform of the previous block on all host threads
// (pipelined; no n-sized draw buffer). The norm is the reference's two_norm:
// amax (exact in any order, folded into the transform), then the sequential
// scaled sum of squares. With `dst`, the normalised vector goes to dst()
// (called once the norm is known) and `out` is scratch.
void random_unit_vector_host(void* engine, int64_t n, double* out,
                             const std::function<double*()>& dst) {
  if (n <= 0) return;
  auto& g = *static_cast<std::mt19937_64*>(engine);
  constexpr int64_t kBlock = int64_t(1) << 18;  // pairs per pipeline block
  std::vector<uint64_t> buf[2];
  buf[0].resize((size_t)(2 * std::min(n, kBlock)));
  buf[1].resize(buf[0].size());
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  // a background draw (ck_start_vector_prefetch) leaves cores to the thread that is
  // uploading and building the operator meanwhile: with every core taken, that thread's
  // launches and stream waits sporadically stalled for 0.3-0.8 s
  const int64_t nthr = std::max<int64_t>(1, std::min<int64_t>((int64_t)hw - tl_rng_reserve_cores, 64));
  // bulk draws from 2^15 words on (text state round trip ~0.1 ms)
  std::unique_ptr<Mt64Bulk> bulk;
  if (n >= (int64_t(1) << 14) && Mt64Bulk::verified()) {
    bulk.reset(new Mt64Bulk(g));
    if (!bulk->ok) bulk.reset();
  }
  const bool raw = bulk != nullptr;
  double nrm = 0.0;
  while (nrm == 0.0) {
    std::vector<double> amax((size_t)nthr, 0.0);
    std::thread worker;
    for (int64_t b0 = 0; b0 < n; b0 += kBlock) {
      const int64_t len = std::min(kBlock, n - b0);
      std::vector<uint64_t>& d = buf[(b0 / kBlock) & 1];
      if (bulk) {
        bulk->fill_raw(d.data(), 2 * len);  // tempered by the transform threads
      } else {
        for (int64_t k = 0; k < 2 * len; ++k) d[(size_t)k] = g();
      }
      if (worker.joinable()) worker.join();
      worker = std::thread([&, b0, len, dp = d.data()] {
        const int64_t chunk = ceil_div(len, nthr);
        std::vector<std::thread> pool;
        for (int64_t t = 0; t < nthr; ++t) {
          const int64_t lo = t * chunk, hi = std::min(len, lo + chunk);
          if (lo >= hi) break;
          pool.emplace_back([&amax, dp, out, b0, lo, hi, t, raw] {
            double m = amax[(size_t)t];
            for (int64_t i = lo; i < hi; ++i) {
              uint64_t w1 = dp[2 * i], w2 = dp[2 * i + 1];
              if (raw) {
                w1 = Mt64Bulk::temper(w1);
                w2 = Mt64Bulk::temper(w2);
              }
              const double u1 = 1.0 - static_cast<double>(w1 >> 11) * 0x1.0p-53;
              const double u2 = static_cast<double>(w2 >> 11) * 0x1.0p-53;
              const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793 * u2);
              out[b0 + i] = z;
              m = std::max(m, std::abs(z));
            }
            amax[(size_t)t] = m;
          });
        }
        for (auto& th : pool) th.join();
      });
    }
    if (worker.joinable()) worker.join();
    double am = 0.0;
    for (double m : amax) am = std::max(am, m);
    if (am == 0.0 || !std::isfinite(am)) {
      nrm = am;
    } else {
      double sq = 0.0;  // two_norm's scaled sum, in order (sparse.hpp:175-186)
      for (int64_t i = 0; i < n; ++i) {
        const double q = out[i] / am;
        sq += q * q;
      }
      nrm = am * std::sqrt(sq);
    }
  }
  if (bulk) bulk->store(g);
  double* to = dst ? dst() : out;  // may wait for the destination to exist
  parallel_for(n, [&](int64_t b, int64_t e) {
    for (int64_t i = b; i < e; ++i) to[i] = out[i] / nrm;
  });
}

// Device allocations from the default stream-ordered pool (ck_common.h).
// CK_PLAIN_MALLOC=1 goes back to cudaMalloc / cudaFree (A/B switch).
namespace {
bool use_pool() {
  static const bool on = std::getenv("CK_PLAIN_MALLOC") == nullptr;
  return on;
}
void pool_configure_once(int dev) {
  static std::mutex mu;
  static std::vector<char> done;
  std::lock_guard<std::mutex> lk(mu);
  if ((int)done.size() <= dev) done.resize(dev + 1, 0);
  if (done[dev]) return;
  cudaMemPool_t pool = nullptr;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = ~0ull;  // freed blocks stay in the pool until device_trim()
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
  done[dev] = 1;
}
}  // namespace

cudaError_t device_alloc(void** p, size_t bytes) {
  if (!use_pool()) return cudaMalloc(p, bytes);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  pool_configure_once(dev);
  e = cudaMallocAsync(p, bytes, cudaStreamPerThread);
  if (e == cudaErrorMemoryAllocation) {  // cached blocks of other sizes in the way: release them and retry
    cudaGetLastError();
    device_trim();
    e = cudaMallocAsync(p, bytes, cudaStreamPerThread);
  }
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(cudaStreamPerThread);  // usable on every stream from here on
}

void device_free(void* p) {
  if (p == nullptr) return;
  if (!use_pool()) {
    cudaFree(p);
    return;
  }
  cudaDeviceSynchronize();  // cudaFree's implicit wait: no stream may still use the block
  cudaFreeAsync(p, cudaStreamPerThread);
}

void device_trim() {
  if (!use_pool()) return;
  int dev = 0;
  cudaMemPool_t pool = nullptr;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    cudaDeviceSynchronize();
    cudaMemPoolTrimTo(pool, 0);
  }
  cudaGetLastError();
}

// Process-wide cache of released pinned staging buffers (ck_common.h).
namespace {
struct PinnedCache {
  std::mutex mu;
  std::vector<std::pair<void*, size_t>> free_list;  // never freed at exit: the driver may be gone
};
PinnedCache& pinned_cache() {
  static PinnedCache* c = new PinnedCache();
  return *c;
}
constexpr size_t kPinnedCacheBuffers = 6;  // staging chunks of pageable uploads + start-vector buffers
constexpr size_t kPinnedCacheBytes = size_t(1) << 30;
}  // namespace

void* pinned_acquire(size_t bytes, size_t* got_bytes) {
  {
    PinnedCache& c = pinned_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    int best = -1;
    // smallest cached buffer that fits, but none more than twice the request: a 32 MB
    // staging chunk must not take the 200 MB start-vector buffer out of the cache
    for (int i = 0; i < (int)c.free_list.size(); ++i)
      if (c.free_list[i].second >= bytes && c.free_list[i].second <= 2 * bytes &&
          (best < 0 || c.free_list[i].second < c.free_list[best].second))
        best = i;
    if (best >= 0) {
      void* p = c.free_list[best].first;
      *got_bytes = c.free_list[best].second;
      c.free_list.erase(c.free_list.begin() + best);
      return p;
    }
  }
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  *got_bytes = bytes;
  return p;
}

void pinned_release(void* p, size_t bytes) {
  if (p == nullptr) return;
  {
    PinnedCache& c = pinned_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    size_t total = bytes;
    for (auto& e : c.free_list) total += e.second;
    if (c.free_list.size() < kPinnedCacheBuffers && total <= kPinnedCacheBytes) {
      c.free_list.emplace_back(p, bytes);
      return;
    }
  }
  cudaFreeHost(p);
}

// ck_start_vector_prefetch's slot: one start vector drawn on a helper thread
// into pageable scratch, then normalised into a pinned buffer (the session
// adopts that buffer as its staging).
namespace {
struct StartPrefetch {
  uint64_t seed = 0;
  int64_t n = 0;
  int device = 0;
  std::mt19937_64 g;
  PinnedBuf<double> pin;
  std::exception_ptr err;
  std::thread th;
  ~StartPrefetch() {
    if (th.joinable()) th.join();
  }
};
std::mutex g_pf_mu;
std::unique_ptr<StartPrefetch> g_pf;
uint64_t g_pf_taken = 0, g_pf_dropped = 0;  // ck_start_vector_prefetch_stats
}  // namespace

// The slot is consumed by the first session that asks: taken when seed and n
// match, dropped (thread joined, pinned buffer freed) otherwise.
bool take_start_prefetch(uint64_t seed, int64_t n, void* engine, PinnedBuf<double>* hx) {
  std::unique_ptr<StartPrefetch> pf;
  bool match = false;
  {
    std::lock_guard<std::mutex> lk(g_pf_mu);
    if (!g_pf) return false;
    match = g_pf->seed == seed && g_pf->n == n;
    pf = std::move(g_pf);
  }
  if (pf->th.joinable()) pf->th.join();
  if (!match || pf->err || pf->pin.p == nullptr) {  // draw it on the caller's thread
    std::lock_guard<std::mutex> lk(g_pf_mu);
    ++g_pf_dropped;
    return false;
  }
  *static_cast<std::mt19937_64*>(engine) = pf->g;
  std::swap(hx->p, pf->pin.p);
  std::swap(hx->n, pf->pin.n);
  std::lock_guard<std::mutex> lk(g_pf_mu);
  ++g_pf_taken;
  return true;
}

}  // namespace ck

extern "C" ck_status ck_start_vector_prefetch(uint64_t seed, int64_t n) {
  using namespace ck;
  return guarded(__func__, [&] {
    if (n <= 0) fail(CK_ERR_INVALID_ARGUMENT, "ck_start_vector_prefetch: n must be positive");
    std::unique_ptr<StartPrefetch> old;
    auto pf = std::make_unique<StartPrefetch>();
    pf->seed = seed;
    pf->n = n;
    pf->g.seed(seed);
    CK_CUDA(cudaGetDevice(&pf->device));
    StartPrefetch* p = pf.get();
    pf->th = std::thread([p] {
      tl_rng_reserve_cores = 3;
      try {
        // The pinned buffer is pinned after the draw, not alongside it: pinning
        // 8n bytes holds the driver for ~0.1 s and stalls whatever upload call
        // runs concurrently (measured: A^T build 30 -> 85-113 ms, e2e
        // 389-412 vs 413-415 it/s)
        std::unique_ptr<double[]> scratch(new double[(size_t)p->n]);
        random_unit_vector_host(&p->g, p->n, scratch.get(), [p]() -> double* {
          CK_CUDA(cudaSetDevice(p->device));
          p->pin.resize(p->n);
          return p->pin.data();
        });
      } catch (...) {
        p->err = std::current_exception();
      }
    });
    std::lock_guard<std::mutex> lk(g_pf_mu);
    old = std::move(g_pf);
    g_pf = std::move(pf);
  });
}

extern "C" ck_status ck_start_vector_prefetch_cancel(void) {
  using namespace ck;
  return guarded(__func__, [&] {
    std::unique_ptr<StartPrefetch> old;
    std::lock_guard<std::mutex> lk(g_pf_mu);
    old = std::move(g_pf);
    if (old) ++g_pf_dropped;
  });
}

extern "C" ck_status ck_start_vector_prefetch_stats(uint64_t* taken, uint64_t* dropped) {
  using namespace ck;
  return guarded(__func__, [&] {
    std::lock_guard<std::mutex> lk(g_pf_mu);
    if (taken) *taken = g_pf_taken;
    if (dropped) *dropped = g_pf_dropped;
  });
}

namespace ck {

// Restart columns per explicit-operator sweep (estimate_norm, cond2, batches).
// Small operators are launch/latency bound and share one sweep among up to 4
// restarts; on large ones the R per-entry gathers bound an R-column sweep and
// two columns per sweep is the measured optimum.
// CK_RESTART_GROUP overrides (A/B switch).
bool matrix_window_ok(ck_matrix_s* m);  // ck_adam.cu
// batch: the operator is a block-diagonal ensemble (config 5). Banded members sweep
// from the shared-memory window, where four columns per sweep pay (config 5:
// 194k member-iterations/s against 191k in pairs; with global gathers 131k vs 165k).
static int restart_group(ck_matrix_s* m, uint64_t restarts, bool batch = false) {
  const char* e = std::getenv("CK_RESTART_GROUP");
  if (e && e[0] >= '1' && e[0] <= '4') return e[0] - '0';
  if (m->nnz < (int64_t(1) << 24)) return kMaxCols;
  if (batch && !std::getenv("CK_NO_WINDOW") && matrix_window_ok(m)) return kMaxCols;
  // large operators (config 4, per step): R = 1 2.24, 2 4.07, 3 6.19, 4 10.45 ms ->
  // three restarts in one sweep, otherwise pairs
  return restarts == 3 ? 3 : 2;
}

static void check_cfg(const ck_adam_cfg* cfg) {
  if (cfg == nullptr) fail(CK_ERR_INVALID_ARGUMENT, "cfg is NULL");
}

static ck_session_s* S(ck_session s) {
  if (s == nullptr) fail(CK_ERR_INVALID_ARGUMENT, "session handle is NULL");
  CK_CUDA(cudaSetDevice(s->device));
  return s;
}

static ck_matrix_s* M(ck_matrix a) {
  if (a == nullptr) fail(CK_ERR_INVALID_ARGUMENT, "matrix handle is NULL");
  CK_CUDA(cudaSetDevice(a->device));
  return a;
}

}  // namespace ck

using namespace ck;

extern "C" {

const char* ck_last_error(void) { return g_last_error.c_str(); }

int32_t ck_abi_version(void) { return 1; }

ck_status ck_device_count(int32_t* count) {
  return guarded(__func__, [&] {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
      cudaGetLastError();
      n = 0;
    } else {
      CK_CUDA(e);
    }
    *count = n;
  });
}

ck_status ck_device_memory(uint64_t* free_bytes, uint64_t* total_bytes, int32_t* sm_count) {
  return guarded(__func__, [&] {
    size_t f = 0, t = 0;
    device_trim();  // cached pool blocks count as free
    CK_CUDA(cudaMemGetInfo(&f, &t));
    int dev = 0, sms = 0;
    CK_CUDA(cudaGetDevice(&dev));
    CK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (free_bytes) *free_bytes = f;
    if (total_bytes) *total_bytes = t;
    if (sm_count) *sm_count = sms;
  });
}

ck_status ck_set_device(int32_t device) {
  return guarded(__func__, [&] {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
      cudaGetLastError();
      fail(CK_ERR_NO_DEVICE, "no CUDA device visible");
    }
    cudaDeviceProp p{};
    CK_CUDA(cudaGetDeviceProperties(&p, device));
    if (p.major != 10) fail(CK_ERR_NO_DEVICE, std::string("device is not sm_100: ") + p.name);
    CK_CUDA(cudaSetDevice(device));
  });
}

ck_status ck_device_synchronize(void) {
  return guarded(__func__, [&] { CK_CUDA(cudaDeviceSynchronize()); });
}

ck_status ck_host_register(void* ptr, uint64_t bytes) {
  return guarded(__func__, [&] {
    if (bytes == 0) return;
    const cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterDefault);
    if (e == cudaErrorHostMemoryAlreadyRegistered) {  // pinned already: nothing to do
      cudaGetLastError();
      return;
    }
    CK_CUDA(e);
  });
}

ck_status ck_host_unregister(void* ptr) {
  return guarded(__func__, [&] { CK_CUDA(cudaHostUnregister(ptr)); });
}

void ck_adam_default(ck_adam_cfg* c) {
  c->alpha = 0.05;
  c->beta1 = 0.9;
  c->beta2 = 0.999;
  c->eps_stab = 1e-8;
  c->max_iter = 2000;
  c->seed = 1;
  c->rel_tol = 1e-12;
  c->patience = 100;
}

uint64_t ck_mix_seed(uint64_t base, uint64_t stream) {
  uint64_t z = base + 0x9E3779B97F4A7C15ull * (stream + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

ck_status ck_random_unit_vectors(uint64_t seed, int64_t n, int64_t count, double* out) {
  return guarded(__func__, [&] {
    if (n < 0 || count < 0) fail(CK_ERR_INVALID_ARGUMENT, "negative size");
    std::mt19937_64 g(seed);
    for (int64_t c = 0; c < count; ++c) random_unit_vector_host(&g, n, out + c * n);
  });
}

ck_status ck_uniform_in(uint64_t seed, int64_t count, double lo, double hi, double* out) {
  return guarded(__func__, [&] {
    if (count < 0) fail(CK_ERR_INVALID_ARGUMENT, "negative size");
    std::mt19937_64 g(seed);
    for (int64_t i = 0; i < count; ++i)
      out[i] = lo + (hi - lo) * (static_cast<double>(g() >> 11) * 0x1.0p-53);
  });
}

// ---------------------------------------------- error_bounds.hpp:59-99
ck_status ck_loose_bounds(double rn, double bn, double kappa, double* lo, double* hi) {
  return guarded(__func__, [&] {
    if (!(rn >= 0.0)) fail(CK_ERR_INVALID_ARGUMENT, "residual norm must be >= 0");
    if (!(kappa >= 1.0)) fail(CK_ERR_INVALID_ARGUMENT, "kappa must be >= 1");
    if (bn == 0.0) fail(CK_ERR_ZERO_RHS, "right-hand side has zero norm");
    if (!(bn > 0.0)) fail(CK_ERR_INVALID_ARGUMENT, "b norm must be >= 0");
    double rho = rn / bn;
    if (rho == 0.0) {
      *lo = 0.0;
      *hi = 0.0;
      return;
    }
    *lo = rho / kappa;
    *hi = kappa * rho;
  });
}

ck_status ck_tight_bounds(double rn, double an, double xn, double kappa, double* lo, double* hi) {
  return guarded(__func__, [&] {
    if (!(rn >= 0.0)) fail(CK_ERR_INVALID_ARGUMENT, "residual norm must be >= 0");
    if (!(kappa >= 1.0)) fail(CK_ERR_INVALID_ARGUMENT, "kappa must be >= 1");
    if (xn == 0.0) fail(CK_ERR_ZERO_SOLUTION, "candidate solution has zero norm");
    if (!(xn > 0.0)) fail(CK_ERR_INVALID_ARGUMENT, "solution norm must be >= 0");
    if (!(an > 0.0)) fail(CK_ERR_INVALID_ARGUMENT, "operator norm must be > 0");
    double rho = rn / (an * xn);
    if (rho == 0.0) {
      *lo = 0.0;
      *hi = 0.0;
      return;
    }
    *lo = rho;
    *hi = kappa * rho;
  });
}

ck_status ck_propagate_bound(double e, double* out) {
  return guarded(__func__, [&] {
    if (!(e >= 0.0)) fail(CK_ERR_INVALID_ARGUMENT, "bound must be >= 0");
    *out = e >= 1.0 ? std::numeric_limits<double>::infinity() : e / (1.0 - e);
  });
}

ck_status ck_singularity_bound(double kappa, double eps, double* out) {
  return guarded(__func__, [&] {
    if (!(kappa >= 1.0)) fail(CK_ERR_INVALID_ARGUMENT, "kappa must be >= 1");
    if (!(eps > 0.0)) fail(CK_ERR_INVALID_ARGUMENT, "eps_mach must be > 0");
    double ke = kappa * eps;
    *out = ke >= 1.0 ? std::numeric_limits<double>::infinity() : 2.0 * ke / (1.0 - ke);
  });
}

// ---------------------------------------------------------- operator
ck_status ck_matrix_upload(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci,
                           const double* va, ck_matrix* out) {
  return guarded(__func__, [&] {
    if (out == nullptr) fail(CK_ERR_INVALID_ARGUMENT, "out is NULL");
    auto* m = new ck_matrix_s();
    try {
      matrix_upload(m, nrows, ncols, rp, ci, va);
    } catch (...) {
      if (m->stream) cudaStreamDestroy(m->stream);
      delete m;
      throw;
    }
    *out = m;
  });
}

ck_status ck_matrix_free(ck_matrix a) {
  return guarded(__func__, [&] {
    if (!a) return;
    cudaSetDevice(a->device);
    cudaStreamSynchronize(a->stream);
    cudaStream_t s = a->stream;
    delete a;
    if (s) cudaStreamDestroy(s);
  });
}
}  // extern "C"

namespace ck {
void matrix_info(const ck_matrix_s* a, ck_matrix_info* info) {
  info->nrows = a->nrows;
  info->ncols = a->ncols;
  info->nnz = a->nnz;
  info->sell_entries_a = a->a.entries;
  info->sell_entries_at = a->at.entries;
  auto sb = [](const Sell& s) {
    return s.slice_ptr.bytes() + s.len.bytes() + s.col.bytes() + s.col16.bytes() + s.cbase.bytes() +
           s.ptab.bytes() + s.poff.bytes() +
           s.val.bytes() + s.perm.bytes() + s.inv.bytes();
  };
  info->device_bytes = sb(a->a) + sb(a->at);
  info->device = a->device;
  info->col_format = (a->a.narrow ? 1 : 0) | (a->at.narrow ? 2 : 0) | (a->a.pattern ? 4 : 0) |
                     (a->at.pattern ? 8 : 0);
}
}  // namespace ck

extern "C" {
ck_status ck_matrix_get_info(ck_matrix a, ck_matrix_info* info) {
  return guarded(__func__, [&] {
    if (!info) fail(CK_ERR_INVALID_ARGUMENT, "info is NULL");
    matrix_info(M(a), info);
  });
}

ck_status ck_spmv(ck_matrix a, const double* x, double* y) {
  return guarded(__func__, [&] { matrix_apply_host(M(a), false, x, y); });
}

ck_status ck_spmv_t(ck_matrix a, const double* x, double* y) {
  return guarded(__func__, [&] { matrix_apply_host(M(a), true, x, y); });
}

ck_status ck_residual_norms(ck_matrix a, const double* x, const double* b, double* rn, double* xn,
                            double* bn) {
  return guarded(__func__, [&] { residual_norms(M(a), x, b, rn, xn, bn); });
}

ck_status ck_loss_explicit(ck_matrix a, const double* x, double* loss) {
  return guarded(__func__, [&] {
    bool deg = false;
    double l = loss_explicit_dev(M(a), x, &deg);
    if (deg) fail(CK_ERR_INVALID_ARGUMENT, "operator maps direction to zero (DegenerateDirection)");
    *loss = l;
  });
}

ck_status ck_grad_explicit(ck_matrix a, const double* x, double* g) {
  return guarded(__func__, [&] {
    bool deg = false;
    grad_explicit_dev(M(a), x, g, &deg);
    if (deg) fail(CK_ERR_INVALID_ARGUMENT, "operator maps direction to zero (DegenerateDirection)");
  });
}

// ------------------------------------------------------ sessions
ck_status ck_session_create(ck_matrix a, const ck_adam_cfg* cfg, const uint64_t* seeds,
                            int32_t ncols, ck_session* out) {
  return guarded(__func__, [&] {
    check_cfg(cfg);
    auto* s = new ck_session_s();
    try {
      session_create(s, M(a), cfg, seeds, ncols);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

ck_status ck_session_run(ck_session s, uint64_t max_steps, int32_t* finished) {
  return guarded(__func__, [&] {
    S(s);
    session_run(s, max_steps, finished);
  });
}

ck_status ck_session_step_observed(ck_session s, ck_step_info* info, double* x, double* x_min) {
  return guarded(__func__, [&] {
    S(s);
    if (s->R != 1) fail(CK_ERR_INVALID_ARGUMENT, "observer mode needs a single-column session");
    session_step_observed(s, info, x, x_min);
  });
}

ck_status ck_session_time(ck_session s, uint64_t steps, int32_t mode, double* ms_total,
                          double* ms_apply, double* ms_transpose) {
  return guarded(__func__, [&] {
    S(s);
    session_time(s, steps, mode, ms_total, ms_apply, ms_transpose);
  });
}

ck_status ck_session_result(ck_session s, int32_t column, ck_norm_result* res, double* witness) {
  return guarded(__func__, [&] {
    S(s);
    session_result(s, column, res, witness);
  });
}

ck_status ck_session_free(ck_session s) {
  return guarded(__func__, [&] {
    if (!s) return;
    cudaSetDevice(s->device);
    cudaStreamSynchronize(s->stream);
    delete s;
  });
}

// projected_adam / norm2, condest.hpp:184-297, 315-317
ck_status ck_projected_adam(ck_matrix a, const ck_adam_cfg* cfg, ck_norm_result* res,
                            double* witness) {
  return guarded(__func__, [&] {
    check_cfg(cfg);
    ck_session_s s;
    uint64_t seed = cfg->seed;
    session_create(&s, M(a), cfg, &seed, 1);
    int32_t fin = 0;
    session_run(&s, 0, &fin);
    session_result(&s, 0, res, witness);
  });
}

// estimate_norm, condest.hpp:301-312: restart r uses seed cfg.seed (r = 0) or
// mix_seed(cfg.seed, r); the first strictly larger value wins. Up to four
// restarts share each device sweep.
ck_status ck_estimate_norm(ck_matrix a, const ck_adam_cfg* cfg, uint64_t restarts,
                           ck_norm_result* res, double* witness) {
  return guarded(__func__, [&] {
    check_cfg(cfg);
    if (restarts == 0) fail(CK_ERR_INVALID_ARGUMENT, "estimate_norm: restarts must be >= 1");
    M(a);
    bool have = false;
    const int group = restart_group(a, restarts);
    for (uint64_t r0 = 0; r0 < restarts; r0 += group) {
      int R = (int)std::min<uint64_t>(group, restarts - r0);
      std::vector<uint64_t> seeds(R);
      for (int c = 0; c < R; ++c) {
        uint64_t r = r0 + c;
        seeds[c] = r == 0 ? cfg->seed : ck_mix_seed(cfg->seed, r);
      }
      ck_session_s s;
      session_create(&s, a, cfg, seeds.data(), R);
      int32_t fin = 0;
      session_run(&s, 0, &fin);
      for (int c = 0; c < R; ++c) {
        ck_norm_result e{};
        session_result(&s, c, &e, nullptr);
        if (!have || e.value > res->value) {
          *res = e;
          have = true;
          if (witness) session_result(&s, c, &e, witness);
        }
      }
    }
  });
}

}  // extern "C"

// ------------------------------------------------------------ LU / InverseOracle
namespace ck {
void lu_factorize(ck_lu_s* f, ck_matrix_s* m, double pivot_tol, int64_t* fail_col,
                  double* fail_pivot);
void lu_solve_launch(ck_lu_s* f, double* const* x, int R, bool transpose, cudaStream_t st);
void lu_build_csr(ck_lu_s* f);
void session_create_inverse(ck_session_s* s, ck_lu_s* lu, const ck_adam_cfg* cfg,
                            const uint64_t* seeds, int R);

static ck_lu_s* LU(ck_lu f) {
  if (f == nullptr) fail(CK_ERR_INVALID_ARGUMENT, "LU handle is NULL");
  CK_CUDA(cudaSetDevice(f->device));
  return f;
}

static void lu_solve_host(ck_lu_s* f, const double* b, double* x, bool transpose) {
  cudaStream_t st = f->stream;
  double* w = f->work.p;
  CK_CUDA(cudaMemcpyAsync(w, b, sizeof(double) * f->n, cudaMemcpyHostToDevice, st));
  double* xs[1] = {w};
  lu_solve_launch(f, xs, 1, transpose, st);
  CK_CUDA(cudaMemcpyAsync(x, w, sizeof(double) * f->n, cudaMemcpyDeviceToHost, st));
  CK_CUDA(cudaStreamSynchronize(st));
}

// InverseOracle restarts run as separate members of one batch session -- one
// CTA each, sharing the factors -- rather than as columns of one sweep: the
// sweeps are a latency chain, so R columns on one CTA cost ~1.5x a single one
// while R CTAs run side by side. Column k of the session is restart k.
void lu_dense_solve_launch(ck_lu_s* f, double* x, bool transpose, cudaStream_t st);
constexpr int kInvRestartGroup = 64;
void session_create_inverse_batch(ck_session_s* s, ck_lu_s* const* lus, int S, const ck_adam_cfg* cfg,
                                  const uint64_t* seeds, int R);
static void inverse_restarts_session(ck_session_s* s, ck_lu_s* f, const ck_adam_cfg* cfg,
                                     const uint64_t* seeds, int restarts) {
  std::vector<ck_lu_s*> lus((size_t)restarts, f);
  session_create_inverse_batch(s, lus.data(), restarts, cfg, seeds, 1);
}

// estimate_norm over an already created session kind (restart groups of <= 4).
template <class MakeSession>
static void estimate_norm_groups(const ck_adam_cfg* cfg, uint64_t restarts, ck_norm_result* res,
                                 double* witness, int group, MakeSession&& make) {
  if (restarts == 0) fail(CK_ERR_INVALID_ARGUMENT, "estimate_norm: restarts must be >= 1");
  bool have = false;
  for (uint64_t r0 = 0; r0 < restarts; r0 += group) {
    const int R = (int)std::min<uint64_t>(group, restarts - r0);
    std::vector<uint64_t> seeds(R);
    for (int c = 0; c < R; ++c) {
      const uint64_t r = r0 + c;
      seeds[c] = r == 0 ? cfg->seed : ck_mix_seed(cfg->seed, r);
    }
    ck_session_s s;
    make(&s, seeds.data(), R);
    int32_t fin = 0;
    session_run(&s, 0, &fin);
    for (int c = 0; c < R; ++c) {
      ck_norm_result e{};
      session_result(&s, c, &e, nullptr);
      if (!have || e.value > res->value) {
        *res = e;
        have = true;
        if (witness) session_result(&s, c, &e, witness);
      }
    }
  }
}
}  // namespace ck

extern "C" {

ck_status ck_lu_factorize(ck_matrix a, double pivot_tol, ck_lu* out, int64_t* fail_col,
                          double* fail_pivot) {
  return guarded(__func__, [&] {
    if (out == nullptr) fail(CK_ERR_INVALID_ARGUMENT, "out is NULL");
    auto* f = new ck_lu_s();
    try {
      lu_factorize(f, M(a), pivot_tol, fail_col, fail_pivot);
    } catch (...) {
      delete f;
      throw;
    }
    *out = f;
  });
}

ck_status ck_lu_factorize_batch(const ck_matrix* a, int32_t nmem, double pivot_tol, ck_lu* out,
                                int32_t* status, int64_t* fail_col, double* fail_pivot) {
  return guarded(__func__, [&] {
    if (nmem < 1 || !a || !out || !status) fail(CK_ERR_INVALID_ARGUMENT, "lu_factorize_batch: bad arguments");
    std::vector<ck_matrix_s*> ms((size_t)nmem);
    for (int g = 0; g < nmem; ++g) ms[g] = M(a[g]);
    std::vector<ck_lu_s*> fs((size_t)nmem, nullptr);
    try {
      for (int g = 0; g < nmem; ++g) fs[g] = new ck_lu_s();
      ck::lu_factorize_batch(fs.data(), ms.data(), nmem, pivot_tol, status, fail_col, fail_pivot);
    } catch (...) {
      for (auto* f : fs) delete f;
      throw;
    }
    for (int g = 0; g < nmem; ++g) {
      if (status[g] == CK_OK) {
        out[g] = fs[g];
      } else {
        delete fs[g];
        out[g] = nullptr;
      }
    }
  });
}

ck_status ck_lu_free(ck_lu f) {
  return guarded(__func__, [&] {
    if (!f) return;
    cudaSetDevice(f->device);
    delete f;
  });
}

ck_status ck_lu_get_info(ck_lu f, int64_t* n, int64_t* kl, int64_t* ku, double* pivot_min,
                         int64_t* device_bytes) {
  return guarded(__func__, [&] {
    LU(f);
    *n = f->n;
    *kl = f->kl;
    *ku = f->ku;
    *pivot_min = f->pivot_min;
    *device_bytes = f->ab.bytes() + f->lb.bytes() + f->ipiv.bytes();
  });
}

ck_status ck_lu_export(ck_lu f, double* ab, int32_t* ipiv) {
  return guarded(__func__, [&] {
    LU(f);
    cudaStream_t st = f->stream;
    if (ab) CK_CUDA(cudaMemcpyAsync(ab, f->ab.p, f->ab.bytes(), cudaMemcpyDeviceToHost, st));
    if (ipiv) CK_CUDA(cudaMemcpyAsync(ipiv, f->ipiv.p, sizeof(int32_t) * f->n, cudaMemcpyDeviceToHost, st));
    CK_CUDA(cudaStreamSynchronize(st));
  });
}

ck_status ck_lu_csr_info(ck_lu f, int64_t* nnz_l, int64_t* nnz_u) {
  return guarded(__func__, [&] {
    LU(f);
    lu_build_csr(f);
    if (nnz_l) *nnz_l = f->nnz_l;
    if (nnz_u) *nnz_u = f->nnz_u;
  });
}

ck_status ck_lu_export_csr(ck_lu f, int64_t* l_rp, int32_t* l_ci, double* l_va, int64_t* u_rp,
                           int32_t* u_ci, double* u_va, int64_t* row_perm) {
  return guarded(__func__, [&] {
    LU(f);
    lu_build_csr(f);
    cudaStream_t st = f->stream;
    const int64_t n = f->n;
    auto get = [&](void* dst, const void* src, int64_t bytes) {
      if (dst && bytes > 0) CK_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToHost, st));
    };
    get(l_rp, f->l_rp.p, 8 * (n + 1));
    get(l_ci, f->l_ci.p, 4 * f->nnz_l);
    get(l_va, f->l_va.p, 8 * f->nnz_l);
    get(u_rp, f->u_rp.p, 8 * (n + 1));
    get(u_ci, f->u_ci.p, 4 * f->nnz_u);
    get(u_va, f->u_va.p, 8 * f->nnz_u);
    std::vector<int32_t> rp32((size_t)(row_perm ? n : 0));
    get(rp32.data(), f->rowperm.p, row_perm ? 4 * n : 0);
    CK_CUDA(cudaStreamSynchronize(st));
    for (int64_t k = 0; row_perm && k < n; ++k) row_perm[k] = rp32[(size_t)k];
  });
}

ck_status ck_lu_solve(ck_lu f, const double* b, double* x) {
  return guarded(__func__, [&] { lu_solve_host(LU(f), b, x, false); });
}

ck_status ck_lu_transpose_solve(ck_lu f, const double* b, double* x) {
  return guarded(__func__, [&] { lu_solve_host(LU(f), b, x, true); });
}

ck_status ck_restart_group(ck_matrix a, uint64_t restarts, int32_t batch, int32_t* group) {
  return guarded(__func__, [&] { *group = restart_group(M(a), restarts, batch != 0); });
}

ck_status ck_lu_dense_info(ck_lu f, int32_t* available, double* growth) {
  return guarded(__func__, [&] {
    ck_lu_s* lu = LU(f);
    if (available) *available = lu->dense_ok ? 1 : 0;
    if (growth) *growth = lu->dense_growth;
  });
}

ck_status ck_lu_dense_solve(ck_lu f, int32_t transpose, const double* b, double* x) {
  return guarded(__func__, [&] {
    ck_lu_s* lu = LU(f);
    if (!lu->dense_ok) fail(CK_ERR_UNSUPPORTED, "dense-block sweeps not available for these factors");
    cudaStream_t st = lu->stream;
    double* w = lu->work.p;
    CK_CUDA(cudaMemcpyAsync(w, b, sizeof(double) * lu->n, cudaMemcpyHostToDevice, st));
    lu_dense_solve_launch(lu, w, transpose != 0, st);
    CK_CUDA(cudaMemcpyAsync(x, w, sizeof(double) * lu->n, cudaMemcpyDeviceToHost, st));
    CK_CUDA(cudaStreamSynchronize(st));
  });
}

ck_status ck_session_create_inverse(ck_lu f, const ck_adam_cfg* cfg, const uint64_t* seeds,
                                    int32_t ncols, ck_session* out) {
  return guarded(__func__, [&] {
    check_cfg(cfg);
    auto* s = new ck_session_s();
    try {
      session_create_inverse(s, LU(f), cfg, seeds, ncols);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

ck_status ck_inv_projected_adam(ck_lu f, const ck_adam_cfg* cfg, ck_norm_result* res,
                                double* witness) {
  return guarded(__func__, [&] {
    check_cfg(cfg);
    ck_session_s s;
    uint64_t seed = cfg->seed;
    session_create_inverse(&s, LU(f), cfg, &seed, 1);
    int32_t fin = 0;
    session_run(&s, 0, &fin);
    session_result(&s, 0, res, witness);
  });
}

ck_status ck_inv_estimate_norm(ck_lu f, const ck_adam_cfg* cfg, uint64_t restarts,
                               ck_norm_result* res, double* witness) {
  return guarded(__func__, [&] {
    check_cfg(cfg);
    LU(f);
    estimate_norm_groups(cfg, restarts, res, witness, kInvRestartGroup, [&](ck_session_s* s, const uint64_t* seeds, int R) {
      inverse_restarts_session(s, f, cfg, seeds, R);
    });
  });
}

// cond2, condest.hpp:341-365: ||A|| by estimate_norm on A, then the LU with
// pivot_tol and ||A^-1|| with seed mix_seed(seed, 0x1234); a singular
// factorisation yields kappa = +inf (no error).
ck_status ck_cond2(ck_matrix a, const ck_adam_cfg* cfg, uint64_t restarts, double pivot_tol,
                   double* kappa, ck_norm_result* fwd, ck_norm_result* inv, int32_t* has_factors) {
  return guarded(__func__, [&] {
    check_cfg(cfg);
    ck_matrix_s* m = M(a);
    if (m->nrows != m->ncols) fail(CK_ERR_DIMENSION, "cond2: matrix must be square");
    estimate_norm_groups(cfg, restarts, fwd, nullptr, restart_group(m, restarts), [&](ck_session_s* s, const uint64_t* seeds, int R) {
      session_create(s, m, cfg, seeds, R);
    });
    *inv = ck_norm_result{};
    *has_factors = 0;
    ck_lu_s f;
    try {
      lu_factorize(&f, m, pivot_tol, nullptr, nullptr);
    } catch (const Error& e) {
      if (e.code == CK_ERR_STRUCT_SINGULAR || e.code == CK_ERR_NUM_SINGULAR) {
        inv->value = std::numeric_limits<double>::infinity();
        *kappa = std::numeric_limits<double>::infinity();
        return;
      }
      throw;
    }
    ck_adam_cfg ci = *cfg;
    ci.seed = ck_mix_seed(cfg->seed, 0x1234);
    estimate_norm_groups(&ci, restarts, inv, nullptr, kInvRestartGroup, [&](ck_session_s* s, const uint64_t* seeds, int R) {
      inverse_restarts_session(s, &f, &ci, seeds, R);
    });
    *kappa = fwd->value * inv->value;
    *has_factors = 1;
  });
}

}  // extern "C"

extern "C" {

// loss / grad of the InverseOracle (condest.hpp:112-123, 142-146) on the device.
ck_status ck_loss_inverse(ck_lu f, const double* x, double* loss) {
  return guarded(__func__, [&] {
    ck_lu_s* F = LU(f);
    cudaStream_t st = F->stream;
    const int64_t n = F->n;
    double* w = F->work.p;
    double* red = F->work.p + 2 * n;
    CK_CUDA(cudaMemcpyAsync(w, x, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    const double xn = device_norm(w, n, red, st);
    double* xs[1] = {w};
    lu_solve_launch(F, xs, 1, false, st);
    const double rn = device_norm(w, n, red, st);
    if (rn == 0.0) fail(CK_ERR_INVALID_ARGUMENT, "operator maps direction to zero (DegenerateDirection)");
    *loss = std::log(xn) - std::log(rn);
  });
}

ck_status ck_grad_inverse(ck_lu f, const double* x, double* g) {
  return guarded(__func__, [&] {
    ck_lu_s* F = LU(f);
    cudaStream_t st = F->stream;
    const int64_t n = F->n;
    double* w = F->work.p;
    double* red = F->work.p + 2 * n;
    CK_CUDA(cudaMemcpyAsync(w, x, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    double* xs[1] = {w};
    lu_solve_launch(F, xs, 1, false, st);
    const double rn = device_norm(w, n, red, st);
    if (rn == 0.0) fail(CK_ERR_INVALID_ARGUMENT, "operator maps direction to zero (DegenerateDirection)");
    lu_solve_launch(F, xs, 1, true, st);
    std::vector<double> s((size_t)n), hx(x, x + n);
    CK_CUDA(cudaMemcpyAsync(s.data(), w, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CK_CUDA(cudaStreamSynchronize(st));
    // ||x|| of the host input (two_norm, exact mirror) and the combine (:117-121)
    const double xn = two_norm_seq(hx.data(), n);
    const double inv_x2 = 1.0 / (xn * xn), inv_r2 = 1.0 / (rn * rn);
    for (int64_t i = 0; i < n; ++i) g[i] = x[i] * inv_x2 - s[(size_t)i] * inv_r2;
  });
}

}  // extern "C"

namespace ck {
void session_create_batch(ck_session_s* s, ck_matrix_s* A, const int64_t* seg_n, int S,
                          const ck_adam_cfg* cfg, const uint64_t* seeds, int R);
void session_create_inverse_batch(ck_session_s* s, ck_lu_s* const* lus, int S,
                                  const ck_adam_cfg* cfg, const uint64_t* seeds, int R);
}

extern "C" {

// S independent operators packed block-diagonally (member g at rows/cols
// [off_g, off_g + n_g), off_g = sum over h < g of round_up(n_h, 256)): one
// session advances every member and restart column with one kernel pair.
ck_status ck_session_create_batch(ck_matrix a, const int64_t* seg_n, int32_t nseg,
                                  const ck_adam_cfg* cfg, const uint64_t* seeds, int32_t ncols,
                                  ck_session* out) {
  return guarded(__func__, [&] {
    check_cfg(cfg);
    auto* s = new ck_session_s();
    try {
      session_create_batch(s, M(a), seg_n, nseg, cfg, seeds, ncols);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

// estimate_norm (condest.hpp:301-312) for every member of a packed batch: member
// g's restarts use seed member_seeds[g] (r = 0) or mix_seed(member_seeds[g], r).
ck_status ck_estimate_norm_batch(ck_matrix a, const int64_t* seg_n, int32_t nseg,
                                 const ck_adam_cfg* cfg, const uint64_t* member_seeds,
                                 uint64_t restarts, ck_norm_result* results) {
  return guarded(__func__, [&] {
    check_cfg(cfg);
    if (restarts == 0) fail(CK_ERR_INVALID_ARGUMENT, "estimate_norm: restarts must be >= 1");
    ck_matrix_s* m = M(a);
    std::vector<char> have((size_t)nseg, 0);
    const int group = restart_group(m, restarts, true);
    for (uint64_t r0 = 0; r0 < restarts; r0 += group) {
      const int R = (int)std::min<uint64_t>(group, restarts - r0);
      std::vector<uint64_t> seeds((size_t)nseg * R);
      for (int g = 0; g < nseg; ++g)
        for (int c = 0; c < R; ++c) {
          const uint64_t r = r0 + c;
          seeds[(size_t)g * R + c] = r == 0 ? member_seeds[g] : ck_mix_seed(member_seeds[g], r);
        }
      ck_session_s s;
      session_create_batch(&s, m, seg_n, nseg, cfg, seeds.data(), R);
      int32_t fin = 0;
      session_run(&s, 0, &fin);
      for (int g = 0; g < nseg; ++g)
        for (int c = 0; c < R; ++c) {
          ck_norm_result e{};
          session_result(&s, g * R + c, &e, nullptr);
          if (!have[g] || e.value > results[g].value) {
            results[g] = e;
            have[g] = 1;
          }
        }
    }
  });
}

// InverseOracle over S independent factorisations: one session, one CTA per
// member per step (the sigma_min half of cond2 for an ensemble, config 5).
ck_status ck_session_create_inverse_batch(const ck_lu* lus, int32_t nmem, const ck_adam_cfg* cfg,
                                          const uint64_t* seeds, int32_t ncols, ck_session* out) {
  return guarded(__func__, [&] {
    check_cfg(cfg);
    if (nmem < 1) fail(CK_ERR_INVALID_ARGUMENT, "at least one member");
    std::vector<ck_lu_s*> f((size_t)nmem);
    for (int g = 0; g < nmem; ++g) f[g] = LU(lus[g]);
    auto* s = new ck_session_s();
    try {
      session_create_inverse_batch(s, f.data(), nmem, cfg, seeds, ncols);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

// estimate_norm on A_g^{-1} for every member g (restart seeds as in
// ck_estimate_norm_batch).
ck_status ck_inv_estimate_norm_batch(const ck_lu* lus, int32_t nmem, const ck_adam_cfg* cfg,
                                     const uint64_t* member_seeds, uint64_t restarts,
                                     ck_norm_result* results) {
  return guarded(__func__, [&] {
    check_cfg(cfg);
    if (restarts == 0) fail(CK_ERR_INVALID_ARGUMENT, "estimate_norm: restarts must be >= 1");
    if (nmem < 1) fail(CK_ERR_INVALID_ARGUMENT, "at least one member");
    std::vector<ck_lu_s*> f((size_t)nmem);
    for (int g = 0; g < nmem; ++g) f[g] = LU(lus[g]);
    std::vector<char> have((size_t)nmem, 0);
    for (uint64_t r0 = 0; r0 < restarts; r0 += kMaxCols) {
      const int R = (int)std::min<uint64_t>(kMaxCols, restarts - r0);
      std::vector<uint64_t> seeds((size_t)nmem * R);
      for (int g = 0; g < nmem; ++g)
        for (int c = 0; c < R; ++c) {
          const uint64_t r = r0 + c;
          seeds[(size_t)g * R + c] = r == 0 ? member_seeds[g] : ck_mix_seed(member_seeds[g], r);
        }
      ck_session_s s;
      session_create_inverse_batch(&s, f.data(), nmem, cfg, seeds.data(), R);
      int32_t fin = 0;
      session_run(&s, 0, &fin);
      for (int g = 0; g < nmem; ++g)
        for (int c = 0; c < R; ++c) {
          ck_norm_result e{};
          session_result(&s, g * R + c, &e, nullptr);
          if (!have[g] || e.value > results[g].value) {
            results[g] = e;
            have[g] = 1;
          }
        }
    }
  });
}

// ---------------------------------------------------------------- scaling
ck_status ck_column_norms(ck_matrix a, double* norms) {
  return guarded(__func__, [&] {
    ck_matrix_s* m = M(a);
    DBuf<double> d(std::max<int64_t>(1, m->ncols));
    matrix_norms(m, true, d.p);
    CK_CUDA(cudaMemcpy(norms, d.p, sizeof(double) * m->ncols, cudaMemcpyDeviceToHost));
  });
}

ck_status ck_row_norms(ck_matrix a, double* norms) {
  return guarded(__func__, [&] {
    ck_matrix_s* m = M(a);
    DBuf<double> d(std::max<int64_t>(1, m->nrows));
    matrix_norms(m, false, d.p);
    CK_CUDA(cudaMemcpy(norms, d.p, sizeof(double) * m->nrows, cudaMemcpyDeviceToHost));
  });
}

// column_scale, sparse.hpp:271-284
ck_status ck_column_scale(ck_matrix a, const int32_t* col_indices, const double* values,
                          double* values_out, double* norms, int64_t* zero_index) {
  return guarded(__func__, [&] {
    ck_matrix_s* m = M(a);
    if (zero_index) *zero_index = -1;
    DBuf<double> d(std::max<int64_t>(1, m->ncols));
    matrix_norms(m, true, d.p);
    std::vector<double> h((size_t)m->ncols);
    CK_CUDA(cudaMemcpy(h.data(), d.p, sizeof(double) * m->ncols, cudaMemcpyDeviceToHost));
    for (int64_t j = 0; j < m->ncols; ++j)
      if (h[j] == 0.0) {
        if (zero_index) *zero_index = j;
        fail(CK_ERR_ZERO_COLUMN, "column " + std::to_string(j) + " has zero norm");
      }
    if (norms) std::memcpy(norms, h.data(), sizeof(double) * m->ncols);
    csr_divide(m, true, nullptr, col_indices, values, d.p, values_out);
  });
}

// row_scale, sparse.hpp:295-311
ck_status ck_row_scale(ck_matrix a, const int64_t* row_offsets, const double* values,
                       double* values_out, const double* b, double* b_out, double* norms,
                       int64_t* zero_index) {
  return guarded(__func__, [&] {
    ck_matrix_s* m = M(a);
    if (zero_index) *zero_index = -1;
    DBuf<double> d(std::max<int64_t>(1, m->nrows));
    matrix_norms(m, false, d.p);
    std::vector<double> h((size_t)m->nrows);
    CK_CUDA(cudaMemcpy(h.data(), d.p, sizeof(double) * m->nrows, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < m->nrows; ++i)
      if (h[i] == 0.0) {
        if (zero_index) *zero_index = i;
        fail(CK_ERR_ZERO_ROW, "row " + std::to_string(i) + " has zero norm");
      }
    if (norms) std::memcpy(norms, h.data(), sizeof(double) * m->nrows);
    csr_divide(m, false, row_offsets, nullptr, values, d.p, values_out);
    if (b && b_out) vector_divide(m->nrows, b, h.data(), b_out, m->stream);
  });
}

ck_status ck_unscale_solution(int64_t n, const double* y, const double* d, double* x) {
  return guarded(__func__, [&] {
    if (n < 0) fail(CK_ERR_INVALID_ARGUMENT, "negative length");
    int cnt = 0;
    if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt == 0) fail(CK_ERR_NO_DEVICE, "no CUDA device");
    cudaStream_t st = nullptr;
    vector_divide(n, y, d, x, st);
  });
}

// ------------------------------------------------------ row-block partitions
ck_status ck_dist_nccl_id(void* id128) {
  return guarded(__func__, [&] { dist_nccl_id(id128); });
}

ck_status ck_dist_create(const ck_dist_part* parts, int32_t nparts, int32_t rank0, int32_t nranks,
                         const void* nccl_id, const ck_adam_cfg* cfg, const uint64_t* seeds,
                         int32_t ncols, ck_dist* out) {
  return guarded(__func__, [&] {
    check_cfg(cfg);
    ck_dist_s* D = dist_new();
    try {
      dist_create(D, parts, nparts, rank0, nranks, nccl_id, cfg, seeds, ncols);
    } catch (...) {
      dist_free(D);
      throw;
    }
    *out = D;
  });
}

ck_status ck_dist_run(ck_dist d, uint64_t max_steps, int32_t* finished) {
  return guarded(__func__, [&] {
    if (!d) fail(CK_ERR_INVALID_ARGUMENT, "dist handle is NULL");
    dist_run(d, max_steps, finished);
  });
}

ck_status ck_dist_time(ck_dist d, uint64_t steps, double* ms) {
  return guarded(__func__, [&] {
    if (!d) fail(CK_ERR_INVALID_ARGUMENT, "dist handle is NULL");
    *ms = dist_time(d, steps);
  });
}

ck_status ck_dist_result(ck_dist d, int32_t col, int32_t part, ck_norm_result* res, double* witness) {
  return guarded(__func__, [&] {
    if (!d) fail(CK_ERR_INVALID_ARGUMENT, "dist handle is NULL");
    dist_result(d, col, part, res, witness);
  });
}

ck_status ck_dist_part_info(ck_dist d, int32_t part, ck_matrix_info* info) {
  return guarded(__func__, [&] {
    if (!d || !info) fail(CK_ERR_INVALID_ARGUMENT, "dist handle or info is NULL");
    matrix_info(dist_part_matrix(d, part), info);
  });
}

ck_status ck_dist_free(ck_dist d) {
  return guarded(__func__, [&] {
    if (d) dist_free(d);
  });
}

}  // extern "C"
