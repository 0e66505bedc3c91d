// Internal definitions shared by the condkit-b200 translation units.
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "condkit_b200.h"

namespace ck {

// Rows handled by one CTA (one thread per row) and rows per sliced-ELL slice.
constexpr int kTile = 256;
constexpr int kSlice = 32;
constexpr int kSlicesPerTile = kTile / kSlice;
constexpr int kMaxCols = 4;  // restarts carried as columns of one multi-vector

// Error carrying a ck_status across the C++ implementation; converted at the ABI.
struct Error : std::runtime_error {
  ck_status code;
  Error(ck_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail(ck_status c, const std::string& msg);
void cuda_check(cudaError_t e, const char* what, const char* file, int line);
#define CK_CUDA(x) ::ck::cuda_check((x), #x, __FILE__, __LINE__)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// NVTX range for the lifetime of a scope (header-only NVTX 3: no cost without
// an attached tool).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Phase timer for the setup paths (CK_TRACE=1): synchronises the stream and
// prints the wall time since the previous mark to stderr.
struct Trace {
  bool on;
  std::chrono::steady_clock::time_point t;
  explicit Trace(const char* tag) : on(false) {
    const char* e = std::getenv("CK_TRACE");
    on = e && e[0] == '1';
    t = std::chrono::steady_clock::now();
    if (on) std::fprintf(stderr, "[ck_trace] %s\n", tag);
  }
  void mark(const char* what, cudaStream_t st) {
    nvtxMarkA(what);
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[ck_trace]   %-28s %9.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// Page-locked host staging memory (start vectors, witnesses). Pinning costs
// ~0.5 ms per MB and holds the driver while it runs -- at config 4 the 200 MB
// start-vector buffer stalls the concurrent operator build by ~0.1 s -- so
// released buffers are kept in a small process-wide cache (ck_api.cu: at most
// six buffers, 1 GiB in total) and the next session reuses them.
void* pinned_acquire(size_t bytes, size_t* got_bytes);  // nullptr: allocation failed
void pinned_release(void* p, size_t bytes);

template <class T>
struct PinnedBuf {
  T* p = nullptr;
  int64_t n = 0;
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  ~PinnedBuf() { reset(); }
  void resize(int64_t count) {
    if (count <= n) return;
    reset();
    size_t got = 0;
    p = static_cast<T*>(pinned_acquire(sizeof(T) * static_cast<size_t>(count), &got));
    if (p == nullptr) fail(CK_ERR_OUT_OF_MEMORY, "cudaMallocHost failed");
    n = static_cast<int64_t>(got / sizeof(T));
  }
  void reset() {
    if (p) pinned_release(p, sizeof(T) * static_cast<size_t>(n));
    p = nullptr;
    n = 0;
  }
  T* data() { return p; }
};

// Device memory comes from the device's stream-ordered pool with the release
// threshold lifted (ck_api.cu): an upload allocates ~14 GB and frees ~8 GB of
// sort scratch at config 4, and plain cudaMalloc / cudaFree of that size
// sporadically stall for 0.1-0.8 s (measured inside the A^T build). The
// semantics of the plain calls are kept: the pointer is usable on any stream
// when device_alloc returns, and device_free waits for the device first.
// device_trim() hands cached memory back (before cudaMemGetInfo decisions).
cudaError_t device_alloc(void** p, size_t bytes);
void device_free(void* p);
void device_trim();

// Device buffer with RAII.
template <class T>
struct DBuf {
  T* p = nullptr;
  int64_t n = 0;
  DBuf() = default;
  explicit DBuf(int64_t count) { alloc(count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    reset();
    p = o.p; n = o.n; o.p = nullptr; o.n = 0;
    return *this;
  }
  ~DBuf() { reset(); }
  void alloc(int64_t count) {
    reset();
    n = count;
    if (count > 0) {
      cudaError_t e = device_alloc(reinterpret_cast<void**>(&p), sizeof(T) * static_cast<size_t>(count));
      if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        p = nullptr;
        n = 0;
        fail(CK_ERR_OUT_OF_MEMORY, "device allocation of " + std::to_string(sizeof(T) * count) + " bytes failed");
      }
      CK_CUDA(e);
    }
  }
  void reset() {
    if (p) device_free(p);
    p = nullptr;
    n = 0;
  }
  int64_t bytes() const { return n * static_cast<int64_t>(sizeof(T)); }
};

// Sliced-ELL (SELL-32-256) layout of a sparse operator. Rows are permuted
// inside each 256-row tile by descending length (stable), so every 32-row slice
// is nearly uniform. Slice widths are even and entries are interleaved in
// pairs: entry j of the slice's lane-th row sits at
//   slice_ptr[s] + 2*lane + 64*(j/2) + (j%2)          (sell_at below),
// so a lane's entries 2m, 2m+1 are adjacent -- one 16-byte value load and one
// 4-byte (narrow) or 8-byte (wide) column load -- and a warp's pair of entry
// rows is one contiguous 512-byte run of values.
//
// Column indices come in two formats, chosen per operator at build time:
//   wide    int32 column (12 bytes per stored entry with the value);
//   narrow  uint16 offset from a per-slice base column, cbase[s] + col16[k]
//           (10 bytes per stored entry). Used whenever every slice's columns
//           span < 65536 -- any operator whose bandwidth (in the permuted
//           spaces) is below ~32k, which covers every banded/stencil operator
//           of the BASELINE configs. Same columns, same order: the arithmetic
//           is unchanged.
struct Sell {
  int64_t nrows = 0;      // logical rows
  int64_t nrows_pad = 0;  // multiple of kTile
  int64_t entries = 0;    // stored entries including slice padding
  DBuf<int64_t> slice_ptr;  // nrows_pad/32 + 1
  DBuf<uint16_t> len;       // per permuted row
  DBuf<int32_t> col;        // wide: column index in the permuted column space
  DBuf<uint16_t> col16;     // narrow: column - cbase[slice]
  DBuf<int32_t> cbase;      // narrow: per-slice base column (nrows_pad/32)
  bool narrow = false;
  // narrow + pattern dictionary: slices with identical uint16 offset blocks (a
  // stencil repeats its handful of slice patterns along every grid row) share
  // one copy in ptab, slice s reads its offsets at ptab[poff[s] + local index]
  // and col16 is dropped: 8 B per stored entry from HBM instead of 10, the same
  // columns in the same order.
  DBuf<uint16_t> ptab;
  DBuf<int64_t> poff;       // per slice: first element of its pattern in ptab
  bool pattern = false;
  DBuf<double> val;
  DBuf<int32_t> perm;       // perm[k] = original row at permuted position k (-1 = pad)
  DBuf<int32_t> inv;        // inv[row] = permuted position
};

// Position of stored entry j of a row whose row base is slice_ptr[s] + 2*lane.
__host__ __device__ __forceinline__ int64_t sell_at(int64_t rowbase, int64_t j) {
  return rowbase + ((j >> 1) << 6) + (j & 1);
}
__host__ __device__ __forceinline__ int64_t sell_rowbase(int64_t slice_start, int64_t row) {
  return slice_start + 2 * (row & 31);
}

struct SellView {
  const int64_t* __restrict__ sp;
  const uint16_t* __restrict__ len;
  const int32_t* __restrict__ col;
  const uint16_t* __restrict__ col16;
  const int32_t* __restrict__ cbase;
  const double* __restrict__ val;
  int narrow;
  const int64_t* __restrict__ poff;  // pattern dictionary: col16 points at the table (else nullptr)
};

inline SellView view(const Sell& s) {
  return {s.slice_ptr.p, s.len.p,   s.col.p, s.pattern ? s.ptab.p : s.col16.p, s.cbase.p, s.val.p,
          s.narrow ? 1 : 0,  s.pattern ? s.poff.p : nullptr};
}

}  // namespace ck

struct ck_matrix_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t nrows = 0, ncols = 0, nnz = 0;
  ck::Sell a;   // rows of A in P order, columns in Q space
  ck::Sell at;  // rows of A^T (= columns of A) in Q order, columns in P space
  // scratch for the standalone ops
  ck::DBuf<double> s_in, s_out, s_perm_in, s_perm_out, s_red;
};
