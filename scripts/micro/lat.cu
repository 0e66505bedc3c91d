// Dependent-chain latencies (cycles) of the FP64 and shuffle operations on
// the band sweeps' head-solve critical path.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  double x = a, y = b;
  long long t0, t1;
  const int lane = threadIdx.x & 31;
#define CHAIN(slot, body)                    \
  __syncwarp();                              \
  t0 = clock64();                            \
  for (int i = 0; i < n; ++i) { body; }      \
  t1 = clock64();                            \
  if (threadIdx.x == 0) cyc[slot] = (t1 - t0);
  CHAIN(0, x = __fma_rn(x, b, a))
  CHAIN(1, x = __dmul_rn(x, b))
  CHAIN(2, x = __dadd_rn(x, b))
  CHAIN(3, x = __shfl_sync(0xffffffffu, x, i & 31))
  CHAIN(4, x = __dsub_rn(x, __dmul_rn(b, __shfl_sync(0xffffffffu, x, i & 31))))
  CHAIN(5, x = __drcp_rn(x))
  CHAIN(6, x = __ddiv_rn(a, x))
  CHAIN(7, x = __shfl_sync(0xffffffffu, x, i & 31) * 1.0000001; if (lane > (i & 31)) x = x - b * y)
  out[threadIdx.x] = x + y;
}

int main() {
  double* out; long long* cyc; long long h[8];
  cudaMalloc(&out, 32 * 8); cudaMalloc(&cyc, 8 * 8);
  const int n = 1024;
  k<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999, n);
  k<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999, n);
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  const char* nm[8] = {"dfma", "dmul", "dadd", "shfl.f64", "shfl+dmul+dsub", "drcp_rn", "ddiv_rn", "shfl+pred sub"};
  for (int i = 0; i < 8; ++i) printf("%-16s %.1f cycles/iter\n", nm[i], (double)h[i] / n);
  return 0;
}
