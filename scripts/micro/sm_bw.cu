// Single-SM streaming bandwidth: one CTA of 1024 threads reads a large array
// (a) with plain coalesced loads, ILP per thread; (b) with cp.async.bulk into a
// multi-stage shared-memory ring. nvcc -gencode arch=compute_100a,code=sm_100a -O3 sm_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int ILP>
__global__ void k_ld(const double* __restrict__ a, int64_t n, double* out) {
  double s = 0.0;
  const int64_t step = (int64_t)blockDim.x * ILP;
  for (int64_t i = threadIdx.x; i < n; i += step) {
    double v[ILP];
#pragma unroll
    for (int u = 0; u < ILP; ++u) v[u] = (i + u * blockDim.x < n) ? __ldcs(a + i + u * blockDim.x) : 0.0;
#pragma unroll
    for (int u = 0; u < ILP; ++u) s += v[u];
  }
  if (s == 1.2345) out[0] = s;
}

template <int NST, int CHUNK>
__global__ void k_tma(const double* __restrict__ a, int64_t n, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ alignas(8) uint64_t bar[NST];
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      uint32_t b = (uint32_t)__cvta_generic_to_shared(bar + s);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int64_t nch = n * 8 / CHUNK;
  auto issue = [&](int64_t c) {
    int s = (int)(c % NST);
    uint32_t b = (uint32_t)__cvta_generic_to_shared(bar + s);
    uint32_t d = (uint32_t)__cvta_generic_to_shared(sm + (int64_t)s * CHUNK);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(CHUNK) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
                 "l"((const char*)a + c * CHUNK), "r"(CHUNK), "r"(b) : "memory");
  };
  if (threadIdx.x == 0)
    for (int64_t c = 0; c < NST && c < nch; ++c) issue(c);
  double s = 0.0;
  uint32_t phase = 0;
  for (int64_t c = 0; c < nch; ++c) {
    int st = (int)(c % NST);
    uint32_t b = (uint32_t)__cvta_generic_to_shared(bar + st);
    uint32_t par = (phase >> st) & 1u, done = 0;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                   : "=r"(done) : "r"(b), "r"(par) : "memory");
    phase ^= 1u << st;
    const double* v = reinterpret_cast<const double*>(sm + (int64_t)st * CHUNK);
    for (int k = threadIdx.x; k < CHUNK / 8; k += blockDim.x) s += v[k];
    __syncthreads();
    if (threadIdx.x == 0 && c + NST < nch) issue(c + NST);
  }
  if (s == 1.2345) out[0] = s;
}

int main() {
  const int64_t n = (int64_t)1 << 27;  // 1 GiB of doubles
  double *a, *o;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&o, 8);
  cudaMemset(a, 0, n * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch, int64_t bytes) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s %8.1f GB/s  (%s)\n", name, bytes / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
  };
  const int64_t m = n / 8;  // 128 MiB per single-CTA test
  run("ld ILP1  1 CTA", [&] { k_ld<1><<<1, 1024>>>(a, m, o); }, m * 8);
  run("ld ILP4  1 CTA", [&] { k_ld<4><<<1, 1024>>>(a, m, o); }, m * 8);
  run("ld ILP8  1 CTA", [&] { k_ld<8><<<1, 1024>>>(a, m, o); }, m * 8);
  run("ld ILP16 1 CTA", [&] { k_ld<16><<<1, 1024>>>(a, m, o); }, m * 8);
  cudaFuncSetAttribute(k_tma<4, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
  cudaFuncSetAttribute(k_tma<6, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
  cudaFuncSetAttribute(k_tma<12, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384);
  cudaFuncSetAttribute(k_tma<3, 65536>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 65536);
  run("tma 4x32K 1 CTA", [&] { k_tma<4, 32768><<<1, 1024, 4 * 32768>>>(a, m, o); }, m * 8);
  run("tma 6x32K 1 CTA", [&] { k_tma<6, 32768><<<1, 1024, 6 * 32768>>>(a, m, o); }, m * 8);
  run("tma 12x16K 1 CTA", [&] { k_tma<12, 16384><<<1, 1024, 12 * 16384>>>(a, m, o); }, m * 8);
  run("tma 3x64K 1 CTA", [&] { k_tma<3, 65536><<<1, 1024, 3 * 65536>>>(a, m, o); }, m * 8);

  return 0;
}
