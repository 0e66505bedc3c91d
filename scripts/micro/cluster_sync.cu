// Latency of cluster.sync() and of a DSMEM broadcast round (leader writes 32
// doubles into every CTA of the cluster, barrier, everyone reads) on B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 cluster_sync.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int C>
__global__ void __cluster_dims__(C, 1, 1) __launch_bounds__(1024) k_sync(int iters, long long* out, double* sink) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double buf[64];
  const int rank = (int)cl.block_rank();
  double acc = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) cl.sync();
  long long t1 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (rank == it % C && threadIdx.x < 32 * C) {  // leader writes its 32 values into every CTA
      const int dst = threadIdx.x / 32;
      double* p = cl.map_shared_rank(buf, dst);
      p[threadIdx.x % 32] = it + threadIdx.x;
    }
    cl.sync();
    if (threadIdx.x < 32) acc += buf[threadIdx.x];
    cl.sync();
  }
  long long t2 = clock64();
  if (threadIdx.x == 0 && rank == 0) {
    out[0] = (t1 - t0) / iters;
    out[1] = (t2 - t1) / iters;
  }
  if (acc == 1.2345) sink[0] = acc;
}

int main() {
  long long* d;
  double* s;
  cudaMalloc(&d, 16);
  cudaMalloc(&s, 8);
  long long h[2];
  k_sync<2><<<2, 1024>>>(1000, d, s);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("C=2: cluster.sync %lld cycles, broadcast round (2 syncs) %lld cycles (%s)\n", h[0], h[1], cudaGetErrorString(cudaGetLastError()));
  k_sync<4><<<4, 1024>>>(1000, d, s);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("C=4: cluster.sync %lld cycles, broadcast round (2 syncs) %lld cycles (%s)\n", h[0], h[1], cudaGetErrorString(cudaGetLastError()));
  k_sync<8><<<8, 1024>>>(1000, d, s);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("C=8: cluster.sync %lld cycles, broadcast round (2 syncs) %lld cycles (%s)\n", h[0], h[1], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
