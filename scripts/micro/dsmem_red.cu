// Microbenchmark: shared-memory red.add throughput, local vs remote (DSMEM) in a cluster.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(1024, 1)
k(int iters, int mode, unsigned *out) {
  extern __shared__ uint32_t sh[];
  cg::cluster_group cl = cg::this_cluster();
  const int n = 48 * 1024;  // 192 KB of counters
  for (int i = threadIdx.x; i < n; i += blockDim.x) sh[i] = 0;
  cl.sync();
  uint32_t rank = cl.block_rank();
  uint32_t x = threadIdx.x * 2654435761u + blockIdx.x * 97u;
  uint32_t local = (uint32_t)__cvta_generic_to_shared(sh);
  uint32_t remote[4];
  for (int r = 0; r < 4; r++) {
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(local), "r"(r));
    remote[r] = a;
  }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < 4; j++) {
      x = x * 1664525u + 1013904223u;
      uint32_t idx = (x >> 8) % n;
      if (mode == 0) {
        asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(local + 4 * idx) : "memory");
      } else {
        uint32_t tgt = (rank + 1 + j % 3) & 3;  // a remote CTA
        if (mode == 2) tgt = j;  // all 4 incl. local via cluster window
        asm volatile("red.shared::cluster.add.u32 [%0], 1;" ::"r"(remote[tgt] + 4 * idx) : "memory");
      }
    }
  }
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = sh[0];
}

int main() {
  unsigned *out;
  cudaMalloc(&out, 4096 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int iters = 2000;
  for (int mode = 0; mode < 3; mode++) {
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(a);
      k<<<132, 1024, 200 * 1024>>>(iters, mode, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double ops = 132.0 * 1024 * iters * 4;
      if (rep) printf("mode %d (%s): %.3f ms, %.2f Gops/s, %.2f ops/clk/SM @1.9GHz\n", mode,
                      mode == 0 ? "local red" : (mode == 1 ? "remote red" : "cluster-window red all"), ms,
                      ops / ms / 1e6, ops / (ms * 1e-3) / 132 / 1.9e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
