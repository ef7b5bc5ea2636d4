// kfold.cu — the paper's K-fold evaluation methodology on the GPU (SURVEY
// §8(f) f4; "we split application inputs into K equal-sized groups.
// A fraction f of groups is used for model training while the rest are used
// for testing ... K-fold creation is repeated 10 times, each time shuffling
// the inputs"; Adaptive-25/50/75 = K = 4 with m = 1/2/3 training groups).
//
//   kfold_weights_kernel  R22: shuffle s permutes the GLOBAL row ids with a
//                         4-round Feistel network on 2h-bit words, cycle-
//                         walking into [0, N); group = floor(pos K / N) (found
//                         from the K+1 integer group bounds, no 64-bit
//                         division); u8 weight 1 iff the group is one of the
//                         fold's training groups.  The level loop trains on the
//                         weights exactly as for forests (weight-0 rows drop
//                         out at the first partition), so no subset is copied.
//   kfold_eval_kernel     per test row (weight 0): the selection against the
//                         row's label and the times of the selected / fastest
//                         variants; one partial per block (a fixed grid), summed
//                         on the host in block order: deterministic.
#include <algorithm>

#include "common.h"

namespace adapt {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // splitmix64 finaliser
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t feistel_pos(uint64_t key, uint64_t N, int h, uint64_t r) {
  const uint64_t mask = (1ull << h) - 1;
  uint64_t x = r;
  do {
    uint64_t L = x >> h, R = x & mask;
#pragma unroll
    for (uint64_t j = 0; j < 4; j++) {
      const uint64_t t = L ^ (mix64(key ^ mix64((R << 2) | j)) & mask);
      L = R;
      R = t;
    }
    x = (L << h) | R;
  } while (x >= N);
  return x;
}

__global__ void kfold_weights_kernel(uint64_t key, uint64_t N, int h, const uint64_t *__restrict__ bnd,
                                     int K, int m, int k, uint64_t lo, int64_t n, uint8_t *__restrict__ w) {
  __shared__ uint64_t sb[kKfoldMaxK + 1];
  for (int i = threadIdx.x; i <= K; i += blockDim.x) sb[i] = bnd[i];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t pos = feistel_pos(key, N, h, lo + (uint64_t)i);
    int g = min(K - 1, (int)((double)pos * (double)K / (double)N));  // then exact, from the bounds
    while (g + 1 < K && pos >= sb[g + 1]) g++;
    while (pos < sb[g]) g--;
    const int off = (g - k + K) % K;  // training groups k, k+1, ..., k+m-1 (mod K)
    w[i] = off < m ? 1 : 0;
  }
}

constexpr int kEvalThreads = 512;

__global__ void __launch_bounds__(kEvalThreads)
    kfold_eval_kernel(const uint8_t *__restrict__ w, const uint8_t *__restrict__ lab,
                      const int32_t *__restrict__ sel, const float *__restrict__ times, int64_t n, int V,
                      KfoldPartial *__restrict__ part) {
  unsigned long long nt = 0, nc = 0;
  double ts = 0.0, tb = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (w[i]) continue;
    const int v = sel[i], y = lab[i];
    nt++;
    nc += v == y;
    ts += (double)__ldg(times + i * V + v);
    tb += (double)__ldg(times + i * V + y);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nt += __shfl_xor_sync(0xffffffffu, nt, o);
    nc += __shfl_xor_sync(0xffffffffu, nc, o);
    ts += __shfl_xor_sync(0xffffffffu, ts, o);
    tb += __shfl_xor_sync(0xffffffffu, tb, o);
  }
  __shared__ KfoldPartial sp[kEvalThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sp[warp] = KfoldPartial{nt, nc, ts, tb};
  __syncthreads();
  if (threadIdx.x == 0) {
    KfoldPartial p = sp[0];
    for (int i = 1; i < kEvalThreads / 32; i++) {  // fixed order
      p.n_test += sp[i].n_test;
      p.n_correct += sp[i].n_correct;
      p.t_selected += sp[i].t_selected;
      p.t_best += sp[i].t_best;
    }
    part[blockIdx.x] = p;
  }
}

int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

}  // namespace

uint64_t kfold_key(uint64_t seed, int shuffle) {
  auto mix = [](uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  return mix(seed ^ mix((uint64_t)shuffle + 0x2545F4914F6CDD1Dull));
}

void launch_kfold_weights(uint64_t seed, int shuffle, uint64_t N, const uint64_t *d_bnd, int K, int m,
                          int k, uint64_t lo, int64_t n, uint8_t *w, cudaStream_t s) {
  if (n == 0) return;
  int h = 1;
  while (h < 31 && (1ull << (2 * h)) < N) h++;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 8);
  kfold_weights_kernel<<<grid, 256, 0, s>>>(kfold_key(seed, shuffle), N, h, d_bnd, K, m, k, lo, n, w);
  CUDA_CHECK(cudaGetLastError());
}

int kfold_eval_blocks() { return sm_count() * 2; }

void launch_kfold_eval(const uint8_t *w, const uint8_t *lab, const int32_t *sel, const float *times,
                       int64_t n, int V, KfoldPartial *part, cudaStream_t s) {
  kfold_eval_kernel<<<kfold_eval_blocks(), kEvalThreads, 0, s>>>(w, lab, sel, times, n, V, part);
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace adapt
