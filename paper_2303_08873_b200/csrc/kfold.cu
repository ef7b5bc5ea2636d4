// kfold.cu — the paper's K-fold evaluation methodology on the GPU (SURVEY
// §8(f) f4; "we split application inputs into K equal-sized groups.
// A fraction f of groups is used for model training while the rest are used
// for testing ... K-fold creation is repeated 10 times, each time shuffling
// the inputs"; Adaptive-25/50/75 = K = 4 with m = 1/2/3 training groups).
//
//   kfold_group_kernel    R22: shuffle s permutes the GLOBAL row ids with a
//                         4-round Feistel network on 2h-bit words, cycle-
//                         walking into [0, N); group = floor(pos K / N) (found
//                         from the K+1 integer group bounds, no 64-bit
//                         division), plus the local group sizes.
//   kfold_scatter_kernel  counting sort of the ingest planes (bins + labels)
//                         by (shuffle, group): group g of shuffle j becomes one
//                         contiguous piece.  Model (j, k)'s root is then the m
//                         pieces of its training groups, and ALL models of a
//                         batch of shuffles grow in ONE frontier of the level
//                         loop (engine.cpp MultiRoot): the first partition
//                         copies each row into the m models that train on it,
//                         so the whole protocol costs D level passes instead of
//                         D per model.
//   kfold_eval_many_kernel  every row walks the trees of the models that hold
//                         it out: the selection against the row's label and the
//                         times of the selected / fastest variants, warp sums
//                         then per-block partials per model.
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

// group of every local row in shuffle s (u8) and the local group sizes
__global__ void kfold_group_kernel(uint64_t key, uint64_t N, int h, const uint64_t *__restrict__ bnd,
                                   int K, uint64_t lo, int64_t n, uint8_t *__restrict__ grp,
                                   unsigned long long *__restrict__ cnt) {
  __shared__ uint64_t sb[kKfoldMaxK + 1];
  __shared__ unsigned int sc[kKfoldMaxK];
  for (int i = threadIdx.x; i <= K; i += blockDim.x) sb[i] = bnd[i];
  for (int i = threadIdx.x; i < K; i += blockDim.x) sc[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t pos = feistel_pos(key, N, h, lo + (uint64_t)i);
    int g = min(K - 1, (int)((double)pos * (double)K / (double)N));
    while (g + 1 < K && pos >= sb[g + 1]) g++;
    while (pos < sb[g]) g--;
    grp[i] = (uint8_t)g;
    atomicAdd(&sc[g], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < K; i += blockDim.x)
    if (sc[i]) atomicAdd(cnt + i, (unsigned long long)sc[i]);
}

// counting-sort scatter of the ingest planes by group: row i of shuffle j goes
// to cursor[j][grp] (warp-aggregated claims); the order inside a group is
// irrelevant (histograms are order-independent integer sums)
__global__ void kfold_scatter_kernel(const uint8_t *__restrict__ bins, size_t pstride_in,
                                     const uint8_t *__restrict__ lab, int64_t n, int planes, int wb,
                                     const uint8_t *__restrict__ grp, int sb, int K,
                                     unsigned int *__restrict__ cursor, uint8_t *__restrict__ obins,
                                     size_t pstride_out, uint8_t *__restrict__ olab) {
  const int lane = threadIdx.x & 31;
  const int64_t total = n * sb;
  for (int64_t t0 = blockIdx.x * (int64_t)blockDim.x; t0 < total; t0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = t0 + threadIdx.x;
    const bool live = t < total;
    const int j = live ? (int)(t / n) : 0;
    const int64_t i = live ? t - (int64_t)j * n : 0;
    const int key = live ? j * K + grp[t] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int leader = __ffs(peers) - 1;
    unsigned base = 0;
    if (live && lane == leader) base = atomicAdd(cursor + key, (unsigned)__popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (!live) continue;
    const uint32_t pos = base + __popc(peers & ((1u << lane) - 1));
    olab[pos] = lab[i];
    if (wb == 4) {
      for (int p = 0; p < planes; p++)
        *reinterpret_cast<uint32_t *>(obins + p * pstride_out + (size_t)pos * 4) =
            *reinterpret_cast<const uint32_t *>(bins + p * pstride_in + (size_t)i * 4);
    } else {
      for (int b = 0; b < wb; b++) obins[(size_t)pos * wb + b] = bins[(size_t)i * wb + b];
    }
  }
}

constexpr int kEvalManyThreads = 256;

// every batch model (shuffle j, fold k) walks its tree for the rows it holds
// out: (g - k) mod K >= m; per-model partials in shared memory, one set per block
__global__ void __launch_bounds__(kEvalManyThreads)
    kfold_eval_many_kernel(const float *__restrict__ X, int64_t n, int F, int V,
                           const float *__restrict__ times, const uint8_t *__restrict__ lab,
                           const uint8_t *__restrict__ grp, int sb, int K, int m,
                           const DNode *__restrict__ nodes, const int32_t *__restrict__ roots,
                           KfoldPartial *__restrict__ part) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  KfoldPartial *sp = reinterpret_cast<KfoldPartial *>(smem_raw);
  const int R = sb * K;
  for (int r = threadIdx.x; r < R; r += blockDim.x) sp[r] = KfoldPartial{0, 0, 0.0, 0.0};
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;  // warp-uniform trip count: lanes past n count nothing
    const bool live = i < n;
    const float *x = X + (live ? i : 0) * F;
    const int y = live ? lab[i] : 0;
    const float ty = live ? __ldg(times + i * V + y) : 0.f;
    for (int j = 0; j < sb; j++) {
      const int g = live ? grp[(int64_t)j * n + i] : 0;
      for (int k = 0; k < K; k++) {
        const bool test = live && (g - k + K) % K >= m;  // else a training row of model (j, k)
        const int r = j * K + k;
        unsigned correct = 0;
        double ts = 0.0, tb = 0.0;
        if (test) {
          int kk = roots[r];
          int2 nd = __ldg(reinterpret_cast<const int2 *>(nodes + kk));
          while (nd.y >= 0) {
            const float xv = __ldg(x + (nd.y & 63));
            kk = (nd.y >> 6) + (xv <= __int_as_float(nd.x) ? 0 : 1);  // NaN -> right (R8)
            nd = __ldg(reinterpret_cast<const int2 *>(nodes + kk));
          }
          const int v = -1 - nd.y;
          correct = v == y;
          ts = (double)__ldg(times + i * V + v);
          tb = (double)ty;
        }
        // warp sums, then one shared-memory update per warp and model
        const unsigned nt = __reduce_add_sync(0xffffffffu, test ? 1u : 0u);
        const unsigned nc = __reduce_add_sync(0xffffffffu, correct);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          ts += __shfl_xor_sync(0xffffffffu, ts, o);
          tb += __shfl_xor_sync(0xffffffffu, tb, o);
        }
        if (lane == 0 && nt) {
          atomicAdd(&sp[r].n_test, (unsigned long long)nt);
          atomicAdd(&sp[r].n_correct, (unsigned long long)nc);
          atomicAdd(&sp[r].t_selected, ts);
          atomicAdd(&sp[r].t_best, tb);
        }
      }
    }
  }
  __syncthreads();
  for (int r = threadIdx.x; r < R; r += blockDim.x) part[(size_t)blockIdx.x * R + r] = sp[r];
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

int kfold_eval_blocks() { return sm_count() * 8; }  // latency-bound tree walks: full occupancy

void launch_kfold_groups(uint64_t seed, int shuffle, uint64_t N, const uint64_t *d_bnd, int K, uint64_t lo,
                         int64_t n, uint8_t *grp, unsigned long long *cnt, cudaStream_t s) {
  if (n == 0) return;
  int h = 1;
  while (h < 31 && (1ull << (2 * h)) < N) h++;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 8);
  kfold_group_kernel<<<grid, 256, 0, s>>>(kfold_key(seed, shuffle), N, h, d_bnd, K, lo, n, grp, cnt); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
}

void launch_kfold_scatter(const uint8_t *bins, size_t pstride_in, const uint8_t *lab, int64_t n, int BS,
                          const uint8_t *grp, int sb, int K, unsigned int *cursor, uint8_t *obins,
                          size_t pstride_out, uint8_t *olab, cudaStream_t s) {
  if (n == 0) return;
  const int planes = BS < 4 ? 1 : BS / 4, wb = BS < 4 ? BS : 4;
  const int grid = (int)std::min<int64_t>((n * sb + 255) / 256, (int64_t)sm_count() * 8);
  kfold_scatter_kernel<<<grid, 256, 0, s>>>(bins, pstride_in, lab, n, planes, wb, grp, sb, K, cursor, obins,
                                            pstride_out, olab); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
}

void launch_kfold_eval_many(const float *X, int64_t n, int F, int V, const float *times, const uint8_t *lab,
                            const uint8_t *grp, int sb, int K, int m, const DNode *nodes, const int32_t *roots,
                            KfoldPartial *part, cudaStream_t s) {
  const size_t smem = (size_t)sb * K * sizeof(KfoldPartial);
  smem_limit(kfold_eval_many_kernel, smem);
  kfold_eval_many_kernel<<<kfold_eval_blocks(), kEvalManyThreads, smem, s>>>(X, n, F, V, times, lab, grp, sb,
                                                                              K, m, nodes, roots, part); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
}


}  // namespace adapt
