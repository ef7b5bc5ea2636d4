// forest.cu — random forests ("rfc": "the
// number of decision trees in the forest" and "the maximum tree depth"; SPEC
// train_rfc / predict).  Each tree is the same level-wise CART trained on a
// bootstrap resample of the table; rows enter the histograms with their
// multiplicity as weight (level.cu), so no resample is ever materialised.
//
//   boot_count_kernel  R19: n draws with replacement over the GLOBAL table;
//                      draw j picks row floor(h_j * n / 2^64),
//                      h_j = splitmix64(key_t ^ splitmix64(j)),
//                      key_t = splitmix64(seed ^ splitmix64(t + 0x5851F42D4C957F2D));
//                      this rank counts the draws that land in its shard;
//   boot_pack_kernel   u32 counts -> the u8 weight plane (a count > 255 is
//                      flagged; for n draws it has probability ~1/255!);
//   select_forest_kernel  a9 for forests: every tree walked per vector, the
//                      majority of their variants, ties -> lowest (R20).
#include <algorithm>

#include "common.h"

namespace adapt {
namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void boot_count_kernel(uint64_t key, uint64_t n_total, uint64_t lo, uint64_t n_local,
                                  uint32_t *cnt) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n_total;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = __umul64hi(splitmix64(key ^ splitmix64(j)), n_total);
    if (i >= lo && i - lo < n_local) atomicAdd(cnt + (i - lo), 1u);
  }
}

__global__ void boot_pack_kernel(const uint32_t *cnt, int64_t n, uint8_t *w, uint32_t *flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t c = cnt[i];
    if (c > 255) atomicOr(flags, kFlagBootstrap);
    w[i] = (uint8_t)min(c, 255u);
  }
}

constexpr int kForestThreads = 256;
constexpr int kForestTop = 8191;  // forest nodes held in smem (64 KB)

__device__ __forceinline__ DNode node_at(const DNode *st, int n_top, const DNode *g, int k) {
  if (k < n_top) return st[k];
  const int2 v = __ldg(reinterpret_cast<const int2 *>(g + k));
  DNode d;
  d.thr = __int_as_float(v.x);
  d.meta = v.y;
  return d;
}

// roots[t] = index of tree t's root in the concatenated node array (children
// indices in DNode::meta are absolute)
__global__ void __launch_bounds__(kForestThreads)
    select_forest_kernel(const DNode *__restrict__ nodes, int n_nodes, const int32_t *roots, int T,
                         const float *__restrict__ X, int64_t m, int F, int32_t *__restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  DNode *st = reinterpret_cast<DNode *>(smem);
  uint8_t *votes = smem + (size_t)kForestTop * sizeof(DNode);  // [T][threads]
  const int n_top = min(n_nodes, kForestTop);
  for (int i = threadIdx.x; i < n_top; i += blockDim.x) st[i] = nodes[i];
  __syncthreads();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < m;
       v += (int64_t)gridDim.x * blockDim.x) {
    const float *x = X + v * F;
    for (int t = 0; t < T; t++) {
      DNode nd = node_at(st, n_top, nodes, roots[t]);
      while (nd.meta >= 0) {
        const float xv = __ldg(x + (nd.meta & 63));
        nd = node_at(st, n_top, nodes, (nd.meta >> 6) + (xv <= nd.thr ? 0 : 1));  // NaN -> right
      }
      votes[t * kForestThreads + threadIdx.x] = (uint8_t)(-1 - nd.meta);
    }
    // majority, ties -> lowest variant (R20)
    int best = 255, best_c = 0;
    for (int t = 0; t < T; t++) {
      const int l = votes[t * kForestThreads + threadIdx.x];
      int c = 0;
      for (int u = 0; u < T; u++) c += votes[u * kForestThreads + threadIdx.x] == l;
      if (c > best_c || (c == best_c && l < best)) {
        best = l;
        best_c = c;
      }
    }
    out[v] = best;
  }
}

int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

}  // namespace

void launch_bootstrap(uint64_t seed, int tree, uint64_t n_total, uint64_t lo, int64_t n_local,
                      uint32_t *cnt, uint8_t *w, uint32_t *flags, cudaStream_t s) {
  if (n_local > 0) CUDA_CHECK(cudaMemsetAsync(cnt, 0, (size_t)n_local * 4, s));
  const uint64_t key = [&] {  // host copy of the same mixer, for the per-tree key
    auto mix = [](uint64_t x) {
      uint64_t z = x + 0x9E3779B97F4A7C15ull;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      return z ^ (z >> 31);
    };
    return mix(seed ^ mix((uint64_t)tree + 0x5851F42D4C957F2Dull));
  }();
  const int sms = sm_count();
  if (n_total > 0 && n_local > 0) {
    const int grid = (int)std::min<uint64_t>((n_total + 255) / 256, (uint64_t)8 * sms);
    boot_count_kernel<<<grid, 256, 0, s>>>(key, n_total, lo, (uint64_t)n_local, cnt);
    CUDA_CHECK(cudaGetLastError());
    const int g2 = (int)std::min<int64_t>((n_local + 255) / 256, (int64_t)8 * sms);
    boot_pack_kernel<<<g2, 256, 0, s>>>(cnt, n_local, w, flags);
    CUDA_CHECK(cudaGetLastError());
  }
}

int forest_max_trees() { return 64; }

void launch_select_forest(const DNode *nodes, int n_nodes, const int32_t *roots, int T,
                          const float *X, int64_t m, int F, int32_t *out, cudaStream_t s) {
  if (m == 0) return;
  const size_t smem = (size_t)kForestTop * sizeof(DNode) + (size_t)T * kForestThreads;
  CUDA_CHECK(cudaFuncSetAttribute(select_forest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  const int grid = (int)std::min<int64_t>((m + kForestThreads - 1) / kForestThreads, 2 * sm_count());
  select_forest_kernel<<<grid, kForestThreads, smem, s>>>(nodes, n_nodes, roots, T, X, m, F, out);
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace adapt
