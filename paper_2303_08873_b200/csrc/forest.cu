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
//                      this rank counts the draws that land in its shard,
//                      straight into the u8 weight plane (packed atomics);
//   boot_sum_kernel    guard: the weights must sum to the draws counted (a
//                      multiplicity of 256+ — probability ~1/256! per row —
//                      would carry into a neighbour and break the sum);
//   select_forest_kernel  a9 for forests: every tree walked per vector, the
//                      majority of their variants, ties -> lowest (R20).
#include <algorithm>
#include <cstdlib>

#include "common.h"
#include "vecreg.cuh"

namespace adapt {
namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// counts are u8 lanes of u32 words (the whole count array of 1e8 rows is
// 100 MB: L2-resident, so the random atomics stay on chip); a count reaching
// 256 would carry into its neighbour, which the caller detects: the bytes must
// sum to the number of draws that landed in this shard (*landed)
__global__ void boot_count_kernel(uint64_t key, uint64_t n_total, uint64_t lo, uint64_t n_local,
                                  uint32_t *cnt4, unsigned long long *landed) {
  uint32_t mine = 0;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n_total;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = __umul64hi(splitmix64(key ^ splitmix64(j)), n_total);
    if (i >= lo && i - lo < n_local) {
      const uint64_t k = i - lo;
      atomicAdd(cnt4 + (k >> 2), 1u << (8 * (k & 3)));
      mine++;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(landed, (unsigned long long)mine);
}

// the byte sum of the counts (must equal *landed; else a count overflowed)
__global__ void boot_sum_kernel(const uint32_t *cnt4, int64_t words, unsigned long long *sum) {
  uint32_t mine = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < words;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t w = cnt4[i];
    mine += (w & 0xFF) + ((w >> 8) & 0xFF) + ((w >> 16) & 0xFF) + (w >> 24);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(sum, (unsigned long long)mine);
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
// indices in DNode::meta are absolute).  Warps own tiles of 32 vectors: the
// tile's rows are loaded coalesced into the warp's odd-stride smem tile, each
// lane walks every tree for its vector, the votes go to the warp's smem, and
// the majority (ties -> lowest) is counted in O(T^2) per vector.
__global__ void __launch_bounds__(kForestThreads)
    select_forest_kernel(const DNode *__restrict__ nodes, int n_nodes, const int32_t *roots, int T,
                         const float *__restrict__ X, int64_t m, int F, int32_t *__restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int W = kForestThreads / 32;
  const int n_top = min(n_nodes, kForestTop);
  const int stride = F | 1;
  DNode *st = reinterpret_cast<DNode *>(smem);
  float *tiles = reinterpret_cast<float *>(smem + (size_t)n_top * sizeof(DNode));
  uint8_t *votes = reinterpret_cast<uint8_t *>(tiles + (size_t)W * 32 * stride);
  __shared__ int32_t s_roots[64];
  for (int i = threadIdx.x; i < n_top; i += blockDim.x) st[i] = nodes[i];
  for (int i = threadIdx.x; i < T; i += blockDim.x) s_roots[i] = roots[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float *tile = tiles + (size_t)warp * 32 * stride;
  uint8_t *vw = votes + (size_t)warp * T * 32;
  const float invF = 1.0f / (float)F;  // row = i / F exactly: i < 2048, F <= 64
  const int64_t ntiles = (m + 31) / 32;
  for (int64_t tl = blockIdx.x * (int64_t)W + warp; tl < ntiles; tl += (int64_t)gridDim.x * W) {
    const int64_t v0 = tl * 32;
    const int rows = m - v0 < 32 ? (int)(m - v0) : 32;
    __syncwarp();
    for (int i = lane; i < rows * F; i += 32) {  // coalesced: the tile is contiguous in X
      const int r = __float2int_rz(((float)i + 0.5f) * invF);
      tile[r * stride + (i - r * F)] = __ldcs(X + v0 * F + i);
    }
    __syncwarp();
    if (lane < rows) {
      const float *x = tile + lane * stride;
      for (int t = 0; t < T; t++) {
        DNode nd = node_at(st, n_top, nodes, s_roots[t]);
        while (nd.meta >= 0) {
          const int k = (nd.meta >> 6) + (x[nd.meta & 63] <= nd.thr ? 0 : 1);  // NaN -> right
          nd = node_at(st, n_top, nodes, k);
        }
        vw[t * 32 + lane] = (uint8_t)(-1 - nd.meta);
      }
      int best = 255, best_c = 0;  // majority, ties -> lowest variant (R20)
      for (int t = 0; t < T; t++) {
        const int l = vw[t * 32 + lane];
        int c = 0;
        for (int u = 0; u < T; u++) c += vw[u * 32 + lane] == l;
        if (c > best_c || (c == best_c && l < best)) {
          best = l;
          best_c = c;
        }
      }
      __stcs(out + v0 + lane, best);
    }
  }
}

// The product forest kernel: one vector per thread, loaded straight from HBM
// (next one in flight) and parked in the thread's own shared-memory column (as
// select.cu's select_kernel_c), every tree walked from the shared-memory top
// (deeper nodes through L1/L2), the T votes in the thread's vote column,
// majority with ties -> lowest variant (R20).  1024 threads per CTA, one CTA
// per SM; the next vector's loads are in flight during the walks.
constexpr int kForestDThreads = 1024;

template <int F>
__global__ void __launch_bounds__(kForestDThreads, 1)
    select_forest_d(const DNode *__restrict__ nodes, int n_nodes, const int32_t *roots, int T,
                    const float *__restrict__ X, int64_t m, int wide, int32_t *__restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int n_top = min(n_nodes, kForestTop);
  DNode *st = reinterpret_cast<DNode *>(smem);
  uint8_t *votes = smem + (size_t)kForestTop * sizeof(DNode);  // [T][kForestDThreads]
  // the thread's vector in its own shared-memory column (conflict-free reads of any feature)
  float *xc = reinterpret_cast<float *>(votes + (size_t)64 * kForestDThreads) + threadIdx.x;
  __shared__ int32_t s_roots[64];
  const int tid = threadIdx.x;
  for (int i = tid; i < n_top; i += kForestDThreads) st[i] = nodes[i];
  for (int i = tid; i < T; i += kForestDThreads) s_roots[i] = roots[i];
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * kForestDThreads;
  int64_t v = blockIdx.x * (int64_t)kForestDThreads + tid;
  float nx[F];
  if (v < m) load_vec<F>(X + v * F, wide, nx);
  for (; v < m; v += stride) {
#pragma unroll
    for (int f = 0; f < F; f++) xc[f * kForestDThreads] = nx[f];
    if (v + stride < m) load_vec<F>(X + (v + stride) * F, wide, nx);
    for (int t = 0; t < T; t++) {
      DNode nd = node_at(st, n_top, nodes, s_roots[t]);
      while (nd.meta >= 0) {
        const int k = (nd.meta >> 6) + (xc[(nd.meta & 63) * kForestDThreads] <= nd.thr ? 0 : 1);  // NaN -> right
        nd = node_at(st, n_top, nodes, k);
      }
      votes[t * kForestDThreads + tid] = (uint8_t)(-1 - nd.meta);
    }
    int best = 255, best_c = 0;  // majority, ties -> lowest variant (R20)
    for (int t = 0; t < T; t++) {
      const int l = votes[t * kForestDThreads + tid];
      int c = 0;
      for (int u = 0; u < T; u++) c += votes[u * kForestDThreads + tid] == l;
      if (c > best_c || (c == best_c && l < best)) {
        best = l;
        best_c = c;
      }
    }
    __stcs(out + v, best);
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
                      uint8_t *w, unsigned long long *sums, cudaStream_t s) {
  // w: the weight plane, used directly as the packed u8 counts (n_local + 4 bytes)
  const int64_t words = (n_local + 3) / 4;
  if (words > 0) CUDA_CHECK(cudaMemsetAsync(w, 0, (size_t)words * 4, s));
  CUDA_CHECK(cudaMemsetAsync(sums, 0, 16, s));
  auto mix = [](uint64_t x) {  // host copy of the mixer, for the per-tree key
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  const uint64_t key = mix(seed ^ mix((uint64_t)tree + 0x5851F42D4C957F2Dull));
  const int sms = sm_count();
  if (n_total > 0 && n_local > 0) {
    const int grid = (int)std::min<uint64_t>((n_total + 255) / 256, (uint64_t)8 * sms);
    boot_count_kernel<<<grid, 256, 0, s>>>(key, n_total, lo, (uint64_t)n_local,
                                           reinterpret_cast<uint32_t *>(w), sums); ++g_kernel_launches;
    CUDA_CHECK(cudaGetLastError());
    const int g2 = (int)std::min<int64_t>((words + 255) / 256, (int64_t)8 * sms);
    boot_sum_kernel<<<g2, 256, 0, s>>>(reinterpret_cast<const uint32_t *>(w), words, sums + 1); ++g_kernel_launches;
    CUDA_CHECK(cudaGetLastError());
  }
}

int forest_max_trees() { return 64; }

void launch_select_forest(const DNode *nodes, int n_nodes, const int32_t *roots, int T,
                          const float *X, int64_t m, int F, int32_t *out, cudaStream_t s) {
  if (m == 0) return;
  static const bool tile = getenv("ADAPT_SEL_TILE") != nullptr;  // the per-warp tile kernel (A/B)
  if (!tile && (reinterpret_cast<uintptr_t>(X) & 15) == 0 && (F == 4 || F == 8 || F == 12 || F == 16)) {
    const int wide = (reinterpret_cast<uintptr_t>(X) & 31) == 0;
    const size_t smem = (size_t)kForestTop * sizeof(DNode) + (size_t)64 * kForestDThreads +
                        (size_t)F * kForestDThreads * 4;  // tree top, vote columns, vector columns
    const int grid = (int)std::min<int64_t>((m + kForestDThreads - 1) / kForestDThreads, sm_count());
    switch (F) {
#define CASE(FF)                                                                                  \
  case FF:                                                                                        \
    smem_limit(select_forest_d<FF>, smem);                                                        \
    select_forest_d<FF><<<grid, kForestDThreads, smem, s>>>(nodes, n_nodes, roots, T, X, m, wide, out); ++g_kernel_launches; \
    break;
      CASE(4) CASE(8) CASE(12) CASE(16)
#undef CASE
    }
    CUDA_CHECK(cudaGetLastError());
    return;
  }
  constexpr int W = kForestThreads / 32;
  const size_t smem = (size_t)std::min(n_nodes, kForestTop) * sizeof(DNode) +
                      (size_t)W * 32 * (F | 1) * 4 + (size_t)W * T * 32;
  smem_limit(select_forest_kernel, smem);
  const int64_t tiles = (m + 31) / 32;
  const int grid = (int)std::min<int64_t>((tiles + W - 1) / W, 2 * sm_count());
  select_forest_kernel<<<grid, kForestThreads, smem, s>>>(nodes, n_nodes, roots, T, X, m, F, out); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace adapt
