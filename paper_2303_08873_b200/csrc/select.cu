// select.cu — a9, batched variant selection (Table 1 get_policy, on many
// feature vectors at once): walk root -> leaf with x[f] <= thr -> left
// (S:224), NaN -> right (R8), output the leaf's variant.
//
// The device tree is a BFS array of 8-byte nodes; the threshold is stored as
// the largest float32 <= the double threshold, which makes the float compare
// exact (V:A5).  The first kTopNodes nodes (the top levels every walk visits;
// a whole depth-12 tree) sit in shared memory, deeper ones are read through
// L1/L2.  Vectors stream through a register-prefetched, double-buffered tile:
// while the block walks tile k out of shared memory (odd row stride: no bank
// conflicts between lanes), the coalesced 16-byte loads of tile k+1 are in
// flight.
#include <algorithm>

#include "common.h"

namespace adapt {
namespace {

constexpr int kSelThreads = 512;
constexpr int kTopNodes = 8191;  // 64 KB

__device__ __forceinline__ DNode ldg_node(const DNode *p) {
  const int2 v = __ldg(reinterpret_cast<const int2 *>(p));
  DNode d;
  d.thr = __int_as_float(v.x);
  d.meta = v.y;
  return d;
}

template <int F>
__global__ void __launch_bounds__(kSelThreads, 2)
    select_kernel(const DNode *__restrict__ gtree, int n_top, const float *__restrict__ X,
                  int64_t m, int32_t *__restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int kStride = F | 1;                   // odd row stride of the tile
  constexpr int kVec = F / 4;                      // float4 per vector
  DNode *st = reinterpret_cast<DNode *>(smem);     // [n_top]
  float *sx = reinterpret_cast<float *>(smem + (size_t)kTopNodes * sizeof(DNode));  // [T][kStride]
  const int t = threadIdx.x;
  for (int i = t; i < n_top; i += kSelThreads) st[i] = gtree[i];

  const int64_t ntiles = (m + kSelThreads - 1) / kSelThreads;
  float4 pre[kVec];  // this thread's share of the next tile (coalesced float4s)
  auto fetch = [&](int64_t tile) {
    const int64_t v0 = tile * kSelThreads;
    const int rows = (m - v0 < kSelThreads) ? (int)(m - v0) : kSelThreads;
    const float4 *src = reinterpret_cast<const float4 *>(X + v0 * F);
#pragma unroll
    for (int k = 0; k < kVec; k++) {
      const int i = t + k * kSelThreads;  // float4 index within the tile
      pre[k] = i < rows * kVec ? __ldcs(src + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto stash = [&]() {
#pragma unroll
    for (int k = 0; k < kVec; k++) {
      const int i = t + k * kSelThreads, r = i / kVec, c = (i % kVec) * 4;
      float *d = sx + r * kStride + c;
      d[0] = pre[k].x;
      d[1] = pre[k].y;
      d[2] = pre[k].z;
      d[3] = pre[k].w;
    }
  };
  int64_t tile = blockIdx.x;
  if (tile < ntiles) fetch(tile);
  __syncthreads();  // tree copy visible
  for (; tile < ntiles; tile += gridDim.x) {
    stash();
    __syncthreads();
    if (tile + gridDim.x < ntiles) fetch(tile + gridDim.x);  // next tile in flight during the walks
    const int64_t v = tile * kSelThreads + t;
    if (v < m) {
      const float *x = sx + t * kStride;
      DNode nd = st[0];
      while (nd.meta >= 0) {
        const float xv = x[nd.meta & 63];
        const int k = (nd.meta >> 6) + (xv <= nd.thr ? 0 : 1);
        nd = k < n_top ? st[k] : ldg_node(gtree + k);
      }
      __stcs(out + v, -1 - nd.meta);
    }
    __syncthreads();
  }
}

// generic F (not a multiple of 4, or an unaligned X): scalar staging
__global__ void __launch_bounds__(kSelThreads, 2)
    select_kernel_any(const DNode *__restrict__ gtree, int n_top, const float *__restrict__ X,
                      int64_t m, int F, int32_t *__restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int stride = F | 1;
  DNode *st = reinterpret_cast<DNode *>(smem);
  float *sx = reinterpret_cast<float *>(smem + (size_t)kTopNodes * sizeof(DNode));
  const int t = threadIdx.x;
  for (int i = t; i < n_top; i += kSelThreads) st[i] = gtree[i];
  for (int64_t v0 = blockIdx.x * (int64_t)kSelThreads; v0 < m; v0 += (int64_t)gridDim.x * kSelThreads) {
    const int rows = (m - v0 < kSelThreads) ? (int)(m - v0) : kSelThreads;
    __syncthreads();
    for (int i = t; i < rows * F; i += kSelThreads) {
      const int r = i / F, c = i - r * F;
      sx[r * stride + c] = __ldcs(X + v0 * F + i);
    }
    __syncthreads();
    if (t < rows) {
      const float *x = sx + t * stride;
      DNode nd = st[0];
      while (nd.meta >= 0) {
        const int k = (nd.meta >> 6) + (x[nd.meta & 63] <= nd.thr ? 0 : 1);
        nd = k < n_top ? st[k] : ldg_node(gtree + k);
      }
      __stcs(out + v0 + t, -1 - nd.meta);
    }
  }
}

}  // namespace

void launch_select(const DNode *tree, int n_nodes, const float *X, int64_t m, int F, int32_t *out,
                   cudaStream_t s) {
  if (m == 0) return;
  const int n_top = std::min(n_nodes, kTopNodes);
  const size_t smem = (size_t)kTopNodes * sizeof(DNode) + (size_t)kSelThreads * (F | 1) * 4;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (m + kSelThreads - 1) / kSelThreads;
  const int grid = (int)std::min<int64_t>(tiles, 2 * sms);
  const bool vec = (reinterpret_cast<uintptr_t>(X) & 15) == 0;
  switch (vec ? F : 0) {
#define CASE(FF)                                                                              \
  case FF:                                                                                    \
    CUDA_CHECK(cudaFuncSetAttribute(select_kernel<FF>,                                        \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));  \
    select_kernel<FF><<<grid, kSelThreads, smem, s>>>(tree, n_top, X, m, out);                \
    break;
    CASE(4) CASE(8) CASE(12) CASE(16) CASE(20) CASE(24) CASE(32) CASE(48) CASE(64)
#undef CASE
    default:
      CUDA_CHECK(cudaFuncSetAttribute(select_kernel_any,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      select_kernel_any<<<grid, kSelThreads, smem, s>>>(tree, n_top, X, m, F, out);
  }
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace adapt
