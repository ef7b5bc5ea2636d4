// select.cu — a9, batched variant selection (Table 1 get_policy, on many
// feature vectors at once): walk root -> leaf with x[f] <= thr -> left
// (S:224), NaN -> right (R8), output the leaf's variant.
//
// The device tree is a BFS array of 8-byte nodes; the threshold is stored as
// the largest float32 <= the double threshold, which makes the float compare
// exact (V:A5).  Vectors are staged through shared memory with coalesced
// 16-byte loads, each thread then walks one vector reading its features from
// a bank-conflict-padded row.
#include "common.h"

namespace adapt {
namespace {

constexpr int kSelThreads = 256;

__global__ void __launch_bounds__(kSelThreads)
    select_kernel(const DNode *__restrict__ gtree, int n_nodes, int tree_in_smem /* = n_top */,
                  const float *__restrict__ X, int64_t m, int F, int32_t *__restrict__ out) {
  extern __shared__ float sx[];  // [kSelThreads][F | 1] (odd stride) | tree copy
  const int stride = F | 1;
  const int t = threadIdx.x;
  // the first n_top nodes (BFS order = the top levels, where every walk
  // passes) live in shared memory; deeper nodes are read through L1/L2
  DNode *st = reinterpret_cast<DNode *>(sx + kSelThreads * stride + (kSelThreads * stride & 1));
  const int n_top = tree_in_smem;
  for (int i = t; i < n_top; i += kSelThreads) st[i] = gtree[i];
  __syncthreads();
  const bool aligned = (reinterpret_cast<uintptr_t>(X) & 15) == 0 && (F & 3) == 0;
  for (int64_t v0 = blockIdx.x * (int64_t)kSelThreads; v0 < m;
       v0 += (int64_t)gridDim.x * kSelThreads) {
    const int rows = (m - v0 < kSelThreads) ? (int)(m - v0) : kSelThreads;
    const float *src = X + v0 * F;
    const int cnt = rows * F;
    if (aligned) {
      const float4 *s4 = reinterpret_cast<const float4 *>(src);
      for (int i = t; i < (cnt >> 2); i += kSelThreads) {
        const float4 v = __ldcs(s4 + i);
        const int e = i << 2, r = e / F, c = e - r * F;  // F % 4 == 0: one row per float4
        float *d = sx + r * stride + c;
        d[0] = v.x;
        d[1] = v.y;
        d[2] = v.z;
        d[3] = v.w;
      }
    } else {
      for (int i = t; i < cnt; i += kSelThreads) {
        const int r = i / F, c = i - r * F;
        sx[r * stride + c] = __ldcs(src + i);
      }
    }
    __syncthreads();
    if (t < rows) {
      const float *x = sx + t * stride;
      DNode nd = n_top > 0 ? st[0] : gtree[0];
      while (nd.meta >= 0) {
        const float v = x[nd.meta & 63];
        const int k = (nd.meta >> 6) + (v <= nd.thr ? 0 : 1);
        nd = k < n_top ? st[k] : gtree[k];
      }
      const int32_t meta = nd.meta;
      __stcs(out + v0 + t, -1 - meta);
    }
    __syncthreads();
  }
}

}  // namespace

void launch_select(const DNode *tree, int n_nodes, const float *X, int64_t m, int F, int32_t *out,
                   cudaStream_t s) {
  if (m == 0) return;
  const size_t xs = ((size_t)kSelThreads * (F | 1) * 4 + 7) / 8 * 8;
  const int n_top = n_nodes < 2048 ? n_nodes : 2047;  // top 11 levels: 16 KB
  const size_t smem = xs + (size_t)n_top * sizeof(DNode);
  CUDA_CHECK(cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  int64_t blocks = (m + kSelThreads - 1) / kSelThreads;
  if (blocks > 148 * 8) blocks = 148 * 8;
  select_kernel<<<(int)blocks, kSelThreads, smem, s>>>(tree, n_nodes, n_top, X, m, F, out);
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace adapt
