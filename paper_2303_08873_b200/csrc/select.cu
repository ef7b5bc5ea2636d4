// select.cu — a9, batched variant selection (Table 1 get_policy, on many
// feature vectors at once): walk root -> leaf with x[f] <= thr -> left
// (S:224), NaN -> right (R8), output the leaf's variant.
//
// Thresholds are stored as the largest float32 <= the double threshold, which
// makes the float compare exact (V:A5).  Two product kernels, both one
// 1024-thread CTA per SM, each lane walking its own vector loaded straight
// from HBM (the next one's loads in flight during the walk):
//   select_kernel_c  trees within the shared-memory top (kSelTopNodes BFS
//                    nodes, e.g. C4's depth 12): the vector parked in the
//                    thread's own shared-memory column, so every feature read
//                    of the walk is one conflict-free wavefront;
//   select_kernel_h  deeper trees (C5's depth 16): the first td <= 14 levels
//                    as a complete heap in shared memory (fixed-trip walk, no
//                    bounds checks or child pointers), the vector in
//                    registers, then 2-level 32-byte bottom blocks (one
//                    256-bit load per 2 levels) — common.h SelTree.
// select_kernel_any serves F not a multiple of 4 or unaligned X.
#include <algorithm>

#include "common.h"
#include "vecreg.cuh"

namespace adapt {
namespace {

constexpr int kSelThreads = 1024;  // one CTA per SM: one smem copy of the tree
constexpr int kAnyThreads = 256;   // generic-F kernel
constexpr int kTopNodes = kSelTopNodes;  // 64 KB

// one bottom block (common.h layout) walked in registers: 3 levels, returns
// the next block (>= 0) or -1 - label
__device__ __forceinline__ int walk_block(const uint4 (&w)[4], const float *x) {
  const float t0 = __uint_as_float(w[0].x);
  const bool g0 = !(x[w[1].w & 63] <= t0);  // NaN -> right (R8)
  const float t1 = __uint_as_float(g0 ? w[0].z : w[0].y);
  const bool g1 = !(x[(g0 ? w[2].y : w[2].x) & 63] <= t1);
  const uint32_t tw = g0 ? (g1 ? w[1].z : w[1].y) : (g1 ? w[1].x : w[0].w);
  const uint32_t fw = g0 ? (g1 ? w[3].y : w[3].x) : (g1 ? w[2].w : w[2].z);
  const bool g2 = !(x[fw & 63] <= __uint_as_float(tw));
  // leaf edges i = 4 g0 + 2 g1 + g2 are words 7..14
  uint32_t r;
  if (g0)
    r = g1 ? (g2 ? w[3].z : w[3].y) : (g2 ? w[3].x : w[2].w);
  else
    r = g1 ? (g2 ? w[2].z : w[2].y) : (g2 ? w[2].x : w[1].w);
  return (int32_t)r >> 6;
}

// two 256-bit loads (LDG.E.256 on sm_100a): each lane touches 2 sectors with 2
// requests, half the L1 request count of four 128-bit loads
__device__ __forceinline__ void load_block(const uint4 *__restrict__ blocks, int b, uint4 (&w)[4]) {
  const uint4 *p = blocks + 4 * (int64_t)b;
#pragma unroll
  for (int i = 0; i < 4; i += 2)
    asm("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[i].x), "=r"(w[i].y), "=r"(w[i].z), "=r"(w[i].w), "=r"(w[i + 1].x),
                   "=r"(w[i + 1].y), "=r"(w[i + 1].z), "=r"(w[i + 1].w)
                 : "l"(p + i));
}


// Trees within the shared-memory top: every lane loads its own vector straight
// from HBM (256-bit loads when rows are 32-byte aligned; the next vector in
// flight during the walk) and parks it in its own shared-memory COLUMN
// (xs[f][tid]: any f of any lane is a distinct bank, so the walk's
// random-feature reads are conflict-free single wavefronts).
__device__ __forceinline__ int walk_block_col(const uint4 (&w)[4], const float *x) {
  constexpr int S = kSelThreads;
  const float t0 = __uint_as_float(w[0].x);
  const bool g0 = !(x[(w[1].w & 63) * S] <= t0);
  const float t1 = __uint_as_float(g0 ? w[0].z : w[0].y);
  const bool g1 = !(x[((g0 ? w[2].y : w[2].x) & 63) * S] <= t1);
  const uint32_t tw = g0 ? (g1 ? w[1].z : w[1].y) : (g1 ? w[1].x : w[0].w);
  const uint32_t fw = g0 ? (g1 ? w[3].y : w[3].x) : (g1 ? w[2].w : w[2].z);
  const bool g2 = !(x[(fw & 63) * S] <= __uint_as_float(tw));
  uint32_t r;
  if (g0)
    r = g1 ? (g2 ? w[3].z : w[3].y) : (g2 ? w[3].x : w[2].w);
  else
    r = g1 ? (g2 ? w[2].z : w[2].y) : (g2 ? w[2].x : w[1].w);
  return (int32_t)r >> 6;
}

template <int F>
__global__ void __launch_bounds__(kSelThreads, 1)
    select_kernel_c(const DNode *__restrict__ gtree, int n_top, const uint4 *__restrict__ blocks,
                    const float *__restrict__ X, int64_t m, int wide, int32_t *__restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  DNode *st = reinterpret_cast<DNode *>(smem);
  const int t = threadIdx.x;
  float *x = reinterpret_cast<float *>(smem + (size_t)kTopNodes * sizeof(DNode)) + t;  // column t
  for (int i = t; i < n_top; i += kSelThreads) st[i] = gtree[i];
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * kSelThreads;
  int64_t v = blockIdx.x * (int64_t)kSelThreads + t;
  float nx[F];
  if (v < m) load_vec<F>(X + v * F, wide, nx);
  for (; v < m; v += stride) {
#pragma unroll
    for (int f = 0; f < F; f++) x[f * kSelThreads] = nx[f];
    if (v + stride < m) load_vec<F>(X + (v + stride) * F, wide, nx);
    DNode nd = st[0];
    int ref = nd.meta;
    while (nd.meta >= 0) {
      const float xv = x[(nd.meta & 63) * kSelThreads];
      const int k = (nd.meta >> 6) + (xv <= nd.thr ? 0 : 1);  // NaN -> right (R8)
      if (k < n_top) {
        nd = st[k];
        ref = nd.meta;
      } else {
        ref = k - n_top;
        break;
      }
    }
    while (ref >= 0) {
      uint4 w[4];
      load_block(blocks, ref, w);
      ref = walk_block_col(w, x);
    }
    __stcs(out + v, -1 - ref);
  }
}

// one 2-level bottom block (32 B): returns the exit ref (>= 0 next block, < 0
// -1 - label)
template <int N>
__device__ __forceinline__ int walk_block2(const uint4 &a, const uint4 &b, const float (&x)[N]) {
  const bool g0 = !(pick<N>(x, a.w & 0xFF) <= __uint_as_float(a.x));  // NaN -> right (R8)
  const float t1 = __uint_as_float(g0 ? a.z : a.y);
  const bool g1 = !(pick<N>(x, (a.w >> (g0 ? 16 : 8)) & 0xFF) <= t1);
  const uint32_t r = g0 ? (g1 ? b.w : b.z) : (g1 ? b.y : b.x);
  return (int32_t)r;
}

// TD > 0: the heap depth at compile time (the full 14-level heap of deep
// trees such as C5's): the top walk unrolls completely
template <int F, int TD = 0>
__global__ void __launch_bounds__(kSelThreads, 1)
    select_kernel_h(const uint2 *__restrict__ gheap, const int32_t *__restrict__ gexits, int td_rt,
                    const uint4 *__restrict__ blocks2, const float *__restrict__ X, int64_t m, int wide,
                    int32_t *__restrict__ out) {
  const int td = TD > 0 ? TD : td_rt;
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int NP = F <= 4 ? 4 : (F <= 8 ? 8 : 16);
  const int nh = (1 << td) - 1;
  uint2 *hs = reinterpret_cast<uint2 *>(smem);
  int32_t *ex = reinterpret_cast<int32_t *>(smem + (size_t)nh * sizeof(uint2));
  const int t = threadIdx.x;
  for (int i = t; i < nh; i += kSelThreads) hs[i] = gheap[i];
  for (int i = t; i <= nh; i += kSelThreads) ex[i] = gexits[i];
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * kSelThreads;
  int64_t v = blockIdx.x * (int64_t)kSelThreads + t;
  float nx[F];
  if (v < m) load_vec<F>(X + v * F, wide, nx);
  for (; v < m; v += stride) {
    float xr[NP];
#pragma unroll
    for (int f = 0; f < NP; f++) xr[f] = f < F ? nx[f] : 0.f;
    if (v + stride < m) load_vec<F>(X + (v + stride) * F, wide, nx);  // next vector in flight
    uint32_t k = 0;
#pragma unroll (TD > 0 ? TD : 2)
    for (int l = 0; l < td; l++) {  // fixed trip count: leaves above td pass through
      const uint2 nd = hs[k];
      k = 2 * k + (pick<NP>(xr, nd.y) <= __uint_as_float(nd.x) ? 1u : 2u);
    }
    int ref = ex[k - nh];
    while (ref >= 0) {
      const uint4 *p = blocks2 + 2 * (int64_t)ref;
      uint4 a, b;
      asm("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
          : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
          : "l"(p));
      ref = walk_block2<NP>(a, b, xr);
    }
    __stcs(out + v, -1 - ref);
  }
}

// generic F (not a multiple of 4, or an unaligned X): scalar staging
__global__ void __launch_bounds__(kAnyThreads, 1)
    select_kernel_any(const DNode *__restrict__ gtree, int n_top, const uint4 *__restrict__ blocks,
                      const float *__restrict__ X,
                      int64_t m, int F, int32_t *__restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int stride = F | 1;
  DNode *st = reinterpret_cast<DNode *>(smem);
  float *sx = reinterpret_cast<float *>(smem + (size_t)kTopNodes * sizeof(DNode));
  const int t = threadIdx.x;
  for (int i = t; i < n_top; i += kAnyThreads) st[i] = gtree[i];
  for (int64_t v0 = blockIdx.x * (int64_t)kAnyThreads; v0 < m; v0 += (int64_t)gridDim.x * kAnyThreads) {
    const int rows = (m - v0 < kAnyThreads) ? (int)(m - v0) : kAnyThreads;
    __syncthreads();
    for (int i = t; i < rows * F; i += kAnyThreads) {
      const int r = i / F, c = i - r * F;
      sx[r * stride + c] = __ldcs(X + v0 * F + i);
    }
    __syncthreads();
    if (t < rows) {
      const float *x = sx + t * stride;
      DNode nd = st[0];
      int ref = nd.meta;
      while (nd.meta >= 0) {
        const int k = (nd.meta >> 6) + (x[nd.meta & 63] <= nd.thr ? 0 : 1);
        if (k < n_top) {
          nd = st[k];
          ref = nd.meta;
        } else {
          ref = k - n_top;
          break;
        }
      }
      while (ref >= 0) {
        uint4 w[4];
        load_block(blocks, ref, w);
        ref = walk_block(w, x);
      }
      __stcs(out + v0 + t, -1 - ref);
    }
  }
}

}  // namespace

void launch_select(const SelTree &tr, const float *X, int64_t m, int F, int32_t *out, cudaStream_t s) {
  if (m == 0) return;
  const DNode *tree = tr.top;
  const uint4 *blocks = tr.blocks;
  const int n_nodes = tr.n_nodes;
  const int n_top = std::min(n_nodes, kTopNodes);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool vec = (reinterpret_cast<uintptr_t>(X) & 15) == 0;
  const size_t tree_b = (size_t)kTopNodes * sizeof(DNode);
  const int wide = (reinterpret_cast<uintptr_t>(X) & 31) == 0;
  const int g = (int)std::min<int64_t>((m + kSelThreads - 1) / kSelThreads, sms);
  switch (vec ? F : 0) {
#define CASE(FF)                                                                                \
  case FF: {                                                                                    \
    if (n_nodes <= kTopNodes) {                                                                 \
      const size_t smem = tree_b + (size_t)kSelThreads * FF * 4;                                \
      smem_limit(select_kernel_c<FF>, smem);                                                    \
      select_kernel_c<FF><<<g, kSelThreads, smem, s>>>(tree, n_top, blocks, X, m, wide, out); ++g_kernel_launches;   \
    } else {                                                                                    \
      const size_t smem = ((size_t)1 << tr.td) * (sizeof(uint2) + 4);                           \
      if (tr.td == kHeapMaxLevels) {                                                            \
        smem_limit(select_kernel_h<FF, kHeapMaxLevels>, smem);                                  \
        select_kernel_h<FF, kHeapMaxLevels><<<g, kSelThreads, smem, s>>>(                       \
            tr.heap, tr.exits, tr.td, tr.blocks2, X, m, wide, out); ++g_kernel_launches;         \
      } else {                                                                                  \
        smem_limit(select_kernel_h<FF>, smem);                                                  \
        select_kernel_h<FF><<<g, kSelThreads, smem, s>>>(tr.heap, tr.exits, tr.td, tr.blocks2, X, m, \
                                                         wide, out); ++g_kernel_launches;                            \
      }                                                                                         \
    }                                                                                           \
    break;                                                                                      \
  }
    CASE(4) CASE(8) CASE(12) CASE(16)
#undef CASE
    default: {
      const size_t smem = tree_b + (size_t)kAnyThreads * (F | 1) * 4;
      const int64_t tiles = (m + kAnyThreads - 1) / kAnyThreads;
      const int grid = (int)std::min<int64_t>(tiles, sms);
      smem_limit(select_kernel_any, smem);
      select_kernel_any<<<grid, kAnyThreads, smem, s>>>(tree, n_top, blocks, X, m, F, out); ++g_kernel_launches;
    }
  }
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace adapt
