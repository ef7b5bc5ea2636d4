// select.cu — a9, batched variant selection (Table 1 get_policy, on many
// feature vectors at once): walk root -> leaf with x[f] <= thr -> left
// (S:224), NaN -> right (R8), output the leaf's variant.
//
// The device tree is a BFS array of 8-byte nodes; the threshold is stored as
// the largest float32 <= the double threshold, which makes the float compare
// exact (V:A5).  The product kernel is select_kernel_d (each lane loads its
// vector straight into registers; below); the tile kernels are kept for A/B
// (ADAPT_SEL_TILE / ADAPT_SEL_SMEMX).  The first kTopNodes nodes (the top levels every walk visits;
// a whole depth-12 tree) sit in shared memory; below them the tree is stored
// as 64-byte blocks of 3 levels (common.h), read with four independent
// 16-byte loads, so a depth-16 walk pays one L2 round trip below the top
// instead of four dependent ones.  Every warp owns its tiles of 64 vectors (no block barriers): the
// coalesced 16-byte loads of the next tile sit in registers while the lanes
// walk the current one out of the warp's odd-stride shared-memory tile, two
// independent walks per lane interleaved to hide the dependent smem latency.
#include <algorithm>
#include <cstdlib>

#include "common.h"
#include "vecreg.cuh"

namespace adapt {
namespace {

constexpr int kSelThreads = 1024;  // one CTA per SM: one smem copy of the tree
#ifndef ADAPT_SEL_CHAINS
#define ADAPT_SEL_CHAINS 2
#endif
constexpr int kSelChains = ADAPT_SEL_CHAINS;  // vectors walked at once per lane
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

template <int F>
__global__ void __launch_bounds__(kSelThreads, 1)
    select_kernel(const DNode *__restrict__ gtree, int n_top, const uint4 *__restrict__ blocks,
                  const float *__restrict__ X,
                  int64_t m, int32_t *__restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int kStride = F | 1;                   // odd row stride of a warp's tile
  constexpr int kVec = F / 4;                      // float4 per vector
  constexpr int kRows = 32 * kSelChains;           // vectors per warp tile
  constexpr int kLd = kRows * kVec / 32;           // float4 loads per lane per tile
  DNode *st = reinterpret_cast<DNode *>(smem);     // [n_top]
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  float *sx = reinterpret_cast<float *>(smem + (size_t)kTopNodes * sizeof(DNode)) +
              (size_t)warp * kRows * kStride;      // this warp's [kRows][kStride]
  for (int i = t; i < n_top; i += kSelThreads) st[i] = gtree[i];
  __syncthreads();  // the only block barrier: tree copy visible

  // warps own tiles of kRows vectors; no block barriers in the loop
  const int64_t ntiles = (m + kRows - 1) / kRows;
  const int64_t nwarps = (int64_t)gridDim.x * (kSelThreads / 32);
  float4 pre[kLd];
  auto fetch = [&](int64_t tile) {
    const int64_t v0 = tile * kRows;
    const int rows = (m - v0 < kRows) ? (int)(m - v0) : kRows;
    const float4 *src = reinterpret_cast<const float4 *>(X + v0 * F);
#pragma unroll
    for (int k = 0; k < kLd; k++) {
      const int i = lane + 32 * k;  // float4 index within the tile: coalesced
      pre[k] = i < rows * kVec ? __ldcs(src + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  int64_t tile = blockIdx.x * (int64_t)(kSelThreads / 32) + warp;
  if (tile < ntiles) fetch(tile);
  for (; tile < ntiles; tile += nwarps) {
    __syncwarp();  // previous tile's walks done before it is overwritten
#pragma unroll
    for (int k = 0; k < kLd; k++) {
      const int i = lane + 32 * k, r = i / kVec, c = (i % kVec) * 4;
      float *d = sx + r * kStride + c;
      d[0] = pre[k].x;
      d[1] = pre[k].y;
      d[2] = pre[k].z;
      d[3] = pre[k].w;
    }
    __syncwarp();
    if (tile + nwarps < ntiles) fetch(tile + nwarps);  // next tile in flight during the walks
    const int64_t v0 = tile * kRows;
    // kSelChains independent walks per lane, interleaved for latency hiding
    const float *x[kSelChains];
    DNode nd[kSelChains];
    int ref[kSelChains];  // -1 - label, or the bottom block the walk continues in
    bool live[kSelChains];
#pragma unroll
    for (int c = 0; c < kSelChains; c++) {
      x[c] = sx + (lane + 32 * c) * kStride;
      nd[c] = st[0];
      ref[c] = nd[c].meta;
      live[c] = v0 + lane + 32 * c < m;
    }
    bool any = true;
    while (any) {  // the shared-memory top
      any = false;
#pragma unroll
      for (int c = 0; c < kSelChains; c++) {
        if (nd[c].meta >= 0) {
          const float xv = x[c][nd[c].meta & 63];
          const int k = (nd[c].meta >> 6) + (xv <= nd[c].thr ? 0 : 1);
          if (k < n_top) {
            nd[c] = st[k];
            ref[c] = nd[c].meta;
            any |= nd[c].meta >= 0;
          } else {
            ref[c] = k - n_top;
            nd[c].meta = -1;
          }
        }
      }
    }
#pragma unroll
    for (int c = 0; c < kSelChains; c++)  // bottom blocks (the prefetched tile holds
      while (ref[c] >= 0) {               // registers: one chain's block at a time)
        uint4 w[4];
        load_block(blocks, ref[c], w);
        ref[c] = walk_block(w, x[c]);
      }
#pragma unroll
    for (int c = 0; c < kSelChains; c++)
      if (live[c]) __stcs(out + v0 + lane + 32 * c, -1 - ref[c]);
  }
}

template <int N>
__device__ __forceinline__ int walk_block_r(const uint4 (&w)[4], const float (&x)[N]) {
  const float t0 = __uint_as_float(w[0].x);
  const bool g0 = !(pick<N>(x, w[1].w & 63) <= t0);  // NaN -> right (R8)
  const float t1 = __uint_as_float(g0 ? w[0].z : w[0].y);
  const bool g1 = !(pick<N>(x, (g0 ? w[2].y : w[2].x) & 63) <= t1);
  const uint32_t tw = g0 ? (g1 ? w[1].z : w[1].y) : (g1 ? w[1].x : w[0].w);
  const uint32_t fw = g0 ? (g1 ? w[3].y : w[3].x) : (g1 ? w[2].w : w[2].z);
  const bool g2 = !(pick<N>(x, fw & 63) <= __uint_as_float(tw));
  uint32_t r;
  if (g0)
    r = g1 ? (g2 ? w[3].z : w[3].y) : (g2 ? w[3].x : w[2].w);
  else
    r = g1 ? (g2 ? w[2].z : w[2].y) : (g2 ? w[2].x : w[1].w);
  return (int32_t)r >> 6;
}

// One vector per lane, its features in REGISTERS: the walk reads only tree
// nodes from shared memory (the random-feature reads of the vector tile were
// half of the LSU wavefronts that bound the smem-x kernel above); the vector
// reaches registers through the same coalesced tile, one uniform-feature (so
// conflict-free) read per feature.
template <int F>
__global__ void __launch_bounds__(kSelThreads, 1)
    select_kernel_r(const DNode *__restrict__ gtree, int n_top, const uint4 *__restrict__ blocks,
                    const float *__restrict__ X, int64_t m, int32_t *__restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int kStride = F | 1;
  constexpr int kVec = F / 4;
  constexpr int kRows = 32;                // one vector per lane
  constexpr int kLd = kRows * kVec / 32;   // float4 loads per lane per tile
  constexpr int NP = F <= 4 ? 4 : (F <= 8 ? 8 : 16);
  DNode *st = reinterpret_cast<DNode *>(smem);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  float *sx = reinterpret_cast<float *>(smem + (size_t)kTopNodes * sizeof(DNode)) + (size_t)warp * kRows * kStride;
  for (int i = t; i < n_top; i += kSelThreads) st[i] = gtree[i];
  __syncthreads();
  const int64_t ntiles = (m + kRows - 1) / kRows;
  const int64_t nwarps = (int64_t)gridDim.x * (kSelThreads / 32);
  float4 pre[kLd];
  auto fetch = [&](int64_t tile) {
    const int64_t v0 = tile * kRows;
    const int rows = (m - v0 < kRows) ? (int)(m - v0) : kRows;
    const float4 *src = reinterpret_cast<const float4 *>(X + v0 * F);
#pragma unroll
    for (int k = 0; k < kLd; k++) {
      const int i = lane + 32 * k;
      pre[k] = i < rows * kVec ? __ldcs(src + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  int64_t tile = blockIdx.x * (int64_t)(kSelThreads / 32) + warp;
  if (tile < ntiles) fetch(tile);
  for (; tile < ntiles; tile += nwarps) {
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kLd; k++) {
      const int i = lane + 32 * k, r = i / kVec, c = (i % kVec) * 4;
      float *d = sx + r * kStride + c;
      d[0] = pre[k].x;
      d[1] = pre[k].y;
      d[2] = pre[k].z;
      d[3] = pre[k].w;
    }
    __syncwarp();
    float xr[NP];
#pragma unroll
    for (int f = 0; f < NP; f++) xr[f] = f < F ? sx[lane * kStride + f] : 0.f;
    if (tile + nwarps < ntiles) fetch(tile + nwarps);  // next tile in flight during the walk
    const int64_t v = tile * kRows + lane;
    DNode nd = st[0];
    int ref = nd.meta;
    while (nd.meta >= 0) {  // the shared-memory top
      const float xv = pick<NP>(xr, nd.meta & 63);
      const int k = (nd.meta >> 6) + (xv <= nd.thr ? 0 : 1);  // NaN -> right (R8)
      if (k < n_top) {
        nd = st[k];
        ref = nd.meta;
      } else {
        ref = k - n_top;
        break;
      }
    }
    while (ref >= 0) {  // bottom blocks
      uint4 w[4];
      load_block(blocks, ref, w);
      ref = walk_block_r<NP>(w, xr);
    }
    if (v < m) __stcs(out + v, -1 - ref);
  }
}

// As select_kernel_r, but every lane loads its own vector straight into
// registers (256-bit loads when the rows are 32-byte aligned): no staging tile,
// no shared-memory stores or feature reads at all; the next vector's loads are
// in flight during the walk.
template <int F>
__global__ void __launch_bounds__(kSelThreads, 1)
    select_kernel_d(const DNode *__restrict__ gtree, int n_top, const uint4 *__restrict__ blocks,
                    const float *__restrict__ X, int64_t m, int wide, int32_t *__restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int NP = F <= 4 ? 4 : (F <= 8 ? 8 : 16);
  DNode *st = reinterpret_cast<DNode *>(smem);
  const int t = threadIdx.x;
  for (int i = t; i < n_top; i += kSelThreads) st[i] = gtree[i];
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
    DNode nd = st[0];
    int ref = nd.meta;
    while (nd.meta >= 0) {
      const float xv = pick<NP>(xr, nd.meta & 63);
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
      ref = walk_block_r<NP>(w, xr);
    }
    __stcs(out + v, -1 - ref);
  }
}

// As select_kernel_d, but the vector parked in the thread's own shared-memory
// COLUMN (xs[f][tid]: any f of any lane is a distinct bank, so the walk's
// random-feature reads are conflict-free single wavefronts) instead of the
// register select tree (A/B: ADAPT_SEL_XCOL=1).
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

void launch_select(const DNode *tree, int n_nodes, const uint4 *blocks, const float *X, int64_t m,
                   int F, int32_t *out, cudaStream_t s) {
  if (m == 0) return;
  const int n_top = std::min(n_nodes, kTopNodes);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool vec = (reinterpret_cast<uintptr_t>(X) & 15) == 0;
  static const bool smem_x = getenv("ADAPT_SEL_SMEMX") != nullptr;  // the smem-x kernel (A/B)
  // default: per-lane vector loads (select_kernel_d); A/B: the tile kernels
  static const bool direct = getenv("ADAPT_SEL_TILE") == nullptr && !smem_x;
  // trees that fit the shared-memory top: the vector in a shared-memory column
  // (C4 select 1.40 -> 1.15 ms); deeper trees: the register kernel, whose
  // bottom-block walks measured faster with the vector in registers (C5)
  static const int xcol_env = getenv("ADAPT_SEL_XCOL") ? atoi(getenv("ADAPT_SEL_XCOL")) : -1;
  const bool xcol = direct && (xcol_env >= 0 ? xcol_env != 0 : n_nodes <= kTopNodes);
  const size_t tree_b = (size_t)kTopNodes * sizeof(DNode);
  // F <= 16, 16-byte aligned X: per-warp tiles, one 1024-thread CTA per SM
  const int64_t wtiles = (m + 32 * kSelChains - 1) / (32 * kSelChains);
  const int vgrid = (int)std::min<int64_t>((wtiles + kSelThreads / 32 - 1) / (kSelThreads / 32), sms);
  switch (vec ? F : 0) {
#define CASE(FF)                                                                               \
  case FF: {                                                                                   \
    if (xcol) {                                                                                \
      const int wide = (reinterpret_cast<uintptr_t>(X) & 31) == 0;                             \
      const int64_t blocks_needed = (m + kSelThreads - 1) / kSelThreads;                       \
      const int g = (int)std::min<int64_t>(blocks_needed, sms);                                \
      const size_t smem = tree_b + (size_t)kSelThreads * FF * 4;                               \
      smem_limit(select_kernel_c<FF>, smem);                                                   \
      select_kernel_c<FF><<<g, kSelThreads, smem, s>>>(tree, n_top, blocks, X, m, wide, out);  \
    } else if (direct) {                                                                       \
      const int wide = (reinterpret_cast<uintptr_t>(X) & 31) == 0;                             \
      const int64_t blocks_needed = (m + kSelThreads - 1) / kSelThreads;                       \
      const int g = (int)std::min<int64_t>(blocks_needed, sms);                                \
      smem_limit(select_kernel_d<FF>, tree_b);                                                 \
      select_kernel_d<FF><<<g, kSelThreads, tree_b, s>>>(tree, n_top, blocks, X, m, wide, out); \
    } else if (smem_x) {                                                                       \
      const size_t smem = tree_b + (size_t)kSelThreads * kSelChains * (FF | 1) * 4;            \
      smem_limit(select_kernel<FF>, smem);                                                     \
      select_kernel<FF><<<vgrid, kSelThreads, smem, s>>>(tree, n_top, blocks, X, m, out);      \
    } else {                                                                                   \
      const size_t smem = tree_b + (size_t)kSelThreads * (FF | 1) * 4;                         \
      const int64_t tiles = (m + 31) / 32;                                                     \
      const int g = (int)std::min<int64_t>((tiles + kSelThreads / 32 - 1) / (kSelThreads / 32), sms); \
      smem_limit(select_kernel_r<FF>, smem);                                                   \
      select_kernel_r<FF><<<g, kSelThreads, smem, s>>>(tree, n_top, blocks, X, m, out);        \
    }                                                                                          \
    break;                                                                                     \
  }
    CASE(4) CASE(8) CASE(12) CASE(16)
#undef CASE
    default: {
      const size_t smem = tree_b + (size_t)kAnyThreads * (F | 1) * 4;
      const int64_t tiles = (m + kAnyThreads - 1) / kAnyThreads;
      const int grid = (int)std::min<int64_t>(tiles, sms);
      smem_limit(select_kernel_any, smem);
      select_kernel_any<<<grid, kAnyThreads, smem, s>>>(tree, n_top, blocks, X, m, F, out);
    }
  }
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace adapt
