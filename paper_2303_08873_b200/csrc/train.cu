// train.cu — the level-wise CART trainer's kernels.
//
// The histogram-side kernels of one tree level (the row passes are in level.cu):
//   zero_slots_kernel the direct nodes' histograms before the row pass;
//   subtract_kernel   the other ("derived") child = parent - direct sibling
//                     (exact integer histogram subtraction, class-remapped:
//                     every node is stored in its own class compaction);
//   split_kernel      a6 per (node, feature): class-chunked block prefix scan
//                     over bins, exact rational Gini score of every cut
//                     between consecutive node-nonempty bins, block argmax;
//   winner_kernel     per node: best feature (ties -> lowest f), plus the class
//                     totals of the node and of the winning left child.
// Every quantity that decides the tree is an integer, so the result does not
// depend on row order, on the number of ranks or on atomic ordering.
#include <algorithm>

#include "common.h"

namespace adapt {
namespace {

constexpr unsigned kFull = 0xffffffffu;

// Per-node matrix jobs are cut into chunks of kChunk elements; block b handles
// chunk b of the flattened list (job found by binary search over the chunk
// prefix), so deep levels with thousands of small nodes launch no idle blocks.
constexpr int kChunk = 4096, kChunkThreads = 256;

__device__ __forceinline__ int find_job(const int32_t *cstart, int n, int b) {
  int lo = 0, hi = n - 1;  // last job with cstart[job] <= b
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (cstart[mid] <= b) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// slots 0..n-1 (the direct nodes): zero their [DS][kc] matrices
__global__ void __launch_bounds__(kChunkThreads)
    zero_slots_kernel(uint32_t *H, const int64_t *soff, const int32_t *skc, int64_t DS,
                      const int32_t *cstart, int n, const int32_t *zslot) {
  const int job = find_job(cstart, n, blockIdx.x);
  const int y = zslot ? zslot[job] : job;  // job -> slot (null: job = slot)
  uint32_t *h = H + soff[y];
  const int64_t E = DS * skc[y];
  const int64_t i0 = (int64_t)(blockIdx.x - cstart[job]) * kChunk;
  const int64_t i1 = min(i0 + kChunk, E);
  for (int64_t i = i0 + threadIdx.x; i < i1; i += kChunkThreads) h[i] = 0;
}

// derived = parent - direct sibling (exact), each in its own class compaction:
// derived column j = parent column map[j].x minus sibling column map[j].y (-1: 0)
__global__ void __launch_bounds__(kChunkThreads)
    subtract_kernel(uint32_t *H, const uint32_t *Hprev, int64_t DS, const SubJob *jobs,
                    const int16_t *maps, const int32_t *cstart, int n) {
  const int y = find_job(cstart, n, blockIdx.x);
  const SubJob jb = jobs[y];
  const short2 *m = reinterpret_cast<const short2 *>(maps) + jb.map;
  uint32_t *d = H + jb.off_d;
  const uint32_t *p = Hprev + jb.off_p;
  const uint32_t *q = H + jb.off_s;
  const int64_t E = DS * jb.kc_d;
  const int64_t i0 = (int64_t)(blockIdx.x - cstart[y]) * kChunk;
  const int64_t i1 = min(i0 + kChunk, E);
  // element i = r * kc_d + j (i < 2^31: a node matrix is DS x kc <= 16384 x 255),
  // advanced by kChunkThreads per step without a division
  const int kcd = jb.kc_d;
  const int dq = kChunkThreads / kcd, dr = kChunkThreads - dq * kcd;
  int r = (int)((i0 + threadIdx.x) / kcd), j = (int)(i0 + threadIdx.x - (int64_t)r * kcd);
  // kSubUnroll elements per thread per step, every load issued before the
  // first subtraction (the element loop is latency-bound otherwise)
  constexpr int kSubUnroll = 4;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += kSubUnroll * kChunkThreads) {
    int rr[kSubUnroll], jj[kSubUnroll];
#pragma unroll
    for (int u = 0; u < kSubUnroll; u++) {
      rr[u] = r;
      jj[u] = j;
      r += dq;
      j += dr;
      if (j >= kcd) {
        j -= kcd;
        r++;
      }
    }
    uint32_t pv[kSubUnroll], sv[kSubUnroll];
#pragma unroll
    for (int u = 0; u < kSubUnroll; u++) {
      pv[u] = 0;
      sv[u] = 0;
      if (i + u * kChunkThreads < i1) {
        const short2 mj = m[jj[u]];
        sv[u] = mj.y >= 0 ? q[(int64_t)rr[u] * jb.kc_s + mj.y] : 0u;
        pv[u] = p[(int64_t)rr[u] * jb.kc_p + mj.x];
      }
    }
#pragma unroll
    for (int u = 0; u < kSubUnroll; u++)
      if (i + u * kChunkThreads < i1) d[i + u * kChunkThreads] = pv[u] - sv[u];
  }
}

// ---- exact comparison of scores num/den (num < 2^97, den < 2^64) ----
struct Key {
  uint64_t hi, lo, den;
  int idx;     // bin rank (split) or feature (winner): lower wins ties
  int valid;
};

__device__ __forceinline__ void mul128x64(uint64_t hi, uint64_t lo, uint64_t d, uint64_t &w2,
                                          uint64_t &w1, uint64_t &w0) {
  w0 = lo * d;
  const uint64_t a = __umul64hi(lo, d);
  const uint64_t b = hi * d;
  const uint64_t c = __umul64hi(hi, d);
  w1 = a + b;
  w2 = c + (w1 < a ? 1 : 0);
}

// true if x is strictly better than y: valid first, larger score, then lower idx
__device__ __forceinline__ bool better(const Key &x, const Key &y) {
  if (x.valid != y.valid) return x.valid > y.valid;
  if (!x.valid) return x.idx < y.idx;
  uint64_t a2, a1, a0, b2, b1, b0;
  mul128x64(x.hi, x.lo, y.den, a2, a1, a0);  // x.num * y.den
  mul128x64(y.hi, y.lo, x.den, b2, b1, b0);  // y.num * x.den
  if (a2 != b2) return a2 > b2;
  if (a1 != b1) return a1 > b1;
  if (a0 != b0) return a0 > b0;
  return x.idx < y.idx;
}

__device__ __forceinline__ Key shfl_key(const Key &k, int src) {
  Key o;
  o.hi = __shfl_sync(kFull, k.hi, src);
  o.lo = __shfl_sync(kFull, k.lo, src);
  o.den = __shfl_sync(kFull, k.den, src);
  o.idx = __shfl_sync(kFull, k.idx, src);
  o.valid = __shfl_sync(kFull, k.valid, src);
  return o;
}

constexpr int kSplitThreads = 256;  // = max bins per feature
constexpr int kClassChunk = 32;

__global__ void __launch_bounds__(kSplitThreads)
    split_kernel(const uint32_t *__restrict__ H, const int64_t *node_off, const int32_t *node_kc,
                 const int32_t *nodes, int F, const int32_t *cumD, const int32_t *nval,
                 SplitCand *out) {
  __shared__ uint32_t tile[kSplitThreads][kClassChunk + 1];
  __shared__ uint32_t segtot[kSplitThreads / 32][kClassChunk];
  __shared__ uint32_t Pk[kClassChunk];
  __shared__ uint64_t nLs[kSplitThreads];
  __shared__ uint32_t nonempty[kSplitThreads / 32];
  __shared__ Key wbest[kSplitThreads / 32];

  const int node = nodes[blockIdx.x], f = blockIdx.y;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int Df = nval[f];
  const int C = node_kc[node];  // the node's classes (compact columns)
  const uint32_t *h = H + node_off[node] + (int64_t)cumD[f] * C;
  uint64_t nl = 0, sl = 0, sr = 0, ntot = 0;
  for (int c0 = 0; c0 < C; c0 += kClassChunk) {
    const int kc = min(kClassChunk, C - c0);
    {  // the chunk's Df x kc counts, flat over all threads: independent loads in
       // flight (contiguous when the node has <= kClassChunk classes)
      const int E = Df * kc;
      const uint32_t tbase = (uint32_t)__cvta_generic_to_shared(&tile[0][0]);
      // element e = r * kc + k, advanced by kSplitThreads per step without a
      // division (r += dq, k += dr, carry)
      const int dq = kSplitThreads / kc, dr = kSplitThreads - dq * kc;
      int r = t / kc, k = t - r * kc;
      for (int e = t; e < E; e += kSplitThreads) {  // async copies: all in flight at once
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                         tbase + 4u * (uint32_t)(r * (kClassChunk + 1) + k)),
                     "l"(h + (size_t)r * C + c0 + k)
                     : "memory");
        r += dq;
        k += dr;
        if (k >= kc) {
          k -= kc;
          r++;
        }
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    }
    __syncthreads();
    // prefix over bins: warp w scans rows [32w, 32w+32) of column `lane`
    const int r0 = w * 32, r1 = min(r0 + 32, Df);
    if (lane < kc) {
      uint32_t acc = 0;
      for (int r = r0; r < r1; r++) {
        acc += tile[r][lane];
        tile[r][lane] = acc;
      }
      segtot[w][lane] = acc;
    }
    __syncthreads();
    if (lane < kc) {
      uint32_t off = 0, tot = 0;
      for (int v = 0; v < kSplitThreads / 32; v++) {
        const uint32_t x = segtot[v][lane];
        if (v < w) off += x;
        tot += x;
      }
      for (int r = r0; r < r1; r++) tile[r][lane] += off;
      if (w == 0) Pk[lane] = tot;
    }
    __syncthreads();
    for (int k = 0; k < kc; k++) ntot += Pk[k];
    if (t < Df) {
      for (int k = 0; k < kc; k++) {
        const uint64_t c = tile[t][k];
        const uint64_t cr = (uint64_t)Pk[k] - c;
        nl += c;
        sl += c * c;
        sr += cr * cr;
      }
    }
    __syncthreads();
  }
  if (t < Df) nLs[t] = nl;
  __syncthreads();
  const uint64_t cnt = t < Df ? nl - (t > 0 ? nLs[t - 1] : 0) : 0;
  const unsigned ne = __ballot_sync(kFull, cnt > 0);
  if (lane == 0) nonempty[w] = ne;
  __syncthreads();
  Key k;
  k.valid = 0;
  k.idx = t;
  k.hi = k.lo = 0;
  k.den = 1;
  int b_hi = -1;
  if (t < Df && cnt > 0 && nl < ntot) {
    // next node-nonempty bin after t
    unsigned m = nonempty[w] & (lane == 31 ? 0u : (kFull << (lane + 1)));
    int ww = w;
    while (!m && ++ww < kSplitThreads / 32) m = nonempty[ww];
    b_hi = ww * 32 + __ffs(m) - 1;
    const uint64_t nR = ntot - nl;
    // num = sl*nR + sr*nl  (128-bit)
    const uint64_t x0 = sl * nR, x1 = __umul64hi(sl, nR);
    const uint64_t y0 = sr * nl, y1 = __umul64hi(sr, nl);
    k.lo = x0 + y0;
    k.hi = x1 + y1 + (k.lo < x0 ? 1 : 0);
    k.den = nl * nR;
    k.valid = 1;
  }
  // block argmax (ties -> lowest bin rank = lowest threshold)
  Key best = k;
  int best_hi = b_hi;
  uint64_t best_nl = nl;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const Key other = shfl_key(best, lane ^ o);
    const int oh = __shfl_sync(kFull, best_hi, lane ^ o);
    const uint64_t on = __shfl_sync(kFull, best_nl, lane ^ o);
    if (better(other, best)) {
      best = other;
      best_hi = oh;
      best_nl = on;
    }
  }
  __shared__ int whi[kSplitThreads / 32];
  __shared__ uint64_t wnl[kSplitThreads / 32];
  if (lane == 0) {
    wbest[w] = best;
    whi[w] = best_hi;
    wnl[w] = best_nl;
  }
  __syncthreads();
  if (t == 0) {
    Key b = wbest[0];
    int bh = whi[0];
    uint64_t bn = wnl[0];
    for (int v = 1; v < kSplitThreads / 32; v++)
      if (better(wbest[v], b)) {
        b = wbest[v];
        bh = whi[v];
        bn = wnl[v];
      }
    SplitCand c;
    c.num_lo = b.lo;
    c.num_hi = b.hi;
    c.den = b.den;
    c.nL = bn;
    c.valid = b.valid;
    c.b_lo = b.idx;
    c.b_hi = bh;
    c.pad = 0;
    out[(size_t)node * F + f] = c;
  }
}

// Nodes with at most kSmallKc classes (most nodes of deep levels): one WARP per
// (node, feature).  The Df x kc counts are staged coalesced into the warp's
// smem tile (bin b at b*kc + b/8: one pad word per 8-bin lane segment, so the
// lanes' segment walks hit distinct banks); lane l owns bins [8l, 8l+8):
// per-class segment sums, warp scans for the prefix offsets and class totals,
// then the same candidate keys, tie rules and exact comparison as split_kernel.
constexpr int kSmallKc = 8;
constexpr int kSmallWarps = 4;

__global__ void __launch_bounds__(kSmallWarps * 32)
    split_small_kernel(const uint32_t *__restrict__ H, const int64_t *node_off,
                       const int32_t *node_kc, const int32_t *nodes, int njobs, int F,
                       const int32_t *cumD, const int32_t *nval, SplitCand *out) {
  __shared__ uint32_t wt[kSmallWarps][kSplitThreads * kSmallKc + 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int job = blockIdx.x * kSmallWarps + warp;
  if (job >= njobs) return;  // warp-uniform; no block barriers below
  const int node = nodes[job / F], f = job % F;
  const int kc = node_kc[node], Df = nval[f];
  const uint32_t *h = H + node_off[node] + (int64_t)cumD[f] * kc;
  uint32_t *tl = wt[warp];
  {  // asynchronous 4-byte copies (no registers held): every load in flight at once
    const int E = Df * kc;
    const float inv = 1.0f / (float)kc;  // exact enough: e < 2048, kc <= 8
    const uint32_t tbase = (uint32_t)__cvta_generic_to_shared(tl);
    for (int e = lane; e < E; e += 32) {
      const int b = __float2int_rz(((float)e + 0.5f) * inv);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(tbase + 4u * (e + (b >> 3))),
                   "l"(h + e)
                   : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  __syncwarp();
  const int b0 = lane * 8;
  const uint32_t *sg = tl + b0 * kc + lane;  // this lane's 8 bins (after lane pad words)
  uint32_t acc[kSmallKc];
  uint32_t bc[8];  // bin counts
#pragma unroll
  for (int k = 0; k < kSmallKc; k++) acc[k] = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < kSmallKc; k++)
      if (k < kc && b0 + i < Df) {
        const uint32_t v = sg[i * kc + k];
        acc[k] += v;
        c += v;
      }
    bc[i] = c;
  }
  uint32_t off[kSmallKc], tot[kSmallKc];
  uint64_t ntot = 0;
#pragma unroll
  for (int k = 0; k < kSmallKc; k++) {
    uint32_t x = acc[k];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    tot[k] = __shfl_sync(kFull, x, 31);
    off[k] = x - acc[k];
    if (k < kc) ntot += tot[k];
  }
  // first node-nonempty bin of this lane, and of the lanes after it
  int first_ne = -1;
#pragma unroll
  for (int i = 7; i >= 0; i--)
    if (bc[i]) first_ne = b0 + i;
  const unsigned has = __ballot_sync(kFull, first_ne >= 0);
  const unsigned later = lane == 31 ? 0u : has & (kFull << (lane + 1));
  const int nf = __shfl_sync(kFull, first_ne, later ? __ffs(later) - 1 : lane);
  int nextb[8];
  {
    int nx = later ? nf : -1;
#pragma unroll
    for (int i = 7; i >= 0; i--) {
      nextb[i] = nx;
      if (bc[i]) nx = b0 + i;
    }
  }
  Key best;
  best.valid = 0;
  best.idx = b0;
  best.hi = best.lo = 0;
  best.den = 1;
  int best_hi = -1;
  uint64_t best_nl = 0;
  uint32_t cl[kSmallKc];
#pragma unroll
  for (int k = 0; k < kSmallKc; k++) cl[k] = off[k];
#pragma unroll
  for (int i = 0; i < 8; i++) {
    uint64_t nl = 0, sl = 0, sr = 0;
#pragma unroll
    for (int k = 0; k < kSmallKc; k++)
      if (k < kc && b0 + i < Df) {
        cl[k] += sg[i * kc + k];
        const uint64_t c = cl[k], r = (uint64_t)tot[k] - cl[k];
        nl += c;
        sl += c * c;
        sr += r * r;
      }
    if (b0 + i < Df && bc[i] > 0 && nl < ntot) {
      const uint64_t nR = ntot - nl;
      Key k;
      const uint64_t x0 = sl * nR, x1 = __umul64hi(sl, nR);
      const uint64_t y0 = sr * nl, y1 = __umul64hi(sr, nl);
      k.lo = x0 + y0;
      k.hi = x1 + y1 + (k.lo < x0 ? 1 : 0);
      k.den = nl * nR;
      k.valid = 1;
      k.idx = b0 + i;
      if (better(k, best)) {  // ascending bins: ties keep the lower one
        best = k;
        best_hi = nextb[i];
        best_nl = nl;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const Key other = shfl_key(best, lane ^ o);
    const int oh = __shfl_sync(kFull, best_hi, lane ^ o);
    const uint64_t on = __shfl_sync(kFull, best_nl, lane ^ o);
    if (better(other, best)) {
      best = other;
      best_hi = oh;
      best_nl = on;
    }
  }
  if (lane == 0) {
    SplitCand c;
    c.num_lo = best.lo;
    c.num_hi = best.hi;
    c.den = best.den;
    c.nL = best_nl;
    c.valid = best.valid;
    c.b_lo = best.valid ? best.idx : -1;
    c.b_hi = best.valid ? best_hi : -1;
    c.pad = 0;
    out[(size_t)node * F + f] = c;
  }
}

__global__ void __launch_bounds__(256)
    winner_kernel(const uint32_t *__restrict__ H, const int64_t *node_off, const int32_t *node_kc,
                  int F, int Cmax, const int32_t *cumD, const int32_t *nval, const SplitCand *cand,
                  uint8_t *res, const int64_t *res_off) {
  __shared__ int s_f;
  __shared__ SplitCand s_c;
  __shared__ unsigned long long s_n;
  const int node = blockIdx.x, t = threadIdx.x;
  __shared__ SplitCand sc[kMaxF];  // the node's F candidates, loaded in parallel
  for (int f = t; f < F; f += blockDim.x) sc[f] = cand[(size_t)node * F + f];
  __syncthreads();
  if (t < 32) {  // warp argmax over the F candidates (ties -> lowest feature)
    Key bk;
    bk.valid = 0;
    bk.idx = 0x7fffffff;
    bk.hi = bk.lo = 0;
    bk.den = 1;
    for (int f = t; f < F; f += 32) {
      const SplitCand &c = sc[f];
      Key k;
      k.valid = c.valid;
      k.idx = f;
      k.hi = c.num_hi;
      k.lo = c.num_lo;
      k.den = c.den;
      if (k.valid && better(k, bk)) bk = k;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const Key other = shfl_key(bk, t ^ o);
      if (better(other, bk)) bk = other;
    }
    if (t == 0) {
      const int bf = bk.valid ? bk.idx : -1;
      s_f = bf;
      if (bf >= 0) s_c = sc[bf];
      s_n = 0;
    }
  }
  __syncthreads();
  const int fsel = s_f >= 0 ? s_f : 0;
  const int blo = s_f >= 0 ? s_c.b_lo : -1;
  const int C = node_kc[node];
  const uint32_t *h = H + node_off[node] + (int64_t)cumD[fsel] * C;
  const int Df = nval[fsel];
  NodeRes *nr = reinterpret_cast<NodeRes *>(res + res_off[node]);
  uint32_t *P = reinterpret_cast<uint32_t *>(nr + 1);
  uint32_t *cL = P + C;  // compact: the node's own class count
  // class totals and left-of-cut totals: thread t sums class t % C over rows
  // t / C, t / C + T, ... (T = threads per class), independent loads in flight
  __shared__ uint32_t sP[kMaxC + 1], sL[kMaxC + 1];
  for (int k = t; k < C; k += blockDim.x) sP[k] = sL[k] = 0;
  __syncthreads();
  if (C <= (int)blockDim.x) {
    const int T = blockDim.x / C, k = t % C, r0 = t / C;
    if (r0 < T) {
      uint32_t tot = 0, left = 0;
#pragma unroll 4
      for (int r = r0; r < Df; r += T) {
        const uint32_t v = __ldg(h + (size_t)r * C + k);
        tot += v;
        left += r <= blo ? v : 0u;
      }
      atomicAdd(&sP[k], tot);
      atomicAdd(&sL[k], left);
    }
  }
  __syncthreads();
  for (int k = t; k < C; k += blockDim.x) {
    P[k] = sP[k];
    cL[k] = sL[k];
    atomicAdd(&s_n, (unsigned long long)sP[k]);
  }
  __syncthreads();
  if (t == 0) {
    nr->n = s_n;
    nr->valid = s_f >= 0;
    nr->feat = s_f;
    nr->nL = s_f >= 0 ? s_c.nL : 0;
    nr->b_lo = s_f >= 0 ? s_c.b_lo : -1;
    nr->b_hi = s_f >= 0 ? s_c.b_hi : -1;
  }
}

}  // namespace

int chunk_count(int64_t elems) { return (int)((elems + kChunk - 1) / kChunk); }

void launch_zero_slots(uint32_t *H, const int64_t *soff, const int32_t *skc, int64_t DS,
                       const int32_t *cstart, int n, int nblocks, cudaStream_t s, const int32_t *zslot) {
  if (n == 0 || nblocks == 0) return;
  zero_slots_kernel<<<nblocks, kChunkThreads, 0, s>>>(H, soff, skc, DS, cstart, n, zslot); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
}

void launch_subtract(uint32_t *H, const uint32_t *Hprev, int64_t DS, const SubJob *jobs,
                     const int16_t *maps, const int32_t *cstart, int n, int nblocks, cudaStream_t s) {
  if (n == 0 || nblocks == 0) return;
  subtract_kernel<<<nblocks, kChunkThreads, 0, s>>>(H, Hprev, DS, jobs, maps, cstart, n); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
}

void launch_split(const uint32_t *H, const int64_t *node_off, const int32_t *node_kc,
                  const int32_t *big_nodes, int nbig, const int32_t *small_nodes, int nsmall,
                  int F, const int32_t *cumD, const int32_t *nval, SplitCand *out, cudaStream_t s) {
  if (nbig > 0) {
    split_kernel<<<dim3(nbig, F), kSplitThreads, 0, s>>>(H, node_off, node_kc, big_nodes, F, cumD,
                                                         nval, out); ++g_kernel_launches;
    CUDA_CHECK(cudaGetLastError());
  }
  if (nsmall > 0) {
    const int njobs = nsmall * F;
    split_small_kernel<<<(njobs + kSmallWarps - 1) / kSmallWarps, kSmallWarps * 32, 0, s>>>(
        H, node_off, node_kc, small_nodes, njobs, F, cumD, nval, out); ++g_kernel_launches;
    CUDA_CHECK(cudaGetLastError());
  }
}

int split_small_max_classes() { return kSmallKc; }

void launch_winner(const uint32_t *H, const int64_t *node_off, const int32_t *node_kc, int nnodes,
                   int F, int C, const int32_t *cumD, const int32_t *nval, const SplitCand *cand,
                   uint8_t *res, const int64_t *res_off, cudaStream_t s) {
  if (nnodes == 0) return;
  winner_kernel<<<nnodes, 256, 0, s>>>(H, node_off, node_kc, F, C, cumD, nval, cand, res,
                                       res_off); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace adapt
