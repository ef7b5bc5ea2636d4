// train.cu — the level-wise CART trainer's kernels.
//
// One tree level = one pass over the rows of the nodes being split:
//   hist_pass_kernel  a7 partition of the previous level's splits (the rows of
//                     a parent span are moved — coalesced reads, warp-contiguous
//                     writes — into the children's spans, left from the front,
//                     right from the back) fused with a4, the
//                     class histogram H[node][f][rank][class] of ONE child per
//                     parent (the smaller, "direct" one), privatised in shared
//                     memory and flushed with integer atomics;
//   subtract_kernel   the other ("derived") child = parent - direct sibling
//                     (exact integer histogram subtraction);
//   split_kernel      a6 per (node, feature): class-chunked block prefix scan
//                     over bins, exact rational Gini score of every cut
//                     between consecutive node-nonempty bins, block argmax;
//   winner_kernel     per node: best feature (ties -> lowest f), plus the class
//                     totals of the node and of the winning left child.
// Every quantity that decides the tree is an integer, so the result does not
// depend on row order, on the number of ranks or on atomic ordering.
#include "common.h"
#include "ptx.h"

namespace adapt {
namespace {

constexpr int kHistThreads = 1024;
constexpr unsigned kFull = 0xffffffffu;

template <int BS>
struct Row {  // one row's bins, BS bytes, in registers
  static constexpr int N = BS >= 4 ? BS / 4 : 1;
  uint32_t w[N];
};

template <int BS>
__device__ __forceinline__ void load_row(const uint8_t *__restrict__ p, Row<BS> &r) {
  if constexpr (BS >= 16) {
#pragma unroll
    for (int i = 0; i < BS / 16; i++) {
      const uint4 v = *(reinterpret_cast<const uint4 *>(p) + i);
      r.w[4 * i + 0] = v.x;
      r.w[4 * i + 1] = v.y;
      r.w[4 * i + 2] = v.z;
      r.w[4 * i + 3] = v.w;
    }
  } else if constexpr (BS == 8) {
    const uint2 v = *reinterpret_cast<const uint2 *>(p);
    r.w[0] = v.x;
    r.w[1] = v.y;
  } else if constexpr (BS == 4) {
    r.w[0] = *reinterpret_cast<const unsigned int *>(p);
  } else if constexpr (BS == 2) {
    r.w[0] = *reinterpret_cast<const unsigned short *>(p);
  } else {
    r.w[0] = *p;
  }
}

template <int BS>
__device__ __forceinline__ void store_row(uint8_t *__restrict__ p, const Row<BS> &r) {
  if constexpr (BS >= 16) {
#pragma unroll
    for (int i = 0; i < BS / 16; i++)
      __stcs(reinterpret_cast<uint4 *>(p) + i,
             make_uint4(r.w[4 * i], r.w[4 * i + 1], r.w[4 * i + 2], r.w[4 * i + 3]));
  } else if constexpr (BS == 8) {
    __stcs(reinterpret_cast<uint2 *>(p), make_uint2(r.w[0], r.w[1]));
  } else if constexpr (BS == 4) {
    __stcs(reinterpret_cast<unsigned int *>(p), r.w[0]);
  } else if constexpr (BS == 2) {
    *reinterpret_cast<unsigned short *>(p) = (unsigned short)r.w[0];
  } else {
    *p = (uint8_t)r.w[0];
  }
}

// select w[i] for a runtime i with a tree of register selects (N = power of 2);
// every array access has a compile-time index, so nothing spills to local memory
template <int N>
__device__ __forceinline__ uint32_t pick(const uint32_t *w, int i) {
  if constexpr (N == 1) {
    return w[0];
  } else {
    constexpr int H = N / 2;
    const uint32_t lo = pick<H>(w, i & (H - 1));
    const uint32_t hi = pick<H>(w + H, i & (H - 1));
    return (i & H) ? hi : lo;
  }
}

template <int BS>
__device__ __forceinline__ int row_byte(const Row<BS> &r, int f) {
  return (int)((pick<Row<BS>::N>(r.w, f >> 2) >> (8 * (f & 3))) & 0xFFu);
}

constexpr int kUnroll = 4;  // rows per thread per iteration (memory-level parallelism)

__device__ __forceinline__ void red_shared_inc(uint32_t addr) {
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// One level pass.  The G CTAs of a "range" (consecutive blockIdx.x, all
// co-resident: one CTA per SM, launched cooperatively) walk the same
// contiguous range of row positions.  CTA g histograms the 4 features of
// 32-bit word w(g) of the bins row for the class slab [k0, k0+kw) — at most 4
// shared-memory atomics per row — and moves the rows of its own contiguous
// G-th of every segment portion into the children's pieces (a7): left rows
// from the front of that sub-portion, right rows from its back, positions
// from shared-memory cursors (no global atomics, no block barriers).  Each
// CTA reports (segment, sub-portion, left/right counts), from which the host
// builds the next level's pieces.  The G CTAs re-synchronise through a
// global counter every kSyncEvery iterations so that a row fetched from HBM
// by one of them is still in L2 for the others.  Counters are indexed by
// PROVISIONAL bin id with an odd class stride; the id -> rank map is applied
// once per counter when a node's histogram is flushed.
constexpr int kSyncEvery = 8;

template <int BS>
__global__ void __launch_bounds__(kHistThreads, 1) hist_pass_kernel(HistPassArgs a) {
  extern __shared__ uint32_t sh[];  // [smem_counters] counters | lut [F*256] bytes
  uint8_t *slut = reinterpret_cast<uint8_t *>(sh + a.smem_counters);
  __shared__ int32_t soff[kMaxF];   // this group's smem offset of feature f, -1 if absent
  __shared__ int32_t sdf[kMaxF];    // distinct values of f
  __shared__ uint32_t s_cur[2];     // left / right cursors of this CTA's sub-portion
  const int tid = threadIdx.x, lane = tid & 31;
  const int G = a.ngroups;
  const int g = blockIdx.x % G;
  const int range = blockIdx.x / G;
  const int4 grp = a.groups[g];  // x: first class, y: classes, z: padded class stride, w: word
  const int k0 = grp.x, kw = grp.y, kwp = grp.z, w0 = grp.w;
  const int C = a.C;
  for (int i = tid; i < a.F * kMaxBins / 4; i += blockDim.x)
    reinterpret_cast<uint32_t *>(slut)[i] = reinterpret_cast<const uint32_t *>(a.lut)[i];
  int gcount = 0;
  for (int f = 0; f < a.F; f++) {
    const int o = a.gsoff[g * a.F + f];
    if (tid == 0) {
      soff[f] = o;
      sdf[f] = a.nval[f];
    }
    if (o >= 0) gcount = max(gcount, o + a.nval[f] * kwp);
  }
  const uint32_t R = (a.total_rows + a.nranges - 1) / a.nranges;
  uint32_t p0 = range * R;
  const uint32_t p1 = min(p0 + R, a.total_rows);
  int s = 0;  // first segment whose span contains position p0
  {
    int lo = 0, hi = a.nseg - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (a.segs[mid].row_base <= p0) lo = mid; else hi = mid - 1;
    }
    s = lo;
  }
  __syncthreads();
  // shared-memory byte address of this group's counter block of each feature of word w0
  const uint32_t sbase = smem_u32(sh);
  uint32_t abase[4];
#pragma unroll
  for (int e = 0; e < 4; e++) {
    const int f = 4 * w0 + e;
    abase[e] = (f < a.F && soff[f] >= 0) ? sbase + 4u * soff[f] : 0xFFFFFFFFu;
  }
  const uint32_t kwp4 = 4u * kwp;
  uint32_t iter = 0, epoch = 0;
  int visits = 0;
  int32_t *my_visits = a.visits + (size_t)blockIdx.x * a.max_visits * 6;
  while (p0 < p1 && s < a.nseg) {
    // ---- one node portion: the node's rows at virtual positions [p0, pe) ----
    const Seg first = a.segs[s];
    const uint32_t pe = min(p1, first.node_base + first.node_len);
    const bool hist_on = first.direct >= 0 && first.hslot >= 0;
    const bool moving = first.feat >= 0 && first.write != 0 && a.bins_out != nullptr;
    // this CTA's share [A, B) of the portion: it moves these rows
    const uint32_t L = pe - p0;
    const uint32_t A = p0 + (uint32_t)(((uint64_t)L * g) / G);
    const uint32_t B = p0 + (uint32_t)(((uint64_t)L * (g + 1)) / G);
    if (hist_on)
      for (int i = tid; i < gcount; i += blockDim.x) sh[i] = 0;
    if (tid == 0) s_cur[0] = s_cur[1] = 0;
    __syncthreads();
    const int s_first = s;
    for (; s < a.nseg && a.segs[s].row_base < pe; s++) {
      const Seg sg = a.segs[s];
      const uint32_t q0 = (p0 > sg.row_base ? p0 - sg.row_base : 0);
      const uint32_t q1 = min(sg.len, pe - sg.row_base);
      for (uint32_t qb = q0; qb < q1; qb += kUnroll * blockDim.x) {
        if (G > 1 && a.sync && ++iter % kSyncEvery == 0) {  // keep the G CTAs within L2 reach
          __syncthreads();
          if (tid == 0) {
            epoch++;
            atomicAdd(a.sync + range, 1u);
            while (ld_acquire_gpu(a.sync + range) < epoch * G) __nanosleep(100);
          }
          __syncthreads();
        }
        Row<BS> r[kUnroll];
        int label[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {  // issue all loads first
          const uint32_t q = qb + u * blockDim.x + tid;
          label[u] = -1;  // -1: no row
          if (q < q1) {
            load_row<BS>(a.bins_in + (size_t)(sg.off + q) * BS, r[u]);
            label[u] = a.lab_in[sg.off + q];
          } else {
#pragma unroll
            for (int i = 0; i < Row<BS>::N; i++) r[u].w[i] = 0;
          }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
          const uint32_t v = sg.row_base + qb + u * blockDim.x + tid;  // virtual position
          bool left = true;
          if (sg.feat >= 0)
            left = slut[sg.feat * kMaxBins + row_byte<BS>(r[u], sg.feat)] <= sg.thr;
          if (moving) {  // a7, warp-aggregated shared-memory cursors
            const bool mine = label[u] >= 0 && v >= A && v < B;
            const unsigned ml = __ballot_sync(kFull, mine && left && (sg.write & 1));
            const unsigned mr = __ballot_sync(kFull, mine && !left && (sg.write & 2));
            uint32_t base = 0;
            if (lane == 0 && ml) base = atomicAdd(&s_cur[0], __popc(ml));
            if (lane == 1 && mr) base = atomicAdd(&s_cur[1], __popc(mr));
            const uint32_t bl = __shfl_sync(kFull, base, 0), br = __shfl_sync(kFull, base, 1);
            const unsigned below = (1u << lane) - 1;
            const bool wl = (ml >> lane) & 1, wr = (mr >> lane) & 1;
            if (wl || wr) {
              const uint32_t pos = wl ? A + bl + __popc(ml & below) : B - 1 - (br + __popc(mr & below));
              store_row<BS>(a.bins_out + (size_t)pos * BS, r[u]);
              __stcs(a.lab_out + pos, (uint8_t)label[u]);
            }
          }
          if (hist_on && label[u] >= 0 && (unsigned)(label[u] - k0) < (unsigned)kw &&
              (sg.direct == 2 || (sg.direct == 0) == left)) {
            const uint32_t w = pick<Row<BS>::N>(r[u].w, w0);
            const uint32_t lk4 = 4u * (label[u] - k0);
#pragma unroll
            for (int e = 0; e < 4; e++)
              if (abase[e] != 0xFFFFFFFFu)
                red_shared_inc(abase[e] + ((w >> (8 * e)) & 0xFF) * kwp4 + lk4);
          }
        }
      }
    }
    __syncthreads();
    if (moving && tid == 0 && visits < a.max_visits) {  // report this share
      int32_t *vv = my_visits + 6 * visits;
      vv[0] = s_first;
      vv[1] = (int32_t)A;
      vv[2] = (int32_t)B;
      vv[3] = (int32_t)s_cur[0];
      vv[4] = (int32_t)s_cur[1];
      vv[5] = 0;
    }
    if (moving) visits++;
    if (hist_on) {  // flush: provisional id -> rank, class slab -> classes
      uint32_t *dst = a.H + (size_t)first.hslot * a.HS;
      for (int f = 0; f < a.F; f++) {
        const int o = soff[f];
        if (o < 0) continue;
        const int n = sdf[f] * kwp;
        const uint8_t *lf = slut + f * kMaxBins;
        uint32_t *df = dst + a.hoff[f];
        for (int i = tid; i < n; i += blockDim.x) {
          const uint32_t val = sh[o + i];
          if (val) {
            const int pp = i / kwp, j = i - pp * kwp;
            atomicAdd(df + (int)lf[pp] * C + k0 + j, val);
          }
        }
      }
      __syncthreads();
    }
    p0 = pe;
  }
}

__global__ void zero_slots_kernel(uint32_t *H, int64_t HS, const int32_t *slots) {
  uint32_t *h = H + (size_t)slots[blockIdx.y] * HS;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < HS;
       i += (int64_t)gridDim.x * blockDim.x)
    h[i] = 0;
}

// triples: (dst slot in H, parent slot in Hprev, direct sibling slot in H)
__global__ void subtract_kernel(uint32_t *H, const uint32_t *Hprev, int64_t HS,
                                const int32_t *triples) {
  const int32_t *t = triples + 3 * blockIdx.y;
  uint32_t *d = H + (size_t)t[0] * HS;
  const uint32_t *p = Hprev + (size_t)t[1] * HS;
  const uint32_t *q = H + (size_t)t[2] * HS;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < HS;
       i += (int64_t)gridDim.x * blockDim.x)
    d[i] = p[i] - q[i];
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
    split_kernel(const uint32_t *__restrict__ H, int64_t HS, const int32_t *node_slot, int F,
                 int C, const int32_t *hoff, const int32_t *nval, SplitCand *out) {
  __shared__ uint32_t tile[kSplitThreads][kClassChunk + 1];
  __shared__ uint32_t segtot[kSplitThreads / 32][kClassChunk];
  __shared__ uint32_t Pk[kClassChunk];
  __shared__ uint64_t nLs[kSplitThreads];
  __shared__ uint32_t nonempty[kSplitThreads / 32];
  __shared__ Key wbest[kSplitThreads / 32];

  const int node = blockIdx.x, f = blockIdx.y;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int Df = nval[f];
  const uint32_t *h = H + (size_t)node_slot[node] * HS + hoff[f];
  uint64_t nl = 0, sl = 0, sr = 0, ntot = 0;
  for (int c0 = 0; c0 < C; c0 += kClassChunk) {
    const int kc = min(kClassChunk, C - c0);
    for (int e = t; e < Df * kc; e += kSplitThreads) {
      const int r = e / kc, k = e - r * kc;
      tile[r][k] = __ldg(h + (size_t)r * C + c0 + k);
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

__global__ void __launch_bounds__(256)
    winner_kernel(const uint32_t *__restrict__ H, int64_t HS, const int32_t *node_slot, int F,
                  int C, const int32_t *hoff, const int32_t *nval, const SplitCand *cand,
                  uint8_t *res, int res_stride) {
  __shared__ int s_f;
  __shared__ SplitCand s_c;
  __shared__ unsigned long long s_n;
  const int node = blockIdx.x, t = threadIdx.x;
  if (t == 0) {
    int bf = -1;
    Key bk;
    bk.valid = 0;
    bk.idx = 0x7fffffff;
    bk.hi = bk.lo = 0;
    bk.den = 1;
    for (int f = 0; f < F; f++) {
      const SplitCand &c = cand[(size_t)node * F + f];
      Key k;
      k.valid = c.valid;
      k.idx = f;
      k.hi = c.num_hi;
      k.lo = c.num_lo;
      k.den = c.den;
      if (k.valid && better(k, bk)) {
        bk = k;
        bf = f;
      }
    }
    s_f = bf;
    if (bf >= 0) s_c = cand[(size_t)node * F + bf];
    s_n = 0;
  }
  __syncthreads();
  const int fsel = s_f >= 0 ? s_f : 0;
  const int blo = s_f >= 0 ? s_c.b_lo : -1;
  const uint32_t *h = H + (size_t)node_slot[node] * HS + hoff[fsel];
  const int Df = nval[fsel];
  NodeRes *nr = reinterpret_cast<NodeRes *>(res + (size_t)node * res_stride);
  uint32_t *P = reinterpret_cast<uint32_t *>(nr + 1);
  uint32_t *cL = P + C;
  for (int k = t; k < C; k += blockDim.x) {
    uint32_t tot = 0, left = 0;
    for (int r = 0; r < Df; r++) {
      const uint32_t v = __ldg(h + (size_t)r * C + k);
      tot += v;
      if (r <= blo) left += v;
    }
    P[k] = tot;
    cL[k] = left;
    atomicAdd(&s_n, (unsigned long long)tot);
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

void launch_hist_pass(const HistPassArgs &a, cudaStream_t s) {
  if (a.total_rows == 0 || a.nseg == 0) return;
  const size_t smem = (size_t)a.smem_counters * 4 + (size_t)a.F * kMaxBins;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.nranges * a.ngroups);
  cfg.blockDim = dim3(kHistThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // co-residency of a range's CTAs (partner sync)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.sync ? 1 : 0;
  switch (a.BS) {
#define CASE(B)                                                                              \
  case B:                                                                                    \
    CUDA_CHECK(cudaFuncSetAttribute(hist_pass_kernel<B>,                                     \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    CUDA_CHECK(cudaLaunchKernelEx(&cfg, hist_pass_kernel<B>, a));                            \
    break;
    CASE(1) CASE(2) CASE(4) CASE(8) CASE(16) CASE(32) CASE(64)
#undef CASE
    default:
      throw Error(-1, "bad bins stride");
  }
  CUDA_CHECK(cudaGetLastError());
}

void launch_zero_slots(uint32_t *H, int64_t HS, const int32_t *slots, int n, cudaStream_t s) {
  if (n == 0) return;
  const int bx = (int)std::min<int64_t>((HS + 1023) / 1024, 64);
  zero_slots_kernel<<<dim3(bx, n), 1024, 0, s>>>(H, HS, slots);
  CUDA_CHECK(cudaGetLastError());
}

void launch_subtract(uint32_t *H, const uint32_t *Hprev, int64_t HS, const int32_t *triples,
                     int n, cudaStream_t s) {
  if (n == 0) return;
  const int bx = (int)std::min<int64_t>((HS + 1023) / 1024, 64);
  subtract_kernel<<<dim3(bx, n), 1024, 0, s>>>(H, Hprev, HS, triples);
  CUDA_CHECK(cudaGetLastError());
}

void launch_split(const uint32_t *H, int64_t HS, const int32_t *node_slot, int nnodes, int F,
                  int C, const int32_t *hoff, const int32_t *nval, SplitCand *out,
                  cudaStream_t s) {
  if (nnodes == 0) return;
  split_kernel<<<dim3(nnodes, F), kSplitThreads, 0, s>>>(H, HS, node_slot, F, C, hoff, nval, out);
  CUDA_CHECK(cudaGetLastError());
}

void launch_winner(const uint32_t *H, int64_t HS, const int32_t *node_slot, int nnodes, int F,
                   int C, const int32_t *hoff, const int32_t *nval, const SplitCand *cand,
                   uint8_t *res, int res_stride, cudaStream_t s) {
  if (nnodes == 0) return;
  winner_kernel<<<nnodes, 256, 0, s>>>(H, HS, node_slot, F, C, hoff, nval, cand, res,
                                       res_stride);
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace adapt
