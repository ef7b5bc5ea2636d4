// small.cu — the whole hot path (a1 labels, a2 value tables, a3 bins, a4-a8
// level-wise CART) for SMALL tables in ONE thread block, one launch: the
// paper's online-training scale (Table 4: a model built at run time
// from tens to hundreds of profiled samples, 60-280 us on the host CPU).  The
// general engine spends two host round trips per level, which dominate at
// this size; here every level stays on chip and the host waits once.
//
// Same definitions as the general path (and the oracle): R2/R3 labels, R4
// canonical -0, R7 node-local midpoint thresholds, R9 ties (score, then lowest
// feature, then lowest threshold), R10 leaf rule, R12 labels, R13x exact
// score comparison — with n <= 512 every cross product fits in 64 bits.
// Anything outside the limits (or any flagged value: NaN / Inf, all-+inf
// rows, > 256 distinct values, a frontier wider than kSmallMaxA) returns
// "fallback" and the caller runs the general path, which also raises the
// errors.
//
// Per level: one thread per (feature, frontier node) walks the feature's
// presorted rows (ascending value, then row) and scans the node's cuts with
// incremental sums of squares (SL += 2 cL_k + 1, SR -= 2 cR_k - 1), keeping
// its best (score, threshold); one thread per node picks the feature.
#include <cstdint>

#include "adapt.h"
#include "common.h"

namespace adapt {
namespace {

constexpr int kT = 512;  // threads; one per row at most

__device__ __forceinline__ uint32_t fkey(float x) {  // order-preserving u32 of a float
  const uint32_t b = __float_as_uint(x);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

struct SmallShared {
  float xs[kSmallMaxF][kSmallMaxN];        // canonical features, feature-major
  int16_t order[kSmallMaxF][kSmallMaxN];   // rows by (node, value, row) per feature
  int16_t order2[kSmallMaxF][kSmallMaxN];  // regrouping buffer
  int16_t seg[kSmallMaxA + 1];             // node j's rows: positions [seg[j], seg[j+1]) of every order[f]
  int16_t cur[kSmallMaxF][kSmallMaxA];     // regrouping cursors
  uint8_t lab[kSmallMaxN];
  int16_t nid[kSmallMaxN];                 // frontier index of the row's node (-1: leaf)
  alignas(16) uint16_t cnt[kSmallMaxA][kSmallMaxC];    // node class totals (u32-pair atomics)
  alignas(16) uint16_t cl[kSmallMaxF * kSmallMaxA][kSmallMaxC];  // a scan thread's left counts
  // per (feature, node) best cut: exact key num/den, threshold values
  uint64_t bnum[kSmallMaxF * kSmallMaxA], bden[kSmallMaxF * kSmallMaxA];
  float blo[kSmallMaxF * kSmallMaxA], bhi[kSmallMaxF * kSmallMaxA];
  int32_t fr_tree[kSmallMaxA], fr_depth[kSmallMaxA];
  int32_t nx_tree[kSmallMaxA], nx_depth[kSmallMaxA];
  int32_t child_of[kSmallMaxA][2];          // next-frontier index of the children (-1: leaf)
  int32_t split_f[kSmallMaxA];
  float split_lo[kSmallMaxA];
  unsigned int cw[kT / 32][kSmallMaxC];    // a scanning warp's running class counts
  alignas(16) uint16_t cnt2[kSmallMaxA][kSmallMaxC];   // next level's class totals
  int32_t nx_n[kSmallMaxA];
  int32_t A, nA, n_nodes, status, old_total;
  uint32_t flags;
};

__device__ void node_stats(const uint16_t *c, int C, adapt_node_t &o) {
  uint64_t n = 0, S = 0;
  int best = 0;
  for (int k = 0; k < C; k++) {
    n += c[k];
    S += (uint64_t)c[k] * c[k];
    if (c[k] > c[best]) best = k;  // ties -> lowest class (R12)
  }
  o.n = (int64_t)n;
  o.label = best;
  o.gini = n ? __dsub_rn(1.0, __ddiv_rn((double)S, __dmul_rn((double)n, (double)n))) : 0.0;
}

__global__ void __launch_bounds__(kT, 1)
    small_train_kernel(const float *__restrict__ X, const float *__restrict__ T, int n, int F, int V, int D,
                       int BS, size_t pstride, uint8_t *__restrict__ bins, uint8_t *__restrict__ labels,
                       SmallOut *__restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  SmallShared &sh = *reinterpret_cast<SmallShared *>(smem_raw);
  const int tid = threadIdx.x;
  if (tid == 0) {
    sh.flags = 0;
    sh.status = 0;
  }
  __syncthreads();
  // ---- a1 labels (one thread per row) and canonical features ----
  for (int i = tid; i < n; i += kT) {
    float best = __int_as_float(0x7f800000);
    int bi = 0;
    bool nan = false;
    for (int v = 0; v < V; v++) {
      const float t = T[(int64_t)i * V + v];
      nan |= t != t;
      if (t < best) {
        best = t;
        bi = v;
      }
    }
    if (nan || best == __int_as_float(0x7f800000)) atomicOr(&sh.flags, 1u);
    sh.lab[i] = (uint8_t)bi;
    labels[i] = (uint8_t)bi;
    for (int f = 0; f < F; f++) {
      float x = X[(int64_t)i * F + f];
      if (x != x || fabsf(x) == __int_as_float(0x7f800000)) atomicOr(&sh.flags, 1u);
      sh.xs[f][i] = x == 0.0f ? 0.0f : x;  // R4
    }
  }
  __syncthreads();
  if (sh.flags) {  // the general path raises the error
    if (tid == 0) out->status = 1;
    return;
  }
  // ---- a2/a3: per feature, position of every row in (value, row) order by
  // counting (n <= 512), then bins = ranks of the distinct values by a block
  // scan of "new value" flags along that order; value tables from the firsts
  __shared__ int warp_tot[kT / 32];
  for (int f = 0; f < F; f++) {
    for (int i = tid; i < n; i += kT) {
      const uint32_t ki = fkey(sh.xs[f][i]);
      int pos = 0;
      for (int j = 0; j < n; j++) {
        const uint32_t kj = fkey(sh.xs[f][j]);
        pos += (kj < ki) || (kj == ki && j < i);
      }
      sh.order[f][pos] = (int16_t)i;
    }
    __syncthreads();
    const int p = tid;  // kT >= n: one sorted position per thread
    int isnew = 0;
    if (p < n)
      isnew = p == 0 || fkey(sh.xs[f][sh.order[f][p]]) != fkey(sh.xs[f][sh.order[f][p - 1]]);
    int incl = isnew;  // inclusive block scan
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if ((tid & 31) >= o) incl += y;
    }
    if ((tid & 31) == 31) warp_tot[tid >> 5] = incl;
    __syncthreads();
    int base = 0;
    for (int w = 0; w < (tid >> 5); w++) base += warp_tot[w];
    const int bin = base + incl - 1;
    if (p < n) {
      const int i = sh.order[f][p];
      if (bin > 255) {
        atomicOr(&sh.flags, 2u);
      } else {
        if (isnew) out->val[f][bin] = sh.xs[f][i];
        if (BS >= 4)
          bins[(size_t)(f / 4) * pstride + (size_t)i * 4 + (f % 4)] = (uint8_t)bin;
        else
          bins[(size_t)i * BS + f] = (uint8_t)bin;
      }
      if (p == n - 1) out->nval[f] = bin + 1;
    }
    __syncthreads();
  }
  if (sh.flags) {  // > 256 distinct values: the general path raises E_TOO_MANY_DISTINCT
    if (tid == 0) out->status = 1;
    return;
  }
  // ---- level loop ----
  if (tid == 0) {
    sh.A = 1;
    sh.fr_tree[0] = 0;
    sh.fr_depth[0] = 0;
    sh.n_nodes = 1;
    adapt_node_t r{};
    r.feature = -1;
    r.left = r.right = -1;
    out->nodes[0] = r;
  }
  for (int i = tid; i < n; i += kT) sh.nid[i] = 0;
  for (int i = tid; i < kSmallMaxC; i += kT) sh.cnt[0][i] = 0;
  if (tid == 0) {
    sh.seg[0] = 0;
    sh.seg[1] = (int16_t)n;
  }
  __syncthreads();
  for (int i = tid; i < n; i += kT)  // root class totals (u16 pairs in u32 words)
    atomicAdd(reinterpret_cast<unsigned int *>(sh.cnt[0]) + (sh.lab[i] >> 1), 1u << (16 * (sh.lab[i] & 1)));
  __syncthreads();
  for (int level = 0; sh.A > 0; level++) {
    const int A = sh.A;
    // a6: one WARP per (feature, node) pair scans the node's rows in value
    // order, 32 at a time: a row's class count before it = the warp's running
    // count + its rank among the chunk's rows of that class (match_any), so the
    // sums of squares after every row are warp prefix sums of 2 c + 1 (left)
    // and 2 (P_k - c) - 1 (right, subtracted); every lane whose next row has a
    // larger value is a cut, compared exactly, ties -> the lowest threshold
    {
      const int w = tid >> 5, lane = tid & 31;
      unsigned int *cw = sh.cw[w];
      for (int pr = w; pr < F * A; pr += kT / 32) {
        const int f = pr / A, j = pr % A;
        const uint16_t *P = sh.cnt[j];
        uint64_t nn = 0, SR = 0;
        for (int k = 0; k < kSmallMaxC; k++) {
          nn += P[k];
          SR += (uint64_t)P[k] * P[k];
        }
        if (lane < kSmallMaxC) cw[lane] = 0;
        __syncwarp();
        const int s0 = sh.seg[j], s1 = sh.seg[j + 1];
        uint64_t SL = 0, nL = 0, bn = 0, bd = 0;
        int bpos = -1;
        float blo = 0.f, bhi = 0.f;
        for (int q0 = s0; q0 < s1; q0 += 32) {
          const int p = q0 + lane;
          const bool valid = p < s1;
          const int i = valid ? sh.order[f][p] : 0;
          const int k = valid ? sh.lab[i] : -1;
          const float x = valid ? sh.xs[f][i] : 0.f;
          const float nx = (p + 1 < s1) ? sh.xs[f][sh.order[f][p + 1]] : x;
          const unsigned peers = __match_any_sync(0xffffffffu, k);
          const int rk = __popc(peers & ((1u << lane) - 1));
          const unsigned cb = valid ? cw[k] + rk : 0;  // class-k rows on the left before this row
          unsigned dl = valid ? 2 * cb + 1 : 0;
          unsigned dr = valid ? 2 * (P[k] - cb) - 1 : 0;
          unsigned cnt = valid ? 1 : 0;
          for (int o = 1; o < 32; o <<= 1) {  // inclusive prefix sums
            const unsigned a1 = __shfl_up_sync(0xffffffffu, dl, o);
            const unsigned a2 = __shfl_up_sync(0xffffffffu, dr, o);
            const unsigned a3 = __shfl_up_sync(0xffffffffu, cnt, o);
            if (lane >= o) {
              dl += a1;
              dr += a2;
              cnt += a3;
            }
          }
          const uint64_t sl = SL + dl, sr = SR - dr, nl = nL + cnt;
          const bool cut = valid && p + 1 < s1 && nx != x;  // a cut between x and nx (R7 node-local)
          uint64_t num = 0, den = 0;
          if (cut) {
            const uint64_t nr = nn - nl;
            num = sl * nr + sr * nl;  // SL/nL + SR/nR (R13x), < 2^46 for n <= 512
            den = nl * nr;
          }
          // warp argmax, ties -> the lower position (lower threshold, R9)
          uint64_t wn = num, wd = den;
          int wp = cut ? p : 0x7fffffff;
          for (int o = 16; o > 0; o >>= 1) {
            const uint64_t on = __shfl_xor_sync(0xffffffffu, wn, o), od = __shfl_xor_sync(0xffffffffu, wd, o);
            const int op = __shfl_xor_sync(0xffffffffu, wp, o);
            if (op != 0x7fffffff &&
                (wp == 0x7fffffff || on * wd > wn * od || (on * wd == wn * od && op < wp))) {
              wn = on;
              wd = od;
              wp = op;
            }
          }
          if (wp != 0x7fffffff && (bpos < 0 || wn * bd > bn * wd)) {  // strict: earlier chunks win ties
            bn = wn;
            bd = wd;
            bpos = wp;
            const float lo = __shfl_sync(0xffffffffu, x, wp - q0);
            const float hi = __shfl_sync(0xffffffffu, nx, wp - q0);
            blo = lo;
            bhi = hi;
          }
          // carry: sums after the chunk's last row, class counts
          SL += __shfl_sync(0xffffffffu, dl, 31);
          SR -= __shfl_sync(0xffffffffu, dr, 31);
          nL += __shfl_sync(0xffffffffu, cnt, 31);
          __syncwarp();
          if (valid && rk == 0) cw[k] += __popc(peers);
          __syncwarp();
        }
        if (lane == 0) {
          sh.bnum[pr] = bpos >= 0 ? bn : 0;
          sh.bden[pr] = bpos >= 0 ? bd : 0;
          sh.blo[pr] = blo;
          sh.bhi[pr] = bhi;
        }
      }
    }
    __syncthreads();
    // decide (one thread, in frontier order: BFS indices are assigned in order)
    if (tid == 0) {
      for (int j = 0; j < A; j++) {
        adapt_node_t &nd = out->nodes[sh.fr_tree[j]];
        const uint16_t *P = sh.cnt[j];
        node_stats(P, kSmallMaxC, nd);
        nd.depth = sh.fr_depth[j];
        sh.child_of[j][0] = sh.child_of[j][1] = -1;
        sh.split_f[j] = -1;
        int np = 0;
        for (int k = 0; k < kSmallMaxC; k++) np += P[k] > 0;
        int bf = -1;
        for (int f = 0; f < F; f++) {
          const int t = f * A + j;
          if (!sh.bden[t]) continue;
          // max score, ties -> lowest feature (R9): strict >
          if (bf < 0 || sh.bnum[t] * sh.bden[bf * A + j] > sh.bnum[bf * A + j] * sh.bden[t]) bf = f;
        }
        if (nd.depth >= D || np <= 1 || bf < 0) continue;  // leaf (R10, R11)
        const int t = bf * A + j;
        nd.feature = bf;
        nd.threshold = __dmul_rn(__dadd_rn((double)sh.blo[t], (double)sh.bhi[t]), 0.5);  // R7
        const int li = sh.n_nodes;
        if (li + 2 > kSmallMaxNodes) {
          sh.status = 1;
          break;
        }
        nd.left = li;
        nd.right = li + 1;
        sh.n_nodes += 2;
        sh.split_f[j] = bf;
        sh.split_lo[j] = sh.blo[t];
        for (int side = 0; side < 2; side++) {
          adapt_node_t c{};
          c.feature = -1;
          c.left = c.right = -1;
          c.depth = nd.depth + 1;
          out->nodes[li + side] = c;
        }
      }
    }
    __syncthreads();
    if (sh.status) break;
    // children's class counts (rows of split nodes by side), then the frontier
    for (int i = tid; i < A * 2 * kSmallMaxC; i += kT)
      sh.cl[i / kSmallMaxC][i % kSmallMaxC] = 0;  // reuse cl[0 .. 2A) as child counts
    __syncthreads();
    for (int i = tid; i < n; i += kT) {
      const int j = sh.nid[i];
      if (j < 0) continue;
      const int f = sh.split_f[j];
      if (f < 0) {
        sh.nid[i] = -1;
        continue;
      }
      const int side = sh.xs[f][i] <= sh.split_lo[j] ? 0 : 1;
      atomicAdd(reinterpret_cast<unsigned int *>(&sh.cl[2 * j + side][0]) + (sh.lab[i] >> 1),
                1u << (16 * (sh.lab[i] & 1)));
    }
    __syncthreads();
    if (tid == 0) {
      int nA = 0;
      for (int j = 0; j < A && !sh.status; j++) {
        if (sh.split_f[j] < 0) continue;
        const adapt_node_t &nd = out->nodes[sh.fr_tree[j]];
        for (int side = 0; side < 2; side++) {
          const uint16_t *c = sh.cl[2 * j + side];
          int np = 0;
          for (int k = 0; k < kSmallMaxC; k++) np += c[k] > 0;
          adapt_node_t &ch = out->nodes[nd.left + side];
          if (nd.depth + 1 < D && np > 1) {  // in the next frontier (stats there)
            if (nA >= kSmallMaxA) {
              sh.status = 1;
              break;
            }
            sh.child_of[j][side] = nA;
            sh.nx_tree[nA] = nd.left + side;
            sh.nx_depth[nA] = nd.depth + 1;
            int nc = 0;
            for (int k = 0; k < kSmallMaxC; k++) nc += c[k];
            sh.nx_n[nA] = nc;
            nA++;
          } else {
            node_stats(c, kSmallMaxC, ch);
          }
        }
      }
      for (int j = 0; j < nA; j++) {
        sh.fr_tree[j] = sh.nx_tree[j];
        sh.fr_depth[j] = sh.nx_depth[j];
      }
      sh.nA = nA;
      sh.old_total = sh.seg[A];
      sh.seg[0] = 0;
      for (int j = 0; j < nA; j++) sh.seg[j + 1] = (int16_t)(sh.seg[j] + sh.nx_n[j]);
    }
    __syncthreads();
    if (sh.status) break;
    for (int i = tid; i < n; i += kT) {  // rows follow their node into the next frontier
      const int j = sh.nid[i];
      if (j < 0) continue;
      const int f = sh.split_f[j];
      const int side = sh.xs[f][i] <= sh.split_lo[j] ? 0 : 1;
      sh.nid[i] = (int16_t)sh.child_of[j][side];
    }
    for (int i = tid; i < kSmallMaxF * kSmallMaxA; i += kT) sh.cur[i / kSmallMaxA][i % kSmallMaxA] = 0;
    // next level's class totals: the children's counts
    for (int i = tid; i < A * 2 * kSmallMaxC; i += kT) {
      const int jj = i / (2 * kSmallMaxC), side = (i / kSmallMaxC) & 1, k = i % kSmallMaxC;
      const int c = sh.child_of[jj][side];
      if (sh.split_f[jj] >= 0 && c >= 0) sh.cnt2[c][k] = sh.cl[2 * jj + side][k];
    }
    __syncthreads();
    // stable regrouping of every feature's order by the rows' next node (one
    // warp per feature, 32 positions at a time: match_any peers give the rank
    // of a row among the chunk's rows of its node); leaf rows drop out
    {
      const int w = tid >> 5, lane = tid & 31;
      for (int f = w; f < F; f += kT / 32) {
        for (int p0 = 0; p0 < sh.old_total; p0 += 32) {
          const int p = p0 + lane;
          const int i = p < sh.old_total ? sh.order[f][p] : -1;
          const int key = i >= 0 ? sh.nid[i] : -1;
          const unsigned peers = __match_any_sync(0xffffffffu, key);
          const int rank = __popc(peers & ((1u << lane) - 1));
          if (key >= 0) sh.order2[f][sh.seg[key] + sh.cur[f][key] + rank] = (int16_t)i;
          __syncwarp();
          if (key >= 0 && rank == 0) sh.cur[f][key] += (int16_t)__popc(peers);
          __syncwarp();
        }
      }
    }
    __syncthreads();
    for (int i = tid; i < F * kSmallMaxN; i += kT) sh.order[i / kSmallMaxN][i % kSmallMaxN] = sh.order2[i / kSmallMaxN][i % kSmallMaxN];
    for (int i = tid; i < kSmallMaxA * kSmallMaxC; i += kT) sh.cnt[i / kSmallMaxC][i % kSmallMaxC] = sh.cnt2[i / kSmallMaxC][i % kSmallMaxC];
    if (tid == 0) sh.A = sh.nA;
    __syncthreads();
  }
  if (tid == 0) {
    out->n_nodes = sh.n_nodes;
    if (!out->status) out->status = sh.status;
  }
}

}  // namespace

size_t small_smem_bytes() { return sizeof(SmallShared); }

void launch_small_train(const float *X, const float *T, int n, int F, int V, int D, int BS, size_t pstride,
                        uint8_t *bins, uint8_t *labels, SmallOut *out, cudaStream_t s) {
  const size_t smem = sizeof(SmallShared);
  smem_limit(small_train_kernel, smem);
  CUDA_CHECK(cudaMemsetAsync(out, 0, sizeof(SmallOut), s));
  small_train_kernel<<<1, kT, smem, s>>>(X, T, n, F, V, D, BS, pstride, bins, labels, out); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace adapt
