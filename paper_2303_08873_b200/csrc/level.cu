// level.cu — the row passes of one tree level.
//
//   partition_kernel  a7: the rows of every split parent are moved from the
//                     input planes into the output planes.  Each CTA owns a
//                     contiguous range of the level's "virtual positions"
//                     (segments = pieces of the parents' rows, concatenated);
//                     inside it, a parent's rows go to [A, ..) if they go left
//                     and (.., B] if right, where [A, B) is the parent's share
//                     of the range, positions from warp-aggregated shared-
//                     memory cursors.  Each CTA reports (parent, A, B, left,
//                     right) — the children's pieces for the next level.
//   hist_kernel       a4: class histogram H[node][f][rank][class] of the rows
//                     of the pieces it is given (the root, or the smaller
//                     child of every split).  A node's histogram (Σ_f D_f × C
//                     u32 counters, 508 KB at C4) does not fit one SM, so G
//                     CTAs share each row range: CTA g owns the 4 features of
//                     32-bit word w(g) of the bins row (× a class slab), i.e.
//                     at most 4 shared-memory reductions per row, reading only
//                     that word's plane (4 bytes per row), so the G CTAs
//                     of a range share only the 1-byte labels and run
//                     unsynchronised.  Per node only the classes present in it get
//                     counters (the host knows them from the parent's split),
//                     with an odd class stride (bank spread); the block's
//                     counters are flushed into the node's global histogram
//                     with integer atomics.
// Every quantity that decides the tree is an integer, so the result does not
// depend on row order, on the number of ranks or on atomic ordering.
#include <algorithm>
#include <map>
#include <utility>

#include "common.h"
#include "ptx.h"

namespace adapt {
namespace {

constexpr unsigned kFull = 0xffffffffu;

template <int BS>
struct Row {  // one row's bins, BS bytes, in registers
  static constexpr int N = BS >= 4 ? BS / 4 : 1;
  uint32_t w[N];
};

// Bins are stored in "word planes": plane p holds bytes [4p, 4p+4) of every
// row's bins (BS >= 4), so any 32-bit word of a row is one coalesced load and a
// pass that needs one word reads 4 bytes per row.  BS < 4: one plane of BS-byte rows.
template <int BS>
__device__ __forceinline__ void load_row(const uint8_t *__restrict__ base, size_t pstride,
                                         uint32_t row, Row<BS> &r) {
  if constexpr (BS >= 4) {
#pragma unroll
    for (int i = 0; i < BS / 4; i++)
      r.w[i] = *reinterpret_cast<const uint32_t *>(base + i * pstride + (size_t)row * 4);
  } else if constexpr (BS == 2) {
    r.w[0] = *reinterpret_cast<const unsigned short *>(base + (size_t)row * 2);
  } else {
    r.w[0] = base[row];
  }
}

template <int BS>
__device__ __forceinline__ void store_row(uint8_t *__restrict__ base, size_t pstride, uint32_t row,
                                          const Row<BS> &r) {
  if constexpr (BS >= 4) {
#pragma unroll
    for (int i = 0; i < BS / 4; i++)
      __stcs(reinterpret_cast<unsigned int *>(base + i * pstride + (size_t)row * 4), r.w[i]);
  } else if constexpr (BS == 2) {
    *reinterpret_cast<unsigned short *>(base + (size_t)row * 2) = (unsigned short)r.w[0];
  } else {
    base[row] = (uint8_t)r.w[0];
  }
}

// predicated streaming stores (no divergent branch around a row's stores);
// no "memory" clobber: nothing in these kernels reads what they write, and a
// clobber would pin the next batch's loads behind every store
__device__ __forceinline__ void st_cs_if(bool p, void *addr, uint32_t v) {
  asm volatile("{\n.reg .pred q;\nsetp.ne.u32 q, %0, 0;\n@q st.global.cs.b32 [%1], %2;\n}" ::"r"((uint32_t)p), "l"(addr),
               "r"(v));
}
__device__ __forceinline__ void st_cs_if_u8(bool p, void *addr, uint32_t v) {
  asm volatile("{\n.reg .pred q;\nsetp.ne.u32 q, %0, 0;\n@q st.global.cs.u8 [%1], %2;\n}" ::"r"((uint32_t)p), "l"(addr),
               "r"(v));
}

// w[i] for a runtime i through a tree of register selects (N = power of 2):
// every array access has a compile-time index, so nothing goes to local memory
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

// no "memory" clobber: the counters are read only after a __syncthreads, so
// other loads (the class map) may move across the reductions
__device__ __forceinline__ void red_shared_add(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v));
}

// (not volatile: the class-map lookups of a thread's rows may be hoisted ahead
// of the reductions — the map is written before the node's rows are counted)
__device__ __forceinline__ uint32_t ld_shared_u8(uint32_t addr) {
  uint32_t v;
  asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ int first_seg(const Seg *segs, int nseg, uint32_t p) {
  int lo = 0, hi = nseg - 1;  // last segment with row_base <= p
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (segs[mid].row_base <= p) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// ------------------------------------------------------------ partition --
#ifndef ADAPT_PART_UNROLL
#define ADAPT_PART_UNROLL 3
#endif
#ifndef ADAPT_HIST_UNROLL
#define ADAPT_HIST_UNROLL 8
#endif
#ifndef ADAPT_PART_THREADS
#define ADAPT_PART_THREADS 1024
#endif
constexpr int kPartThreads = ADAPT_PART_THREADS;
constexpr int kPartMinBlocks = 1024 / ADAPT_PART_THREADS;  // 1024 threads per SM
constexpr int kPartUnroll = ADAPT_PART_UNROLL;  // rows in flight per thread

template <int BS>
__global__ void __launch_bounds__(kPartThreads, kPartMinBlocks) partition_kernel(PartArgs a) {
  __shared__ uint32_t s_cur[2];
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t R = (a.total_rows + gridDim.x - 1) / gridDim.x;
  uint32_t p0 = blockIdx.x * R;
  const uint32_t p1 = min(p0 + R, a.total_rows);
  int s = p0 < p1 ? first_seg(a.segs, a.nseg, p0) : a.nseg;
  int32_t *my_visits = a.visits + (size_t)blockIdx.x * a.max_visits * 6;
  int visits = 0;
  __syncthreads();
  while (p0 < p1 && s < a.nseg) {
    // ---- one parent's rows at virtual positions [p0, pe): its share [A, B) = [p0, pe) ----
    const Seg first = a.segs[s];
    const uint32_t pe = min(p1, first.node_base + first.node_len);
    const uint32_t A = p0, B = pe;
    if (tid == 0) s_cur[0] = s_cur[1] = 0;
    __syncthreads();
    const int s_first = s;
    for (; s < a.nseg && a.segs[s].row_base < pe; s++) {
      const Seg sg = a.segs[s];
      if (!sg.write) continue;  // a parent that does not split (or whose children are leaves)
      const uint32_t q0 = p0 > sg.row_base ? p0 - sg.row_base : 0;
      const uint32_t q1 = min(sg.len, pe - sg.row_base);
      // rows in flight: kPartUnroll per thread, loaded one batch ahead of the
      // batch being placed (software pipeline: the next batch's loads are in
      // flight during this batch's ballots and stores)
      Row<BS> r[kPartUnroll], rn[kPartUnroll];
      int label[kPartUnroll], labn[kPartUnroll];
      uint8_t wgt[kPartUnroll], wgn[kPartUnroll];
      auto load = [&](uint32_t qb, Row<BS>(&rr)[kPartUnroll], int(&ll)[kPartUnroll],
                      uint8_t(&ww)[kPartUnroll]) {
#pragma unroll
        for (int u = 0; u < kPartUnroll; u++) {
          // branch-free: a lane past the segment's end re-reads its last row
          // (q clamped; q0 < q1 here) and is marked invalid by its label
          const uint32_t q = qb + u * kPartThreads + tid;
          const uint32_t qc = min(q, q1 - 1);
          load_row<BS>(a.bins_in, a.pstride, sg.off + qc, rr[u]);
          const int lb = __ldcs(a.lab_in + sg.off + qc);
          ll[u] = q < q1 ? lb : -1;
          // bootstrap weight (forests): rows drawn 0 times leave the tree here
          ww[u] = a.w_in ? __ldcs(a.w_in + sg.off + qc) : (uint8_t)1;
        }
      };
      if (q0 < q1) load(q0, r, label, wgt);
      for (uint32_t qb = q0; qb < q1; qb += kPartUnroll * kPartThreads) {
        const bool more = qb + kPartUnroll * kPartThreads < q1;
        if (more) load(qb + kPartUnroll * kPartThreads, rn, labn, wgn);
#pragma unroll
        for (int u = 0; u < kPartUnroll; u++) {
          const bool valid = label[u] >= 0 && wgt[u] > 0;
          const bool left = row_byte<BS>(r[u], sg.feat) <= sg.thr;  // bins are ranks
          const unsigned ml = __ballot_sync(kFull, valid && left && (sg.write & 1));
          const unsigned mr = __ballot_sync(kFull, valid && !left && (sg.write & 2));
          uint32_t base = 0;
          if (lane == 0 && ml) base = atomicAdd(&s_cur[0], __popc(ml));
          if (lane == 1 && mr) base = atomicAdd(&s_cur[1], __popc(mr));
          const bool wl = (ml >> lane) & 1, wr = (mr >> lane) & 1;
          const uint32_t bb = __shfl_sync(kFull, base, wl ? 0 : 1);  // lane 0: left base, 1: right
          const unsigned below = (1u << lane) - 1;
          const uint32_t pos = wl ? A + bb + __popc(ml & below) : B - 1 - (bb + __popc(mr & below));
          const bool w = wl || wr;
          if constexpr (BS >= 4) {  // predicated stores: no branch around them
            uint8_t *o = a.bins_out + (size_t)pos * 4;
#pragma unroll
            for (int i = 0; i < BS / 4; i++) st_cs_if(w, o + i * a.pstride, r[u].w[i]);
            st_cs_if_u8(w, a.lab_out + pos, (uint32_t)label[u]);
            if (a.w_out) st_cs_if_u8(w, a.w_out + pos, wgt[u]);
          } else if (w) {
            store_row<BS>(a.bins_out, a.pstride, pos, r[u]);
            __stcs(a.lab_out + pos, (uint8_t)label[u]);
            if (a.w_out) __stcs(a.w_out + pos, wgt[u]);
          }
        }
        if (more) {
#pragma unroll
          for (int u = 0; u < kPartUnroll; u++) {
            r[u] = rn[u];
            label[u] = labn[u];
            wgt[u] = wgn[u];
          }
        }
      }
    }
    __syncthreads();
    if (tid == 0 && visits < a.max_visits) {  // report this parent's share
      int32_t *v = my_visits + 6 * visits;
      v[0] = s_first;
      v[1] = (int32_t)A;
      v[2] = (int32_t)B;
      v[3] = (int32_t)s_cur[0];
      v[4] = (int32_t)s_cur[1];
      v[5] = 0;
    }
    visits++;
    p0 = pe;
  }
}

// ---------------------------------------------------- two-level moves --
// DESIGN.md §6 "two-level row moves": the rows move every other level.  The
// TAG pass runs where a partition would, over the same segments and ranges,
// but moves nothing: it reads the split feature's word plane and the labels,
// writes each row's label with bit 7 = "goes to the parent's direct child"
// into lab_tag (same position), and reports per parent share the counts of
// ALL rows going left / right.  The next level's histogram pass counts the
// marked rows straight from the parent's pieces; one level later MOVE4 moves
// every row to its grandchild's piece.
template <int BS>
__device__ __forceinline__ uint32_t feat_word(const uint8_t *__restrict__ base, size_t pstride, uint32_t row,
                                              int f, int &shift) {
  if constexpr (BS >= 4) {
    shift = 8 * (f & 3);
    return __ldcs(reinterpret_cast<const unsigned int *>(base + (size_t)(f >> 2) * pstride + (size_t)row * 4));
  } else if constexpr (BS == 2) {
    shift = 8 * f;
    return __ldcs(reinterpret_cast<const unsigned short *>(base + (size_t)row * 2));
  } else {
    shift = 0;
    return __ldcs(base + row);
  }
}

constexpr int kTagUnroll = 4;  // rows in flight per thread

template <int BS>
__global__ void __launch_bounds__(kPartThreads, kPartMinBlocks) tag_kernel(PartArgs a) {
  __shared__ uint32_t s_cnt[2];
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t R = (a.total_rows + gridDim.x - 1) / gridDim.x;
  uint32_t p0 = blockIdx.x * R;
  const uint32_t p1 = min(p0 + R, a.total_rows);
  int s = p0 < p1 ? first_seg(a.segs, a.nseg, p0) : a.nseg;
  int32_t *my_visits = a.visits + (size_t)blockIdx.x * a.max_visits * 6;
  int visits = 0;
  __syncthreads();
  while (p0 < p1 && s < a.nseg) {
    const Seg first = a.segs[s];
    const uint32_t pe = min(p1, first.node_base + first.node_len);
    if (tid == 0) s_cnt[0] = s_cnt[1] = 0;
    __syncthreads();
    const int s_first = s;
    uint32_t nl = 0, nr = 0;
    for (; s < a.nseg && a.segs[s].row_base < pe; s++) {
      const Seg sg = a.segs[s];
      if (!sg.write) continue;  // a parent that does not split (or whose children are leaves)
      const uint32_t q0 = p0 > sg.row_base ? p0 - sg.row_base : 0;
      const uint32_t q1 = min(sg.len, pe - sg.row_base);
      const uint32_t mark_left = sg.hslot == 0 ? 0x80u : 0u, mark_right = sg.hslot == 1 ? 0x80u : 0u;
      if constexpr (BS >= 4) {
        // the 4-aligned body as quads: one 16-byte load of the split feature's
        // word plane, one 4-byte label load and store per 4 rows; head / tail per row
        const uint32_t r0 = sg.off + q0, r1 = sg.off + q1;
        const uint32_t a4 = min((r0 + 3u) & ~3u, r1), b4 = max(a4, r1 & ~3u);
        const int shift = 8 * (sg.feat & 3);
        const uint8_t *plane = a.bins_in + (size_t)(sg.feat >> 2) * a.pstride;
        auto one = [&](uint32_t row) {
          const uint32_t w = *reinterpret_cast<const uint32_t *>(plane + (size_t)row * 4);
          const bool left = (int)((w >> shift) & 0xFFu) <= sg.thr;
          nl += left;
          nr += !left;
          a.lab_tag[row] = (uint8_t)(a.lab_in[row] | (left ? mark_left : mark_right));
        };
        if (tid < (int)(a4 - r0)) one(r0 + tid);
        if (tid >= 64 && tid < 64 + (int)(r1 - b4)) one(b4 + tid - 64);
        const uint32_t nq = (b4 - a4) >> 2;
        const uint4 *wq = reinterpret_cast<const uint4 *>(plane + (size_t)a4 * 4);
        const uint32_t *lq = reinterpret_cast<const uint32_t *>(a.lab_in + a4);
        uint32_t *oq = reinterpret_cast<uint32_t *>(a.lab_tag + a4);
#ifndef ADAPT_TAG_QU
#define ADAPT_TAG_QU 4
#endif
        constexpr int QU = ADAPT_TAG_QU;  // quads in flight per thread
        for (uint32_t qb = 0; qb < nq; qb += QU * kPartThreads) {
          uint4 w[QU];
          uint32_t l[QU];
#pragma unroll
          for (int u = 0; u < QU; u++) {
            const uint32_t qi = qb + u * kPartThreads + tid;
            if (qi < nq) {
              w[u] = __ldcs(wq + qi);
              l[u] = __ldcs(lq + qi);
            }
          }
#pragma unroll
          for (int u = 0; u < QU; u++) {
            const uint32_t qi = qb + u * kPartThreads + tid;
            if (qi < nq) {
              const uint32_t x[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
              uint32_t mark = 0;
#pragma unroll
              for (int c = 0; c < 4; c++) {
                const bool left = (int)((x[c] >> shift) & 0xFFu) <= sg.thr;
                nl += left;
                nr += !left;
                mark |= (left ? mark_left : mark_right) << (8 * c);
              }
              __stcs(oq + qi, l[u] | mark);
            }
          }
        }
      } else {
        for (uint32_t qb = q0; qb < q1; qb += kTagUnroll * kPartThreads) {
          uint32_t w[kTagUnroll], lab[kTagUnroll];
          int sh[kTagUnroll];
#pragma unroll
          for (int u = 0; u < kTagUnroll; u++) {  // all loads first
            const uint32_t q = qb + u * kPartThreads + tid;
            sh[u] = 0;
            w[u] = 0;
            lab[u] = 0;
            if (q < q1) {
              w[u] = feat_word<BS>(a.bins_in, a.pstride, sg.off + q, sg.feat, sh[u]);
              lab[u] = __ldcs(a.lab_in + sg.off + q);
            }
          }
#pragma unroll
          for (int u = 0; u < kTagUnroll; u++) {
            const uint32_t q = qb + u * kPartThreads + tid;
            if (q < q1) {
              const bool left = (int)((w[u] >> sh[u]) & 0xFFu) <= sg.thr;  // bins are ranks
              nl += left;
              nr += !left;
              __stcs(a.lab_tag + sg.off + q, (uint8_t)(lab[u] | (left ? mark_left : mark_right)));
            }
          }
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      nl += __shfl_xor_sync(kFull, nl, o);
      nr += __shfl_xor_sync(kFull, nr, o);
    }
    if (lane == 0 && (nl | nr)) {
      atomicAdd(&s_cnt[0], nl);
      atomicAdd(&s_cnt[1], nr);
    }
    __syncthreads();
    if (tid == 0 && visits < a.max_visits) {  // report this parent's share
      int32_t *v = my_visits + 6 * visits;
      v[0] = s_first;
      v[1] = (int32_t)p0;
      v[2] = (int32_t)pe;
      v[3] = (int32_t)s_cnt[0];
      v[4] = (int32_t)s_cnt[1];
      v[5] = 0;
    }
    visits++;
    p0 = pe;
  }
}

// MOVE4: one level after the TAG pass, over its segments and ranges.  A parent's
// share [A, B) splits at M = A + cL (cL = the TAG pass's left count of this
// share): left-left rows from A up, left-right from M down, right-left from M
// up, right-right from B down, positions from warp-aggregated cursors as in
// partition_kernel; rows of a grandchild that is not in the frontier stay behind.
#ifndef ADAPT_P4_UNROLL
#define ADAPT_P4_UNROLL 2
#endif
template <int BS>
__global__ void __launch_bounds__(kPartThreads, kPartMinBlocks) partition4_kernel(PartArgs a) {
  constexpr int kPartUnroll = ADAPT_P4_UNROLL;  // rows in flight per thread (this kernel)
  __shared__ uint32_t s_cur[4];
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t R = (a.total_rows + gridDim.x - 1) / gridDim.x;
  uint32_t p0 = blockIdx.x * R;
  const uint32_t p1 = min(p0 + R, a.total_rows);
  int s = p0 < p1 ? first_seg(a.segs, a.nseg, p0) : a.nseg;
  int32_t *my_visits = a.visits + (size_t)blockIdx.x * a.max_visits * 8;
  const int32_t *tag_visits = a.tag_visits + (size_t)blockIdx.x * a.max_visits * 6;
  int visits = 0;
  __syncthreads();
  while (p0 < p1 && s < a.nseg) {
    const Seg first = a.segs[s];
    const uint32_t pe = min(p1, first.node_base + first.node_len);
    const uint32_t A = p0, B = pe;
    // the TAG pass visited the same parents in the same order
    const uint32_t M = A + (visits < a.max_visits ? (uint32_t)tag_visits[6 * visits + 3] : 0u);
    if (tid < 4) s_cur[tid] = 0;
    __syncthreads();
    const int s_first = s;
    for (; s < a.nseg && a.segs[s].row_base < pe; s++) {
      const Seg sg = a.segs[s];
      if (!sg.write) continue;
      const int4 kl = a.kids[2 * s], kr = a.kids[2 * s + 1];
      if (!(kl.z | kr.z)) continue;  // no grandchild stays in the frontier
      const uint32_t q0 = p0 > sg.row_base ? p0 - sg.row_base : 0;
      const uint32_t q1 = min(sg.len, pe - sg.row_base);
      Row<BS> r[kPartUnroll], rn[kPartUnroll];
      int label[kPartUnroll], labn[kPartUnroll];
      auto load = [&](uint32_t qb, Row<BS>(&rr)[kPartUnroll], int(&ll)[kPartUnroll]) {
#pragma unroll
        for (int u = 0; u < kPartUnroll; u++) {
          const uint32_t q = qb + u * kPartThreads + tid;
          ll[u] = -1;
          if (q < q1) {
            load_row<BS>(a.bins_in, a.pstride, sg.off + q, rr[u]);
            ll[u] = __ldcs(a.lab_in + sg.off + q);
          } else {
#pragma unroll
            for (int i = 0; i < Row<BS>::N; i++) rr[u].w[i] = 0;
          }
        }
      };
      if (q0 < q1) load(q0, r, label);
      for (uint32_t qb = q0; qb < q1; qb += kPartUnroll * kPartThreads) {
        const bool more = qb + kPartUnroll * kPartThreads < q1;
        if (more) load(qb + kPartUnroll * kPartThreads, rn, labn);
#pragma unroll
        for (int u = 0; u < kPartUnroll; u++) {
          const bool left = row_byte<BS>(r[u], sg.feat) <= sg.thr;
          const int4 k = left ? kl : kr;
          const bool gl = k.x >= 0 && row_byte<BS>(r[u], max(k.x, 0)) <= k.y;
          const int code = (left ? 0 : 2) | (gl ? 0 : 1);
          const bool wr = label[u] >= 0 && (k.z & (gl ? 1 : 2));
          // the four grandchildren's lane masks from three ballots
          const unsigned bw = __ballot_sync(kFull, wr), b1 = __ballot_sync(kFull, wr && (code & 1)),
                         b2 = __ballot_sync(kFull, wr && (code & 2));
          const unsigned m[4] = {bw & ~(b1 | b2), b1 & ~b2, b2 & ~b1, b1 & b2};
          uint32_t base = 0;
          const unsigned ml = (lane & 2) ? ((lane & 1) ? m[3] : m[2]) : ((lane & 1) ? m[1] : m[0]);
          if (lane < 4 && ml) base = atomicAdd(&s_cur[lane], __popc(ml));
          const uint32_t bc = __shfl_sync(kFull, base, code);  // lane c holds code c's base
          // the lane's position without branches (selects on the code bits):
          // codes 0 / 2 grow up from A / M, codes 1 / 3 down from M / B
          const bool c1 = code & 1, c2 = code & 2;
          const unsigned mc = c2 ? (c1 ? m[3] : m[2]) : (c1 ? m[1] : m[0]);
          const uint32_t rk = bc + __popc(mc & ((1u << lane) - 1));
          const uint32_t edge = c2 ? (c1 ? B : M) : (c1 ? M : A);
          const uint32_t pos = c1 ? edge - 1 - rk : edge + rk;
          if (wr) {
            store_row<BS>(a.bins_out, a.pstride, pos, r[u]);
            __stcs(a.lab_out + pos, (uint8_t)label[u]);
          }
        }
        if (more) {
#pragma unroll
          for (int u = 0; u < kPartUnroll; u++) {
            r[u] = rn[u];
            label[u] = labn[u];
          }
        }
      }
    }
    __syncthreads();
    if (tid == 0 && visits < a.max_visits) {  // this parent's share and its four pieces
      int32_t *v = my_visits + 8 * visits;
      v[0] = s_first;
      v[1] = (int32_t)A;
      v[2] = (int32_t)B;
      v[3] = (int32_t)(M - A);
      v[4] = (int32_t)s_cur[0];
      v[5] = (int32_t)s_cur[1];
      v[6] = (int32_t)s_cur[2];
      v[7] = (int32_t)s_cur[3];
    }
    visits++;
    p0 = pe;
  }
}

// ------------------------------------------------------------ histogram --
constexpr int kHistThreads = 1024;
constexpr int kHistUnroll = ADAPT_HIST_UNROLL;  // rows in flight per thread (latency-bound otherwise)

// WEIGHTED (forests): rows add their bootstrap weight; a separate instance so
// the plain path keeps its registers (the weights cost 16 more per thread)
template <int BS, bool WEIGHTED>
__global__ void __launch_bounds__(kHistThreads, 1) hist_kernel(HistArgs a) {
  constexpr int UNROLL = WEIGHTED ? kHistUnroll / 2 : kHistUnroll;
  extern __shared__ uint32_t sh[];  // [smem_counters] counters
  __shared__ uint8_t s_cmap[kMaxC + 1];  // this node: class -> compact index (255: absent)
  const int tid = threadIdx.x;
  const HistCta ct = a.ctas[blockIdx.x];
  const int g = ct.g;
  const int4 grp = a.groups[g];  // x: first compact class, y: classes, w: bins word
  const int k0 = grp.x, kw = grp.y, w0 = grp.w;
  const int C = a.C;
  int Dw[4];  // distinct values of the 4 features of word w0 (0: absent)
#pragma unroll
  for (int e = 0; e < 4; e++) Dw[e] = (4 * w0 + e < a.F) ? a.nval[4 * w0 + e] : 0;
  uint32_t p0 = ct.p0;
  const uint32_t p1 = ct.p1;
  int s = p0 < p1 ? (ct.s0 >= 0 ? ct.s0 : first_seg(a.segs, a.nseg, p0)) : a.nseg;
  const uint32_t sbase = smem_u32(sh);
  while (p0 < p1 && s < a.nseg) {
    // ---- one node's rows at virtual positions [p0, pe) ----
    const Seg first = a.segs[s];
    if (first.len == 0) {  // an empty slot (device-built segments): the next one starts here too
      s++;
      continue;
    }
    const uint32_t pe = min(p1, first.node_base + first.node_len);
    // the node's classes are its compact columns; this CTA counts [k0, k0 + kn)
    const int kcn = first.ncls;
    const int kn = min(kw, kcn - k0);
    if (kn <= 0) {  // none of this node's classes fall in this CTA's slab
      while (s < a.nseg && a.segs[s].row_base < pe) s++;
      p0 = pe;
      continue;
    }
    const int kwp = kn | 1;  // odd stride: bank spread
    int gneed = 0;           // counters the smem path would zero and flush
#pragma unroll
    for (int e = 0; e < 4; e++) gneed += Dw[e] * kwp;
    if ((int64_t)(pe - p0) * 16 < gneed) {
      // a tiny portion (deep levels): count straight into the node's global
      // matrix (zeroed by zero_slots) — no smem zero/flush, no block barrier
      const uint8_t *m = a.cmaps + (size_t)first.cmap * C;
      uint32_t *dst = a.H + a.soff[first.hslot] + k0;
      int64_t fb[4];
#pragma unroll
      for (int e = 0; e < 4; e++) fb[e] = Dw[e] ? (int64_t)a.cumD[4 * w0 + e] * kcn : -1;
      for (; s < a.nseg && a.segs[s].row_base < pe; s++) {
        const Seg sg = a.segs[s];
        const uint32_t q0 = p0 > sg.row_base ? p0 - sg.row_base : 0;
        const uint32_t q1 = min(sg.len, pe - sg.row_base);
        for (uint32_t q = q0 + tid; q < q1; q += kHistThreads) {
          const uint32_t row = sg.off + q;
          uint32_t w;
          if constexpr (BS >= 4)
            w = *reinterpret_cast<const uint32_t *>(a.bins_in + w0 * a.pstride + (size_t)row * 4);
          else if constexpr (BS == 2)
            w = *reinterpret_cast<const unsigned short *>(a.bins_in + (size_t)row * 2);
          else
            w = a.bins_in[row];
          const uint32_t lb = a.lab_in[row];
          const int lk = (!a.tagged ? (int)__ldg(m + lb) : (lb & 0x80u) ? (int)__ldg(m + (lb & 0x7Fu)) : 255) - k0;
          const uint32_t wv = a.w_in ? a.w_in[row] : 1u;
          if ((unsigned)lk >= (unsigned)kn) continue;
#pragma unroll
          for (int e = 0; e < 4; e++)
            if (fb[e] >= 0) atomicAdd(dst + fb[e] + (int64_t)((w >> (8 * e)) & 0xFF) * kcn + lk, wv);
        }
      }
      p0 = pe;
      continue;
    }
    {
      const uint8_t *m = a.cmaps + (size_t)first.cmap * C;
      if (a.tagged)  // only labels marked by the TAG pass (bit 7) count
        for (int k = tid; k < kMaxC + 1; k += kHistThreads) s_cmap[k] = k >= 128 && k - 128 < C ? m[k - 128] : 255;
      else
        for (int k = tid; k < C; k += kHistThreads) s_cmap[k] = m[k];
    }
    uint32_t abase[4];
    int gcount = 0;
#pragma unroll
    for (int e = 0; e < 4; e++) {
      abase[e] = Dw[e] ? sbase + 4u * gcount : 0xFFFFFFFFu;
      gcount += Dw[e] * kwp;
    }
    const bool all4 = Dw[0] && Dw[1] && Dw[2] && Dw[3];
    const uint32_t kwp4 = 4u * kwp;
    for (int i = tid; i < gcount; i += kHistThreads) sh[i] = 0;
    if (tid == 0) s_cmap[255] = 255;  // label sentinel of the padded quad lanes
    __syncthreads();
    // one row: its word w (4 features), label, weight -> up to 4 reductions
    const uint32_t cmap_base = smem_u32(s_cmap);
    // a row's compact class column in this CTA's slab (kn or more: skip)
    auto column = [&](int label) { return (int)ld_shared_u8(cmap_base + label) - k0; };
    auto count_col = [&](uint32_t w, int lk, uint32_t wv) {
      if ((unsigned)lk >= (unsigned)kn) return;  // another CTA's class slab (or padding)
      const uint32_t lk4 = 4u * lk;
      if (all4) {
        red_shared_add(abase[0] + __byte_perm(w, 0, 0x4440) * kwp4 + lk4, wv);
        red_shared_add(abase[1] + __byte_perm(w, 0, 0x4441) * kwp4 + lk4, wv);
        red_shared_add(abase[2] + __byte_perm(w, 0, 0x4442) * kwp4 + lk4, wv);
        red_shared_add(abase[3] + __byte_perm(w, 0, 0x4443) * kwp4 + lk4, wv);
      } else {
#pragma unroll
        for (int e = 0; e < 4; e++)
          if (abase[e] != 0xFFFFFFFFu)
            red_shared_add(abase[e] + ((w >> (8 * e)) & 0xFF) * kwp4 + lk4, wv);
      }
    };
    auto count = [&](uint32_t w, int label, uint32_t wv) { count_col(w, column(label), wv); };
    auto load_word = [&](uint32_t row) -> uint32_t {
      if constexpr (BS >= 4)
        return *reinterpret_cast<const uint32_t *>(a.bins_in + w0 * a.pstride + (size_t)row * 4);
      else if constexpr (BS == 2)
        return *reinterpret_cast<const unsigned short *>(a.bins_in + (size_t)row * 2);
      else
        return a.bins_in[row];
    };
    for (; s < a.nseg && a.segs[s].row_base < pe; s++) {
      const Seg sg = a.segs[s];
      const uint32_t q0 = p0 > sg.row_base ? p0 - sg.row_base : 0;
      const uint32_t q1 = min(sg.len, pe - sg.row_base);
      if constexpr (BS >= 4) {
        // rows [r0, r1): the 4-aligned body as quads (one 16-byte word load and
        // one 4-byte label load per 4 rows), the unaligned head / tail per row
        const uint32_t r0 = sg.off + q0, r1 = sg.off + q1;
        const uint32_t a4 = min((r0 + 3u) & ~3u, r1), b4 = max(a4, r1 & ~3u);
        if (tid < (int)(a4 - r0)) {
          const uint32_t row = r0 + tid;
          count(load_word(row), a.lab_in[row], WEIGHTED ? a.w_in[row] : 1u);
        }
        if (tid >= 64 && tid < 64 + (int)(r1 - b4)) {
          const uint32_t row = b4 + tid - 64;
          count(load_word(row), a.lab_in[row], WEIGHTED ? a.w_in[row] : 1u);
        }
        const uint32_t nq = (b4 - a4) >> 2;
        const uint4 *wq = reinterpret_cast<const uint4 *>(a.bins_in + w0 * a.pstride + (size_t)a4 * 4);
        const uint32_t *lq = reinterpret_cast<const uint32_t *>(a.lab_in + a4);
        const uint32_t *vq = WEIGHTED ? reinterpret_cast<const uint32_t *>(a.w_in + a4) : nullptr;
        constexpr int QU = UNROLL / 4 > 0 ? UNROLL / 4 : 1;  // quads in flight per thread
        for (uint32_t qb = 0; qb < nq; qb += QU * kHistThreads) {
          uint4 w[QU];
          uint32_t l[QU], v[WEIGHTED ? QU : 1];
#pragma unroll
          for (int u = 0; u < QU; u++) {  // all loads first
            const uint32_t qi = qb + u * kHistThreads + tid;
            l[u] = 0xFFFFFFFFu;
            w[u] = make_uint4(0, 0, 0, 0);
            if (qi < nq) {
              w[u] = __ldcs(wq + qi);
              l[u] = __ldcs(lq + qi);
              if constexpr (WEIGHTED) v[u] = __ldcs(vq + qi);
            }
          }
          int lk[QU][4];  // every class-map lookup first (independent), then the reductions
#pragma unroll
          for (int u = 0; u < QU; u++)
#pragma unroll
            for (int c = 0; c < 4; c++) lk[u][c] = column((l[u] >> (8 * c)) & 0xFF);
#pragma unroll
          for (int u = 0; u < QU; u++) {
            count_col(w[u].x, lk[u][0], WEIGHTED ? (v[u] & 0xFF) : 1u);
            count_col(w[u].y, lk[u][1], WEIGHTED ? ((v[u] >> 8) & 0xFF) : 1u);
            count_col(w[u].z, lk[u][2], WEIGHTED ? ((v[u] >> 16) & 0xFF) : 1u);
            count_col(w[u].w, lk[u][3], WEIGHTED ? (v[u] >> 24) : 1u);
          }
        }
      } else {
        for (uint32_t qb = q0; qb < q1; qb += UNROLL * kHistThreads) {
          uint32_t w[UNROLL];
          int label[UNROLL];
          uint32_t wv[UNROLL];
#pragma unroll
          for (int u = 0; u < UNROLL; u++) {  // all loads first: only this CTA's word
            const uint32_t q = qb + u * kHistThreads + tid;
            label[u] = 255;
            w[u] = 0;
            wv[u] = 1;
            if (q < q1) {
              const uint32_t row = sg.off + q;
              w[u] = load_word(row);
              label[u] = a.lab_in[row];
              if constexpr (WEIGHTED) wv[u] = a.w_in[row];
            }
          }
#pragma unroll
          for (int u = 0; u < UNROLL; u++) count(w[u], label[u], wv[u]);
        }
      }
    }
    __syncthreads();
    {  // flush into the node's [DS][kcn] matrix: row cumD[f] + rank, column k0 + j.
       // A CTA that saw ALL of the node's rows (the common case at deep levels)
       // owns its columns: plain stores of every counter, no atomics.
      const bool sole = p0 <= first.node_base && pe >= first.node_base + first.node_len;
      uint32_t *dst = a.H + a.soff[first.hslot];
      // the word's features are consecutive rows of both layouts (smem stride
      // kwp, global stride kcn), so the flush is ONE flat pass over Rt rows;
      // each thread steps its (row, column) by the block size without dividing
      const int Rt = Dw[0] + Dw[1] + Dw[2] + Dw[3];
      uint32_t *df = dst + (int64_t)a.cumD[4 * w0] * kcn + k0;
      const int width = sole ? kn : kwp;
      const int n = Rt * width;
      const int qs = kHistThreads / width, rs = kHistThreads - qs * width;
      int rk = tid / width, j = tid - rk * width;
#pragma unroll 4
      for (int i = tid; i < n; i += kHistThreads) {
        if (sole) {  // dense [rank][kn] block of this CTA's columns
          df[rk * kcn + j] = sh[rk * kwp + j];
        } else {
          const uint32_t val = sh[i];
          if (val) atomicAdd(df + rk * kcn + j, val);
        }
        rk += qs;
        j += rs;
        if (j >= width) j -= width, rk++;
      }
    }
    __syncthreads();
    p0 = pe;
  }
}

// Histogram segments from the partition's share reports (SegBuildArgs), one
// CTA: scatter every report's direct-child piece into its slot, then an
// exclusive scan of the slot lengths per list gives the virtual positions; a
// node whose first slot does not start at its planned base (or a list whose
// total differs) flags an error for the host.
constexpr int kBuildThreads = 1024;
__global__ void __launch_bounds__(kBuildThreads) build_hist_segs_kernel(SegBuildArgs a) {
  __shared__ uint32_t s_warp[kBuildThreads / 32];
  __shared__ uint32_t s_carry;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nent = a.nranges * a.max_visits;
  for (int i = tid; i < nent && !a.mode4; i += blockDim.x) {
    const int32_t *e = a.visits + (size_t)i * 6;
    if (e[0] < 0) continue;
    const int4 info = a.bseg[e[0]];
    if (info.x < 0) continue;
    Seg &sg = a.segs[info.y][info.z + i / a.max_visits];
    sg.off = info.x == 0 ? (uint32_t)e[1] : (uint32_t)(e[2] - e[4]);
    sg.len = (uint32_t)(info.x == 0 ? e[3] : e[4]);
  }
  // MOVE4: a share [A, B) split at M = A + cL holds LL [A, +n0), LR
  // [M - n1, M), RL [M, +n2), RR [B - n3, B); each child's direct grandchild
  for (int i = tid; i < nent && a.mode4; i += blockDim.x) {
    const int32_t *e = a.visits + (size_t)i * 8;
    if (e[0] < 0) continue;
    const uint32_t A = (uint32_t)e[1], B = (uint32_t)e[2], M = A + (uint32_t)e[3];
#pragma unroll
    for (int c = 0; c < 2; c++) {
      const int4 info = a.bseg[2 * e[0] + c];
      if (info.x < 0) continue;
      Seg &sg = a.segs[info.y][info.z + i / a.max_visits];
      const uint32_t n = (uint32_t)e[4 + info.x];
      sg.off = info.x == 0 ? A : info.x == 1 ? M - n : info.x == 2 ? M : B - n;
      sg.len = n;
    }
  }
  __syncthreads();
  for (int l = 0; l < 2; l++) {
    Seg *sg = a.segs[l];
    const int n = a.nslot[l];
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (int c0 = 0; c0 < n; c0 += blockDim.x) {
      const int i = c0 + tid;
      const uint32_t len = i < n ? sg[i].len : 0u;
      uint32_t x = len;  // inclusive warp scan, then across warps
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_warp[wid] = x;
      __syncthreads();
      if (wid == 0) {
        uint32_t w = s_warp[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, w, o);
          if (lane >= o) w += y;
        }
        s_warp[lane] = w;  // inclusive over warps
      }
      __syncthreads();
      const uint32_t carry = s_carry;
      const uint32_t excl = carry + (wid ? s_warp[wid - 1] : 0u) + x - len;
      if (i < n) {
        sg[i].row_base = excl;
        if ((i == 0 || sg[i - 1].hslot != sg[i].hslot) && excl != sg[i].node_base) *a.err = 1;
      }
      __syncthreads();
      if (tid == 0) s_carry = carry + s_warp[31];
      __syncthreads();
    }
    if (tid == 0 && s_carry != a.total[l]) *a.err = 1;
    __syncthreads();
  }
}

// Small direct nodes (deep levels): a flat pass over their rows, one thread
// per row and all F features, counting straight into each node's global
// matrix (zeroed by zero_slots).  A node's smem block would cost more to zero
// and flush than its few rows cost in global atomics.
template <int BS>
__global__ void __launch_bounds__(256) hist_flat_kernel(HistArgs a) {
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < a.total_rows;
       p = (uint32_t)min((uint64_t)p + gridDim.x * blockDim.x, (uint64_t)a.total_rows)) {
    const Seg sg = a.segs[first_seg(a.segs, a.nseg, p)];
    const uint32_t row = sg.off + (p - sg.row_base);
    Row<BS> r;
    load_row<BS>(a.bins_in, a.pstride, row, r);
    const int kcn = sg.ncls;
    const uint32_t lb = a.lab_in[row];
    if (a.tagged && !(lb & 0x80u)) continue;  // not the direct child's row
    const int lk = (int)__ldg(a.cmaps + (size_t)sg.cmap * a.C + (a.tagged ? lb & 0x7Fu : lb));
    const uint32_t wv = a.w_in ? a.w_in[row] : 1u;
    uint32_t *dst = a.H + a.soff[sg.hslot] + lk;
#pragma unroll
    for (int i = 0; i < Row<BS>::N; i++)
#pragma unroll
      for (int e = 0; e < (BS >= 4 ? 4 : BS); e++) {
        const int f = 4 * i + e;
        if (f < a.F)
          atomicAdd(dst + (int64_t)(__ldg(a.cumD + f) + (int)((r.w[i] >> (8 * e)) & 0xFF)) * kcn, wv);
      }
  }
}

// The next partition's decisions on the device, straight from the winner
// records (so it launches right behind the winner kernel, without a host round
// trip): per segment (a piece of frontier node j = seg.direct), the split
// feature / rank and which children stay in the frontier, by the rule the host
// applies to the same records (engine.cpp decide, R10 / R11): a node splits
// when depth < D, it has a cut, and more than one class is present; a child
// stays when depth + 1 < D and it holds more than one class.
// node j's split (feat, rank) and which children stay (write bits), from its record
__device__ __forceinline__ int decide_node(const uint8_t *res, const int64_t *rec_off, const int32_t *node_kc,
                                           const int32_t *node_depth, int D, int j, bool last_rule, int *feat,
                                           int *thr, int *side) {
  const NodeRes *nr = reinterpret_cast<const NodeRes *>(res + rec_off[j]);
  const uint32_t *Pd = reinterpret_cast<const uint32_t *>(nr + 1);
  const int kc = node_kc[j];
  const uint32_t *cLd = Pd + kc;
  int np = 0, npl = 0, npr = 0;
  for (int k = 0; k < kc; k++) {
    const uint32_t p = Pd[k], l = cLd[k];
    np += p > 0;
    npl += l > 0;
    npr += p - l > 0;
  }
  const int depth = node_depth[j];
  int write = 0;
  *side = -1;
  if (depth < D && np > 1 && nr->valid) {
    write = (depth + 1 < D && npl > 1 ? 1 : 0) | (depth + 1 < D && npr > 1 ? 2 : 0);
    // the direct child: the smaller when both stay (ties left — the host's rule)
    *side = write == 3 ? (nr->nL <= nr->n - nr->nL ? 0 : 1) : write == 1 ? 0 : write == 2 ? 1 : -1;
    // children on the LAST frontier level (depth D - 1) are never partitioned
    // again: only the direct child's rows are needed
    if (last_rule && depth + 2 == D && write == 3) write = *side == 0 ? 1 : 2;
    *feat = nr->feat;
    *thr = nr->b_lo;
  }
  return write;
}

__global__ void __launch_bounds__(256) decide_kids_kernel(const int2 *kid_j, int nseg, const uint8_t *res,
                                                          const int64_t *rec_off, const int32_t *node_kc,
                                                          const int32_t *node_depth, int D, int4 *kids) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nseg) return;
  const int2 jj = kid_j[i];
#pragma unroll
  for (int c = 0; c < 2; c++) {
    const int j = c ? jj.y : jj.x;
    int feat = -1, thr = 0, side = -1, write = 0;
    if (j >= 0) write = decide_node(res, rec_off, node_kc, node_depth, D, j, true, &feat, &thr, &side);
    kids[2 * i + c] = make_int4(write ? feat : -1, thr, write, 0);
  }
}

__global__ void __launch_bounds__(256) decide_segs_kernel(Seg *segs, int nseg, const uint8_t *res,
                                                          const int64_t *rec_off, const int32_t *node_kc,
                                                          const int32_t *node_depth, int D, int tag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nseg) return;
  Seg &sg = segs[i];
  const int j = sg.direct;
  if (tag) {  // TAG pass: both children's rows are marked / counted; hslot = the direct side
    int feat = -1, thr = 0, side = -1;
    sg.write = decide_node(res, rec_off, node_kc, node_depth, D, j, false, &feat, &thr, &side);
    if (sg.write) sg.feat = feat, sg.thr = thr;
    sg.hslot = side;
    return;
  }
  const NodeRes *nr = reinterpret_cast<const NodeRes *>(res + rec_off[j]);
  const uint32_t *Pd = reinterpret_cast<const uint32_t *>(nr + 1);
  const int kc = node_kc[j];
  const uint32_t *cLd = Pd + kc;
  int np = 0, npl = 0, npr = 0;
  for (int k = 0; k < kc; k++) {
    const uint32_t p = Pd[k], l = cLd[k];
    np += p > 0;
    npl += l > 0;
    npr += p - l > 0;
  }
  const int depth = node_depth[j];
  int write = 0;
  if (depth < D && np > 1 && nr->valid) {
    write = (depth + 1 < D && npl > 1 ? 1 : 0) | (depth + 1 < D && npr > 1 ? 2 : 0);
    // children on the LAST frontier level (depth D - 1) are histogrammed and
    // split-searched but never partitioned again: only the direct (smaller,
    // ties left — the host's rule) child's rows are needed; the other child's
    // histogram is parent - direct
    if (depth + 2 == D && write == 3) write = nr->nL <= nr->n - nr->nL ? 1 : 2;
    sg.feat = nr->feat;
    sg.thr = nr->b_lo;
  }
  sg.write = write;
}

}  // namespace

void launch_build_hist_segs(const SegBuildArgs &a, cudaStream_t s) {
  build_hist_segs_kernel<<<1, kBuildThreads, 0, s>>>(a); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
}


void launch_decide_segs(Seg *segs, int nseg, const uint8_t *res, const int64_t *rec_off,
                        const int32_t *node_kc, const int32_t *node_depth, int D, cudaStream_t s, int tag) {
  if (nseg == 0) return;
  decide_segs_kernel<<<(nseg + 255) / 256, 256, 0, s>>>(segs, nseg, res, rec_off, node_kc, node_depth, D, tag); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
}

void launch_decide_kids(const int2 *kid_j, int nseg, const uint8_t *res, const int64_t *rec_off,
                        const int32_t *node_kc, const int32_t *node_depth, int D, int4 *kids, cudaStream_t s) {
  if (nseg == 0) return;
  decide_kids_kernel<<<(nseg + 255) / 256, 256, 0, s>>>(kid_j, nseg, res, rec_off, node_kc, node_depth, D, kids); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
}

void launch_tag(const PartArgs &a, cudaStream_t s) {
  if (a.total_rows == 0 || a.nseg == 0) return;
  switch (a.BS) {
#define CASE(B)                                                                               \
  case B:                                                                                     \
    tag_kernel<B><<<a.nranges, kPartThreads, 0, s>>>(a); ++g_kernel_launches;                 \
    break;
    CASE(1) CASE(2) CASE(4) CASE(8) CASE(16) CASE(32) CASE(64)
#undef CASE
    default:
      throw Error(-1, "bad bins stride");
  }
  CUDA_CHECK(cudaGetLastError());
}

void launch_partition4(const PartArgs &a, cudaStream_t s) {
  if (a.total_rows == 0 || a.nseg == 0) return;
  switch (a.BS) {
#define CASE(B)                                                                               \
  case B:                                                                                     \
    partition4_kernel<B><<<a.nranges, kPartThreads, 0, s>>>(a); ++g_kernel_launches;          \
    break;
    CASE(1) CASE(2) CASE(4) CASE(8) CASE(16) CASE(32) CASE(64)
#undef CASE
    default:
      throw Error(-1, "bad bins stride");
  }
  CUDA_CHECK(cudaGetLastError());
}

void ensure_smem_limit(const void *func, size_t bytes) {
  // cudaFuncSetAttribute applies per device: cache per (device, function)
  static std::map<std::pair<int, const void *>, size_t> set;
  int dev = 0;
  CUDA_CHECK(cudaGetDevice(&dev));
  size_t &cur = set[{dev, func}];
  if (bytes <= cur) return;
  CUDA_CHECK(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  cur = bytes;
}

int partition_ranges(int sms, uint32_t total_rows) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((total_rows + 4095) / 4096,
                                                      (int64_t)kPartMinBlocks * sms));
}

void launch_partition(const PartArgs &a, cudaStream_t s) {
  if (a.total_rows == 0 || a.nseg == 0) return;
  switch (a.BS) {
#define CASE(B)                                                                               \
  case B:                                                                                     \
    partition_kernel<B><<<a.nranges, kPartThreads, 0, s>>>(a); ++g_kernel_launches;                                \
    break;
    CASE(1) CASE(2) CASE(4) CASE(8) CASE(16) CASE(32) CASE(64)
#undef CASE
    default:
      throw Error(-1, "bad bins stride");
  }
  CUDA_CHECK(cudaGetLastError());
}

void launch_hist_flat(const HistArgs &a, cudaStream_t s) {
  if (a.total_rows == 0 || a.nseg == 0) return;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>((a.total_rows + 255) / 256, 8 * sms);
  switch (a.BS) {
#define CASE(B)                                                 \
  case B:                                                       \
    hist_flat_kernel<B><<<grid, 256, 0, s>>>(a); ++g_kernel_launches;                \
    break;
    CASE(1) CASE(2) CASE(4) CASE(8) CASE(16) CASE(32) CASE(64)
#undef CASE
    default:
      throw Error(-1, "bad bins stride");
  }
  CUDA_CHECK(cudaGetLastError());
}

void launch_hist(const HistArgs &a, cudaStream_t s) {
  if (a.total_rows == 0 || a.nseg == 0 || a.nctas == 0) return;
  const size_t smem = (size_t)a.smem_counters * 4;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.nctas);
  cfg.blockDim = dim3(kHistThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.numAttrs = 0;
  switch (a.BS) {
#define CASE(B)                                                                              \
  case B:                                                                                    \
    if (a.w_in) {                                                                            \
      smem_limit(hist_kernel<B, true>, smem);                                                \
      CUDA_CHECK(cudaLaunchKernelEx(&cfg, hist_kernel<B, true>, a)); ++g_kernel_launches;                         \
    } else {                                                                                 \
      smem_limit(hist_kernel<B, false>, smem);                                               \
      CUDA_CHECK(cudaLaunchKernelEx(&cfg, hist_kernel<B, false>, a)); ++g_kernel_launches;                        \
    }                                                                                        \
    break;
    CASE(1) CASE(2) CASE(4) CASE(8) CASE(16) CASE(32) CASE(64)
#undef CASE
    default:
      throw Error(-1, "bad bins stride");
  }
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace adapt
