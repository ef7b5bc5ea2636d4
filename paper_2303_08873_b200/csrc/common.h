// common.h — internal declarations shared by the engine's host code and its
// sm_100a kernels.  Not part of the C ABI (see include/adapt.h).
#pragma once
#include <cuda_runtime.h>

#include "adapt.h"

#include <cstdint>
#include <stdexcept>
#include <string>

namespace adapt {
// every kernel this library launches bumps this (host side, under the library
// lock): the profile's per-phase launch counts are differences of it
extern long long g_kernel_launches;

constexpr int kMaxF = 64;          // features per region (adapt.h)
constexpr int kMaxC = 255;         // variants = classes (adapt.h)
constexpr int kMaxBins = 256;      // lossless bins per feature (R14)
constexpr int kGSlots = 1024;      // global value-discovery hash slots per feature
constexpr uint32_t kEmptyKey = 0xFFFFFFFFu;  // a NaN pattern: never a valid (finite) key
constexpr uint32_t kPendingId = 0xFFFFFFFFu;

// ingest error flags (atomicOr'ed by the kernels)
constexpr uint32_t kFlagBadFeature = 1;   // NaN/Inf feature (R4)
constexpr uint32_t kFlagNanTime = 2;      // NaN time (R3)
constexpr uint32_t kFlagAllInf = 4;       // every variant unmeasured (R3)
constexpr uint32_t kFlagTooMany = 8;      // > 256 distinct values of a feature (R14)
constexpr uint32_t kFlagBadVariant = 16;  // recorded variant outside [0, V)
constexpr uint32_t kFlagUnseen = 32;      // bin pass met a value the (sampled) discovery missed

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char *what);
#define CUDA_CHECK(x) ::adapt::cuda_check((x), #x)

// ---- one segment of a row pass (host-built, read by level.cu's kernels) ----
// A segment is one piece [off, off+len) of a parent node's rows in the level's
// input planes (a node's rows may lie in several pieces, consecutive in the
// segment list).  Concatenating the segments gives every row a "virtual
// position"; the output planes are indexed by it.  The pass moves the rows
// (feat >= 0): each CTA takes a contiguous share [A, B) of a node's virtual
// positions inside its range and writes that share's left rows at [A, ...)
// and right rows at [..., B) — the children's pieces for the next level — and
// accumulates the class histogram of the "direct" child (or of all rows for
// the root pass).
struct Seg {
  uint32_t off;        // piece start (row position in the level's input planes)
  uint32_t len;        // rows of this rank in the piece
  uint32_t row_base;   // virtual position: prefix sum of len over previous segments
  uint32_t node_base;  // virtual position of the first piece of this segment's node
  uint32_t node_len;   // rows of the node (all its pieces)
  int32_t feat;        // split feature, -1 = no partition (root pass)
  int32_t thr;         // rank b_lo: rank <= thr goes left
  int32_t direct;      // 0: histogram rows going left, 1: right, 2: all rows, -1: none
  int32_t hslot;       // histogram slot of the direct child (-1: none)
  int32_t write;       // bit0: move left rows to the output planes, bit1: right rows
  int32_t cmap;        // histogram pass: this node's class map (index into HistArgs::cmaps)
  int32_t ncls;        // histogram pass: classes present in the node
};

// best cut of one (node, feature), exact key num/den (R13x)
struct SplitCand {
  uint64_t num_lo, num_hi;  // SL*nR + SR*nL  (< 2^97)
  uint64_t den;             // nL*nR          (< 2^64)
  uint64_t nL;              // rows at or left of the cut (global)
  int32_t valid;            // a cut exists
  int32_t b_lo, b_hi;       // ranks of the consecutive node-nonempty bins around the cut
  int32_t pad;
};

// per-node outcome of the split search (device -> host once per level)
struct NodeRes {
  uint64_t n;               // rows in node (global)
  uint64_t nL;              // rows left of the winning cut
  int32_t valid, feat, b_lo, b_hi;
  // followed in memory by uint32 P[kc] (class totals) and uint32 cL[kc], compact
  // class order (node j's record starts at res_off[j]: sizeof(NodeRes) + 8 kc_j, 8-aligned)
};

// Raise a kernel's dynamic shared-memory limit only when a launch needs more
// than what was set before (cudaFuncSetAttribute costs microseconds per call;
// launchers run under the library's mutex).
void ensure_smem_limit(const void *func, size_t bytes);
template <class K>
inline void smem_limit(K *kernel, size_t bytes) {
  ensure_smem_limit(reinterpret_cast<const void *>(kernel), bytes);
}

// ---- kernel launchers (records.cu): long-format records -> wide rows ----
size_t rec_table_slots(int64_t m);  // hash-set slots for m records (power of two >= 2m)
int rec_scan_blocks(int64_t m);     // blocks of the group-id scan
// groups the m records; *d_groups (device) = number of distinct vectors
void launch_rec_group(const float *feat, const int32_t *var, int64_t m, int F, int V,
                      uint32_t *slot_rep, uint32_t *slot_first, size_t slots, uint32_t *slot_of,
                      uint32_t *flag, uint32_t *bsum, uint32_t *d_groups, uint32_t *flags,
                      cudaStream_t s);
// wide rows in order of first appearance; *pairs (device, optional) = measured cells
void launch_rec_wide(const float *feat, const int32_t *var, const uint64_t *ns, int64_t m, int F,
                     int V, const uint32_t *slot_of, uint32_t *slot_gid, const uint32_t *flag,
                     const uint32_t *bsum, int64_t groups, unsigned long long *sum, uint32_t *cnt,
                     float *wide_feat, float *wide_times, uint32_t *pairs, cudaStream_t s);

// ---- kernel launchers (ingest.cu) ----
int lookup_table_bytes(int F);  // size of the per-feature key -> rank perfect hashes
// n rows; chunk_rows > 0: a sampled view, row i -> i + (i / chunk_rows) * gap_rows
void launch_discover(const float *feat, int64_t n, int F, uint32_t *gkey, uint32_t *gcount,
                     uint32_t *flags, int64_t chunk_rows, int64_t gap_rows, cudaStream_t s);
void launch_collect_values(const uint32_t *gkey, const uint32_t *gcount, int F, float *local_vals,
                           int32_t *local_cnt, cudaStream_t s);
void launch_merge_values(const float *all_vals, const int32_t *all_cnt, int world, int F,
                         float *val, int32_t *nval, uint32_t *flags, cudaStream_t s);
bool build_value_hash(const float *vals, int D, uint32_t mul[2], uint8_t *tab, uint32_t *slot_keys);
int lookup_slots();  // hash slots per feature (slot_keys entries)
void launch_label_bin(const float *feat, const float *times, int64_t n, int F, int V, int BS,
                      const uint8_t *tab, const uint32_t *lk_mul, const uint32_t *slot_keys,
                      int verify, uint32_t *flags, uint8_t *bins, size_t pstride, uint8_t *labels,
                      cudaStream_t s);
void launch_bins_out(const uint8_t *bins, size_t pstride, int64_t n, int F, int BS, uint8_t *out,
                     cudaStream_t s);
// bytes between the bins word planes of an n-row buffer (plane p = bytes [4p, 4p+4) of each row)
inline size_t bins_plane_stride(int64_t n, int BS) {
  const size_t wb = BS < 4 ? BS : 4;
  return (((size_t)(n + 16) * wb) + 255) & ~(size_t)255;
}
inline size_t bins_bytes(int64_t n, int BS) {
  return bins_plane_stride(n, BS) * (BS < 4 ? 1 : BS / 4);
}

// ---- kernel launchers (level.cu) ----
struct PartArgs {            // a7: move the split parents' rows into the children's pieces
  const Seg *segs;           // pieces of the split parents (feat, thr, write set)
  int nseg;
  uint32_t total_rows;       // sum of the pieces' lengths (virtual positions)
  const uint8_t *bins_in, *lab_in;  // input: bins word planes (see level.cu), labels [pos]
  uint8_t *bins_out, *lab_out;      // output planes, indexed by virtual position
  const uint8_t *w_in;              // forests: bootstrap weight plane (null: every row weighs 1);
  uint8_t *w_out;                   //   rows of weight 0 are dropped, the plane moves with the rows
  size_t pstride;                   // bytes between bins word planes
  int BS, F;
  int32_t *visits;           // [nranges][max_visits][6]: seg, share [A, B), left, right moved
                             //   (two-level move: [8]: seg, A, B, cL, LL, LR, RL, RR moved)
  int max_visits;
  int nranges;               // CTAs, one row range each
  // Two-level schedule (DESIGN.md §6 "two-level row moves"): the rows move only
  // every other level.  TAG pass (launch_tag): no row moves; each split
  // parent's row gets bit 7 of its label set in lab_tag[row] (same position as
  // the input planes) when it goes to the parent's direct child (seg.hslot =
  // that side, 0 left / 1 right), and the share reports count every left /
  // right row.  MOVE4 pass (launch_partition4): the same segments and ranges
  // one level later; each row goes to one of its parent's four grandchildren
  // (kids[2 s + c] = child c's (feat, thr, write) from its winner record), the
  // parent's share [A, B) split at A + cL (cL from the tag pass's reports).
  uint8_t *lab_tag;          // TAG: tagged labels out
  const int32_t *tag_visits; // MOVE4: the TAG pass's share reports ([6] per visit)
  const int4 *kids;          // MOVE4: per segment, per child
};
int partition_ranges(int sms, uint32_t total_rows);
void launch_partition(const PartArgs &a, cudaStream_t s);
void launch_tag(const PartArgs &a, cudaStream_t s);
void launch_partition4(const PartArgs &a, cudaStream_t s);
// MOVE4's per-child decisions from the tagged level's winner records:
// kid_j[s] = the two children (frontier indices, -1: none) of segment s's
// parent; kids[2 s + c] = (feat, thr, write, 0) by decide_segs' rule
void launch_decide_kids(const int2 *kid_j, int nseg, const uint8_t *res, const int64_t *rec_off,
                        const int32_t *node_kc, const int32_t *node_depth, int D, int4 *kids,
                        cudaStream_t s);
// the partition's per-segment split / write decisions from the winner records
// (node j's record at res + rec_off[j]); segs[i].direct = the segment's node
// tag != 0 (TAG pass): also seg.hslot = the side of the parent's direct child
// (0 left, 1 right, -1 none), and the last-level single-child rule is not applied
void launch_decide_segs(Seg *segs, int nseg, const uint8_t *res, const int64_t *rec_off,
                        const int32_t *node_kc, const int32_t *node_depth, int D, cudaStream_t s,
                        int tag = 0);

// The histogram segments built on the device from the partition's share
// reports (single-rank, unweighted levels: the host planned every node's size
// and slot range from the winners, so nothing waits for the host between the
// partition and the histogram).  Slot slot0 + b of a direct child holds its
// piece from partition range b; row_base = exclusive prefix of the slots' len.
struct SegBuildArgs {
  int mode4;                 // MOVE4 reports ([8] per visit) with two bseg entries per segment
                             // (one per child of the parent: x = code of its direct grandchild)
  const int32_t *visits;     // the partition's share reports [nranges][max_visits][6]
  int nranges, max_visits;
  const int4 *bseg;          // per partition segment: x side of the parent's direct
                             // child (0 left, 1 right, -1 none), y list (0 big, 1 small), z slot0 - b0
  Seg *segs[2];              // per list: slot templates (node fields set, len 0) -> filled
  int nslot[2];
  uint32_t total[2];         // planned rows per list
  int32_t *err;              // set to 1 when the pieces disagree with the planned sizes
};
void launch_build_hist_segs(const SegBuildArgs &a, cudaStream_t s);

// Node histograms are stored class-compacted: node j with kc_j present classes
// (ascending class ids) is a [DS][kc_j] u32 matrix, DS = sum_f D_f; feature f's
// rows are [cumD_f, cumD_f + D_f), row = rank, column = compact class index.
// A level's nodes are concatenated: node j at element offset off_j.
struct HistCta {             // one histogram CTA's work: group g, virtual rows [p0, p1)
  int32_t g;                 // from segment s0 on (the segment holding p0)
  uint32_t p0, p1;
  int32_t s0;
};
struct HistArgs {            // a4: class histograms of the given pieces' rows
  const Seg *segs;           // pieces (off, len, row_base, node_base/len, hslot, cmap, ncls), grouped by node
  int nseg;
  uint32_t total_rows;
  const uint8_t *bins_in, *lab_in;
  const uint8_t *w_in;       // forests: row weights (bootstrap multiplicities); null: 1
  size_t pstride;            // bytes between bins word planes
  int BS, F, C;
  const int32_t *cumD;       // [F] first histogram row of feature f
  const int32_t *nval;       // [F] distinct values of f
  const int4 *groups;        // [ngroups] x: first compact class, y: classes, z: padded stride, w: bins word
  const uint8_t *cmaps;      // [direct nodes][C]: class -> compact index (255: absent)
  int ngroups;
  int smem_counters;         // max counters of a group
  uint32_t *H;               // level histograms
  const int64_t *soff;       // [slots] element offset of a slot's matrix in H
  const HistCta *ctas;       // [nctas] per-CTA work (cost-balanced on the host)
  int nctas;
  int tagged;                // rows are the PARENT's pieces; count only labels with bit 7
                             // (the TAG pass's mark of the direct child), class = label & 127
};
void launch_hist(const HistArgs &a, cudaStream_t s);
void launch_hist_flat(const HistArgs &a, cudaStream_t s);  // small nodes: thread per row

struct SubJob {              // derived node = parent - direct sibling, class-remapped
  int64_t off_d, off_p, off_s;  // element offsets: derived (H), parent (Hprev), sibling (H)
  int32_t kc_d, kc_p, kc_s;     // their class counts
  int32_t map;                  // first entry in the map array: per derived class
};                              // (parent column, sibling column or -1) as int16 pairs

// ---- kernel launchers (train.cu) ----
// zero / subtract work in chunks: cstart[j] = first chunk of job j (prefix of
// chunk_count(elements of job j)), nblocks = total chunks
int chunk_count(int64_t elems);
// zslot (optional): job k zeroes slot zslot[k] (else slot k)
void launch_zero_slots(uint32_t *H, const int64_t *soff, const int32_t *skc, int64_t DS,
                       const int32_t *cstart, int n, int nblocks, cudaStream_t s,
                       const int32_t *zslot = nullptr);
void launch_subtract(uint32_t *H, const uint32_t *Hprev, int64_t DS, const SubJob *jobs,
                     const int16_t *maps, const int32_t *cstart, int n, int nblocks, cudaStream_t s);
// nodes with <= split_small_max_classes() classes go to the warp-per-(node, f)
// kernel, the others to the block-per-(node, f) kernel
int split_small_max_classes();
void launch_split(const uint32_t *H, const int64_t *node_off, const int32_t *node_kc,
                  const int32_t *big_nodes, int nbig, const int32_t *small_nodes, int nsmall,
                  int F, const int32_t *cumD, const int32_t *nval, SplitCand *out, cudaStream_t s);
void launch_winner(const uint32_t *H, const int64_t *node_off, const int32_t *node_kc, int nnodes,
                   int F, int C, const int32_t *cumD, const int32_t *nval, const SplitCand *cand,
                   uint8_t *res, const int64_t *res_off, cudaStream_t s);

// ---- kernel launchers (select.cu) ----
struct DNode {     // device inference node, 8 bytes
  float thr;       // largest float32 <= threshold (x <= thr_f64  <=>  x <= thr_f32, V:A5)
  int32_t meta;    // >= 0: (left << 6) | feature ; < 0: -1 - label
};

// ---- kernel launchers (forest.cu): random forests ----
// u8 bootstrap weights of this rank's rows [lo, lo + n_local) for tree `tree` (R19)
// sums[0] = draws landing in the shard, sums[1] = sum of the weights (equal unless
// a multiplicity overflowed u8); w needs n_local + 4 bytes
void launch_bootstrap(uint64_t seed, int tree, uint64_t n_total, uint64_t lo, int64_t n_local,
                      uint8_t *w, unsigned long long *sums, cudaStream_t s);
int forest_max_trees();
// majority vote of the T trees rooted at roots[t] in the concatenated node array
void launch_select_forest(const DNode *nodes, int n_nodes, const int32_t *roots, int T,
                          const float *X, int64_t m, int F, int32_t *out, cudaStream_t s);

// ---- quantile.cu: lossy binning of features with > 256 distinct values (R23) ----
size_t sort_unique_temp_bytes(int64_t n);
void launch_column_keys(const float *X, int64_t n, int F, int f, uint32_t *keys, cudaStream_t s);
void sort_unique_keys(const uint32_t *keys, int64_t n, uint32_t *sorted, uint32_t *out, int *d_count,
                      void *temp, size_t temp_bytes, cudaStream_t s);
void launch_edges(const uint32_t *ukeys, int64_t D, float *lb, float *prev, cudaStream_t s);
void launch_quantize(const float *X, int64_t n, int F, uint64_t qmask, const float *lb, float *Xq,
                     cudaStream_t s);

// ---- small.cu: the whole path for small tables in one thread block ----
constexpr int kSmallMaxN = 512, kSmallMaxF = 8, kSmallMaxC = 16, kSmallMaxA = 64, kSmallMaxNodes = 2112;
struct SmallOut {
  int32_t status;   // 0: trained; 1: outside the limits or a flagged value (use the general path)
  int32_t n_nodes;
  int32_t nval[kSmallMaxF];
  float val[kSmallMaxF][256];
  adapt_node_t nodes[kSmallMaxNodes];
};
size_t small_smem_bytes();
// labels -> labels[n], bins -> word planes (BS, pstride) like the ingest, tree -> out
void launch_small_train(const float *X, const float *T, int n, int F, int V, int D, int BS, size_t pstride,
                        uint8_t *bins, uint8_t *labels, SmallOut *out, cudaStream_t s);

// ---- kernel launchers (kfold.cu): the K-fold harness ----
constexpr int kKfoldMaxK = 64;
struct KfoldPartial {
  unsigned long long n_test, n_correct;
  double t_selected, t_best;
};
int kfold_eval_blocks();
// groups of the local rows in one shuffle (u8 [n]) and their local sizes (cnt [K], accumulated);
// d_bnd[j] = ceil(j N / K), j = 0..K (the first position of group j)
void launch_kfold_groups(uint64_t seed, int shuffle, uint64_t N, const uint64_t *d_bnd, int K, uint64_t lo,
                         int64_t n, uint8_t *grp, unsigned long long *cnt, cudaStream_t s);
// ingest planes -> per-(shuffle j, group g) contiguous copies at cursor[j*K+g]
void launch_kfold_scatter(const uint8_t *bins, size_t pstride_in, const uint8_t *lab, int64_t n, int BS,
                          const uint8_t *grp, int sb, int K, unsigned int *cursor, uint8_t *obins,
                          size_t pstride_out, uint8_t *olab, cudaStream_t s);
// held-out evaluation of the sb*K batch models (trees concatenated, roots[r]);
// part: [kfold_eval_blocks()][sb*K]
void launch_kfold_eval_many(const float *X, int64_t n, int F, int V, const float *times, const uint8_t *lab,
                            const uint8_t *grp, int sb, int K, int m, const DNode *nodes, const int32_t *roots,
                            KfoldPartial *part, cudaStream_t s);

// a single tree: the first kSelTopNodes BFS nodes (DNode) are staged in shared
// memory; a child index k >= n_top of a top node names bottom block k - n_top.
// A bottom block (64 B, 16 words) holds 3 levels in heap order: words 0..6 =
// the thresholds of its nodes p = 0..6 (children 2p+1, 2p+2; a leaf above the
// bottom is a pass-through whose 8 descendants all carry its label), words
// 7..14 = (ref_i << 6) | feature_p (feature of node p = i for i < 7), ref_i of
// leaf edge i = 2(p-3) + right for p = 3..6: >= 0 the next block, < 0 -1 - label.
constexpr int kSelTopNodes = 8191;
// Trees deeper than that top (select_kernel_h): the first `td` levels as a
// complete heap in shared memory, node h = {float bits of thr_f32, feature},
// children 2h+1 / 2h+2 (a leaf above level td is a pass-through node whose
// whole subtree leads to it), so the walk is td fixed steps with no bounds
// checks; exits[h - (2^td - 1)] after the top: >= 0 a 2-level bottom block,
// < 0 -1 - label.  A 2-level block is 32 bytes (one 256-bit load): words 0..2
// the thresholds of its root, left and right child, word 3 their features
// (bytes 0..2), words 4..7 the refs of its 4 exits (LL, LR, RL, RR; a leaf
// child passes through to both of its exits).
constexpr int kHeapMaxLevels = 14;  // 16383 nodes (128 KB) + 16384 exits (64 KB)
struct SelTree {
  const DNode *top;      // BFS nodes (the first kSelTopNodes are staged)
  int n_nodes;
  const uint4 *blocks;   // 3-level bottom blocks of the BFS layout
  const uint2 *heap;     // [2^td - 1]
  const int32_t *exits;  // [2^td]
  const uint4 *blocks2;  // 2-level blocks, 2 x uint4 each
  int td;                // heap levels (0: no heap layout)
};
void launch_select(const SelTree &t, const float *X, int64_t m, int F, int32_t *out, cudaStream_t s);

}  // namespace adapt
