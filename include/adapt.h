/*
 * adapt.h — C ABI of the B200-native model-building engine behind
 * machine-learning-driven adaptive OpenMP (arXiv 2303.08873).
 *
 * Citations: P:NNN = PAPER.md line; S:NNN = SPEC.md line; R# = reading in
 * DESIGN.md §3.  The library (libadapt.so) is hand-written CUDA for sm_100a;
 * every step of record -> label -> train -> select runs in its kernels.  There
 * is no CPU fallback: with no usable GPU every compute call returns ADAPT_E_CUDA.
 *
 * The calls follow the paper's statement of the problem — collect profiling
 * records, train a model (Table 1 "__apollo_region_train"),
 * query the policy (Table 1 "__apollo_region_get_policy") — plus a
 * Table-1-shaped shim (bottom of this file).
 *
 * Conventions for every call below unless stated otherwise:
 *  - returns ADAPT_OK (0) or a negative adapt_status; adapt_last_error() gives
 *    a thread-local message for the last failing call of this thread;
 *  - all calls are thread-safe (one library-wide mutex);
 *  - the library owns region handles and its internal device buffers; the
 *    caller owns every pointer it passes.  Host pointers are read during the
 *    call only.  Device pointers passed to adapt_record_table(on_device=1) are
 *    BORROWED until adapt_train() returns; device pointers passed to
 *    adapt_select_batch() must stay valid until the stream passes the call;
 *  - "stream" is a cudaStream_t passed as void* (NULL = legacy default stream);
 *  - row-major layouts; float = IEEE binary32, double = binary64.
 */
#ifndef ADAPT_H
#define ADAPT_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ADAPT_OK = 0,
  ADAPT_E_INVALID_ARG = -1,       /* null pointer, n<0, F not in [1,64], V not in [1,255], depth not in [0,24] */
  ADAPT_E_USAGE = -2,             /* begin twice, end/set_feature without begin */
  ADAPT_E_ARITY = -3,             /* wrong number of features */
  ADAPT_E_INSUFFICIENT_DATA = -4, /* train with zero samples */
  ADAPT_E_SPEC_MISMATCH = -5,     /* re-create an id with a different spec */
  ADAPT_E_BAD_VALUE = -6,         /* NaN/Inf feature, NaN time, all-+inf time row, variant out of range (R3, R4) */
  ADAPT_E_TOO_MANY_DISTINCT = -7, /* a feature has more than 256 distinct values over all ranks (R14) */
  ADAPT_E_NOT_TRAINED = -8,       /* select before train */
  ADAPT_E_CUDA = -9,              /* CUDA error or no usable device */
  ADAPT_E_NCCL = -10,             /* NCCL error (world > 1) */
  ADAPT_E_OOM = -11               /* device allocation failed */
} adapt_status;

typedef struct adapt_region adapt_region_t; /* opaque, owned by the library */

/* One node of a trained tree in canonical breadth-first order: root = 0, the
 * children of a split node are appended left then right (SURVEY §8(c) step
 * 2.9).  x <= threshold goes left (R8).  48 bytes. */
typedef struct {
  int32_t feature;  /* split feature, -1 for a leaf */
  int32_t left;     /* BFS index of the left child, -1 for a leaf */
  int32_t right;    /* BFS index of the right child, -1 for a leaf */
  int32_t label;    /* majority variant of the node's training rows, ties -> lowest (R12) */
  int32_t depth;    /* root = 0 (R11) */
  int32_t pad_;
  double threshold; /* ((double)u_lo + (double)u_hi)/2 of consecutive node-local values (R7); 0 for a leaf */
  int64_t n;        /* training rows in the node, summed over ranks */
  double gini;      /* 1 - S/(n*n), S = sum_k c_k^2 */
} adapt_node_t;

/* Per-phase device time of the engine's own kernels (CUDA events on the
 * launching stream), accumulated since the last adapt_profile_reset(). */
typedef struct {
  char name[32];     /* "ingest", "values", "hist", "subtract", "split", "winner", "select", ... */
  int64_t launches;  /* kernel launches in this phase */
  double ms;         /* summed event time */
  double bytes;      /* algorithmic bytes moved (DESIGN.md §6 per-unit figures x units) */
} adapt_phase_t;

/* ---- lifetime ----------------------------------------------------------- */
/* Bind this process to CUDA device `device` as rank `rank` of `world`.
 * world == 1: nccl_unique_id may be NULL.  world > 1: nccl_unique_id points to
 * the 128-byte ncclUniqueId produced by adapt_nccl_unique_id() on rank 0 and
 * shipped to every rank (the Python layer uses torch.distributed for that).
 * NCCL is resolved at run time (dlopen "libnccl.so.2"); failure -> ADAPT_E_NCCL.
 * Calling again with the same arguments is a no-op; different ones -> E_USAGE
 * until adapt_finalize(). */
int adapt_init(int device, int rank, int world, const void *nccl_unique_id);
/* Writes a fresh 128-byte ncclUniqueId into out (rank 0, before adapt_init). */
int adapt_nccl_unique_id(void *out128);

/* Host-staged collectives: the same multi-rank training (value
 * tables all-gathered, per-level histograms and error flags summed) over a
 * transport the CALLER provides instead of NCCL, e.g. torch.distributed gloo
 * or MPI.  Used to run several ranks on ONE device (NCCL refuses duplicate
 * GPUs), which is how the P-invariance of the tree is tested on a 1-GPU box.
 * The library synchronises its stream, copies the operand to pinned host
 * memory, calls the hook, and copies the result back; no kernel changes.
 *   all_gather(send, recv, bytes, user): recv[r*bytes .. (r+1)*bytes) = rank r's
 *     send (bytes each, rank order); recv has world*bytes bytes.
 *   all_reduce_u64(buf, count, user): buf[i] = sum over ranks of buf[i]
 *     (in place; the library widens its u32 operands to u64 for the call).
 * Hooks return 0 on success; any other value -> ADAPT_E_NCCL.  The struct is
 * copied; `user` is passed through untouched and must outlive adapt_finalize.
 * Same rules as adapt_init otherwise (world >= 1, rank in [0,world)). */
typedef struct {
  int (*all_gather)(const void *send, void *recv, size_t bytes, void *user);
  int (*all_reduce_u64)(uint64_t *buf, size_t count, void *user);
  void *user;
} adapt_host_comm_t;
int adapt_init_host_comm(int device, int rank, int world, const adapt_host_comm_t *comm);
/* Destroys every region and the NCCL communicator; frees device memory. */
int adapt_finalize(void);
const char *adapt_last_error(void);
/* Library build identity, e.g. "adapt sm_100a <git>". */
const char *adapt_version(void);

/* ---- regions (Table 1 "__apollo_region_create") ---------------- */
/* id: unique region name.  num_features F in [1,64]; num_variants V in [1,255]
 * (variants are enumerated 0..V-1 in declaration order).
 * model_params: "dtree" | "dtree,depth=D" | "dtree,D" | "DecisionTree[,explore=RoundRobin]"
 * (P:142); NULL or "" -> dtree depth 2.  D in [0,24].
 * Random forest ("rfc"): "rfc" | "rfc,T,D" | "rfc(T,D)" |
 * "rfc,trees=T,depth=D,seed=S" | "RandomForest[...]": T trees (default 10,
 * [1,64]) of depth D (default 2), each trained on a bootstrap resample of the
 * table drawn from a counter RNG keyed by (seed, tree) (R19, default seed 0);
 * selection = majority vote, ties -> lowest variant (R20).
 * Lossy bins (DESIGN R23): ",bins=quantile" on a dtree or
 * rfc spec quantises every feature with more than 256 distinct values (over
 * all ranks) into 256 bins of equal numbers of distinct values; splits on it
 * report raw thresholds at the bin cut points.  Default ",bins=exact": such a
 * table fails with ADAPT_E_TOO_MANY_DISTINCT (R14).
 * min_train_data <= 0 -> V.
 * Same id and same spec -> the same handle; same id with a different
 * spec -> ADAPT_E_SPEC_MISMATCH. */
int adapt_region_create(const char *id, int num_features, int num_variants,
                        const char *model_params, int min_train_data, adapt_region_t **out);
int adapt_region_destroy(adapt_region_t *h);
/* Reads back the spec (any out pointer may be NULL). */
int adapt_region_info(adapt_region_t *h, int *num_features, int *num_variants, int *max_depth,
                      int *min_train_data, int64_t *num_rows, int *trained);

/* ---- record samples ("elapsed execution time between pairs of
 * begin/end calls, stored in a persistent database of per region records") -- */
/* Long format: one profiled execution, features[F] (host), variant in
 * [0,V), elapsed_ns.  Copied.  Aggregated to wide rows at train time: one row
 * per distinct feature vector (exact float32 bits, -0 == +0), each variant's
 * time = mean of its records rounded to float32, unmeasured = +inf (R1, R4). */
int adapt_record(adapt_region_t *h, const float *features, int variant, uint64_t elapsed_ns);
/* Long format in bulk (the GPU record path): m records
 * features [m][F] float32, variants [m] int32 in [0,V), elapsed_ns [m] uint64.
 * on_device = 1: device pointers, 0: host pointers; either way the records are
 * COPIED into the region's device store (stream-ordered on `stream`, complete
 * when the call returns).  At adapt_train() every record — the device store
 * first, then the adapt_record() ones in call order — is aggregated ON THE GPU
 * into one wide row per distinct feature vector in order of first appearance
 * (exact float32 bits, -0 == +0; time = (double)sum_ns/(double)count rounded to
 * float32; +inf = never recorded; R1, R3, R4).  A variant outside [0,V)
 * -> ADAPT_E_BAD_VALUE at train time; NaN/Inf features -> ADAPT_E_BAD_VALUE at
 * train time.  Record-path aggregation is rank-local (world > 1: each rank's
 * own records).  Total records < 2^32 (else ADAPT_E_INVALID_ARG). */
int adapt_record_batch(adapt_region_t *h, const float *features, const int32_t *variants,
                       const uint64_t *elapsed_ns, int64_t m, int on_device, void *stream);
/* The wide table the last adapt_train() built from records (host copies):
 * *n = rows; copies features [n][F] and times [n][V] when cap >= n (else only
 * sets *n).  ADAPT_E_NOT_TRAINED before training; ADAPT_E_USAGE when the last
 * train used adapt_record_table (or adapt_distinct_pairs re-aggregated since). */
int adapt_get_wide_table(adapt_region_t *h, float *features, float *times, int64_t cap,
                         int64_t *n);
/* Wide format (the profiling table): features [n][F] float32 and times
 * [n][V] float32 nanoseconds, +inf = unmeasured (R3).  With world > 1 this is
 * the calling rank's contiguous shard; the table is the concatenation over
 * ranks.  on_device = 0: host pointers, copied to the device on `stream`
 * before returning.  on_device = 1: device pointers, borrowed (not copied)
 * until adapt_train() returns.  Replaces any previous table; appends nothing. */
int adapt_record_table(adapt_region_t *h, const float *features, const float *times, int64_t n,
                       int on_device, void *stream);
/* Number of distinct (feature vector, variant) pairs among the long-format
 * records ("uniqueness is defined as collecting profiling data of
 * different features and variants").  With device-batch records this runs
 * the GPU aggregation (measured cells of the wide table). */
int adapt_distinct_pairs(adapt_region_t *h, int64_t *count);

/* ---- train (Table 1 "__apollo_region_train"; P:173 + P:253-255) --------- */
/* Labels every row with its fastest variant (a1), builds the value tables
 * (a2) and bins (a3), then grows the tree level by level (a4-a7) and
 * finalizes it (a8).  Collective over all ranks when world > 1 (every rank
 * gets the identical tree).  Blocks until the tree is on the host.
 * Errors: E_INSUFFICIENT_DATA (no rows on any rank), E_BAD_VALUE,
 * E_TOO_MANY_DISTINCT, E_CUDA, E_NCCL, E_OOM.  On error the region keeps its
 * previous model, if any. */
int adapt_train(adapt_region_t *h, void *cuda_stream);
/* k independent regions trained in one call (C2's "3 regions"; R15).  When
 * k >= 2 decision-tree regions share (F, V, D), are not in bins=quantile
 * mode and each holds a recorded wide table, they are trained FUSED: one
 * ingest over the union of their tables and one level loop whose frontier
 * starts with k roots.  Trees and labels are each region's own (thresholds
 * are node-local midpoints, R7, so the union's value tables only re-index
 * the bins); adapt_get_value_table / adapt_get_bins of such a region report
 * the union's value tables and ranks in them.  If the union has more than 256
 * distinct values of a feature, or a region has no rows, or the specs differ,
 * the regions are trained one by one (adapt_train each, in order). */
int adapt_train_many(adapt_region_t *const *hs, int k, void *cuda_stream);

/* ---- select (Table 1 "__apollo_region_get_policy") ---------------- */
/* One vector, host tree walk: variant = leaf label, x <= thr -> left,
 * NaN -> right (R8).  E_NOT_TRAINED before train. */
int adapt_select(adapt_region_t *h, const float *features, int32_t *variant);
/* m vectors on the device: d_X [m][F] float32 -> d_out [m] int32.  Async,
 * ordered on `stream`; rank-local (no communication). */
int adapt_select_batch(adapt_region_t *h, const float *d_X, int64_t m, int32_t *d_out,
                       void *cuda_stream);
/* Same from pinned or pageable HOST buffers X [m][F] -> out [m]: chunked
 * host->device copies, the select kernel and device->host copies, overlapped on
 * internal streams.  Returns when out is written. */
int adapt_select_batch_host(adapt_region_t *h, const float *X, int64_t m, int32_t *out,
                            void *cuda_stream);
/* The selections of every row of the region's recorded wide table (the
 * profiled feature vectors themselves: "which variant does the model pick for
 * each configuration it was trained on"), from the library's device copy of a
 * HOST-recorded table (adapt_record_table with on_device = 0 keeps it until the
 * next record), so the vectors cross PCIe once.  out [n] int32 (n = the rows
 * recorded on this rank): device memory when out_on_device != 0 (async on
 * `stream`), else host memory (returns when written).  E_NOT_TRAINED before
 * train; E_USAGE when the table was borrowed device memory (released when
 * train returned: use adapt_select_batch with the caller's buffer) or came
 * from long-format records. */
int adapt_select_table(adapt_region_t *h, int32_t *out, int out_on_device, void *cuda_stream);

/* ---- model exchange / parity introspection ------------------------------ */
/* Canonical BFS node array; *n_nodes receives the node count even when cap is
 * too small (then ADAPT_E_INVALID_ARG). */
int adapt_get_tree(adapt_region_t *h, adapt_node_t *out, int32_t cap, int32_t *n_nodes);
/* Forests: number of trees (1 for a decision tree), and tree t in canonical
 * BFS order (same layout and rules as adapt_get_tree; adapt_get_tree returns
 * tree 0).  ADAPT_E_INVALID_ARG for t out of range or cap too small. */
int adapt_forest_size(adapt_region_t *h, int32_t *trees);
int adapt_get_forest_tree(adapt_region_t *h, int32_t t, adapt_node_t *out, int32_t cap,
                          int32_t *n_nodes);
/* ---- K-fold harness (DESIGN R22) ----
 * The paper's evaluation methodology: "split application inputs into K
 * equal-sized groups. A fraction f of groups is used for model training while
 * the rest are used for testing ... K-fold creation is repeated 10 times, each
 * time shuffling the inputs" (Adaptive-25/50/75 = K 4, m 1/2/3).  Inputs are
 * the rows of the recorded table (all ranks: a collective call, like
 * adapt_train).  Shuffle s permutes the global row ids (4-round Feistel on
 * 2h-bit words, 4^h >= N, cycle-walking, keyed by (seed, s)); group of row r
 * = floor(pos(r) K / N); model (s, k) = the region's dtree trained on the rows
 * of groups {(k + j) mod K : j < train_groups} and tested on the others.
 * out[s * K + k] (caller-owned, shuffles * K entries) gets the model's counts
 * summed over ranks; t_selected / t_best are double sums of the test rows'
 * float32 times of the selected / the fastest variant (summation order
 * differs from the oracle's exactly rounded sum: DESIGN R22 bounds it).
 * The region's own model is left as it was.  Borrowed device tables stay
 * borrowed until this call returns (as for adapt_train).
 * Errors: ADAPT_E_INVALID_ARG for K not in [2,64], train_groups not in
 * [1,K-1], shuffles < 1 or NULL out; ADAPT_E_USAGE on a forest region;
 * ADAPT_E_INSUFFICIENT_DATA for fewer than K rows; as adapt_train otherwise. */
typedef struct {
  int32_t shuffle, fold;   /* model (s, k) */
  int32_t n_nodes, pad_;   /* size of its tree (adapt_get_kfold_tree) */
  int64_t n_train, n_test; /* global rows */
  int64_t n_correct;       /* test rows whose selection is their label (the fastest variant) */
  double t_selected;       /* sum over test rows of times[i][selected] (ns) */
  double t_best;           /* sum over test rows of times[i][label] (ns) */
} adapt_kfold_result_t;
int adapt_kfold(adapt_region_t *h, int K, int train_groups, int shuffles, uint64_t seed,
                adapt_kfold_result_t *out, void *cuda_stream);
/* Tree of model `model` (= s * K + k) of the last adapt_kfold, canonical BFS. */
int adapt_get_kfold_tree(adapt_region_t *h, int32_t model, adapt_node_t *out, int32_t cap,
                         int32_t *n_nodes);
/* Install a tree (model reuse across runs; synthetic trees for the
 * selection benchmark).  Validates BFS structure, features and labels. */
int adapt_set_tree(adapt_region_t *h, const adapt_node_t *nodes, int32_t n_nodes);
/* Labels (a1) of this rank's rows, u8 [n], from the last adapt_train. */
int adapt_get_labels(adapt_region_t *h, uint8_t *out, int64_t n);
/* Sorted distinct values of feature f over all ranks (a2): vals[<=256],
 * *count = D_f. */
int adapt_get_value_table(adapt_region_t *h, int f, float *vals, int *count);
/* Rank of each value in its feature's value table (a3), u8 [n][F]. */
int adapt_get_bins(adapt_region_t *h, uint8_t *out, int64_t n);

/* ---- measurement -------------------------------------------------------- */
/* enable != 0: record CUDA events around every engine kernel (adds no sync). */
int adapt_profile_enable(int enable);
int adapt_profile_reset(void);
/* Copies up to cap phases; *n receives the number of phases. Synchronizes
 * the recorded events. */
int adapt_profile_get(adapt_phase_t *out, int cap, int *n);
/* Per-level statistics of the last adapt_train on this rank (SURVEY §8(d)
 * per-level reporting): for level d, out[6d] = frontier nodes, out[6d+1] =
 * rows histogrammed, out[6d+2] = rows partitioned, out[6d+3] = bytes of the
 * level's node histograms (class-compacted, direct + derived), out[6d+4] =
 * bytes through the level's collectives on this rank (0 on one rank; the
 * all-reduce input, or the reduce-scatter input plus the gathered winner
 * records with ADAPT_HIST_COMM=rs), out[6d+5] = bytes of the DIRECT nodes'
 * histograms (what the default all-reduce sums when world > 1; reported on
 * one rank too, for scaling projections).  *levels receives the level count
 * (forests / K-fold: the levels of every tree / batch, in order). */
int adapt_train_stats(adapt_region_t *h, int64_t *out, int cap, int *levels);

/* ---- Apollo Table-1 shim (lowering order P:558-569) ------------- */
/* void calls record errors in adapt_last_error(); get_policy returns 0 on error.
 * create: NULL on error.  begin starts a monotonic clock, set_feature
 * appends (Table 1: float), get_policy returns the trained tree's choice
 * or, untrained, the round-robin exploration cursor, end
 * records (features, policy, elapsed) and auto-trains once min_train_data
 * distinct (features, variant) pairs exist. */
void *__adapt_region_create(const char *id, int num_features, int num_policies,
                            const char *model_type_params, int min_train_data);
void __adapt_region_begin(void *region);
void __adapt_region_end(void *region);
void __adapt_region_set_feature(void *region, float value);
int __adapt_region_get_policy(void *region);
void __adapt_region_train(void *region);

#ifdef __cplusplus
}
#endif
#endif /* ADAPT_H */
