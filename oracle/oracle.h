/*
 * oracle.h — CPU oracle for the adaptive-OpenMP model-building path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the C-ABI library
 * under paper_2303_08873_b200/, its Python binding) may include, link, load or
 * call anything declared here.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py use it.  It shares no code
 * with the CUDA path (no common headers, helpers or tables).
 *
 * It is plain, single-threaded C written straight from the paper and the
 * readings in DESIGN.md §3:
 *   P:NNN = /root/reference/PAPER.md line, S:NNN = SPEC.md line,
 *   R#    = reading number in DESIGN.md §3 ("readings of the paper").
 *
 * What it computes:
 *   step 0  long -> wide aggregation of profiling records   (R1, R4)
 *   step 1  fastest-variant label per sample                (R2, R3)
 *   a2      sorted distinct values of a feature             (R7, R14)
 *   step 2  exact greedy CART, breadth first, Gini          (R6-R12)
 *   step 3  tree walk ("get_policy" on a trained model)     (R8)
 *
 * Parity pins: every function is pinned by tests/test_oracle_*.py against
 * brute force in exact rational arithmetic (tests/exact_checker.py), closed
 * forms and the worked examples in tests/golden/.  None is "parity unpinned".
 *
 * Return codes follow include/adapt.h's numbering so tests can compare error
 * behaviour, but the values are restated here, not included from there.
 */
#ifndef ORACLE_H
#define ORACLE_H
#include <stdint.h>

#define ORACLE_OK 0
#define ORACLE_E_INVALID_ARG (-1)
#define ORACLE_E_INSUFFICIENT_DATA (-4)
#define ORACLE_E_BAD_VALUE (-6)
#define ORACLE_E_TOO_MANY_DISTINCT (-7)
#define ORACLE_E_CAPACITY (-12)

/* One tree node, canonical breadth-first order (root = 0; children of a node
 * are appended left then right when the node is split, R9 of SURVEY §8(c)). */
typedef struct {
  int32_t feature;   /* -1 for a leaf */
  int32_t left;      /* BFS index of left child, -1 for a leaf */
  int32_t right;     /* BFS index of right child, -1 for a leaf */
  int32_t label;     /* majority class of the node's rows, ties -> lowest */
  int32_t depth;     /* root = 0 */
  int32_t pad_;
  double threshold;  /* (double)x <= threshold -> left; 0.0 for a leaf */
  int64_t n;         /* rows in the node */
  double gini;       /* 1 - S/(n*n), S = sum_k c_k^2 */
} oracle_node_t;

/* -0.0 -> +0.0 and reject NaN/+-Inf (R4).  X is [n][F] row-major; out may
 * alias X.  Returns ORACLE_E_BAD_VALUE at the first non-finite value. */
int oracle_canon_features(const float *X, int64_t n, int F, float *out);

/* Step 1 ("finds the fastest execution policies per feature values"):
 * label[i] = min{ v : times[i][v] == min_u times[i][u] } under IEEE float <.
 * +inf = unmeasured (R3); a NaN time or an all-+inf row is BAD_VALUE. */
int oracle_labels(const float *times, int64_t n, int V, uint8_t *label);

/* Step 0 ("persistent database of per region records"; R1 mean, R4
 * exact-bits grouping).  Records r = 0..R-1: features feat[r][F], variant
 * var[r], elapsed ns[r].  Output: one wide row per distinct feature vector in
 * order of first appearance: out_feat[n][F], out_times[n][V] (mean as
 * (double)sum/(double)count rounded to float32; +inf when unmeasured).
 * *n_out receives the row count; cap = capacity in rows. */
int oracle_aggregate(const float *feat, const int32_t *var, const uint64_t *ns,
                     int64_t R, int F, int V, float *out_feat, float *out_times,
                     int64_t cap, int64_t *n_out);

/* Number of distinct (feature vector, variant) pairs ("uniqueness is
 * defined as collecting profiling data of different features and variants"). */
int64_t oracle_distinct_pairs(const float *feat, const int32_t *var, int64_t R, int F);

/* a2: sorted distinct values of column f of X[n][F] (after canonicalisation).
 * Writes at most cap values; *count receives the true number.  Returns
 * ORACLE_E_TOO_MANY_DISTINCT if the count exceeds 256 (R14). */
int oracle_value_table(const float *X, int64_t n, int F, int f, float *vals,
                       int cap, int *count);

/* Step 2: exact greedy CART (readings R6-R12, R13x).  X[n][F] finite floats,
 * y[n] in [0, C).  D = max depth (root = depth 0).  Writes at most cap nodes. */
int oracle_train(const float *X, const uint8_t *y, int64_t n, int F, int C, int D,
                 oracle_node_t *out, int32_t cap, int32_t *n_nodes);

/* Step 3: out[i] = leaf label reached from the root by (double)x[f] <= thr -> left
 * (NaN compares false -> right, R8). */
int oracle_select(const oracle_node_t *tree, int32_t n_nodes, const float *X,
                  int64_t m, int F, int32_t *out);

/* Random forest ("rfc"; SPEC train_rfc; readings R19-R21).
 * Bootstrap multiplicities of tree t (R19): n draws with replacement,
 * draw j picks row floor(h_j * n / 2^64), h_j = splitmix64(key_t ^ splitmix64(j)),
 * key_t = splitmix64(seed ^ splitmix64(t + 0x5851F42D4C957F2D)); w[i] = number of
 * draws of row i (sum = n).  The forest itself is plain: tree t = oracle_train on
 * the resample (rows repeated w[i] times), vote = majority, ties -> lowest
 * (R20) — composed in oracle/__init__.py from this and oracle_train/select. */
int oracle_bootstrap(uint64_t seed, int tree, int64_t n, uint32_t *w);

/* Helper used by the pins: Gini of a class-count vector, 1 - S/(n*n). */
double oracle_gini_counts(const int64_t *counts, int C);

/* K-fold harness ("split application inputs into K equal-sized
 * groups ... repeated 10 times, each time shuffling the inputs"; R22).
 * oracle_kfold_pos: the position of global row r in shuffle `shuffle` (a
 * bijection of [0, N): 4-round Feistel on 2h bits, cycle-walking), -1 on bad
 * arguments.  oracle_kfold_groups: group[r] = floor(pos(r) * K / N).  Model
 * (shuffle, fold k) trains on groups {(k + j) mod K : j < m} and is tested on
 * the others — composed in oracle/__init__.py from these and oracle_train/select. */
int64_t oracle_kfold_pos(uint64_t seed, int shuffle, int64_t N, int64_t r);
int oracle_kfold_groups(uint64_t seed, int shuffle, int64_t N, int K, int32_t *group);

#endif
