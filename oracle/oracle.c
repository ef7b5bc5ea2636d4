/*
 * oracle.c — plain CPU oracle.  TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Written for obviousness, not speed: per node and feature the node's rows are
 * sorted and scanned, every candidate is scored exactly, and the best one is
 * chosen under an explicit total order.  No binning, no histograms, no
 * subtraction, nothing shared with the CUDA path.
 *
 * Compile with -ffp-contract=off (build() does): no FMA may fuse the
 * few double expressions below.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

static float canon(float x) { return x == 0.0f ? 0.0f : x; } /* -0 -> +0 (R4) */

static uint32_t fbits(float x) {
  uint32_t b;
  memcpy(&b, &x, 4);
  return b;
}

int oracle_canon_features(const float *X, int64_t n, int F, float *out) {
  if (n < 0 || F < 1) return ORACLE_E_INVALID_ARG;
  for (int64_t i = 0; i < n * F; i++) {
    float x = X[i];
    if (isnan(x) || isinf(x)) return ORACLE_E_BAD_VALUE; /* R4 */
    out[i] = canon(x);
  }
  return ORACLE_OK;
}

/* ---- step 1: labels (R2, R3) ------------------ */
int oracle_labels(const float *times, int64_t n, int V, uint8_t *label) {
  if (n < 0 || V < 1 || V > 255) return ORACLE_E_INVALID_ARG;
  for (int64_t i = 0; i < n; i++) {
    const float *t = times + i * (int64_t)V;
    /* the minimum under IEEE '<' over the measured (+inf = unmeasured) times */
    float m = INFINITY;
    for (int v = 0; v < V; v++) {
      if (isnan(t[v])) return ORACLE_E_BAD_VALUE;
      if (t[v] < m) m = t[v];
    }
    if (isinf(m) && m > 0) return ORACLE_E_BAD_VALUE; /* all unmeasured (R3) */
    /* lowest variant index attaining it (R2) */
    int best = -1;
    for (int v = 0; v < V; v++)
      if (t[v] == m) { best = v; break; }
    label[i] = (uint8_t)best;
  }
  return ORACLE_OK;
}

/* ---- step 0: long -> wide aggregation (R1, R4) ------------------ */
typedef struct {
  const float *feat;
  int F;
} sort_ctx_t;
static sort_ctx_t g_ctx; /* single-threaded oracle: a static context is fine */

static int cmp_rows_then_index(const void *a, const void *b) {
  int64_t ia = *(const int64_t *)a, ib = *(const int64_t *)b;
  for (int f = 0; f < g_ctx.F; f++) {
    uint32_t xa = fbits(canon(g_ctx.feat[ia * g_ctx.F + f]));
    uint32_t xb = fbits(canon(g_ctx.feat[ib * g_ctx.F + f]));
    if (xa != xb) return xa < xb ? -1 : 1;
  }
  return ia < ib ? -1 : (ia > ib);
}

static int same_vector(const float *feat, int F, int64_t a, int64_t b) {
  for (int f = 0; f < F; f++)
    if (fbits(canon(feat[a * F + f])) != fbits(canon(feat[b * F + f]))) return 0;
  return 1;
}

static int cmp_i64(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return x < y ? -1 : (x > y);
}

int oracle_aggregate(const float *feat, const int32_t *var, const uint64_t *ns,
                     int64_t R, int F, int V, float *out_feat, float *out_times,
                     int64_t cap, int64_t *n_out) {
  if (R < 0 || F < 1 || V < 1 || V > 255) return ORACLE_E_INVALID_ARG;
  *n_out = 0;
  if (R == 0) return ORACLE_E_INSUFFICIENT_DATA;
  for (int64_t r = 0; r < R; r++) {
    if (var[r] < 0 || var[r] >= V) return ORACLE_E_BAD_VALUE;
    for (int f = 0; f < F; f++) {
      float x = feat[r * F + f];
      if (isnan(x) || isinf(x)) return ORACLE_E_BAD_VALUE;
    }
  }
  int64_t *idx = malloc(sizeof(int64_t) * R);
  for (int64_t r = 0; r < R; r++) idx[r] = r;
  g_ctx.feat = feat;
  g_ctx.F = F;
  qsort(idx, R, sizeof(int64_t), cmp_rows_then_index);
  /* group heads: the first (lowest) record index of each distinct vector */
  int64_t *first = malloc(sizeof(int64_t) * R);
  int64_t G = 0;
  for (int64_t k = 0; k < R; k++)
    if (k == 0 || !same_vector(feat, F, idx[k - 1], idx[k])) first[G++] = idx[k];
  free(idx);
  if (G > cap) {
    free(first);
    return ORACLE_E_CAPACITY;
  }
  qsort(first, G, sizeof(int64_t), cmp_i64); /* order of first appearance */
  uint64_t *sum = calloc((size_t)V, sizeof(uint64_t));
  int64_t *cnt = calloc((size_t)V, sizeof(int64_t));
  for (int64_t g = 0; g < G; g++) {
    int64_t h = first[g];
    memset(sum, 0, sizeof(uint64_t) * V);
    memset(cnt, 0, sizeof(int64_t) * V);
    for (int64_t r = 0; r < R; r++) /* plain O(R*G) scan */
      if (same_vector(feat, F, h, r)) {
        sum[var[r]] += ns[r];
        cnt[var[r]] += 1;
      }
    for (int f = 0; f < F; f++) out_feat[g * F + f] = canon(feat[h * F + f]);
    for (int v = 0; v < V; v++)
      out_times[g * V + v] =
          cnt[v] ? (float)((double)sum[v] / (double)cnt[v]) : INFINITY; /* R1, R3 */
  }
  free(sum);
  free(cnt);
  free(first);
  *n_out = G;
  return ORACLE_OK;
}

int64_t oracle_distinct_pairs(const float *feat, const int32_t *var, int64_t R, int F) {
  int64_t d = 0;
  for (int64_t r = 0; r < R; r++) { /* plain O(R^2): count first occurrences */
    int seen = 0;
    for (int64_t q = 0; q < r && !seen; q++)
      if (var[q] == var[r] && same_vector(feat, F, q, r)) seen = 1;
    if (!seen) d++;
  }
  return d;
}

/* ---- a2: sorted distinct values (R7, R14) ---------------------------------- */
static int cmp_float(const void *a, const void *b) {
  float x = *(const float *)a, y = *(const float *)b;
  return x < y ? -1 : (x > y);
}

int oracle_value_table(const float *X, int64_t n, int F, int f, float *vals, int cap,
                       int *count) {
  if (n < 0 || f < 0 || f >= F) return ORACLE_E_INVALID_ARG;
  float *col = malloc(sizeof(float) * (n ? n : 1));
  for (int64_t i = 0; i < n; i++) {
    float x = X[i * F + f];
    if (isnan(x) || isinf(x)) {
      free(col);
      return ORACLE_E_BAD_VALUE;
    }
    col[i] = canon(x);
  }
  qsort(col, n, sizeof(float), cmp_float);
  int c = 0;
  for (int64_t i = 0; i < n; i++)
    if (i == 0 || col[i] != col[i - 1]) {
      if (c < cap) vals[c] = col[i];
      c++;
    }
  free(col);
  *count = c;
  return c > 256 ? ORACLE_E_TOO_MANY_DISTINCT : ORACLE_OK;
}

/* ---- step 2: exact greedy CART ---------------------- */
double oracle_gini_counts(const int64_t *counts, int C) {
  int64_t n = 0, S = 0;
  for (int k = 0; k < C; k++) {
    n += counts[k];
    S += counts[k] * counts[k];
  }
  if (n == 0) return 0.0;
  return 1.0 - (double)S / ((double)n * (double)n);
}

/* Stop rule (R10): a node is a leaf iff it is pure, at depth D, or has no
 * candidate cut.  Otherwise the best candidate is taken even if its gain is
 * zero (XOR-like nodes), so a depth-unlimited tree reproduces the labels of
 * distinct training vectors (north_star invariant).  Improving candidates have
 * score > S/n and zero-gain ones exactly S/n, so any improving candidate wins.
 *
 * A candidate's key is the exact rational score SL/nL + SR/nR = num/den with
 * num = SL*nR + SR*nL and den = nL*nR (R13x).  Maximising it minimises the
 * weighted child Gini, since weighted Gini = 1 - score/n. */
typedef struct {
  int valid;
  u128 num, den;
  int f;
  double thr;
  int64_t nL;
} cand_t;

/* exact num1/den1 > num2/den2 via quotient and remainder; den < 2^64 */
static int frac_gt(u128 n1, u128 d1, u128 n2, u128 d2) {
  u128 q1 = n1 / d1, q2 = n2 / d2;
  if (q1 != q2) return q1 > q2;
  u128 r1 = n1 % d1, r2 = n2 % d2; /* r < d < 2^64, so r*d < 2^128 */
  return r1 * d2 > r2 * d1;
}
static int frac_eq(u128 n1, u128 d1, u128 n2, u128 d2) {
  return !frac_gt(n1, d1, n2, d2) && !frac_gt(n2, d2, n1, d1);
}

/* key order: score desc, then f asc, then thr asc (R9) */
static int better(const cand_t *a, const cand_t *b) {
  if (!b->valid) return 1;
  if (frac_gt(a->num, a->den, b->num, b->den)) return 1;
  if (!frac_eq(a->num, a->den, b->num, b->den)) return 0;
  if (a->f != b->f) return a->f < b->f;
  return a->thr < b->thr;
}

typedef struct {
  float x;
  uint8_t y;
} pair_t;
static int cmp_pair(const void *a, const void *b) {
  float x = ((const pair_t *)a)->x, y = ((const pair_t *)b)->x;
  return x < y ? -1 : (x > y);
}

typedef struct {
  int64_t *rows;
  int64_t n;
} rowset_t;

int oracle_train(const float *X, const uint8_t *y, int64_t n, int F, int C, int D,
                 oracle_node_t *out, int32_t cap, int32_t *n_nodes) {
  *n_nodes = 0;
  if (n < 0 || F < 1 || C < 1 || C > 255 || D < 0 || cap < 1) return ORACLE_E_INVALID_ARG;
  if (n == 0) return ORACLE_E_INSUFFICIENT_DATA;
  if (n >= ((int64_t)1 << 32)) return ORACLE_E_INVALID_ARG;
  for (int64_t i = 0; i < n * F; i++)
    if (isnan(X[i]) || isinf(X[i])) return ORACLE_E_BAD_VALUE;
  for (int64_t i = 0; i < n; i++)
    if (y[i] >= C) return ORACLE_E_INVALID_ARG;

  rowset_t *sets = calloc((size_t)cap, sizeof(rowset_t));
  sets[0].rows = malloc(sizeof(int64_t) * n);
  for (int64_t i = 0; i < n; i++) sets[0].rows[i] = i;
  sets[0].n = n;
  memset(&out[0], 0, sizeof(oracle_node_t));
  out[0].depth = 0;
  int32_t count = 1;
  int rc = ORACLE_OK;
  int64_t *cnt = malloc(sizeof(int64_t) * C);
  /* one sort buffer per thread: the all-cores build (-fopenmp, liboracle_omp.so,
   * bench timing only) scans the features of a node in parallel; the plain
   * build has one thread and the pragma below is ignored */
  int nthr = 1;
#ifdef _OPENMP
  nthr = omp_get_max_threads();
#endif
  pair_t **tpairs = malloc(sizeof(pair_t *) * nthr);
  int64_t **tcL = malloc(sizeof(int64_t *) * nthr);
  for (int t = 0; t < nthr; t++) {
    tpairs[t] = malloc(sizeof(pair_t) * n);
    tcL[t] = malloc(sizeof(int64_t) * C);
  }
  cand_t *fbest = malloc(sizeof(cand_t) * F);

  /* nodes are processed in index order; children are appended, so this is BFS */
  for (int32_t k = 0; k < count; k++) {
    oracle_node_t *nd = &out[k];
    int64_t *rows = sets[k].rows;
    int64_t m = sets[k].n;
    memset(cnt, 0, sizeof(int64_t) * C);
    for (int64_t i = 0; i < m; i++) cnt[y[rows[i]]]++;
    int label = 0, present = 0;
    for (int c = 0; c < C; c++) {
      if (cnt[c] > cnt[label]) label = c; /* strict > keeps the lowest on ties (R12) */
      if (cnt[c] > 0) present++;
    }
    nd->label = label;
    nd->n = m;
    nd->gini = oracle_gini_counts(cnt, C);
    nd->feature = -1;
    nd->left = nd->right = -1;
    nd->threshold = 0.0;
    if (nd->depth >= D || present <= 1) { /* depth cap or pure (R10, R11) */
      free(rows);
      sets[k].rows = NULL;
      continue;
    }
    /* best candidate of each feature, then the best over features in f order */
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int f = 0; f < F; f++) {
      int t = 0;
#ifdef _OPENMP
      t = omp_get_thread_num();
#endif
      pair_t *pairs = tpairs[t];
      int64_t *cL = tcL[t];
      cand_t best;
      memset(&best, 0, sizeof(best));
      for (int64_t i = 0; i < m; i++) {
        pairs[i].x = canon(X[rows[i] * F + f]);
        pairs[i].y = y[rows[i]];
      }
      qsort(pairs, m, sizeof(pair_t), cmp_pair);
      memset(cL, 0, sizeof(int64_t) * C);
      int64_t nL = 0;
      for (int64_t i = 0; i < m; i++) {
        cL[pairs[i].y]++;
        nL++;
        /* a candidate cut after each run of equal values u_j with a next u_{j+1};
         * every candidate competes, zero-gain ones included (R10) */
        if (i + 1 < m && pairs[i + 1].x != pairs[i].x) {
          int64_t nR = m - nL;
          u128 SL = 0, SR = 0;
          for (int c = 0; c < C; c++) {
            SL += (u128)cL[c] * (u128)cL[c];
            SR += (u128)(cnt[c] - cL[c]) * (u128)(cnt[c] - cL[c]);
          }
          cand_t cd;
          cd.valid = 1;
          cd.num = SL * (u128)nR + SR * (u128)nL;
          cd.den = (u128)nL * (u128)nR;
          cd.f = f;
          cd.thr = ((double)pairs[i].x + (double)pairs[i + 1].x) / 2; /* R7 */
          cd.nL = nL;
          if (better(&cd, &best)) best = cd;
        }
      }
      fbest[f] = best;
    }
    cand_t best;
    memset(&best, 0, sizeof(best));
    for (int f = 0; f < F; f++)
      if (fbest[f].valid && better(&fbest[f], &best)) best = fbest[f];
    if (!best.valid) { /* no candidate cut: all rows share every feature value (R10) */
      free(rows);
      sets[k].rows = NULL;
      continue;
    }
    if (count + 2 > cap) {
      rc = ORACLE_E_CAPACITY;
      break;
    }
    int32_t l = count, r = count + 1;
    count += 2;
    nd->feature = best.f;
    nd->threshold = best.thr;
    nd->left = l;
    nd->right = r;
    sets[l].rows = malloc(sizeof(int64_t) * best.nL);
    sets[r].rows = malloc(sizeof(int64_t) * (m - best.nL));
    sets[l].n = sets[r].n = 0;
    for (int64_t i = 0; i < m; i++) {
      double x = (double)canon(X[rows[i] * F + best.f]);
      rowset_t *s = (x <= best.thr) ? &sets[l] : &sets[r]; /* R8: <= goes left */
      s->rows[s->n++] = rows[i];
    }
    memset(&out[l], 0, sizeof(oracle_node_t));
    memset(&out[r], 0, sizeof(oracle_node_t));
    out[l].depth = out[r].depth = nd->depth + 1;
    free(rows);
    sets[k].rows = NULL;
  }
  for (int32_t k = 0; k < count; k++) free(sets[k].rows);
  free(sets);
  free(cnt);
  for (int t = 0; t < nthr; t++) {
    free(tpairs[t]);
    free(tcL[t]);
  }
  free(tpairs);
  free(tcL);
  free(fbest);
  *n_nodes = count;
  return rc;
}

/* ---- step 3: tree walk (R8) ----------------------------------------- */
int oracle_select(const oracle_node_t *tree, int32_t n_nodes, const float *X, int64_t m,
                  int F, int32_t *out) {
  if (n_nodes < 1 || m < 0 || F < 1) return ORACLE_E_INVALID_ARG;
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
  for (int64_t i = 0; i < m; i++) {
    int32_t k = 0;
    while (tree[k].feature >= 0) {
      double x = (double)X[i * F + tree[k].feature];
      k = (x <= tree[k].threshold) ? tree[k].left : tree[k].right;
    }
    out[i] = tree[k].label;
  }
  return ORACLE_OK;
}

/* ---- random forest bootstrap (R19) ---- */
static uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int oracle_bootstrap(uint64_t seed, int tree, int64_t n, uint32_t *w) {
  if (n < 0 || tree < 0 || (n > 0 && !w)) return ORACLE_E_INVALID_ARG;
  for (int64_t i = 0; i < n; i++) w[i] = 0;
  const uint64_t key = splitmix64(seed ^ splitmix64((uint64_t)tree + 0x5851F42D4C957F2Dull));
  for (int64_t j = 0; j < n; j++) {
    const uint64_t h = splitmix64(key ^ splitmix64((uint64_t)j));
    const int64_t i = (int64_t)(((unsigned __int128)h * (uint64_t)n) >> 64);
    w[i] += 1;
  }
  return 0;
}

/* ---- K-fold harness (R22): the permutation of the inputs ----
 * Shuffle s permutes the N global rows with a 4-round Feistel network on
 * 2h-bit words (the smallest h >= 1 with 4^h >= N), cycle-walking until the
 * image falls inside [0, N); group of row r = floor(pos(r) * K / N). */
int64_t oracle_kfold_pos(uint64_t seed, int shuffle, int64_t N, int64_t r) {
  if (N <= 0 || r < 0 || r >= N || shuffle < 0) return -1;
  int h = 1;
  while (h < 31 && ((uint64_t)1 << (2 * h)) < (uint64_t)N) h++;
  const uint64_t mask = ((uint64_t)1 << h) - 1;
  const uint64_t key = splitmix64(seed ^ splitmix64((uint64_t)shuffle + 0x2545F4914F6CDD1Dull));
  uint64_t x = (uint64_t)r;
  do {
    uint64_t L = x >> h, R = x & mask;
    for (uint64_t j = 0; j < 4; j++) {
      const uint64_t f = splitmix64(key ^ splitmix64((R << 2) | j)) & mask;
      const uint64_t t = L ^ f;
      L = R;
      R = t;
    }
    x = (L << h) | R;
  } while (x >= (uint64_t)N);
  return (int64_t)x;
}

int oracle_kfold_groups(uint64_t seed, int shuffle, int64_t N, int K, int32_t *group) {
  if (N < 0 || K < 2 || shuffle < 0 || (N > 0 && !group)) return ORACLE_E_INVALID_ARG;
  for (int64_t r = 0; r < N; r++) {
    const int64_t pos = oracle_kfold_pos(seed, shuffle, N, r);
    group[r] = (int32_t)(((unsigned __int128)pos * (unsigned)K) / (uint64_t)N);
  }
  return ORACLE_OK;
}
