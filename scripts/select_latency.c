/* Host get_policy latency through the C ABI, no Python in the loop (the
 * paper's Table 4 "inference" overhead, 7-20 ns per call).
 *
 *   select_latency X.f32 T.f32 n F V params reps
 *
 * Reads the wide table (features [n][F], times [n][V], float32 files), trains
 * the region on the GPU (adapt_record_table + adapt_train), then times `reps`
 * passes of adapt_select over the n feature vectors with CLOCK_MONOTONIC and
 * prints one JSON object.  Built by __graft_entry__.build(); run by bench.py. */
#include <stdio.h>
#include <stdlib.h>
#include <time.h>

#include "adapt.h"

static float *load(const char *path, size_t count) {
  FILE *f = fopen(path, "rb");
  if (!f) return NULL;
  float *p = malloc(count * sizeof(float));
  size_t got = fread(p, sizeof(float), count, f);
  fclose(f);
  if (got != count) {
    free(p);
    return NULL;
  }
  return p;
}

int main(int argc, char **argv) {
  if (argc != 8) {
    fprintf(stderr, "usage: %s X.f32 T.f32 n F V params reps\n", argv[0]);
    return 2;
  }
  const long n = atol(argv[3]);
  const int F = atoi(argv[4]), V = atoi(argv[5]), reps = atoi(argv[7]);
  float *X = load(argv[1], (size_t)n * F), *T = load(argv[2], (size_t)n * V);
  if (!X || !T) return 3;
  adapt_region_t *h = NULL;
  if (adapt_init(0, 0, 1, NULL) || adapt_region_create("select_latency", F, V, argv[6], 0, &h) ||
      adapt_record_table(h, X, T, n, 0, NULL) || adapt_train(h, NULL)) {
    fprintf(stderr, "setup failed: %s\n", adapt_last_error());
    return 4;
  }
  int32_t v = 0;
  long long acc = 0;
  for (long i = 0; i < n; i++) { /* warm-up */
    adapt_select(h, X + i * F, &v);
    acc += v;
  }
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (int r = 0; r < reps; r++)
    for (long i = 0; i < n; i++) {
      adapt_select(h, X + i * F, &v);
      acc += v;
    }
  clock_gettime(CLOCK_MONOTONIC, &t1);
  const double ns = (t1.tv_sec - t0.tv_sec) * 1e9 + (t1.tv_nsec - t0.tv_nsec);
  printf("{\"ns_per_call\": %.2f, \"calls\": %lld, \"checksum\": %lld}\n", ns / ((double)reps * n),
         (long long)reps * n, acc);
  adapt_region_destroy(h);
  adapt_finalize();
  return 0;
}
