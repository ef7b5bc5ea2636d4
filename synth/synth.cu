// synth.cu — device twin of synth/__init__.py's generate() (the input recipe of
// DESIGN.md §4).  Makes inputs only: no labelling, binning or tree arithmetic.
// Every double operation is written with an explicit _rn intrinsic so nvcc can
// not contract it into an FMA; the host twin does the same operations in the
// same order in numpy, so the float32 tables are byte-identical.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += kGolden;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t u24(uint64_t seed, uint64_t row, uint64_t col) {
  return splitmix64(seed ^ splitmix64(row * kGolden + col)) >> 40;
}

#define MUL __dmul_rn
#define ADD __dadd_rn
#define SUB __dsub_rn
#define DIV __ddiv_rn

constexpr int kMaxF = 16;
constexpr int kMaxV = 48;

__device__ void costs(int cid, const double *x, uint64_t row, double *out) {
  if (cid == 1) {
    out[0] = ADD(MUL(x[0], 1.0), 2000.0);
    out[1] = ADD(MUL(x[0], 0.02), 30000.0);
    return;
  }
  if (cid == 2) {
    const double N = x[0], m = x[1], s = x[2], cls = x[3];
    const int r = (int)(row % 3);
    const double w = r == 0 ? 1.0 : (r == 1 ? 2.5 : 0.6);
    const double o = r == 0 ? 3000.0 : (r == 1 ? 1500.0 : 6000.0);
    for (int v = 0; v < 7; v++) {
      const double p = (double)(1 << v);
      double a = SUB(1.0, s);
      double b = DIV(a, p);
      double c = ADD(s, b);
      double t1 = MUL(N, w);
      t1 = MUL(t1, c);
      double t2 = MUL(o, cls);
      t2 = MUL(t2, p);
      double bwp = fmin(MUL(p, 8.0), 96.0);
      double t3 = MUL(N, m);
      t3 = DIV(t3, bwp);
      out[v] = ADD(ADD(t1, t2), t3);
    }
    return;
  }
  // cid 3 and 4 share the block-size model
  const double N = x[0], regs = x[1], smem = x[2], flops = x[3], byts = x[4];
  const double w1 = MUL(flops, 0.5);
  const double w2 = MUL(byts, 0.25);
  const double work = MUL(N, ADD(w1, w2));
  const double cap = DIV(65536.0, regs);
  double sm = DIV(smem, 32.0);
  sm = ADD(1.0, sm);
  if (cid == 3) {
    for (int v = 0; v < 6; v++) {
      const double T = (double)(32 << v);
      double conc = fmin(T, cap);
      double t = DIV(work, conc);
      double g = MUL(2000.0, T);
      g = MUL(g, sm);
      out[v] = ADD(t, g);
    }
    return;
  }
  const double cores = x[8], res = x[9], xfer = x[10], numa = x[11];
  for (int v = 0; v < 48; v++) {
    const int dev = v / 24;
    const double th = (double)(8 << ((v / 6) % 4));
    const double blk = (double)(32 << (v % 6));
    double t;
    if (dev == 0) {
      t = DIV(work, fmin(th, cores));
      double nf = MUL(numa, 0.25);
      nf = ADD(1.0, nf);
      t = MUL(t, nf);
      double s1 = DIV(N, blk);
      s1 = MUL(s1, 40.0);
      t = ADD(t, s1);
      double s2 = MUL(blk, ADD(w1, w2));
      t = ADD(t, s2);
      t = ADD(t, MUL(th, 800.0));
    } else {
      const double mm = DIV(th, 8.0);
      double conc = fmin(blk, cap);
      conc = MUL(conc, mm);
      conc = MUL(conc, 16.0);
      t = DIV(work, conc);
      double g = MUL(2000.0, blk);
      g = MUL(g, sm);
      g = DIV(g, mm);
      t = ADD(t, g);
      double xr = SUB(1.0, res);
      double xb = MUL(N, xfer);
      xb = DIV(xb, 25.0);
      xb = MUL(xb, xr);
      t = ADD(t, xb);
      t = ADD(t, 20000.0);
      t = ADD(t, MUL(mm, 3000.0));
    }
    out[v] = t;
  }
}

__global__ void gen_kernel(int cid, uint64_t seed, int64_t row0, int64_t n, int F, int V,
                           const float *__restrict__ grids, const int *__restrict__ off,
                           double noise, float *__restrict__ feat, float *__restrict__ times) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t row = (uint64_t)(row0 + i);
    double x[kMaxF];
    for (int f = 0; f < F; f++) {
      const uint64_t G = (uint64_t)(off[f + 1] - off[f]);
      const uint64_t k = (u24(seed, row, (uint64_t)f) * G) >> 24;
      const float v = grids[off[f] + k];
      feat[i * F + f] = v;
      x[f] = (double)v;
    }
    if (times == nullptr) continue;
    double c[kMaxV];
    costs(cid, x, row, c);
    for (int v = 0; v < V; v++) {
      double t = c[v];
      if (noise != 0.0) {
        double u = MUL((double)u24(seed, row, 1000 + (uint64_t)v), 5.9604644775390625e-08);
        double fac = MUL(2.0, u);
        fac = SUB(fac, 1.0);
        fac = MUL(noise, fac);
        fac = ADD(1.0, fac);
        t = MUL(t, fac);
      }
      times[i * V + v] = __double2float_rn(t);
    }
  }
}

}  // namespace

extern "C" int synth_generate(int cid, uint64_t seed, int64_t row0, int64_t n, int F, int V,
                              const float *d_grids, const int *d_off, double noise, float *d_feat,
                              float *d_times, void *stream) {
  if (F > kMaxF || V > kMaxV || n < 0) return -1;
  if (n == 0) return 0;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 64) blocks = 148 * 64;
  gen_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(cid, seed, row0, n, F, V, d_grids, d_off,
                                                       noise, d_feat, d_times);
  return cudaGetLastError() == cudaSuccess ? 0 : -9;
}
