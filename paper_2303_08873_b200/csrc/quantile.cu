// quantile.cu — lossy binning for features with more than 256 distinct values
// (DESIGN R23), opt-in with the model parameter
// "bins=quantile" (the exact path rejects such tables, R14).
//
// Quantizer of feature f (global over ranks): u_0 < ... < u_{D-1} are its
// sorted distinct values; bin b (0..255) holds the distinct values with index
// in [e_b, e_{b+1}), e_b = floor(b D / 256) — equal numbers of distinct values
// per bin; lb_b = u_{e_b}.  Every value x becomes x' = lb_{q(x)},
// q(x) = #{b : lb_b <= x} - 1, so the quantised column has exactly 256
// distinct values and the exact (lossless) path trains on it; a split between
// node bins a < b' reports the raw threshold ((double)u_{e_{a+1}-1} +
// (double)u_{e_{a+1}}) / 2 (engine.cpp), which routes every raw x exactly as
// q(x) <= a.
//
//   column_keys_kernel  strided column -> order-preserving u32 keys (-0 -> +0)
//   cub radix sort + unique (library primitives) -> the sorted distinct keys
//   edges_kernel        lb_b and u_{e_b - 1} from the sorted distinct keys
//   quantize_kernel     X' = X with the quantised columns replaced (binary
//                       search of the 256 lower bounds in shared memory)
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include "adapt.h"
#include "common.h"

namespace adapt {
namespace {

__device__ __forceinline__ uint32_t f2key(float x) {
  uint32_t b = __float_as_uint(x == 0.0f ? 0.0f : x);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ float key2f(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

__global__ void column_keys_kernel(const float *__restrict__ X, int64_t n, int F, int f,
                                   uint32_t *__restrict__ keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = f2key(__ldg(X + i * F + f));
}

// lb[b] = u[e_b], prev[b] = u[e_b - 1] (b >= 1; prev[0] = lb[0])
__global__ void edges_kernel(const uint32_t *__restrict__ ukeys, int64_t D, float *lb, float *prev) {
  const int b = threadIdx.x;  // 256 threads
  const int64_t e = (int64_t)(((unsigned __int128)b * (uint64_t)D) / kMaxBins);
  lb[b] = key2f(ukeys[e]);
  prev[b] = key2f(ukeys[b ? e - 1 : e]);
}

__global__ void quantize_kernel(const float *__restrict__ X, int64_t n, int F, uint64_t qmask,
                                const float *__restrict__ lb /*[F][256]*/, float *__restrict__ Xq) {
  extern __shared__ float s_lb[];  // [F][256] (quantised features only are read)
  for (int i = threadIdx.x; i < F * kMaxBins; i += blockDim.x)
    if ((qmask >> (i / kMaxBins)) & 1) s_lb[i] = lb[i];
  __syncthreads();
  const int64_t total = n * F;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)(i % F);
    float x = __ldg(X + i);
    if ((qmask >> f) & 1) {
      x = x == 0.0f ? 0.0f : x;
      const float *t = s_lb + f * kMaxBins;
      int lo = 0;  // largest b with t[b] <= x (t[0] is the minimum: x >= t[0])
#pragma unroll
      for (int step = 128; step > 0; step >>= 1)
        if (t[lo + step] <= x) lo += step;
      x = t[lo];
    }
    Xq[i] = x;
  }
}

int grid_for(int64_t work) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, (int64_t)sms * 16));
}

}  // namespace

size_t sort_unique_temp_bytes(int64_t n) {
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, a, (const uint32_t *)nullptr, (uint32_t *)nullptr, (int)n);
  cub::DeviceSelect::Unique(nullptr, b, (const uint32_t *)nullptr, (uint32_t *)nullptr, (int *)nullptr,
                            (int)n);
  return std::max(a, b);
}

void launch_column_keys(const float *X, int64_t n, int F, int f, uint32_t *keys, cudaStream_t s) {
  if (n == 0) return;
  column_keys_kernel<<<grid_for(n), 256, 0, s>>>(X, n, F, f, keys); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
}

// keys [n] -> sorted distinct keys in out [<= n], count in *d_count (device int)
void sort_unique_keys(const uint32_t *keys, int64_t n, uint32_t *sorted, uint32_t *out, int *d_count,
                      void *temp, size_t temp_bytes, cudaStream_t s) {
  if (n >= (int64_t)1 << 31) throw Error(ADAPT_E_INVALID_ARG, "quantile binning: more than 2^31 rows per rank");
  size_t t = temp_bytes;
  CUDA_CHECK(cub::DeviceRadixSort::SortKeys(temp, t, keys, sorted, (int)n, 0, 32, s));
  t = temp_bytes;
  CUDA_CHECK(cub::DeviceSelect::Unique(temp, t, sorted, out, d_count, (int)n, s));
}

void launch_edges(const uint32_t *ukeys, int64_t D, float *lb, float *prev, cudaStream_t s) {
  edges_kernel<<<1, kMaxBins, 0, s>>>(ukeys, D, lb, prev); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
}

void launch_quantize(const float *X, int64_t n, int F, uint64_t qmask, const float *lb, float *Xq,
                     cudaStream_t s) {
  if (n == 0) return;
  const size_t smem = (size_t)F * kMaxBins * 4;
  smem_limit(quantize_kernel, smem);
  quantize_kernel<<<grid_for(n * F), 256, smem, s>>>(X, n, F, qmask, lb, Xq); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace adapt
