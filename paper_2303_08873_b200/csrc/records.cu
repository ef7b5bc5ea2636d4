// records.cu — the long-format record path on the GPU (
// SURVEY §8(c) step 0, "elapsed execution time between pairs of
// begin/end calls, stored ... per region records" -> "finds the fastest
// execution policies per feature values").
//
// m records (features[F] float32, variant, elapsed ns) become one wide row per
// distinct feature vector (exact float32 bits after -0 -> +0, R4), in order of
// first appearance, with time[v] = (double)sum_ns / (double)count
// rounded to float32, +inf when variant v was never recorded (R1, R3):
//   rec_group_kernel   hash-set insert of every record's vector (open
//                      addressing on a 64-bit hash of the F keys, equality on
//                      the keys themselves; a slot remembers one member) and
//                      atomicMin of the group's first record index;
//   rec_head_kernel    flag[r] = record r is its group's first record;
//   scan kernels       exclusive scan of the flags = dense group id in order
//                      of first appearance (block sums, one-block scan, add);
//   rec_sum_kernel     per (group, variant) u64 sum of ns and u32 count
//                      (integer atomics: exact, order-independent);
//   rec_mean_kernel    the wide times.
// Every result is a pure function of the record list, bit-identical to the
// oracle's sort-based grouping (tests/test_gpu_records.py).
#include <algorithm>

#include "common.h"

namespace adapt {
namespace {

constexpr uint32_t kEmptySlot = 0xFFFFFFFFu;
constexpr int kScanThreads = 1024, kScanItems = 4;  // 4096 records per scan block

__device__ __forceinline__ uint32_t canon_bits(float x) {
  return x == 0.0f ? 0u : __float_as_uint(x);  // -0 -> +0 (R4)
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 33;
  z *= 0xff51afd7ed558ccdull;
  z ^= z >> 33;
  z *= 0xc4ceb9fe1a85ec53ull;
  z ^= z >> 33;
  return z;
}

__device__ __forceinline__ bool same_vec(const float *feat, int F, uint32_t a, uint32_t b) {
  const float *x = feat + (size_t)a * F, *y = feat + (size_t)b * F;
  for (int f = 0; f < F; f++)
    if (canon_bits(x[f]) != canon_bits(y[f])) return false;
  return true;
}

__global__ void rec_group_kernel(const float *__restrict__ feat, const int32_t *__restrict__ var,
                                 uint32_t m, int F, int V, uint32_t mask, uint32_t *slot_rep,
                                 uint32_t *slot_first, uint32_t *slot_of, uint32_t *flags) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r = (uint32_t)min((uint64_t)r + gridDim.x * blockDim.x, (uint64_t)m)) {
    if ((unsigned)var[r] >= (unsigned)V) atomicOr(flags, kFlagBadVariant);
    uint64_t hsh = 0x9E3779B97F4A7C15ull;
    for (int f = 0; f < F; f++) hsh = mix64(hsh ^ canon_bits(feat[(size_t)r * F + f]));
    uint32_t s = (uint32_t)hsh & mask;
    for (;;) {
      uint32_t cur = slot_rep[s];
      if (cur == kEmptySlot) {
        cur = atomicCAS(slot_rep + s, kEmptySlot, r);
        if (cur == kEmptySlot) break;  // r represents a new group
      }
      if (same_vec(feat, F, cur, r)) break;
      s = (s + 1) & mask;
    }
    slot_of[r] = s;
    atomicMin(slot_first + s, r);
  }
}

// flag[r] = 1 iff r is the first record of its group
__global__ void rec_head_kernel(const uint32_t *slot_of, const uint32_t *slot_first, uint32_t m,
                                uint32_t *flag) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r = (uint32_t)min((uint64_t)r + gridDim.x * blockDim.x, (uint64_t)m))
    flag[r] = slot_first[slot_of[r]] == r ? 1u : 0u;
}

// ---- exclusive scan of u32 flags (m < 2^32) ----
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t x, uint32_t *warp_sums,
                                                         uint32_t &total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t v = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) warp_sums[w] = v;
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    uint32_t s = lane < nw ? warp_sums[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) warp_sums[lane] = s;
  }
  __syncthreads();
  total = warp_sums[(blockDim.x >> 5) - 1];
  const uint32_t before = w ? warp_sums[w - 1] : 0u;
  __syncthreads();
  return before + v - x;
}

__global__ void __launch_bounds__(kScanThreads) scan_block_sums_kernel(const uint32_t *flag, uint32_t m,
                                                                       uint32_t *bsum) {
  __shared__ uint32_t ws[32];
  const uint32_t base = blockIdx.x * (uint32_t)(kScanThreads * kScanItems);
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; i++) {
    const uint32_t r = base + i * kScanThreads + threadIdx.x;
    acc += r < m ? flag[r] : 0u;
  }
  uint32_t tot;
  block_exclusive_scan(acc, ws, tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanThreads) scan_sums_kernel(uint32_t *bsum, int nb, uint32_t *total) {
  __shared__ uint32_t ws[32];
  uint32_t carry = 0;
  for (int b0 = 0; b0 < nb; b0 += kScanThreads) {
    const int b = b0 + threadIdx.x;
    const uint32_t x = b < nb ? bsum[b] : 0u;
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan(x, ws, tot);
    if (b < nb) bsum[b] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *total = carry;
}

// group ids for the heads (rank in first-appearance order) and the wide features
__global__ void __launch_bounds__(kScanThreads)
    scan_apply_kernel(const uint32_t *flag, uint32_t m, const uint32_t *bsum,
                      const uint32_t *slot_of, uint32_t *slot_gid, const float *feat, int F,
                      float *wide_feat) {
  __shared__ uint32_t ws[32];
  const uint32_t base = blockIdx.x * (uint32_t)(kScanThreads * kScanItems);
  // each thread owns kScanItems consecutive records (scan order = record order)
  const uint32_t r0 = base + threadIdx.x * kScanItems;
  uint32_t fl[kScanItems], acc = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; i++) {
    fl[i] = r0 + i < m ? flag[r0 + i] : 0u;
    acc += fl[i];
  }
  uint32_t tot;
  uint32_t g = bsum[blockIdx.x] + block_exclusive_scan(acc, ws, tot);
#pragma unroll
  for (int i = 0; i < kScanItems; i++) {
    if (fl[i]) {
      const uint32_t r = r0 + i;
      slot_gid[slot_of[r]] = g;
      for (int f = 0; f < F; f++)
        wide_feat[(size_t)g * F + f] = __uint_as_float(canon_bits(feat[(size_t)r * F + f]));
      g++;
    }
  }
}

__global__ void rec_sum_kernel(const int32_t *var, const uint64_t *ns, const uint32_t *slot_of,
                               const uint32_t *slot_gid, uint32_t m, int V,
                               unsigned long long *sum, uint32_t *cnt) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r = (uint32_t)min((uint64_t)r + gridDim.x * blockDim.x, (uint64_t)m)) {
    const int v = var[r];
    if ((unsigned)v >= (unsigned)V) continue;  // flagged by rec_group_kernel
    const size_t i = (size_t)slot_gid[slot_of[r]] * V + v;
    atomicAdd(sum + i, (unsigned long long)ns[r]);
    atomicAdd(cnt + i, 1u);
  }
}

// wide times; optionally counts the measured cells (= distinct (vector,
// variant) pairs) into *pairs
__global__ void rec_mean_kernel(const unsigned long long *sum, const uint32_t *cnt, size_t n,
                                float *wide_times, uint32_t *pairs) {
  uint32_t mine = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    wide_times[i] = cnt[i] ? __double2float_rn(__ddiv_rn((double)sum[i], (double)cnt[i]))
                           : __int_as_float(0x7f800000);  // +inf: unmeasured (R3)
    mine += cnt[i] != 0;
  }
  if (pairs) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(pairs, mine);
  }
}

int grid_for(int64_t n, int threads) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 8 * sms));
}

}  // namespace

size_t rec_table_slots(int64_t m) {
  size_t t = 1024;
  while (t < (size_t)(2 * m)) t <<= 1;
  return t;
}

int rec_scan_blocks(int64_t m) {
  return (int)((m + kScanThreads * kScanItems - 1) / (kScanThreads * kScanItems));
}

void launch_rec_group(const float *feat, const int32_t *var, int64_t m, int F, int V,
                      uint32_t *slot_rep, uint32_t *slot_first, size_t slots, uint32_t *slot_of,
                      uint32_t *flag, uint32_t *bsum, uint32_t *d_groups, uint32_t *flags,
                      cudaStream_t s) {
  CUDA_CHECK(cudaMemsetAsync(slot_rep, 0xFF, slots * 4, s));
  CUDA_CHECK(cudaMemsetAsync(slot_first, 0xFF, slots * 4, s));
  rec_group_kernel<<<grid_for(m, 256), 256, 0, s>>>(feat, var, (uint32_t)m, F, V,
                                                     (uint32_t)(slots - 1), slot_rep, slot_first,
                                                     slot_of, flags); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
  rec_head_kernel<<<grid_for(m, 256), 256, 0, s>>>(slot_of, slot_first, (uint32_t)m, flag); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
  const int nb = rec_scan_blocks(m);
  scan_block_sums_kernel<<<nb, kScanThreads, 0, s>>>(flag, (uint32_t)m, bsum); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
  scan_sums_kernel<<<1, kScanThreads, 0, s>>>(bsum, nb, d_groups); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
}

void launch_rec_wide(const float *feat, const int32_t *var, const uint64_t *ns, int64_t m, int F,
                     int V, const uint32_t *slot_of, uint32_t *slot_gid, const uint32_t *flag,
                     const uint32_t *bsum, int64_t groups, unsigned long long *sum, uint32_t *cnt,
                     float *wide_feat, float *wide_times, uint32_t *pairs, cudaStream_t s) {
  const int nb = rec_scan_blocks(m);
  scan_apply_kernel<<<nb, kScanThreads, 0, s>>>(flag, (uint32_t)m, bsum, slot_of, slot_gid, feat,
                                                 F, wide_feat); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
  CUDA_CHECK(cudaMemsetAsync(sum, 0, (size_t)groups * V * 8, s));
  CUDA_CHECK(cudaMemsetAsync(cnt, 0, (size_t)groups * V * 4, s));
  rec_sum_kernel<<<grid_for(m, 256), 256, 0, s>>>(var, ns, slot_of, slot_gid, (uint32_t)m, V, sum,
                                                   cnt); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
  if (pairs) CUDA_CHECK(cudaMemsetAsync(pairs, 0, 4, s));
  rec_mean_kernel<<<grid_for(groups * V, 256), 256, 0, s>>>(sum, cnt, (size_t)groups * V,
                                                            wide_times, pairs); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace adapt
