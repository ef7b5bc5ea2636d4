// ingest.cu — steps a1 (label), a2 (value tables) and a3 (bin) in ONE pass
// over the profiling table.
//
// a1  label[i] = lowest v attaining min_v times[i][v] under IEEE '<'; +inf is
//     "unmeasured" and an all-+inf or NaN row is an error (R2, R3).
// a2  the distinct float32 values of every feature are discovered on the fly
//     in a per-feature hash table in global memory (fronted by a per-block
//     shared-memory cache); each new value gets a provisional id in order of
//     discovery.  After the pass a tiny kernel sorts the <= 256 values
//     (merged over ranks) into the value table and maps provisional ids to
//     ranks (R7, R14).
// a3  the bin of x[i][f] is its provisional id; the rank LUT turns it into
//     the rank in the sorted table wherever a rank is needed.  So features are
//     read exactly once: 4F + 4V bytes in, RS bytes (bins + label) out per row.
//
// Output record of row i (RS = F+1 rounded up to a power of two bytes):
//     rec[i*RS + f] = provisional bin of feature f, rec[i*RS + F] = label.
#include "common.h"

namespace adapt {
namespace {

constexpr int kIngestThreads = 256;  // threads per block; a tile holds TR <= 256 rows

__device__ __forceinline__ uint32_t hash_slot(uint32_t key, int log2slots) {
  return (key * 2654435761u) >> (32 - log2slots);
}

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t *p) {
  return *(volatile const uint32_t *)p;
}

// Global, race-free insert-or-find.  The winner of the key CAS takes the next
// id from the per-feature counter and publishes it; losers wait for it.
__device__ uint32_t global_lookup(uint32_t *gkey, uint32_t *gid, uint32_t *gcount,
                                  uint32_t *flags, int f, uint32_t key) {
  uint32_t *K = gkey + (size_t)f * kGSlots;
  uint32_t *I = gid + (size_t)f * kGSlots;
  uint32_t h = hash_slot(key, 10);
  static_assert(kGSlots == 1024, "hash width");
  for (int p = 0; p < kGSlots; p++) {
    uint32_t k = ld_volatile(K + h);
    if (k == kEmptyKey) {
      const uint32_t old = atomicCAS(K + h, kEmptyKey, key);
      if (old == kEmptyKey) {
        const uint32_t id = atomicAdd(gcount + f, 1u);
        if (id >= (uint32_t)kMaxBins) atomicOr(flags, kFlagTooMany);
        atomicExch(I + h, id);
        return id < (uint32_t)kMaxBins ? id : kMaxBins - 1;
      }
      k = old;
    }
    if (k == key) {
      uint32_t id;
      while ((id = ld_volatile(I + h)) == kPendingId) __nanosleep(32);
      return id < (uint32_t)kMaxBins ? id : kMaxBins - 1;
    }
    h = (h + 1) & (kGSlots - 1);
  }
  atomicOr(flags, kFlagTooMany);  // table full: far more than 256 values
  return kMaxBins - 1;
}

template <int RS>
__global__ void __launch_bounds__(kIngestThreads)
    ingest_kernel(const float *__restrict__ feat, const float *__restrict__ times, int64_t n,
                  int F, int V, int TR, int log2sl, uint32_t *gkey, uint32_t *gid, uint32_t *gcount,
                  uint32_t *flags, uint8_t *__restrict__ rec) {
  extern __shared__ uint4 smem_u4[];
  const int SL = 1 << log2sl;
  uint32_t *skey = reinterpret_cast<uint32_t *>(smem_u4);
  uint16_t *sid = reinterpret_cast<uint16_t *>(skey + F * SL);
  float *tile_t = reinterpret_cast<float *>(
      reinterpret_cast<uint4 *>(smem_u4) + ((F * SL * 6 + 15) / 16));
  float *tile_f = tile_t + TR * V;
  uint8_t *srec = reinterpret_cast<uint8_t *>(tile_f + TR * F);

  const int tid = threadIdx.x;
  for (int i = tid; i < F * SL; i += blockDim.x) {
    skey[i] = kEmptyKey;
    sid[i] = 0xFFFF;
  }
  uint32_t local_flags = 0;
  const bool aligned_t = (reinterpret_cast<uintptr_t>(times) & 15) == 0;
  const bool aligned_f = (reinterpret_cast<uintptr_t>(feat) & 15) == 0;
  __syncthreads();

  const int64_t ntiles = (n + TR - 1) / TR;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * TR;
    const int rows = (n - row0 < TR) ? (int)(n - row0) : TR;
    // ---- stage the tile: coalesced 16-byte streaming loads ----
    {
      const float *src = times + row0 * V;
      const int cnt = rows * V;
      int done = 0;
      if (aligned_t) {
        const float4 *s4 = reinterpret_cast<const float4 *>(src);
        float4 *d4 = reinterpret_cast<float4 *>(tile_t);
        const int n4 = cnt >> 2;
        for (int i = tid; i < n4; i += kIngestThreads) d4[i] = __ldcs(s4 + i);
        done = n4 << 2;
      }
      for (int i = done + tid; i < cnt; i += kIngestThreads) tile_t[i] = __ldcs(src + i);
    }
    {
      const float *src = feat + row0 * F;
      const int cnt = rows * F;
      int done = 0;
      if (aligned_f) {
        const float4 *s4 = reinterpret_cast<const float4 *>(src);
        float4 *d4 = reinterpret_cast<float4 *>(tile_f);
        const int n4 = cnt >> 2;
        for (int i = tid; i < n4; i += kIngestThreads) d4[i] = __ldcs(s4 + i);
        done = n4 << 2;
      }
      for (int i = done + tid; i < cnt; i += kIngestThreads) tile_f[i] = __ldcs(src + i);
    }
    __syncthreads();

    if (tid < rows) {
      // ---- a1: argmin with lowest-index ties; the row is read starting at a
      // thread-dependent rotation so the 32 lanes hit (almost) distinct banks.
      const float *tr = tile_t + tid * V;
      float best = __int_as_float(0x7f800000);  // +inf
      int bi = 0x7fffffff;
      bool nan = false;
      int j = tid % V;
      for (int k = 0; k < V; k++) {
        const float x = tr[j];
        nan |= (x != x);
        if (x < best || (x == best && j < bi)) {
          best = x;
          bi = j;
        }
        j = (j + 1 == V) ? 0 : j + 1;
      }
      if (nan) local_flags |= kFlagNanTime;
      if (best == __int_as_float(0x7f800000)) local_flags |= kFlagAllInf;
      uint8_t *my = srec + tid * RS;
      my[F] = (uint8_t)bi;
      for (int p = F + 1; p < RS; p++) my[p] = 0;
      // ---- a2 + a3: provisional id of each feature value ----
      const float *fr = tile_f + tid * F;
      int f = tid % F;
      for (int k = 0; k < F; k++) {
        const float x = fr[f];
        uint32_t key = __float_as_uint(x);
        if ((key & 0x7f800000u) == 0x7f800000u) {
          local_flags |= kFlagBadFeature;
          key = 0;
        }
        if (x == 0.0f) key = 0;  // -0 -> +0 (R4)
        uint32_t *sk = skey + f * SL;
        uint16_t *si = sid + f * SL;
        uint32_t h = hash_slot(key, log2sl);
        int id = -1;
        for (int p = 0; p < SL; p++) {
          const uint32_t kk = sk[h];
          if (kk == key) {
            const uint16_t v = si[h];
            if (v != 0xFFFF) id = v;
            break;
          }
          if (kk == kEmptyKey) break;
          h = (h + 1) & (SL - 1);
        }
        if (id < 0) {
          id = (int)global_lookup(gkey, gid, gcount, flags, f, key);
          // publish in the block cache (best effort; a full cache just misses)
          uint32_t hh = hash_slot(key, log2sl);
          for (int p = 0; p < SL; p++) {
            const uint32_t old = atomicCAS(sk + hh, kEmptyKey, key);
            if (old == kEmptyKey) {
              si[hh] = (uint16_t)id;
              break;
            }
            if (old == key) break;
            hh = (hh + 1) & (SL - 1);
          }
        }
        my[f] = (uint8_t)id;
        f = (f + 1 == F) ? 0 : f + 1;
      }
    }
    __syncthreads();
    // ---- write the tile's records: contiguous, 16-byte stores ----
    {
      uint8_t *dst = rec + row0 * RS;
      const int bytes = rows * RS;
      if (RS >= 16) {
        const uint4 *s4 = reinterpret_cast<const uint4 *>(srec);
        uint4 *d4 = reinterpret_cast<uint4 *>(dst);
        for (int i = tid; i < (bytes >> 4); i += kIngestThreads) __stcs(d4 + i, s4[i]);
      } else {
        for (int i = tid; i < bytes; i += kIngestThreads) dst[i] = srec[i];
      }
    }
    __syncthreads();
  }
  if (local_flags) atomicOr(flags, local_flags);
}

__global__ void collect_values_kernel(const uint32_t *gkey, const uint32_t *gid,
                                      const uint32_t *gcount, float *local_vals,
                                      int32_t *local_cnt) {
  const int f = blockIdx.x;
  for (int s = threadIdx.x; s < kGSlots; s += blockDim.x) {
    const uint32_t k = gkey[(size_t)f * kGSlots + s];
    if (k == kEmptyKey) continue;
    const uint32_t id = gid[(size_t)f * kGSlots + s];
    if (id < (uint32_t)kMaxBins) local_vals[f * kMaxBins + id] = __uint_as_float(k);
  }
  if (threadIdx.x == 0) local_cnt[f] = (int32_t)min(gcount[f], (uint32_t)kMaxBins + 1);
}

// Union of every rank's distinct values of feature f, sorted; lut maps this
// rank's provisional ids to ranks in the union (the value table, a2).
__global__ void merge_values_kernel(const float *all_vals, const int32_t *all_cnt, int world,
                                    int rank, int F, float *val, int32_t *nval, uint8_t *lut,
                                    uint32_t *flags) {
  extern __shared__ float cand[];  // [world*256]
  uint8_t *rep = reinterpret_cast<uint8_t *>(cand + world * kMaxBins);
  __shared__ int s_nrep;
  const int f = blockIdx.x;
  int M = 0;
  for (int p = 0; p < world; p++) {
    const int c = all_cnt[p * F + f];
    if (c > kMaxBins && threadIdx.x == 0) atomicOr(flags, kFlagTooMany);
    M += min(c, kMaxBins);
  }
  for (int c = threadIdx.x; c < M; c += blockDim.x) {
    int p = 0, i = c;
    while (i >= min(all_cnt[p * F + f], kMaxBins)) {
      i -= min(all_cnt[p * F + f], kMaxBins);
      p++;
    }
    cand[c] = all_vals[((size_t)p * F + f) * kMaxBins + i];
  }
  if (threadIdx.x == 0) s_nrep = 0;
  __syncthreads();
  for (int c = threadIdx.x; c < M; c += blockDim.x) {
    const uint32_t b = __float_as_uint(cand[c]);
    bool first = true;
    for (int e = 0; e < c && first; e++) first = __float_as_uint(cand[e]) != b;
    rep[c] = first;
    if (first) atomicAdd(&s_nrep, 1);
  }
  __syncthreads();
  const int D = s_nrep;
  if (threadIdx.x == 0) {
    nval[f] = D;
    if (D > kMaxBins) atomicOr(flags, kFlagTooMany);
  }
  int base = 0;  // offset of this rank's candidates
  for (int p = 0; p < rank; p++) base += min(all_cnt[p * F + f], kMaxBins);
  const int mine = min(all_cnt[rank * F + f], kMaxBins);
  for (int c = threadIdx.x; c < M; c += blockDim.x) {
    const float x = cand[c];
    int r = 0;
    for (int e = 0; e < M; e++) r += (rep[e] && cand[e] < x);
    if (rep[c] && r < kMaxBins) val[f * kMaxBins + r] = x;
    if (c >= base && c < base + mine) lut[f * kMaxBins + (c - base)] = (uint8_t)min(r, 255);
  }
}

__global__ void bins_out_kernel(const uint8_t *rec, int64_t n, int F, int RS, const uint8_t *lut,
                                uint8_t *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * F;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / F;
    const int f = (int)(i % F);
    out[i] = lut[f * kMaxBins + rec[r * RS + f]];
  }
}

__global__ void labels_out_kernel(const uint8_t *rec, int64_t n, int F, int RS, uint8_t *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = rec[i * RS + F];
}

int grid_for(int64_t work, int per_block, int cap) {
  int64_t b = (work + per_block - 1) / per_block;
  if (b < 1) b = 1;
  return (int)(b < cap ? b : cap);
}

}  // namespace

void launch_ingest(const float *feat, const float *times, int64_t n, int F, int V, int RS,
                   uint32_t *gkey, uint32_t *gid, uint32_t *gcount, uint32_t *flags,
                   uint8_t *rec, cudaStream_t s) {
  if (n == 0) return;
  // per-block value cache: 512 slots/feature (<= 50% load at 256 values) when it fits
  int log2sl = 9;
  while (log2sl > 5 && (size_t)F * (6u << log2sl) > 48 * 1024) log2sl--;
  const size_t cache = (((size_t)F * (6u << log2sl)) + 15) / 16 * 16;
  int TR = kIngestThreads;  // tile rows: keep the block under ~100 KB of smem
  while (TR > 32 && cache + (size_t)TR * ((V + F) * 4 + RS) > 100 * 1024) TR >>= 1;
  const size_t smem = cache + (size_t)TR * ((V + F) * 4 + RS);
  const int grid = grid_for(n, TR, 148 * 8);
  switch (RS) {
#define CASE(R)                                                                              \
  case R: {                                                                                  \
    CUDA_CHECK(cudaFuncSetAttribute(ingest_kernel<R>,                                        \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    ingest_kernel<R><<<grid, kIngestThreads, smem, s>>>(feat, times, n, F, V, TR, log2sl,    \
                                                        gkey, gid, gcount, flags, rec);      \
    break;                                                                                   \
  }
    CASE(2) CASE(4) CASE(8) CASE(16) CASE(32) CASE(64) CASE(128)
#undef CASE
    default:
      throw Error(-1, "bad record stride");
  }
  CUDA_CHECK(cudaGetLastError());
}

void launch_collect_values(const uint32_t *gkey, const uint32_t *gid, const uint32_t *gcount,
                           int F, float *local_vals, int32_t *local_cnt, cudaStream_t s) {
  collect_values_kernel<<<F, 256, 0, s>>>(gkey, gid, gcount, local_vals, local_cnt);
  CUDA_CHECK(cudaGetLastError());
}

void launch_merge_values(const float *all_vals, const int32_t *all_cnt, int world, int rank,
                         int F, float *val, int32_t *nval, uint8_t *lut, uint32_t *flags,
                         cudaStream_t s) {
  const size_t smem = (size_t)world * kMaxBins * 5;
  CUDA_CHECK(cudaFuncSetAttribute(merge_values_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  merge_values_kernel<<<F, 1024, smem, s>>>(all_vals, all_cnt, world, rank, F, val, nval, lut,
                                            flags);
  CUDA_CHECK(cudaGetLastError());
}

void launch_bins_out(const uint8_t *rec, int64_t n, int F, int RS, const uint8_t *lut,
                     uint8_t *out, cudaStream_t s) {
  if (n == 0) return;
  bins_out_kernel<<<grid_for(n * F, 256, 148 * 16), 256, 0, s>>>(rec, n, F, RS, lut, out);
  CUDA_CHECK(cudaGetLastError());
}

void launch_labels_out(const uint8_t *rec, int64_t n, int F, int RS, uint8_t *out,
                       cudaStream_t s) {
  if (n == 0) return;
  labels_out_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(rec, n, F, RS, out);
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace adapt
