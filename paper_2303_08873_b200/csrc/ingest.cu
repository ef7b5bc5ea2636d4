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
//     read exactly once: 4F + 4V bytes in, BS + 1 bytes out per row.
//
// Output planes (BS = F rounded up to a power of two bytes):
//     bins[i*BS + f] = provisional bin of feature f, labels[i] = label.
#include <algorithm>

#include "common.h"
#include "ptx.h"

namespace adapt {
namespace {

constexpr int kIngestThreads = 1024;

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

// One CTA per SM, persistent over row tiles of TR rows.  Thread 0 keeps
// kStages tiles of (times, features) in flight with 1-D TMA bulk copies that
// complete on "full" mbarriers.  Every warp owns TR/32 rows of a tile (P = 4
// lanes per row for TR = 256): it labels them, bins them, writes its rows'
// bins and labels straight to global memory (coalesced) and arrives on the
// stage's "empty" mbarrier — no block-wide barrier in the loop.
//
// The per-block value cache is bucketised: a feature value hashes to a bucket
// of 4 slots whose 4 keys (16 B) and 4 provisional ids (8 B) are fetched with
// one 128-bit and one 64-bit shared load, so a hit costs one round trip.
constexpr int kStages = 2;
constexpr int kWarps = kIngestThreads / 32;
constexpr uint16_t kNoId = 0xFFFF;

struct IngestArgs {
  const float *feat, *times;
  int64_t n;
  int F, V, BS, TR, P, log2nb, use_tma;
  uint32_t *gkey, *gid, *gcount, *flags;
  uint8_t *bins, *labels;
};

__device__ __forceinline__ int bucket_find(const uint4 K, const uint2 I, uint32_t key) {
  // id of `key` in the bucket, -1 if absent or not yet published
  int id = -1;
  if (K.x == key) id = I.x & 0xFFFF;
  if (K.y == key) id = I.x >> 16;
  if (K.z == key) id = I.y & 0xFFFF;
  if (K.w == key) id = I.y >> 16;
  return id == kNoId ? -1 : id;
}

__device__ __noinline__ int cache_miss(uint32_t *keys, uint16_t *ids, int log2nb, uint32_t key,
                                       const IngestArgs &a, int f) {
  const int NB = 1 << log2nb;
  const uint32_t b0 = hash_slot(key, log2nb);
  for (int p = 1; p < NB; p++) {  // later buckets of the probe sequence
    const uint32_t b = (b0 + p) & (NB - 1);
    const int id = bucket_find(reinterpret_cast<const uint4 *>(keys)[b],
                               reinterpret_cast<const uint2 *>(ids)[b], key);
    if (id >= 0) return id;
    if (keys[4 * b + 3] == kEmptyKey) break;  // a bucket with room ends the sequence
  }
  const uint32_t id = global_lookup(a.gkey, a.gid, a.gcount, a.flags, f, key);
  for (int p = 0; p < NB; p++) {  // publish (best effort: a full cache just misses)
    const uint32_t b = (b0 + p) & (NB - 1);
    for (int e = 0; e < 4; e++) {
      const uint32_t old = atomicCAS(keys + 4 * b + e, kEmptyKey, key);
      if (old == kEmptyKey) {
        ids[4 * b + e] = (uint16_t)id;
        return (int)id;
      }
      if (old == key) return (int)id;
    }
  }
  return (int)id;
}

__device__ __forceinline__ uint32_t canon_key(float x, uint32_t &flags) {
  uint32_t key = __float_as_uint(x);
  if ((key & 0x7f800000u) == 0x7f800000u) {
    flags |= kFlagBadFeature;
    key = 0;
  }
  return x == 0.0f ? 0u : key;  // -0 -> +0 (R4)
}

__device__ __forceinline__ int lookup(uint32_t *keys, uint16_t *ids, int log2nb, uint32_t key,
                                      const IngestArgs &a, int f) {
  const uint32_t b = hash_slot(key, log2nb);
  const int id = bucket_find(reinterpret_cast<const uint4 *>(keys)[b],
                             reinterpret_cast<const uint2 *>(ids)[b], key);
  return id >= 0 ? id : cache_miss(keys, ids, log2nb, key, a, f);
}

__global__ void __launch_bounds__(kIngestThreads, 1) ingest_kernel(IngestArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int F = a.F, V = a.V, BS = a.BS, TR = a.TR, P = a.P;
  const int NB = 1 << a.log2nb;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem);
  uint64_t *empty = full + kStages;
  uint32_t *ckeys = reinterpret_cast<uint32_t *>(smem + 128);   // [F][NB][4]
  uint16_t *cids = reinterpret_cast<uint16_t *>(ckeys + F * NB * 4);  // [F][NB][4]
  const size_t o1 = 128 + (size_t)F * NB * 24;
  float *stT = reinterpret_cast<float *>(smem + o1);
  float *stF = stT + (size_t)kStages * TR * V;

  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < F * NB * 4; i += blockDim.x) {
    ckeys[i] = kEmptyKey;
    cids[i] = kNoId;
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int64_t ntiles = (a.n + TR - 1) / TR;
  const int64_t nfull = a.n / TR;  // tiles that TMA can load whole
  const int64_t first = blockIdx.x, stride = gridDim.x;
  const int64_t K = first < ntiles ? (ntiles - 1 - first) / stride + 1 : 0;
  const uint32_t bytesT = (uint32_t)TR * V * 4, bytesF = (uint32_t)TR * F * 4;
  auto issue = [&](int64_t k) {  // thread 0 only
    const int64_t t = first + k * stride;
    if (!a.use_tma || t >= nfull) return;
    const int s = (int)(k % kStages);
    if (k >= kStages) mbar_wait(&empty[s], (uint32_t)(((k / kStages) - 1) & 1));
    mbar_arrive_expect_tx(&full[s], bytesT + bytesF);
    tma_load_1d(stT + (size_t)s * TR * V, a.times + t * TR * V, bytesT, &full[s]);
    tma_load_1d(stF + (size_t)s * TR * F, a.feat + t * TR * F, bytesF, &full[s]);
  };
  if (tid == 0)
    for (int64_t k = 0; k < K && k < kStages; k++) issue(k);

  uint32_t local_flags = 0;
  const int r = tid / P, q = tid % P;
  const bool vec_t = (V & 3) == 0;
  const int per = F / P;                        // features per lane when F % P == 0
  const bool vec_f = (F % P) == 0 && (per & 3) == 0;
  for (int64_t k = 0; k < K; k++) {
    const int64_t t = first + k * stride;
    const int64_t row0 = t * TR;
    const int rows = (a.n - row0 < TR) ? (int)(a.n - row0) : TR;
    const int s = (int)(k % kStages);
    float *tT = stT + (size_t)s * TR * V;
    float *tF = stF + (size_t)s * TR * F;
    if (a.use_tma && t < nfull) {
      mbar_wait(&full[s], (uint32_t)((k / kStages) & 1));
    } else {  // partial last tile or unaligned inputs: plain loads, block-synchronous
      __syncthreads();
      for (int i = tid; i < rows * V; i += blockDim.x) tT[i] = __ldcs(a.times + row0 * V + i);
      for (int i = tid; i < rows * F; i += blockDim.x) tF[i] = __ldcs(a.feat + row0 * F + i);
      __syncthreads();
    }
    // ---- a1: label = lowest index of the minimum (P lanes per row) ----
    float best = __int_as_float(0x7f800000);
    int bi = 0x7fffffff;
    bool nan = false;
    const bool live = r < rows;
    if (live) {
      const float *tr = tT + (size_t)r * V;
      if (vec_t) {
        const float4 *t4 = reinterpret_cast<const float4 *>(tr);
        for (int c = q; c < (V >> 2); c += P) {
          const float4 x = t4[c];
          nan |= (x.x != x.x) | (x.y != x.y) | (x.z != x.z) | (x.w != x.w);
          // ascending index within this lane: strict '<' keeps the lowest
          if (x.x < best) { best = x.x; bi = 4 * c; }
          if (x.y < best) { best = x.y; bi = 4 * c + 1; }
          if (x.z < best) { best = x.z; bi = 4 * c + 2; }
          if (x.w < best) { best = x.w; bi = 4 * c + 3; }
        }
      } else {
        for (int v = q; v < V; v += P) {
          const float x = tr[v];
          nan |= x != x;
          if (x < best) {
            best = x;
            bi = v;
          }
        }
      }
    }
    for (int o = 1; o < P; o <<= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob < best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if (live) {
      if (nan) local_flags |= kFlagNanTime;
      if (q == 0) {
        if (best == __int_as_float(0x7f800000)) local_flags |= kFlagAllInf;
        a.labels[row0 + r] = (uint8_t)(bi < V ? bi : 0);
      }
      // ---- a2 + a3: provisional ids of this lane's features ----
      const float *fr = tF + (size_t)r * F;
      uint8_t *dst = a.bins + (row0 + r) * BS;
      if (vec_f) {
        for (int c = 0; c < per; c += 4) {
          const int f = q * per + c;
          const float4 x = *reinterpret_cast<const float4 *>(fr + f);
          const uint32_t key[4] = {canon_key(x.x, local_flags), canon_key(x.y, local_flags),
                                   canon_key(x.z, local_flags), canon_key(x.w, local_flags)};
          uint4 Kb[4];
          uint2 Ib[4];
#pragma unroll
          for (int e = 0; e < 4; e++) {  // the 4 features' buckets, loaded together
            const uint32_t b = hash_slot(key[e], a.log2nb);
            Kb[e] = reinterpret_cast<const uint4 *>(ckeys + (size_t)(f + e) * NB * 4)[b];
            Ib[e] = reinterpret_cast<const uint2 *>(cids + (size_t)(f + e) * NB * 4)[b];
          }
          uint32_t packed = 0;
#pragma unroll
          for (int e = 0; e < 4; e++) {
            int id = bucket_find(Kb[e], Ib[e], key[e]);
            if (id < 0)
              id = cache_miss(ckeys + (size_t)(f + e) * NB * 4, cids + (size_t)(f + e) * NB * 4,
                              a.log2nb, key[e], a, f + e);
            packed |= (uint32_t)(id & 0xFF) << (8 * e);
          }
          *reinterpret_cast<uint32_t *>(dst + f) = packed;
        }
      } else {
        for (int f = q; f < F; f += P)
          dst[f] = (uint8_t)lookup(ckeys + (size_t)f * NB * 4, cids + (size_t)f * NB * 4, a.log2nb,
                                   canon_key(fr[f], local_flags), a, f);
        for (int f = F + q; f < BS; f += P) dst[f] = 0;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s
    if (tid == 0 && k + kStages < K) issue(k + kStages);
  }
  if (local_flags) atomicOr(a.flags, local_flags);
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
                                uint8_t *out) {  // rec = bins plane, RS = its row stride
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * F;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / F;
    const int f = (int)(i % F);
    out[i] = lut[f * kMaxBins + rec[r * RS + f]];
  }
}

int grid_for(int64_t work, int per_block, int cap) {
  int64_t b = (work + per_block - 1) / per_block;
  if (b < 1) b = 1;
  return (int)(b < cap ? b : cap);
}

}  // namespace

void launch_ingest(const float *feat, const float *times, int64_t n, int F, int V, int BS,
                   uint32_t *gkey, uint32_t *gid, uint32_t *gcount, uint32_t *flags,
                   uint8_t *bins, uint8_t *labels, cudaStream_t s) {
  if (n == 0) return;
  IngestArgs a;
  a.feat = feat;
  a.times = times;
  a.n = n;
  a.F = F;
  a.V = V;
  a.BS = BS;
  a.gkey = gkey;
  a.gid = gid;
  a.gcount = gcount;
  a.flags = flags;
  a.bins = bins;
  a.labels = labels;
  // per-block value cache: 128 buckets x 4 slots per feature (load <= 1/2 at
  // 256 values), fewer when F is large
  a.log2nb = 7;
  while (a.log2nb > 3 && (size_t)F * (24u << a.log2nb) > 48 * 1024) a.log2nb--;
  const size_t cache = 128 + (size_t)F * (24u << a.log2nb);
  // P threads per row, TR = threads / P rows per tile: the largest tile whose
  // kStages (times, features) buffers fit next to the cache
  a.P = 4;
  while (a.P < 32 && cache + (size_t)kStages * (kIngestThreads / a.P) * (V + F) * 4 > 220 * 1024)
    a.P <<= 1;
  a.TR = kIngestThreads / a.P;
  a.use_tma = ((reinterpret_cast<uintptr_t>(feat) | reinterpret_cast<uintptr_t>(times)) & 15) == 0;
  const size_t smem = cache + (size_t)kStages * a.TR * (V + F) * 4;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ntiles = (n + a.TR - 1) / a.TR;
  const int grid = (int)std::min<int64_t>(ntiles, sms);
  CUDA_CHECK(cudaFuncSetAttribute(ingest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  ingest_kernel<<<grid, kIngestThreads, smem, s>>>(a);
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

}  // namespace adapt
