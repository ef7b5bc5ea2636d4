// ingest.cu — steps a1 (label), a2 (value tables) and a3 (bin) of SURVEY §8(a).
//
// Two streaming passes over the profiling table:
//   discover_kernel   reads the features once (4F bytes/row) and collects the
//                     distinct canonical float32 values of every feature in a
//                     per-CTA shared-memory set backed by a global lock-free
//                     hash set (R4: -0 -> +0; NaN/Inf flagged; > 256 flagged, R14).
//   merge_values_kernel  sorts the union of the (per-rank) sets into the value
//                     table val[f][rank] (a2) and builds, per feature, a
//                     perfect hash key -> rank ("hash and displace": 64
//                     displacements + 512 one-byte slots, collision-free for the
//                     feature's own keys — the only keys the next pass meets).
//   label_bin_kernel  streams (times, features) tiles with 1-D TMA bulk copies
//                     (mbarrier pipeline, one persistent CTA per SM): a1 label =
//                     lowest index of the minimum time, +inf = unmeasured (P:173,
//                     R2, R3); a3 bin = rank of the value through the perfect
//                     hash (two dependent byte loads, no misses, no atomics).  Writes the
//                     bins as word planes (plane p = bytes [4p, 4p+4) of every row's
//                     BS = F-rounded-up-to-a-power-of-two bins) and labels [N].
// So every later pass works directly in rank space (bins == ranks).
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.h"
#include "ptx.h"

namespace adapt {
namespace {

__device__ __forceinline__ uint32_t hash_bits(uint32_t key, uint32_t mul, int log2n) {
  return (key * mul) >> (32 - log2n);
}

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t *p) {
  return *(volatile const uint32_t *)p;
}

__device__ __forceinline__ uint32_t canon_key(float x, uint32_t &flags, uint32_t bad) {
  uint32_t key = __float_as_uint(x);
  if ((key & 0x7f800000u) == 0x7f800000u) {
    flags |= bad;
    key = 0;
  }
  return x == 0.0f ? 0u : key;  // -0 -> +0 (R4)
}

// perfect-hash geometry per feature: 64 displacements (u16) + 512 slot ranks (u8)
constexpr int kPhLog2Buckets = 6, kPhLog2Slots = 9;
constexpr int kPhBuckets = 1 << kPhLog2Buckets, kPhSlots = 1 << kPhLog2Slots;
constexpr int kPhBytes = kPhBuckets * 2 + kPhSlots;  // 640

// ------------------------------------------------------------ discovery --
constexpr int kDiscThreads = 512;
constexpr uint32_t kMul = 2654435761u;

__device__ void global_insert(uint32_t *gkey, uint32_t *gcount, uint32_t *flags, int f, uint32_t key) {
  uint32_t *K = gkey + (size_t)f * kGSlots;
  uint32_t h = hash_bits(key, kMul, 10);
  static_assert(kGSlots == 1024, "hash width");
  for (int p = 0; p < kGSlots; p++) {
    uint32_t k = ld_volatile(K + h);
    if (k == kEmptyKey) {
      k = atomicCAS(K + h, kEmptyKey, key);
      if (k == kEmptyKey) {
        if (atomicAdd(gcount + f, 1u) >= (uint32_t)kMaxBins) atomicOr(flags, kFlagTooMany);
        return;
      }
    }
    if (k == key) return;
    h = (h + 1) & (kGSlots - 1);
  }
  atomicOr(flags, kFlagTooMany);  // table full: far more than 256 values
}

// The per-CTA value set of a feature: NB buckets of 4 keys; a key lives in
// the first bucket of its probe sequence h, h+1, ... with a free slot, so a
// lookup of a present key is one 16-byte shared load in the common case.
// Slow path: walk the sequence, insert, publish globally.
__device__ __noinline__ void see_slow(uint32_t *S, int log2nb, uint32_t key, uint32_t *gkey,
                                      uint32_t *gcount, uint32_t *flags, int f) {
  const int NB = 1 << log2nb;
  uint32_t b = hash_bits(key, kMul, log2nb);
  for (int p = 0; p < NB; p++) {
    for (int e = 0; e < 4; e++) {
      uint32_t k = S[4 * b + e];
      if (k == key) return;
      if (k == kEmptyKey) {
        k = atomicCAS(S + 4 * b + e, kEmptyKey, key);
        if (k == kEmptyKey) {  // first sighting in this CTA: publish globally
          global_insert(gkey, gcount, flags, f, key);
          return;
        }
        if (k == key) return;
      }
    }
    b = (b + 1) & (NB - 1);
  }
  global_insert(gkey, gcount, flags, f, key);  // CTA set full: always ask the global one
}

constexpr int kDiscUnroll = 4;  // float4 loads in flight per thread

// n rows of a possibly sampled view: sample row i is table row
// i + (i / chunk_rows) * gap_rows (chunks of chunk_rows rows, gap_rows apart)
__global__ void __launch_bounds__(kDiscThreads) discover_kernel(const float *__restrict__ feat,
                                                               int64_t n, int F, int log2nb,
                                                               uint32_t *gkey, uint32_t *gcount,
                                                               uint32_t *flags, int64_t chunk_rows,
                                                               int64_t gap_rows) {
  extern __shared__ uint4 sset4[];  // [F][NB] buckets of 4 keys seen by this CTA
  uint32_t *sset = reinterpret_cast<uint32_t *>(sset4);
  const int NB = 1 << log2nb;
  for (int i = threadIdx.x; i < F * NB * 4; i += blockDim.x) sset[i] = kEmptyKey;
  __syncthreads();
  uint32_t local_flags = 0;
  // fast path: the value is in its home bucket (almost always, once warm)
  auto see = [&](int f, uint32_t key) {
    const uint4 K = sset4[f * NB + hash_bits(key, kMul, log2nb)];
    if (K.x != key && K.y != key && K.z != key && K.w != key)
      see_slow(sset + f * NB * 4, log2nb, key, gkey, gcount, flags, f);
  };
  const int64_t total = n * F;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  // every thread runs the same number of iterations and the warp re-converges
  // at the end of each, so the loads stay coalesced even though the set
  // insertions diverge
  if ((F & 3) == 0 && (reinterpret_cast<uintptr_t>(feat) & 15) == 0) {
    // float4 j holds features 4j % F .. +3 of one row (coalesced)
    const float4 *f4 = reinterpret_cast<const float4 *>(feat);
    const int64_t n4 = total / 4;
    int f0 = (int)((4 * tid0) % F);
    const int df = (int)((4 * stride) % F);
    for (int64_t base = 0; base < n4; base += kDiscUnroll * stride) {
      float4 x[kDiscUnroll];
#pragma unroll
      for (int u = 0; u < kDiscUnroll; u++) {
        const int64_t j = base + u * stride + tid0;
        x[u] = j < n4 ? __ldcs(f4 + j + ((4 * j) / F / chunk_rows) * gap_rows * (F / 4))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kDiscUnroll; u++) {
        if (base + u * stride + tid0 < n4) {
          see(f0, canon_key(x[u].x, local_flags, kFlagBadFeature));
          see(f0 + 1, canon_key(x[u].y, local_flags, kFlagBadFeature));
          see(f0 + 2, canon_key(x[u].z, local_flags, kFlagBadFeature));
          see(f0 + 3, canon_key(x[u].w, local_flags, kFlagBadFeature));
        }
        f0 += df;
        if (f0 >= F) f0 -= F;
      }
      __syncwarp();
    }
  } else {
    int f0 = (int)(tid0 % F);
    const int df = (int)(stride % F);
    for (int64_t base = 0; base < total; base += stride) {
      const int64_t i = base + tid0;
      if (i < total)
        see(f0, canon_key(__ldcs(feat + i + (i / F / chunk_rows) * gap_rows * F), local_flags,
                          kFlagBadFeature));
      f0 += df;
      if (f0 >= F) f0 -= F;
      __syncwarp();
    }
  }
  if (local_flags) atomicOr(flags, local_flags);
}

__global__ void collect_values_kernel(const uint32_t *gkey, const uint32_t *gcount,
                                      float *local_vals, int32_t *local_cnt) {
  __shared__ uint32_t cnt;
  const int f = blockIdx.x;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int s = threadIdx.x; s < kGSlots; s += blockDim.x) {
    const uint32_t k = gkey[(size_t)f * kGSlots + s];
    if (k == kEmptyKey) continue;
    const uint32_t i = atomicAdd(&cnt, 1u);
    if (i < (uint32_t)kMaxBins) local_vals[f * kMaxBins + i] = __uint_as_float(k);
  }
  if (threadIdx.x == 0) local_cnt[f] = (int32_t)min(gcount[f], (uint32_t)kMaxBins + 1);
}

// Union of every rank's distinct values of feature f, sorted into val[f][*] (a2).
__global__ void merge_values_kernel(const float *all_vals, const int32_t *all_cnt, int world, int F,
                                    float *val, int32_t *nval, uint32_t *flags) {
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
  for (int c = threadIdx.x; c < M; c += blockDim.x) {
    if (!rep[c]) continue;
    const float x = cand[c];
    int r = 0;
    for (int e = 0; e < M; e++) r += (rep[e] && cand[e] < x);
    if (r < kMaxBins) val[f * kMaxBins + r] = x;
  }
}

// ------------------------------------------------------------ label + bin --
// One CTA per SM, persistent over row tiles of TR rows.  Thread 0 keeps
// kStages tiles of (times, features) in flight with 1-D TMA bulk copies that
// complete on "full" mbarriers.  Every warp owns TR/32 rows of a tile (P
// lanes per row): it labels them, bins them, writes its rows' bins and labels
// straight to global memory and arrives on the stage's "empty" mbarrier.
constexpr int kIngestThreads = 1024;
#ifndef ADAPT_INGEST_STAGES
#define ADAPT_INGEST_STAGES 2
#endif
constexpr int kStages = ADAPT_INGEST_STAGES;  // TMA tile stages (tuning knob)
constexpr int kWarps = kIngestThreads / 32;

struct LabelBinArgs {
  const float *feat, *times;
  int64_t n;
  int F, V, BS, TR, P, use_tma;
  const uint8_t *tab;       // [F][kPhBytes] perfect hashes
  const uint32_t *lk_mul;   // [F][2] their multipliers
  const uint32_t *slot_keys;  // [F][512] the key of every hash slot (0xFFFFFFFF: empty)
  int keys_in_smem;           // copy them to smem (else read through L1: wide tables)
  int verify;                 // check every key (the tables came from a sample)
  uint32_t *flags;
  uint8_t *bins, *labels;
  size_t pstride;           // bytes between bins word planes
};

// VQ / FQ: float4 chunks of times / features per lane when known at compile
// time (the common shapes; 0 = runtime loops): fully unrolled, constant offsets
template <int VQ, int FQ>
__global__ void __launch_bounds__(kIngestThreads, 1) label_bin_kernel(LabelBinArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  // the compile-time shape (VQ, FQ > 0: C4's 48 variants and 16 features, 4
  // lanes per row, 256-row tiles) folds the tile / stage address arithmetic
  constexpr bool kFixed = VQ > 0 && FQ > 0;
  const int P = kFixed ? 4 : a.P;
  const int TR = kFixed ? kIngestThreads / 4 : a.TR;
  const int V = kFixed ? 16 * VQ : a.V, F = kFixed ? 16 * FQ : a.F;
  const int BS = kFixed ? 16 * FQ : a.BS;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem);
  uint64_t *empty = full + kStages;
  uint32_t *lmul = reinterpret_cast<uint32_t *>(smem + 128);  // [F][2]
  uint8_t *tab = smem + 128 + 8 * kMaxF;                     // [F][kPhBytes]
  const size_t o0 = (128 + 8 * kMaxF + (size_t)F * kPhBytes + 15) & ~(size_t)15;
  uint32_t *skeys = reinterpret_cast<uint32_t *>(smem + o0);  // [F][kPhSlots]
  const size_t o1 = o0 + (a.keys_in_smem ? (size_t)F * kPhSlots * 4 : 0);
  float *stT = reinterpret_cast<float *>(smem + o1);
  float *stF = stT + (size_t)kStages * TR * V;

  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < F * kPhBytes / 4; i += blockDim.x)
    reinterpret_cast<uint32_t *>(tab)[i] = reinterpret_cast<const uint32_t *>(a.tab)[i];
  for (int i = tid; i < 2 * F; i += blockDim.x) lmul[i] = a.lk_mul[i];
  if (a.keys_in_smem)
    for (int i = tid; i < F * kPhSlots; i += blockDim.x) skeys[i] = a.slot_keys[i];
  const uint32_t *kk = a.keys_in_smem ? skeys : a.slot_keys;
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
  // every tile's empty-barrier phase is waited exactly once by thread 0: tile
  // k - kStages's here (before stage s is refilled), the last kStages after the
  // loop, TMA-loaded or not (synccheck: no arrival phase left unconsumed)
  auto issue = [&](int64_t k) {  // thread 0 only
    const int64_t t = first + k * stride;
    const int s = (int)(k % kStages);
    if (k >= kStages) mbar_wait(&empty[s], (uint32_t)(((k / kStages) - 1) & 1));
    if (!a.use_tma || t >= nfull) return;
    mbar_arrive_expect_tx(&full[s], bytesT + bytesF);
    tma_load_1d(stT + (size_t)s * TR * V, a.times + t * TR * V, bytesT, &full[s]);
    tma_load_1d(stF + (size_t)s * TR * F, a.feat + t * TR * F, bytesF, &full[s]);
  };
  if (tid == 0)
    for (int64_t k = 0; k < K && k < kStages; k++) issue(k);

  uint32_t local_flags = 0;
  const int r = tid / P, q = tid % P;
  const bool vec_t = kFixed || (V & 3) == 0;
  const int per = F / P;  // features per lane when F % P == 0
  const bool vec_f = kFixed || ((F % P) == 0 && (per & 3) == 0);
  // perfect hash: the displacement, then the slot's rank and key (independent
  // loads); a key that is not the slot's is a value the discovery (sample)
  // missed: flagged, the caller re-discovers the whole table
  uint32_t miss = 0;  // OR of (slot key ^ key): nonzero iff some value was not in the tables
  auto rank_of = [&](int f, uint32_t key) -> int {
    const uint8_t *t = tab + f * kPhBytes;
    const uint32_t d = reinterpret_cast<const uint16_t *>(t)[hash_bits(key, lmul[2 * f], kPhLog2Buckets)];
    const uint32_t sl = (hash_bits(key, lmul[2 * f + 1], kPhLog2Slots) + d) & (kPhSlots - 1);
    if (a.verify) miss |= kk[f * kPhSlots + sl] ^ key;
    return t[kPhBuckets * 2 + sl];
  };
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
        auto chunk = [&](int c) {
          const float4 x = t4[c];
          nan |= (x.x != x.x) | (x.y != x.y) | (x.z != x.z) | (x.w != x.w);
          // ascending index within this lane: strict '<' keeps the lowest
          if (x.x < best) { best = x.x; bi = 4 * c; }
          if (x.y < best) { best = x.y; bi = 4 * c + 1; }
          if (x.z < best) { best = x.z; bi = 4 * c + 2; }
          if (x.w < best) { best = x.w; bi = 4 * c + 3; }
        };
        if constexpr (VQ > 0) {
#pragma unroll
          for (int i = 0; i < VQ; i++) chunk(q + i * P);
        } else {
          for (int c = q; c < (V >> 2); c += P) chunk(c);
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
      // ---- a3: rank of each of this lane's feature values ----
      const float *fr = tF + (size_t)r * F;
      const int64_t row = row0 + r;
      if (vec_f) {
#pragma unroll
        for (int c = 0; c < (FQ > 0 ? 4 * FQ : per); c += 4) {
          const int f = q * per + c;
          const float4 x = *reinterpret_cast<const float4 *>(fr + f);
          const int r0 = rank_of(f, canon_key(x.x, local_flags, kFlagBadFeature));
          const int r1 = rank_of(f + 1, canon_key(x.y, local_flags, kFlagBadFeature));
          const int r2 = rank_of(f + 2, canon_key(x.z, local_flags, kFlagBadFeature));
          const int r3 = rank_of(f + 3, canon_key(x.w, local_flags, kFlagBadFeature));
          *reinterpret_cast<uint32_t *>(a.bins + (f / 4) * a.pstride + row * 4) =  // word plane f/4
              (uint32_t)(r0 & 0xFF) | ((uint32_t)(r1 & 0xFF) << 8) | ((uint32_t)(r2 & 0xFF) << 16) |
              ((uint32_t)(r3 & 0xFF) << 24);
        }
      } else {
        const int wb = BS < 4 ? BS : 4;  // bytes per plane element
        for (int f = q; f < BS; f += P)
          a.bins[(BS < 4 ? 0 : f / 4) * a.pstride + row * wb + (BS < 4 ? f : f % 4)] =
              f < F ? (uint8_t)rank_of(f, canon_key(fr[f], local_flags, kFlagBadFeature)) : 0;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s
    if (tid == 0 && k + kStages < K) issue(k + kStages);
  }
  // drain: the last kStages tiles' empty phases (see issue)
  if (tid == 0)
    for (int64_t k = K > kStages ? K - kStages : 0; k < K; k++)
      mbar_wait(&empty[k % kStages], (uint32_t)((k / kStages) & 1));
  if (miss) local_flags |= kFlagUnseen;
  if (local_flags) atomicOr(a.flags, local_flags);
}

__global__ void bins_out_kernel(const uint8_t *bins, size_t pstride, int64_t n, int F, int BS,
                                uint8_t *out) {
  const int wb = BS < 4 ? BS : 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * F;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / F;
    const int f = (int)(i - r * F);
    out[i] = bins[(BS < 4 ? 0 : f / 4) * pstride + r * wb + (BS < 4 ? f : f % 4)];
  }
}

int grid_for(int64_t work, int per_block, int cap) {
  int64_t b = (work + per_block - 1) / per_block;
  if (b < 1) b = 1;
  return (int)(b < cap ? b : cap);
}

int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

}  // namespace

int lookup_table_bytes(int F) { return F * kPhBytes; }
int lookup_slots() { return kPhSlots; }

// Perfect hash of one feature's sorted values (host; <= 256 keys): bucket
// h1(key) of 64 gets a displacement d so that slot (h2(key) + d) mod 512 is
// distinct for every key; buckets are placed largest first.  Same hash_bits
// as the device.  Returns false only if no seed works (never seen).
bool build_value_hash(const float *vals, int D, uint32_t mul[2], uint8_t *tab, uint32_t *slot_keys) {
  // hash-and-displace, allocation-free (it runs on the host between the
  // discovery and the bin pass, with the GPU idle): buckets by the first
  // hash, largest first (ties in bucket order), each bucket gets the
  // smallest displacement d that puts all its keys on free slots
  auto hb = [](uint32_t key, uint32_t m, int l) { return (key * m) >> (32 - l); };
  uint32_t keys[kMaxBins], h2[kMaxBins];
  int members[kMaxBins];
  for (int r = 0; r < D; r++) memcpy(&keys[r], &vals[r], 4);
  for (uint32_t seed = 0; seed < 1024; seed++) {
    const uint32_t m1 = (0x9E3779B1u + 0x85EBCA6Bu * seed) | 1u;
    const uint32_t m2 = (0xC2B2AE35u + 0x27D4EB2Fu * seed) | 1u;
    int cnt[kPhBuckets] = {0}, start[kPhBuckets + 1], fill[kPhBuckets];
    uint8_t bk[kMaxBins];
    int maxc = 0;
    for (int r = 0; r < D; r++) {
      bk[r] = (uint8_t)hb(keys[r], m1, kPhLog2Buckets);
      h2[r] = hb(keys[r], m2, kPhLog2Slots);
      maxc = std::max(maxc, ++cnt[bk[r]]);
    }
    start[0] = 0;
    for (int b = 0; b < kPhBuckets; b++) start[b + 1] = start[b] + cnt[b];
    for (int b = 0; b < kPhBuckets; b++) fill[b] = start[b];
    for (int r = 0; r < D; r++) members[fill[bk[r]]++] = r;  // rows in order within a bucket
    uint8_t used[kPhSlots] = {0};
    uint16_t disp[kPhBuckets] = {0};
    uint8_t slot_rank[kPhSlots] = {0};
    uint32_t skey[kPhSlots];
    for (int i = 0; i < kPhSlots; i++) skey[i] = 0xFFFFFFFFu;  // NaN bits: never a canonical key
    bool ok = true;
    for (int size = maxc; size >= 1 && ok; size--)
      for (int b = 0; b < kPhBuckets && ok; b++) {
        if (cnt[b] != size) continue;
        int found = -1;
        uint32_t taken[kMaxBins];
        for (int d = 0; d < kPhSlots && found < 0; d++) {
          bool good = true;
          int nt = 0;
          for (int q = start[b]; q < start[b + 1] && good; q++) {
            const uint32_t sl = (h2[members[q]] + d) & (kPhSlots - 1);
            if (used[sl]) good = false;
            for (int t = 0; t < nt && good; t++) good = taken[t] != sl;
            taken[nt++] = sl;
          }
          if (good) found = d;
        }
        if (found < 0) {
          ok = false;
          break;
        }
        disp[b] = (uint16_t)found;
        for (int q = start[b]; q < start[b + 1]; q++) {
          const int r = members[q];
          const uint32_t sl = (h2[r] + found) & (kPhSlots - 1);
          used[sl] = 1;
          slot_rank[sl] = (uint8_t)r;
          skey[sl] = keys[r];
        }
      }
    if (!ok) continue;
    memcpy(tab, disp, sizeof disp);
    memcpy(tab + kPhBuckets * 2, slot_rank, kPhSlots);
    memcpy(slot_keys, skey, kPhSlots * 4);
    mul[0] = m1;
    mul[1] = m2;
    return true;
  }
  return false;
}

void launch_discover(const float *feat, int64_t n, int F, uint32_t *gkey, uint32_t *gcount,
                     uint32_t *flags, int64_t chunk_rows, int64_t gap_rows, cudaStream_t s) {
  if (n == 0) return;
  int log2nb = 8;  // 256 buckets x 4 keys per feature (~1 key per bucket at 256 values)
  while (log2nb > 4 && (size_t)F * (16u << log2nb) > 64 * 1024) log2nb--;
  const size_t smem = (size_t)F * (16u << log2nb);
  smem_limit(discover_kernel, smem);
  const int grid = grid_for(n * F / 4 + 1, kDiscThreads * 4, sm_count() * 2);
  discover_kernel<<<grid, kDiscThreads, smem, s>>>(feat, n, F, log2nb, gkey, gcount, flags,
                                                   chunk_rows > 0 ? chunk_rows : n + 1, gap_rows); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
}

void launch_collect_values(const uint32_t *gkey, const uint32_t *gcount, int F, float *local_vals,
                           int32_t *local_cnt, cudaStream_t s) {
  collect_values_kernel<<<F, 256, 0, s>>>(gkey, gcount, local_vals, local_cnt); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
}

void launch_merge_values(const float *all_vals, const int32_t *all_cnt, int world, int F,
                         float *val, int32_t *nval, uint32_t *flags, cudaStream_t s) {
  const size_t smem = (size_t)world * kMaxBins * 5;
  smem_limit(merge_values_kernel, smem);
  merge_values_kernel<<<F, 1024, smem, s>>>(all_vals, all_cnt, world, F, val, nval, flags); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
}

void launch_label_bin(const float *feat, const float *times, int64_t n, int F, int V, int BS,
                      const uint8_t *tab, const uint32_t *lk_mul, const uint32_t *slot_keys,
                      int verify, uint32_t *flags, uint8_t *bins, size_t pstride, uint8_t *labels,
                      cudaStream_t s) {
  if (n == 0) return;
  LabelBinArgs a;
  a.feat = feat;
  a.times = times;
  a.n = n;
  a.F = F;
  a.V = V;
  a.BS = BS;
  a.tab = tab;
  a.lk_mul = lk_mul;
  a.slot_keys = slot_keys;
  a.verify = verify;
  a.flags = flags;
  a.bins = bins;
  a.pstride = pstride;
  a.labels = labels;
  size_t table = (128 + 8 * kMaxF + (size_t)F * kPhBytes + 15) & ~(size_t)15;
  // slot keys in smem when they leave room for 4-lane rows (always at F <= 16)
  a.keys_in_smem = table + (size_t)F * kPhSlots * 4 +
                           (size_t)kStages * (kIngestThreads / 4) * (V + F) * 4 <= 220 * 1024;
  if (a.keys_in_smem) table += (size_t)F * kPhSlots * 4;
  // P threads per row, TR = threads / P rows per tile: the largest tile whose
  // kStages (times, features) buffers fit next to the table
  a.P = 4;
  while (a.P < 32 && table + (size_t)kStages * (kIngestThreads / a.P) * (V + F) * 4 > 220 * 1024)
    a.P <<= 1;
  a.TR = kIngestThreads / a.P;
  a.use_tma = ((reinterpret_cast<uintptr_t>(feat) | reinterpret_cast<uintptr_t>(times)) & 15) == 0;
  const size_t smem = table + (size_t)kStages * a.TR * (V + F) * 4;
  const int64_t ntiles = (n + a.TR - 1) / a.TR;
  const int grid = (int)std::min<int64_t>(ntiles, sm_count());
  // compile-time chunk counts for C4's shape (V = 48, F = 16 at 4 lanes per row)
  const bool c4 = a.P == 4 && V == 48 && F == 16;
  if (c4) {
    smem_limit(label_bin_kernel<3, 1>, smem);
    label_bin_kernel<3, 1><<<grid, kIngestThreads, smem, s>>>(a); ++g_kernel_launches;
  } else {
    smem_limit(label_bin_kernel<0, 0>, smem);
    label_bin_kernel<0, 0><<<grid, kIngestThreads, smem, s>>>(a); ++g_kernel_launches;
  }
  CUDA_CHECK(cudaGetLastError());
}

void launch_bins_out(const uint8_t *bins, size_t pstride, int64_t n, int F, int BS, uint8_t *out,
                     cudaStream_t s) {
  if (n == 0) return;
  bins_out_kernel<<<grid_for(n * F, 256, 148 * 16), 256, 0, s>>>(bins, pstride, n, F, BS, out); ++g_kernel_launches;
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace adapt
