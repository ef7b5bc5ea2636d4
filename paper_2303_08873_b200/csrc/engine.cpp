// engine.cpp — host side of libadapt.so: the C ABI of include/adapt.h, the
// region registry, the level-by-level training loop that drives the kernels
// of ingest.cu / train.cu / select.cu, NCCL plumbing for world > 1, per-phase
// CUDA-event profiling, and the Apollo Table-1 shim.
//
// Host work here is bookkeeping only (a few hundred bytes per tree node per
// level): every per-row step runs in the kernels.  The one row-level host
// routine is the long -> wide aggregation of adapt_record() profiling records
// (P:172-173), which is the small interactive path of the Table-1 shim; wide
// tables (adapt_record_table) never touch the host.
#include <dlfcn.h>
#include <nccl.h>
#include <time.h>

#include <algorithm>
#include <deque>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/adapt.h"
#include "common.h"

namespace adapt {

void cuda_check(cudaError_t e, const char *what) {
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    throw Error(ADAPT_E_OOM, std::string("out of device memory: ") + what);
  }
  if (e != cudaSuccess) throw Error(ADAPT_E_CUDA, std::string(cudaGetErrorString(e)) + ": " + what);
}

namespace {

// ------------------------------------------------------------ utilities --
bool trace_allocs() {  // ADAPT_TRACE_HOST=3: report every buffer (re)allocation
  static const bool on = getenv("ADAPT_TRACE_HOST") && atoi(getenv("ADAPT_TRACE_HOST")) >= 3;
  return on;
}

struct DevBuf {
  void *p = nullptr;
  size_t cap = 0;
  void ensure(size_t bytes) {
    if (bytes <= cap) return;
    if (trace_allocs()) fprintf(stderr, "[adapt] cudaMalloc %zu (had %zu)\n", bytes, cap);
    release();
    size_t want = std::max<size_t>(bytes, 256);
    CUDA_CHECK(cudaMalloc(&p, want));
    cap = want;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  // per-level buffers whose size varies level to level and call to call:
  // 1.5x headroom, so a later level / call rarely pays a (synchronising) cudaMalloc
  void grow(size_t bytes) {
    if (bytes > cap) ensure(std::max(bytes, cap + cap / 2));
  }
  template <class T>
  T *as() const { return static_cast<T *>(p); }
  ~DevBuf() { release(); }
};

struct HostBuf {  // pinned staging for small D2H copies
  void *p = nullptr;
  size_t cap = 0;
  void ensure(size_t bytes) {
    if (bytes <= cap) return;
    if (trace_allocs()) fprintf(stderr, "[adapt] cudaMallocHost %zu (had %zu)\n", bytes, cap);
    if (p) cudaFreeHost(p);
    p = nullptr;
    CUDA_CHECK(cudaMallocHost(&p, std::max<size_t>(bytes, 4096)));
    cap = std::max<size_t>(bytes, 4096);
  }
  // (cudaMallocHost pins pages: milliseconds per call) 1.5x headroom
  void grow(size_t bytes) {
    if (bytes > cap) ensure(std::max(bytes, cap + cap / 2));
  }
  template <class T>
  T *as() const { return static_cast<T *>(p); }
  ~HostBuf() {
    if (p) cudaFreeHost(p);
  }
};

// Per-level small host -> device arrays, gathered into one pinned buffer and
// uploaded with ONE async copy (a pageable cudaMemcpyAsync per array cost
// ~15 us of host time each, with the GPU idle).  Offsets are stable; device
// pointers are formed after flush().  The caller synchronises the stream
// before the next put() round (every level does).
struct Arena {
  HostBuf pinned;   // written directly by put() (no pageable staging copy)
  DevBuf dev;
  size_t used = 0;
  template <class T>
  size_t put(const std::vector<T> &v) {
    const size_t off = (used + 15) & ~size_t(15);
    const size_t end = off + v.size() * sizeof(T) + 16;
    if (end > pinned.cap) {  // grow geometrically (>= 4 MB), keeping what was put so far
      HostBuf nb;
      nb.ensure(std::max<size_t>({end, 2 * pinned.cap, (size_t)4 << 20}));
      if (used) memcpy(nb.p, pinned.p, used);
      std::swap(nb.p, pinned.p);
      std::swap(nb.cap, pinned.cap);
    }
    if (!v.empty()) memcpy(static_cast<uint8_t *>(pinned.p) + off, v.data(), v.size() * sizeof(T));
    used = end;
    return off;
  }
  void flush(cudaStream_t s) {
    if (!used) return;
    if (used > dev.cap) dev.ensure(std::max<size_t>({used, 2 * dev.cap, (size_t)4 << 20}));
    CUDA_CHECK(cudaMemcpyAsync(dev.p, pinned.p, used, cudaMemcpyHostToDevice, s));
    if (!copied) CUDA_CHECK(cudaEventCreateWithFlags(&copied, cudaEventDisableTiming));
    CUDA_CHECK(cudaEventRecord(copied, s));
    in_flight = true;
  }
  template <class T>
  T *ptr(size_t off) const { return reinterpret_cast<T *>(static_cast<uint8_t *>(dev.p) + off); }
  // the pinned buffer is the SOURCE of the last flush's async copy: before it is
  // written again that copy must have run (it can sit behind queued kernels)
  void reset() {
    if (in_flight) CUDA_CHECK(cudaEventSynchronize(copied));
    in_flight = false;
    used = 0;
  }
  ~Arena() {
    if (copied) cudaEventDestroy(copied);
  }
  cudaEvent_t copied = nullptr;
  bool in_flight = false;
};

thread_local std::string g_last_error;
std::recursive_mutex g_mu;

// ------------------------------------------------------------ profiling --
struct Prof {
  bool on = false;
  struct Rec {
    int phase;
    cudaEvent_t a, b;
    double bytes;
    long long kernels;  // kernels launched inside the phase
  };
  std::vector<std::string> names;
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  struct Acc {
    int64_t launches = 0;
    double ms = 0, bytes = 0;
  };
  std::vector<Acc> acc;
  int id(const char *n) {
    for (size_t i = 0; i < names.size(); i++)
      if (names[i] == n) return (int)i;
    names.push_back(n);
    acc.emplace_back();
    return (int)names.size() - 1;
  }
  cudaEvent_t ev() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    CUDA_CHECK(cudaEventCreate(&e));
    return e;
  }
  void drain() {
    for (auto &r : pending) {
      float ms = 0;
      CUDA_CHECK(cudaEventSynchronize(r.b));
      CUDA_CHECK(cudaEventElapsedTime(&ms, r.a, r.b));
      acc[r.phase].launches += r.kernels;
      acc[r.phase].ms += ms;
      acc[r.phase].bytes += r.bytes;
      pool.push_back(r.a);
      pool.push_back(r.b);
    }
    pending.clear();
  }
};
Prof g_prof;
}  // namespace
long long g_kernel_launches = 0;
namespace {

// RAII: events around the kernel(s) launched in its scope, on `s`
struct Phase {
  int ph = -1;
  cudaEvent_t a{}, b{};
  cudaStream_t s;
  double bytes;
  long long k0 = 0;  // g_kernel_launches at the start
  Phase(const char *name, cudaStream_t st, double by) : s(st), bytes(by) {
    if (!g_prof.on) return;
    ph = g_prof.id(name);
    a = g_prof.ev();
    b = g_prof.ev();
    k0 = g_kernel_launches;
    CUDA_CHECK(cudaEventRecord(a, s));
  }
  ~Phase() {
    if (ph < 0) return;
    cudaEventRecord(b, s);
    g_prof.pending.push_back({ph, a, b, bytes, g_kernel_launches - k0});
  }
};

// ------------------------------------------------------------ NCCL (dlopen) --
struct Nccl {
  void *h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                            ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                                ncclComm_t, cudaStream_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  void load() {
    if (h) return;
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *n : names)
      if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) throw Error(ADAPT_E_NCCL, "cannot dlopen libnccl.so.2");
#define SYM(field, name)                                                     \
  field = reinterpret_cast<decltype(field)>(dlsym(h, name));                 \
  if (!field) throw Error(ADAPT_E_NCCL, std::string("missing NCCL symbol ") + name);
    SYM(GetUniqueId, "ncclGetUniqueId");
    SYM(CommInitRank, "ncclCommInitRank");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(AllReduce, "ncclAllReduce");
    SYM(AllGather, "ncclAllGather");
    SYM(ReduceScatter, "ncclReduceScatter");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
  }
  void check(ncclResult_t r, const char *what) {
    if (r != ncclSuccess)
      throw Error(ADAPT_E_NCCL, std::string(what) + ": " + (GetErrorString ? GetErrorString(r) : "?"));
  }
};
Nccl g_nccl;

struct Ctx {
  bool inited = false;
  int device = 0, rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  bool host_comm = false;  // collectives through caller hooks (adapt_init_host_comm)
  adapt_host_comm_t hooks{};
};
Ctx g_ctx;

// ---- the three collectives of SURVEY §8(e), over NCCL or the host hooks ----
// (ADAPT_NCCL_SELF=1 gives a world-1 run a 1-rank NCCL communicator so the
// NCCL path is exercised on one GPU; collectives are then real NCCL calls)
bool collectives_on() { return g_ctx.world > 1 || g_ctx.comm != nullptr; }

// per-level histogram exchange: with more than one rank, the
// reduce-scatter by node ownership + owner split search + winner all-gather
// (the split search, node-bound at deep levels, divides by the rank count);
// ADAPT_HIST_COMM=allreduce selects the all-reduce of the direct nodes'
// histograms (every rank searches every split), ADAPT_HIST_COMM=rs forces the
// reduce-scatter also on a 1-rank NCCL communicator
bool hist_comm_rs() {
  if (!collectives_on()) return false;
  const char *m = getenv("ADAPT_HIST_COMM");
  if (m && !strcmp(m, "allreduce")) return false;
  if (m && !strcmp(m, "rs")) return true;
  return g_ctx.world > 1;
}

void host_hook(int rc, const char *what) {
  if (rc != 0) throw Error(ADAPT_E_NCCL, std::string(what) + ": host collective hook returned " +
                                            std::to_string(rc));
}

// sum of `count` u32 (or u64 when wide) over ranks, in place on the device
void comm_allreduce_sum(void *dbuf, size_t count, bool wide, cudaStream_t s, const char *what) {
  if (!collectives_on() || count == 0) return;
  if (!g_ctx.host_comm) {
    g_nccl.check(g_nccl.AllReduce(dbuf, dbuf, count, wide ? ncclUint64 : ncclUint32, ncclSum,
                                  g_ctx.comm, s), what);
    return;
  }
  std::vector<uint64_t> w(count);
  if (wide) {
    CUDA_CHECK(cudaMemcpyAsync(w.data(), dbuf, count * 8, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  } else {
    std::vector<uint32_t> n(count);
    CUDA_CHECK(cudaMemcpyAsync(n.data(), dbuf, count * 4, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    for (size_t i = 0; i < count; i++) w[i] = n[i];
  }
  host_hook(g_ctx.hooks.all_reduce_u64(w.data(), count, g_ctx.hooks.user), what);
  if (wide) {
    CUDA_CHECK(cudaMemcpyAsync(dbuf, w.data(), count * 8, cudaMemcpyHostToDevice, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  } else {
    std::vector<uint32_t> n(count);
    for (size_t i = 0; i < count; i++) {
      if (w[i] > 0xFFFFFFFFull) throw Error(ADAPT_E_NCCL, std::string(what) + ": u32 sum overflow");
      n[i] = (uint32_t)w[i];
    }
    CUDA_CHECK(cudaMemcpyAsync(dbuf, n.data(), count * 4, cudaMemcpyHostToDevice, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
}

// drecv[0, count) = sum over ranks of dsend[rank * count, (rank + 1) * count)
// (u32): rank r receives the reduced chunk r (histograms summed
// only at the owner of their nodes)
void comm_reduce_scatter(const void *dsend, void *drecv, size_t count, cudaStream_t s,
                         const char *what) {
  if (!collectives_on()) {
    CUDA_CHECK(cudaMemcpyAsync(drecv, dsend, count * 4, cudaMemcpyDeviceToDevice, s));
    return;
  }
  if (count == 0) return;
  if (!g_ctx.host_comm) {
    g_nccl.check(g_nccl.ReduceScatter(dsend, drecv, count, ncclUint32, ncclSum, g_ctx.comm, s), what);
    return;
  }
  // host hooks: the element-wise sum of the whole buffer, then this rank's chunk
  const size_t total = count * (size_t)g_ctx.world;
  std::vector<uint32_t> n(total);
  CUDA_CHECK(cudaMemcpyAsync(n.data(), dsend, total * 4, cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  std::vector<uint64_t> w(n.begin(), n.end());
  host_hook(g_ctx.hooks.all_reduce_u64(w.data(), total, g_ctx.hooks.user), what);
  const size_t o = count * (size_t)g_ctx.rank;
  for (size_t i = 0; i < count; i++) {
    if (w[o + i] > 0xFFFFFFFFull) throw Error(ADAPT_E_NCCL, std::string(what) + ": u32 sum overflow");
    n[i] = (uint32_t)w[o + i];
  }
  CUDA_CHECK(cudaMemcpyAsync(drecv, n.data(), count * 4, cudaMemcpyHostToDevice, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
}

// drecv[r*bytes, (r+1)*bytes) = rank r's dsend, on the device
void comm_allgather(const void *dsend, void *drecv, size_t bytes, cudaStream_t s, const char *what) {
  if (!collectives_on()) {
    CUDA_CHECK(cudaMemcpyAsync(drecv, dsend, bytes, cudaMemcpyDeviceToDevice, s));
    return;
  }
  if (!g_ctx.host_comm) {
    g_nccl.check(g_nccl.AllGather(dsend, drecv, bytes, ncclUint8, g_ctx.comm, s), what);
    return;
  }
  std::vector<uint8_t> snd(bytes), rcv(bytes * g_ctx.world);
  CUDA_CHECK(cudaMemcpyAsync(snd.data(), dsend, bytes, cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  host_hook(g_ctx.hooks.all_gather(snd.data(), rcv.data(), bytes, g_ctx.hooks.user), what);
  CUDA_CHECK(cudaMemcpyAsync(drecv, rcv.data(), rcv.size(), cudaMemcpyHostToDevice, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
}

void ensure_init() {
  if (g_ctx.inited) return;
  int dev = 0;
  CUDA_CHECK(cudaGetDevice(&dev));
  int n = 0;
  CUDA_CHECK(cudaGetDeviceCount(&n));
  if (n == 0) throw Error(ADAPT_E_CUDA, "no CUDA device");
  cudaDeviceProp prop;
  CUDA_CHECK(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10) throw Error(ADAPT_E_CUDA, "libadapt is built for sm_100a (B200) only");
  g_ctx.device = dev;
  g_ctx.rank = 0;
  g_ctx.world = 1;
  g_ctx.inited = true;
}

// ------------------------------------------------------------ regions --
constexpr int kHistSmemBudget = 200 * 1024;  // counters + LUT per level-pass CTA (1 CTA/SM)

struct ClassSet {  // classes present in a node (C <= 255), ascending = compact order
  uint64_t bits[4] = {0, 0, 0, 0};
  void add(int c) { bits[c >> 6] |= 1ull << (c & 63); }
  bool has(int c) const { return (bits[c >> 6] >> (c & 63)) & 1; }
  int count() const {
    return __builtin_popcountll(bits[0]) + __builtin_popcountll(bits[1]) +
           __builtin_popcountll(bits[2]) + __builtin_popcountll(bits[3]);
  }
  int rank(int c) const {  // compact column of class c (number of present classes below it)
    int r = 0;
    for (int w = 0; w < (c >> 6); w++) r += __builtin_popcountll(bits[w]);
    return r + __builtin_popcountll(bits[c >> 6] & ((1ull << (c & 63)) - 1));
  }
  template <class Fn>
  void each(Fn fn) const {  // fn(class, compact column), ascending
    int k = 0;
    for (int w = 0; w < 4; w++)
      for (uint64_t b = bits[w]; b; b &= b - 1) fn(64 * w + __builtin_ctzll(b), k++);
  }
};

// a4 work split over the histogram CTAs (one per SM).  Cost model, measured on
// B200 with per-CTA timers at C4 (DESIGN.md §6 "histogram CTA balance"): a row
// costs row_ns of its group (its word's shared-memory reductions), a node
// portion kNodeNs (three block barriers and the pipeline refill) plus kCtrNs per
// counter it zeroes and flushes.  CTAs go to the groups in proportion to their
// total cost; within a group the virtual rows are cut at equal cost, a node
// split only where the piece carries enough rows to pay its own overhead.
constexpr double kNodeNs = 2200.0, kCtrNs = 0.13;
struct HistGroupCost {
  double row_ns;  // per counted row (all classes of the node in this slab)
  int k0, kw, dsw;  // class slab and the word's distinct values (counters = dsw * (kn | 1))
};
struct PlanNode {
  int fs, ls;  // its segments [fs, ls) (fs = -1: not known yet, the kernel searches)
  uint32_t base, len;
  int kc;
  double cf = 1.0;  // fraction of the rows read that are counted (tagged levels: child / parent rows)
};
std::vector<HistCta> plan_hist_ctas(const std::vector<PlanNode> &nodes, const std::vector<Seg> &segs,
                                    uint32_t total, const std::vector<HistGroupCost> &gc, int nct);
std::vector<HistCta> plan_hist_ctas(const std::vector<Seg> &segs, uint32_t total,
                                    const std::vector<HistGroupCost> &gc, int nct,
                                    const std::vector<double> *cf_of_slot = nullptr) {
  std::vector<PlanNode> nodes;
  for (int i = 0; i < (int)segs.size();) {
    int k = i;
    while (k < (int)segs.size() && segs[k].hslot == segs[i].hslot) k++;
    nodes.push_back(PlanNode{i, k, segs[i].node_base, segs[i].node_len, segs[i].ncls,
                             cf_of_slot ? (*cf_of_slot)[segs[i].hslot] : 1.0});
    i = k;
  }
  return plan_hist_ctas(nodes, segs, total, gc, nct);
}
std::vector<HistCta> plan_hist_ctas(const std::vector<PlanNode> &nodes, const std::vector<Seg> &segs,
                                    uint32_t total, const std::vector<HistGroupCost> &gc, int nct) {
  std::vector<HistCta> out;
  const int G = (int)gc.size();
  if (!total || nodes.empty() || G == 0) return out;
  using N = PlanNode;
  auto kn_of = [&](const HistGroupCost &c, int kc) { return std::min(c.kw, kc - c.k0); };
  auto row_of = [&](const HistGroupCost &c, int kc, double cf) {  // rows of other slabs (or
    // unmarked rows of a tagged level) are only loaded
    return c.row_ns * (0.3 + 0.7 * cf * (double)std::max(0, kn_of(c, kc)) / std::max(1, kc));
  };
  auto ovh = [&](const HistGroupCost &c, int kc) {
    const int kn = kn_of(c, kc);
    return kn > 0 ? kNodeNs + kCtrNs * (double)c.dsw * (kn | 1) : 0.0;
  };
  std::vector<double> T(G, 0.0);
  double sum = 0;
  for (int g = 0; g < G; g++) {
    for (const auto &n : nodes)
      if (kn_of(gc[g], n.kc) > 0) T[g] += ovh(gc[g], n.kc) + n.len * row_of(gc[g], n.kc, n.cf);
    sum += T[g];
  }
  // CTAs per group: proportional to cost, at least one for a group with work
  nct = std::max(nct, G);
  std::vector<int> ng(G, 0);
  int used = 0;
  for (int g = 0; g < G; g++)
    if (T[g] > 0) used += ng[g] = std::max(1, (int)std::lround(nct * T[g] / sum));
  while (used < nct && used > 0) {  // rounding shortfall: the group with the dearest CTAs
    int b = 0;
    for (int g = 1; g < G; g++)
      if (T[g] / std::max(ng[g], 1) > T[b] / std::max(ng[b], 1)) b = g;
    ng[b]++, used++;
  }
  while (used > nct) {  // rounding overshoot: trim the group with the cheapest CTAs
    int b = -1;
    for (int g = 0; g < G; g++)
      if (ng[g] > 1 && (b < 0 || T[g] / ng[g] < T[b] / ng[b])) b = g;
    if (b < 0) break;
    ng[b]--, used--;
  }
  auto seg_at = [&](const N &n, uint32_t p) {
    if (n.fs < 0) return -1;
    int k = n.fs;
    while (k + 1 < n.ls && segs[k + 1].row_base <= p) k++;
    return k;
  };
  // one group's greedy cut at `target` cost per CTA; returns the overhead the
  // node splits added (each extra piece of a node pays its zero/flush again)
  auto walk = [&](int g, double target, std::vector<HistCta> *emit) {
    int made = 0;
    double acc = 0, extra = 0;
    uint32_t start = 0;
    int s_start = 0;
    bool open = false;  // the current CTA holds rows
    auto close = [&](uint32_t end, int s_next, uint32_t next) {
      if (end > start) {
        if (emit) emit->push_back(HistCta{g, start, end, s_start});
        made++;
      }
      start = next;
      s_start = s_next;
      acc = 0;
      open = false;
    };
    for (const auto &n : nodes) {
      const int kn = kn_of(gc[g], n.kc);
      if (kn <= 0) continue;
      const double O = ovh(gc[g], n.kc), r = row_of(gc[g], n.kc, n.cf);
      uint32_t pos = n.base, left = n.len;
      if (!open) start = pos, s_start = n.fs;  // skip rows no CTA of g needs
      open = true;
      while (left > 0) {
        if (made == ng[g] - 1) {  // the last CTA takes the rest
          left = 0;
          break;
        }
        const double all = O + left * r;
        if (acc + all <= target) {
          acc += all;
          left = 0;
          break;
        }
        const double room = target - acc - O;
        const uint32_t take = room > 0 ? (uint32_t)std::min<double>(room / r, left) : 0u;
        if (take >= 4096 && take < left) {  // split the node here
          pos += take;
          left -= take;
          extra += O;
          close(pos, emit ? seg_at(n, pos) : 0, pos);
          open = true;
        } else if (acc > 0) {  // the node starts the next CTA
          close(pos, emit ? seg_at(n, pos) : 0, pos);
          open = true;
        } else {  // a fresh CTA that cannot split it usefully takes it whole
          acc += all;
          left = 0;
        }
      }
    }
    close(total, 0, total);
    return extra;
  };
  for (int g = 0; g < G; g++) {
    if (!ng[g]) continue;
    double extra = 0;  // the target from the cost including the splits' overheads
    for (int it = 0; it < 2; it++) extra = walk(g, (T[g] + extra) / ng[g], nullptr);
    walk(g, (T[g] + extra) / ng[g], &out);
  }
  return out;
}

struct FNode {  // a frontier node: histogrammed and split-searched at this level
  int32_t tree_idx;
  int32_t depth;
  int32_t slot;  // histogram slot at this level
  bool direct;   // histogrammed from its rows (else parent - sibling)
  ClassSet cls;  // classes present; the node's histogram columns
  int64_t rows = -1;  // its rows (the parent's winner record; single rank, unweighted)
  int32_t par = -1, side = 0;  // parent's index in the previous frontier, left (0) / right (1) child
};

}  // namespace
}  // namespace adapt

struct adapt_region {
  std::string id;
  int F = 0, V = 0, D = 2, min_train = 0;
  // long-format records: adapt_record (host, one at a time) and
  // adapt_record_batch (device store, rec_n records)
  std::vector<float> rfeat;
  std::vector<int32_t> rvar;
  std::vector<uint64_t> rns;
  adapt::DevBuf rec_feat, rec_var, rec_ns;
  int64_t rec_n = 0, rec_cap = 0;
  adapt::DevBuf slot_rep, slot_first, slot_of, rflag, rbsum, rgroups, slot_gid, rsum, rcnt;
  adapt::DevBuf agg_feat, agg_times;  // their wide rows (GPU aggregation output)
  bool aggregated = false;  // the last train used the record path (adapt_get_wide_table)
  // wide table
  int64_t n = 0;
  bool have_table = false;
  const float *d_feat = nullptr, *d_times = nullptr;
  adapt::DevBuf own_feat, own_times;
  // products of the last train
  int BS = 0;                   // bins per row incl. padding (F rounded up to a power of two)
  size_t pstride = 0;           // bytes between the bins word planes
  int64_t trained_n = 0;
  adapt::DevBuf bins, labels;   // ingest output in row order (kept for introspection)
  adapt::DevBuf binsA, binsB, labA, labB;  // level planes, rows grouped by node span
  // random forest (kind 1): T trees of depth D on bootstrap resamples (R19-R21)
  int kind = 0;        // 0: dtree, 1: rfc
  int T = 1;
  uint64_t seed = 0;
  std::vector<std::vector<adapt_node_t>> forest;  // canonical BFS trees
  adapt::DevBuf d_forest, d_roots;                 // concatenated device nodes, root indices
  int forest_nodes = 0;
  adapt::DevBuf wcnt, wplane, wA, wB;              // bootstrap counts / weight planes
  std::vector<float> val;       // [F][256]
  std::vector<int32_t> nval;    // [F]
  std::vector<adapt_node_t> tree;
  adapt::DevBuf d_tree, d_blocks;  // device tree: DNode top + bottom blocks (select.cu)
  adapt::DevBuf d_heap, d_exits, d_blocks2;  // deep trees: heap top + 2-level blocks (common.h)
  int heap_td = 0;
  // lossy quantile bins (quantile.cu, R23): features in qmask were quantised;
  // qprev[f][b] = the largest distinct value of bin b-1 (threshold midpoints)
  bool quantile = false;
  uint64_t qmask = 0;
  std::vector<float> qprev;
  adapt::DevBuf qfeat, qlb, qprevd;
  // K-fold harness (kfold.cu): set for the duration of adapt_kfold
  struct KfoldSpec {
    int K, m, shuffles;
    uint64_t seed;
    adapt_kfold_result_t *out;
  };
  const KfoldSpec *kfold = nullptr;
  // adapt_train_many (fused): this internal region's table is the union of k
  // regions' tables; multi_n[r] = region r's rows on this rank, in order
  const std::vector<int64_t> *multi_n = nullptr;
  std::vector<std::vector<adapt_node_t>> multi_trees;
  std::vector<std::vector<adapt_node_t>> kfold_trees;
  adapt::DevBuf flagsum;  // error-flag sums over ranks
  adapt::DevBuf dsmall;   // small.cu result (SmallOut)
  adapt::DevBuf kbnd, kpart, kgrp, kcnt, kcur, ksb, klab, knodes, kroots;
  bool trained = false;
  std::vector<int64_t> stats;
  // scratch
  adapt::DevBuf gkey, gcount, flags, lvals, lcnt, avals, acnt, dval, dnval,
      H0, H1, Hg, reso, resall, segs,
      hsegs, visits, slots, triples, nslot, cand, res, hoff, grp, gsoff, cmaps, xa, xb, oa, ob;
  adapt::HostBuf hres, hsmall, hvis, hgat;  // winners, scalars, partition share reports, gathered winners
  adapt::Arena stage_p, stage_a, stage_b, stage_r;  // per-level uploads: partition, its tables,
                                                     // histogram segments, owner split lists
  adapt::Arena stage_k;                  // two-level moves: MOVE4's per-segment children
  adapt::Arena stage_i;                  // ingest: the value hashes (one upload)
  adapt::DevBuf labT, visits2, kids;     // TAG pass labels, MOVE4 share reports, MOVE4 decisions
  cudaEvent_t sel_evt = nullptr;  // recorded after every device select (upload_tree waits)
  cudaEvent_t win_evt = nullptr;  // a level's winner records are on the host
  cudaEvent_t vis_evt = nullptr;  // a partition's share reports are on the host
  adapt::DevBuf dseg_err;  // the device-built histogram segments disagree with the plan
  adapt::HostBuf hseg_err;
  ~adapt_region() {
    if (sel_evt) cudaEventDestroy(sel_evt);
    if (win_evt) cudaEventDestroy(win_evt);
    if (vis_evt) cudaEventDestroy(vis_evt);
  }
  std::unordered_set<std::string> pair_set;  // distinct (features, variant) of the host records
  int64_t autotrain_failed_at = -1;          // pair count of the last failed auto-train
  // Table-1 shim state
  bool active = false;
  std::vector<float> ctx_feat;
  int ctx_policy = -1;
  timespec t0{};
  int cursor = 0;
};

namespace adapt {
namespace {

std::map<std::string, std::unique_ptr<adapt_region>> g_regions;
// adapt_train_many's union region (buffers reused across calls; freed by adapt_finalize)
std::unique_ptr<adapt_region> g_multi;

// model_type: "dtree[,D]" / "dtree,depth=D" /
// "DecisionTree[,explore=RoundRobin]"; "rfc[,T[,D]]" / "rfc(T,D)" /
// "rfc,trees=T,depth=D,seed=S" / "RandomForest[...]" ("model_type(rfc,
// 10, 4)": trees, then depth).  Defaults: dtree depth 2; rfc 10 trees
// of depth 2, seed 0 (R21).
int parse_params(const char *p, int *depth, int *kind, int *trees, uint64_t *seed, bool *quantile) {
  *quantile = false;
  *depth = 2;
  *kind = 0;
  *trees = 1;
  *seed = 0;
  if (!p || !*p) return 0;
  std::string s(p);
  for (char &c : s)
    if (c == '(') c = ',';
  s.erase(std::remove(s.begin(), s.end(), ')'), s.end());
  std::vector<std::string> tok;
  size_t st = 0;
  while (true) {
    size_t c = s.find(',', st);
    std::string t = s.substr(st, c == std::string::npos ? std::string::npos : c - st);
    t.erase(0, t.find_first_not_of(" \t"));
    t.erase(t.find_last_not_of(" \t") + 1);
    tok.push_back(t);
    if (c == std::string::npos) break;
    st = c + 1;
  }
  if (tok[0] == "rfc" || tok[0] == "RandomForest") {
    *kind = 1;
    *trees = 10;
  } else if (tok[0] != "dtree" && tok[0] != "DecisionTree") {
    throw Error(ADAPT_E_INVALID_ARG, "model kind '" + tok[0] + "' not supported (dtree, rfc)");
  }
  auto num = [&](const std::string &v, const std::string &t) {
    char *end = nullptr;
    const long long d = strtoll(v.c_str(), &end, 10);
    if (v.empty() || *end) throw Error(ADAPT_E_INVALID_ARG, "bad model parameter '" + t + "'");
    return d;
  };
  int positional = 0;
  for (size_t i = 1; i < tok.size(); i++) {
    const std::string &t = tok[i];
    if (t.empty()) continue;
    if (t.rfind("explore=", 0) == 0) {
      if (t != "explore=RoundRobin") throw Error(ADAPT_E_INVALID_ARG, "only explore=RoundRobin");
      continue;
    }
    if (t.rfind("bins=", 0) == 0) {  // R23: lossy quantile bins for > 256 distinct values
      if (t != "bins=quantile" && t != "bins=exact")
        throw Error(ADAPT_E_INVALID_ARG, "bins must be 'exact' or 'quantile'");
      *quantile = t == "bins=quantile";
      continue;
    }
    long long d;
    if (t.rfind("depth=", 0) == 0) d = num(t.substr(6), t), *depth = (int)d;
    else if (t.rfind("max_depth=", 0) == 0) d = num(t.substr(10), t), *depth = (int)d;
    else if (*kind == 1 && t.rfind("trees=", 0) == 0) d = num(t.substr(6), t), *trees = (int)d;
    else if (*kind == 1 && t.rfind("seed=", 0) == 0) *seed = (uint64_t)num(t.substr(5), t);
    else if (*kind == 1 && positional == 0) d = num(t, t), *trees = (int)d, positional++;
    else d = num(t, t), *depth = (int)d, positional++;
    if (*depth < 0 || *depth > 24) throw Error(ADAPT_E_INVALID_ARG, "depth must be in [0,24]");
    if (*trees < 1 || *trees > forest_max_trees())
      throw Error(ADAPT_E_INVALID_ARG, "trees must be in [1,64]");
  }
  return 0;
}

adapt_region *checked(adapt_region *h) {
  if (!h) throw Error(ADAPT_E_INVALID_ARG, "null region");
  for (auto &kv : g_regions)
    if (kv.second.get() == h) return h;
  throw Error(ADAPT_E_INVALID_ARG, "unknown region handle");
}

float canon(float x) { return x == 0.0f ? 0.0f : x; }

// long -> wide: one row per distinct feature vector (exact bits,
// -0 == +0), in order of first appearance; mean time per variant (R1).
float round_down_f32(double t) {  // largest float32 <= t (V:A5)
  float f = (float)t;
  if ((double)f > t) f = std::nextafter(f, -INFINITY);
  return f;
}

// selects still in flight on any stream read the device tree: wait for the
// last one (a concurrent select must never walk a half-written tree)
void wait_selects(adapt_region *h) {
  if (h->sel_evt) CUDA_CHECK(cudaEventSynchronize(h->sel_evt));
}

void upload_tree(adapt_region *h, cudaStream_t s) {
  wait_selects(h);
  std::vector<DNode> d(h->tree.size());
  for (size_t k = 0; k < h->tree.size(); k++) {
    const adapt_node_t &nd = h->tree[k];
    if (nd.feature >= 0) {
      d[k].thr = round_down_f32(nd.threshold);
      d[k].meta = (nd.left << 6) | nd.feature;
    } else {
      d[k].thr = 0;
      d[k].meta = -1 - nd.label;
    }
  }
  h->d_tree.ensure(d.size() * sizeof(DNode));
  CUDA_CHECK(cudaMemcpyAsync(h->d_tree.p, d.data(), d.size() * sizeof(DNode),
                             cudaMemcpyHostToDevice, s));
  // bottom blocks (common.h): the nodes below the shared-memory top, 3 levels
  // per 64-byte block, so a walk below the top costs one L2 round trip per 3
  // levels instead of one per level
  const auto &tr = h->tree;
  const int n_top = std::min<int>((int)tr.size(), kSelTopNodes);
  std::vector<uint32_t> blk;
  if ((int)tr.size() > n_top) {
    int c_end = n_top;  // children of top nodes: entry blocks [0, c_end - n_top)
    for (int k = 0; k < n_top; k++)
      if (tr[k].feature >= 0) c_end = std::max(c_end, tr[k].right + 1);
    blk.assign((size_t)16 * (c_end - n_top), 0u);
    std::deque<std::pair<int64_t, int>> work;  // (block, tree node at its root)
    for (int k = 0; k < n_top; k++)
      if (tr[k].feature >= 0)
        for (int c : {tr[k].left, tr[k].right})
          if (c >= n_top) work.emplace_back(c - n_top, c);
    while (!work.empty()) {
      const auto [b, root] = work.front();
      work.pop_front();
      int pos[15];
      pos[0] = root;
      uint32_t w[16] = {};
      for (int p = 0; p < 7; p++) {
        const adapt_node_t &nd = tr[pos[p]];
        if (nd.feature >= 0) {
          const float t = round_down_f32(nd.threshold);
          memcpy(&w[p], &t, 4);
          w[7 + p] = (uint32_t)nd.feature;
          pos[2 * p + 1] = nd.left;
          pos[2 * p + 2] = nd.right;
        } else {  // pass-through: both subtrees end in this leaf
          pos[2 * p + 1] = pos[2 * p + 2] = pos[p];
        }
      }
      for (int i = 0; i < 8; i++) {
        const adapt_node_t &nd = tr[pos[7 + i]];
        int32_t ref;
        if (nd.feature < 0) {
          ref = -1 - nd.label;
        } else {
          ref = (int32_t)(blk.size() / 16);
          if (ref >= (1 << 25)) throw Error(ADAPT_E_INVALID_ARG, "tree too large for the select layout");
          blk.resize(blk.size() + 16, 0u);
          work.emplace_back(ref, pos[7 + i]);
        }
        w[7 + i] |= (uint32_t)ref << 6;
      }
      memcpy(&blk[(size_t)b * 16], w, sizeof(w));
    }
  }
  h->d_blocks.ensure(std::max<size_t>(blk.size() * 4, 64));
  if (!blk.empty())
    CUDA_CHECK(cudaMemcpyAsync(h->d_blocks.p, blk.data(), blk.size() * 4, cudaMemcpyHostToDevice, s));
  // trees deeper than the BFS top: the heap-top layout of select_kernel_h
  h->heap_td = 0;
  if ((int)tr.size() > kSelTopNodes) {
    int maxd = 0;
    for (const auto &nd : tr) maxd = std::max(maxd, nd.depth);
    const int td = std::min(kHeapMaxLevels, maxd);
    const int nh = (1 << td) - 1;
    std::vector<uint2> heap((size_t)std::max(nh, 1), make_uint2(0u, 0u));
    std::vector<int32_t> exits((size_t)1 << td, 0);
    std::vector<uint32_t> b2;  // 8 words per block
    std::deque<std::pair<int64_t, int>> q2;  // (block, tree node at its root)
    auto ref_of = [&](int t) -> int32_t {   // exit to tree node t: its label, or a new block
      if (tr[t].feature < 0) return -1 - tr[t].label;
      const int64_t b = (int64_t)(b2.size() / 8);
      if (b >= (1ll << 30)) throw Error(ADAPT_E_INVALID_ARG, "tree too large for the select layout");
      b2.resize(b2.size() + 8, 0u);
      q2.emplace_back(b, t);
      return (int32_t)b;
    };
    // heap fill: (heap position, tree node, level); leaves above td pass through
    std::vector<std::array<int, 3>> st{{0, 0, 0}};
    while (!st.empty()) {
      const auto [hp, t, lv] = st.back();
      st.pop_back();
      if (lv == td) {
        exits[(size_t)(hp - nh)] = ref_of(t);
        continue;
      }
      const adapt_node_t &nd = tr[t];
      if (nd.feature >= 0) {
        const float th = round_down_f32(nd.threshold);
        uint32_t bits;
        memcpy(&bits, &th, 4);
        heap[hp] = make_uint2(bits, (uint32_t)nd.feature);
      }
      st.push_back({2 * hp + 2, nd.feature >= 0 ? nd.right : t, lv + 1});
      st.push_back({2 * hp + 1, nd.feature >= 0 ? nd.left : t, lv + 1});
    }
    while (!q2.empty()) {  // 2-level blocks, breadth first
      const auto [b, root] = q2.front();
      q2.pop_front();
      uint32_t w[8] = {};
      const adapt_node_t &r = tr[root];
      const int kids[2] = {r.left, r.right};
      auto thr_bits = [&](const adapt_node_t &nd) {
        const float th = round_down_f32(nd.threshold);
        uint32_t bits;
        memcpy(&bits, &th, 4);
        return bits;
      };
      w[0] = thr_bits(r);
      w[3] = (uint32_t)r.feature;
      for (int c = 0; c < 2; c++) {
        const adapt_node_t &ch = tr[kids[c]];
        if (ch.feature >= 0) {
          w[1 + c] = thr_bits(ch);
          w[3] |= (uint32_t)ch.feature << (8 * (c + 1));
          const int32_t l = ref_of(ch.left), rr = ref_of(ch.right);
          w[4 + 2 * c] = (uint32_t)l;
          w[5 + 2 * c] = (uint32_t)rr;
        } else {  // pass-through: both exits of this child are its leaf
          const int32_t lf = -1 - ch.label;
          w[4 + 2 * c] = w[5 + 2 * c] = (uint32_t)lf;
        }
      }
      memcpy(&b2[(size_t)b * 8], w, sizeof(w));
    }
    h->d_heap.ensure(heap.size() * sizeof(uint2));
    h->d_exits.ensure(exits.size() * 4);
    h->d_blocks2.ensure(std::max<size_t>(b2.size() * 4, 64));
    CUDA_CHECK(cudaMemcpyAsync(h->d_heap.p, heap.data(), heap.size() * sizeof(uint2), cudaMemcpyHostToDevice, s));
    CUDA_CHECK(cudaMemcpyAsync(h->d_exits.p, exits.data(), exits.size() * 4, cudaMemcpyHostToDevice, s));
    if (!b2.empty())
      CUDA_CHECK(cudaMemcpyAsync(h->d_blocks2.p, b2.data(), b2.size() * 4, cudaMemcpyHostToDevice, s));
    h->heap_td = td;
  }
  CUDA_CHECK(cudaStreamSynchronize(s));
}

// forest: trees concatenated, child indices made absolute; roots[t] = offset
void upload_forest(adapt_region *h, cudaStream_t s) {
  wait_selects(h);
  std::vector<DNode> d;
  std::vector<int32_t> roots;
  for (const auto &tr : h->forest) {
    const int32_t off = (int32_t)d.size();
    roots.push_back(off);
    for (const auto &nd : tr) {
      DNode x;
      if (nd.feature >= 0) {
        x.thr = round_down_f32(nd.threshold);
        x.meta = ((nd.left + off) << 6) | nd.feature;
      } else {
        x.thr = 0;
        x.meta = -1 - nd.label;
      }
      d.push_back(x);
    }
  }
  if (d.size() >= (1u << 25)) throw Error(ADAPT_E_INVALID_ARG, "forest too large (2^25 nodes)");
  h->forest_nodes = (int)d.size();
  h->d_forest.ensure(d.size() * sizeof(DNode) + 16);
  h->d_roots.ensure(roots.size() * 4 + 16);
  CUDA_CHECK(cudaMemcpyAsync(h->d_forest.p, d.data(), d.size() * sizeof(DNode), cudaMemcpyHostToDevice, s));
  CUDA_CHECK(cudaMemcpyAsync(h->d_roots.p, roots.data(), roots.size() * 4, cudaMemcpyHostToDevice, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
}

template <class T>
void h2d(DevBuf &b, const std::vector<T> &v, cudaStream_t s) {
  b.ensure(v.size() * sizeof(T) + 16);
  if (!v.empty())
    CUDA_CHECK(cudaMemcpyAsync(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
}

// ------------------------------------------------------------ records --
// grow a device buffer keeping its first `keep` bytes
void grow_keep(DevBuf &b, size_t bytes, size_t keep, cudaStream_t s) {
  if (bytes <= b.cap) return;
  DevBuf nb;
  nb.ensure(bytes);
  if (keep) CUDA_CHECK(cudaMemcpyAsync(nb.p, b.p, keep, cudaMemcpyDeviceToDevice, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  std::swap(b.p, nb.p);
  std::swap(b.cap, nb.cap);
}

void reserve_records(adapt_region *h, int64_t need, cudaStream_t s) {
  if (need <= h->rec_cap) return;
  const int64_t cap = std::max<int64_t>(need, std::max<int64_t>(2 * h->rec_cap, 1024));
  grow_keep(h->rec_feat, (size_t)cap * h->F * 4, (size_t)h->rec_n * h->F * 4, s);
  grow_keep(h->rec_var, (size_t)cap * 4, (size_t)h->rec_n * 4, s);
  grow_keep(h->rec_ns, (size_t)cap * 8, (size_t)h->rec_n * 8, s);
  h->rec_cap = cap;
}

// SURVEY §8(c) step 0 on the GPU (records.cu): every record (the device
// store, then the host-recorded ones) -> wide rows in agg_feat / agg_times.
// Returns the number of wide rows; *pairs (optional) = distinct (vector,
// variant) pairs = measured cells of the wide table.
int64_t gpu_aggregate(adapt_region *h, cudaStream_t s, int64_t *pairs) {
  const int F = h->F, V = h->V;
  const int64_t hn = (int64_t)h->rvar.size(), m = h->rec_n + hn;
  if (m == 0) return 0;
  if (m >= (int64_t)0xFFFFFFFFll) throw Error(ADAPT_E_INVALID_ARG, "more than 2^32-1 records");
  reserve_records(h, m, s);
  if (hn) {  // host records after the device store (re-uploaded by every call)
    CUDA_CHECK(cudaMemcpyAsync(h->rec_feat.as<float>() + h->rec_n * F, h->rfeat.data(),
                               (size_t)hn * F * 4, cudaMemcpyHostToDevice, s));
    CUDA_CHECK(cudaMemcpyAsync(h->rec_var.as<int32_t>() + h->rec_n, h->rvar.data(), (size_t)hn * 4,
                               cudaMemcpyHostToDevice, s));
    CUDA_CHECK(cudaMemcpyAsync(h->rec_ns.as<uint64_t>() + h->rec_n, h->rns.data(), (size_t)hn * 8,
                               cudaMemcpyHostToDevice, s));
  }
  const size_t slots = rec_table_slots(m);
  h->slot_rep.ensure(slots * 4);
  h->slot_first.ensure(slots * 4);
  h->slot_gid.ensure(slots * 4);
  h->slot_of.ensure((size_t)m * 4);
  h->rflag.ensure((size_t)m * 4);
  h->rbsum.ensure((size_t)rec_scan_blocks(m) * 4 + 16);
  h->rgroups.ensure(16);
  h->flags.ensure(16);
  CUDA_CHECK(cudaMemsetAsync(h->flags.p, 0, 16, s));
  uint32_t *hs = h->hsmall.as<uint32_t>();
  {
    Phase ph("records", s, (double)m * (4.0 * F + 12));
    launch_rec_group(h->rec_feat.as<float>(), h->rec_var.as<int32_t>(), m, F, V,
                     h->slot_rep.as<uint32_t>(), h->slot_first.as<uint32_t>(), slots,
                     h->slot_of.as<uint32_t>(), h->rflag.as<uint32_t>(), h->rbsum.as<uint32_t>(),
                     h->rgroups.as<uint32_t>(), h->flags.as<uint32_t>(), s);
  }
  CUDA_CHECK(cudaMemcpyAsync(hs, h->rgroups.p, 4, cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaMemcpyAsync(hs + 1, h->flags.p, 4, cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  if (hs[1] & kFlagBadVariant) throw Error(ADAPT_E_BAD_VALUE, "recorded variant out of range");
  const int64_t G = hs[0];
  h->agg_feat.ensure((size_t)G * F * 4 + 16);
  h->agg_times.ensure((size_t)G * V * 4 + 16);
  h->rsum.ensure((size_t)G * V * 8 + 16);
  h->rcnt.ensure((size_t)G * V * 4 + 16);
  {
    Phase ph("records", s, 0);
    launch_rec_wide(h->rec_feat.as<float>(), h->rec_var.as<int32_t>(), h->rec_ns.as<uint64_t>(), m,
                    F, V, h->slot_of.as<uint32_t>(), h->slot_gid.as<uint32_t>(),
                    h->rflag.as<uint32_t>(), h->rbsum.as<uint32_t>(), G,
                    h->rsum.as<unsigned long long>(), h->rcnt.as<uint32_t>(), h->agg_feat.as<float>(),
                    h->agg_times.as<float>(), pairs ? h->rgroups.as<uint32_t>() + 1 : nullptr, s);
  }
  if (pairs) {
    CUDA_CHECK(cudaMemcpyAsync(hs, h->rgroups.as<uint32_t>() + 1, 4, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    *pairs = hs[0];
  }
  return G;
}

// K-fold models grown in one frontier (kfold.cu, R22): root r's rows are the
// pieces pieces[r] of the planes (bins word planes with stride pstride, labels)
struct MultiRoot {
  int R;
  const uint8_t *bins, *labs;
  size_t pstride;
  int64_t rows_out;  // rows the level passes may write (sum of the roots' rows)
  std::vector<std::vector<std::pair<uint32_t, uint32_t>>> pieces;
};

// ------------------------------------------------------------ training --
void train_region(adapt_region *h, cudaStream_t s) {
  const int F = h->F, V = h->V, C = V, D = h->D;
  static const bool trace = getenv("ADAPT_TRACE_HOST") != nullptr;  // host-side time per level
  auto now_us = []() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e6 + ts.tv_nsec * 1e-3;
  };
  double tr[8] = {0};
  if (trace) {
    CUDA_CHECK(cudaStreamSynchronize(s));
    tr[7] = now_us();
  }
  const int world = g_ctx.world;
  // 0. source table (wide, or long records aggregated on the host)
  const float *feat = h->d_feat, *times = h->d_times;
  int64_t n = h->n;
  h->hsmall.ensure(1 << 16);
  h->aggregated = !h->have_table;
  if (!h->have_table) {  // long-format records -> wide rows, on the GPU
    n = gpu_aggregate(h, s, nullptr);
    feat = h->agg_feat.as<float>();
    times = h->agg_times.as<float>();
  }
  uint64_t n_total = (uint64_t)n;
  h->hsmall.ensure(1 << 16);
  if (collectives_on()) {
    DevBuf tmp;
    tmp.ensure(8);
    CUDA_CHECK(cudaMemcpyAsync(tmp.p, &n_total, 8, cudaMemcpyHostToDevice, s));
    comm_allreduce_sum(tmp.p, 1, true, s, "allreduce n");
    CUDA_CHECK(cudaMemcpyAsync(&n_total, tmp.p, 8, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  if (n_total == 0) throw Error(ADAPT_E_INSUFFICIENT_DATA, "no training rows");
  if (n_total >= (1ull << 32)) throw Error(ADAPT_E_INVALID_ARG, "more than 2^32-1 rows");
  int BS = 1;
  while (BS < F) BS <<= 1;
  h->BS = BS;

  // 1. a2 discovery pass, value tables merged over ranks, then a1 + a3 in one
  //    pass over (times, features); bins are ranks in the merged value table
  h->gkey.ensure((size_t)F * kGSlots * 4);
  h->gcount.ensure((size_t)F * 4);
  h->flags.ensure(16);
  const size_t pstride = bins_plane_stride(n, BS);
  h->pstride = pstride;
  h->bins.ensure(bins_bytes(n, BS));
  h->labels.ensure((size_t)std::max<int64_t>(n, 1) + 64);
  // small tables (the paper's run-time scale): the whole path in one thread
  // block, one launch, one wait (small.cu); falls through to the general path
  // when a limit or a flagged value says so
  static const bool no_small = getenv("ADAPT_NO_SMALL") != nullptr;
  if (!no_small && !collectives_on() && h->kind == 0 && !h->quantile && !h->kfold && !h->multi_n &&
      n >= 1 && n <= kSmallMaxN && F <= kSmallMaxF && V <= kSmallMaxC) {
    h->hres.ensure(sizeof(SmallOut));
    h->dsmall.ensure(sizeof(SmallOut));
    {
      Phase ph("small", s, (double)n * (4.0 * F + 4.0 * V + F + 1));
      launch_small_train(feat, times, (int)n, F, V, D, BS, pstride, h->bins.as<uint8_t>(),
                         h->labels.as<uint8_t>(), h->dsmall.as<SmallOut>(), s);
    }
    SmallOut *so = h->hres.as<SmallOut>();
    CUDA_CHECK(cudaMemcpyAsync(so, h->dsmall.p, sizeof(SmallOut), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    if (so->status == 0) {
      h->val.assign((size_t)F * kMaxBins, 0.f);
      h->nval.assign(F, 0);
      for (int f = 0; f < F; f++) {
        h->nval[f] = so->nval[f];
        memcpy(&h->val[(size_t)f * kMaxBins], so->val[f], (size_t)so->nval[f] * 4);
      }
      h->qmask = 0;
      h->tree.assign(so->nodes, so->nodes + so->n_nodes);
      h->forest.clear();
      h->stats.clear();
      h->trained_n = n;
      h->trained = true;
      upload_tree(h, s);
      return;
    }
  }
  h->lvals.ensure((size_t)F * kMaxBins * 4);
  h->lcnt.ensure((size_t)F * 4);
  h->avals.ensure((size_t)world * F * kMaxBins * 4);
  h->acnt.ensure((size_t)world * F * 4);
  h->dval.ensure((size_t)F * kMaxBins * 4);
  h->dnval.ensure((size_t)F * 4);
  // error flags, summed over ranks so that all ranks fail (or retry) together
  uint32_t *hs = h->hsmall.as<uint32_t>();
  auto check_flags = [&](bool allow_too_many = false) -> uint32_t {
    CUDA_CHECK(cudaMemcpyAsync(hs, h->flags.p, 4, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    uint32_t bits[6];
    for (int b = 0; b < 6; b++) bits[b] = (hs[0] >> b) & 1;
    if (collectives_on()) {
      DevBuf &fl = h->flagsum;
      fl.ensure(32);
      CUDA_CHECK(cudaMemcpyAsync(fl.p, bits, 24, cudaMemcpyHostToDevice, s));
      comm_allreduce_sum(fl.p, 6, false, s, "allreduce flags");
      CUDA_CHECK(cudaMemcpyAsync(bits, fl.p, 24, cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
    }
    if (bits[0]) throw Error(ADAPT_E_BAD_VALUE, "NaN or Inf feature value");
    if (bits[1]) throw Error(ADAPT_E_BAD_VALUE, "NaN time");
    if (bits[2]) throw Error(ADAPT_E_BAD_VALUE, "row with every variant unmeasured (+inf)");
    if (bits[3] && !allow_too_many)
      throw Error(ADAPT_E_TOO_MANY_DISTINCT, "a feature has more than 256 distinct values");
    uint32_t m = 0;
    for (int b = 0; b < 6; b++) m |= (bits[b] ? 1u : 0u) << b;
    return m;
  };
  // Discovery reads a SAMPLE of a large table first (kSampleChunks contiguous
  // chunks spread over it): the bin pass checks every value against the
  // resulting tables and flags any value the sample missed, and only then the
  // whole table is discovered and binned again — the tables and bins are the
  // exact ones either way, typically for a 1% read.
  constexpr int64_t kSampleChunk = 1 << 15, kSampleChunks = 32;
  const bool sampled = n > 4 * kSampleChunk * kSampleChunks;
  h->qmask = 0;
  // R23 (bins=quantile): the features with > 256 distinct values over all ranks
  // are replaced by their quantised copies (quantile.cu), then ingest restarts
  auto quantize_features = [&]() {
    std::vector<int32_t> nv(F), ac((size_t)world * F);
    CUDA_CHECK(cudaMemcpyAsync(nv.data(), h->dnval.p, (size_t)F * 4, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaMemcpyAsync(ac.data(), h->acnt.p, (size_t)world * F * 4, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    uint64_t qm = 0;
    for (int f = 0; f < F; f++) {
      bool over = nv[f] > kMaxBins;
      for (int p = 0; p < world; p++) over |= ac[(size_t)p * F + f] > kMaxBins;
      if (over) qm |= 1ull << f;
    }
    h->qlb.ensure((size_t)F * kMaxBins * 4);
    h->qprevd.ensure((size_t)F * kMaxBins * 4);
    CUDA_CHECK(cudaMemsetAsync(h->qlb.p, 0, (size_t)F * kMaxBins * 4, s));
    CUDA_CHECK(cudaMemsetAsync(h->qprevd.p, 0, (size_t)F * kMaxBins * 4, s));
    DevBuf keys, sorted, uniq, dcnt, temp, cnt8, all8, gath;
    const int64_t nn = std::max<int64_t>(n, 1);
    keys.ensure((size_t)nn * 4);
    sorted.ensure((size_t)nn * 4);
    uniq.ensure((size_t)nn * 4);
    dcnt.ensure(16);
    cnt8.ensure(8);
    all8.ensure((size_t)world * 8);
    for (int f = 0; f < F; f++) {
      if (!((qm >> f) & 1)) continue;
      Phase ph("quantile", s, (double)n * 4.0);
      size_t tb = sort_unique_temp_bytes(nn);
      temp.ensure(tb);
      int c = 0;
      if (n) {
        launch_column_keys(feat, n, F, f, keys.as<uint32_t>(), s);
        sort_unique_keys(keys.as<uint32_t>(), n, sorted.as<uint32_t>(), uniq.as<uint32_t>(), dcnt.as<int>(),
                         temp.p, tb, s);
        CUDA_CHECK(cudaMemcpyAsync(&c, dcnt.p, 4, cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
      }
      const uint32_t *u = uniq.as<uint32_t>();
      int64_t D = c;
      if (collectives_on()) {  // union of the ranks' sorted distinct keys (padded all-gather)
        const uint64_t mine = (uint64_t)c;
        CUDA_CHECK(cudaMemcpyAsync(cnt8.p, &mine, 8, cudaMemcpyHostToDevice, s));
        comm_allgather(cnt8.p, all8.p, 8, s, "allgather distinct counts");
        std::vector<uint64_t> cs(world);
        CUDA_CHECK(cudaMemcpyAsync(cs.data(), all8.p, (size_t)world * 8, cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        const int64_t mx = std::max<int64_t>(1, (int64_t)*std::max_element(cs.begin(), cs.end()));
        DevBuf send, recv, rs, ru;
        send.ensure((size_t)mx * 4);
        recv.ensure((size_t)world * mx * 4);
        rs.ensure((size_t)world * mx * 4);
        ru.ensure((size_t)world * mx * 4);
        CUDA_CHECK(cudaMemsetAsync(send.p, 0xFF, (size_t)mx * 4, s));  // pad: no finite key
        if (c) CUDA_CHECK(cudaMemcpyAsync(send.p, uniq.p, (size_t)c * 4, cudaMemcpyDeviceToDevice, s));
        comm_allgather(send.p, recv.p, (size_t)mx * 4, s, "allgather distinct keys");
        tb = sort_unique_temp_bytes((int64_t)world * mx);
        temp.ensure(tb);
        sort_unique_keys(recv.as<uint32_t>(), (int64_t)world * mx, rs.as<uint32_t>(), ru.as<uint32_t>(),
                         dcnt.as<int>(), temp.p, tb, s);
        uint32_t last = 0;
        CUDA_CHECK(cudaMemcpyAsync(&c, dcnt.p, 4, cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        CUDA_CHECK(cudaMemcpyAsync(&last, ru.as<uint32_t>() + c - 1, 4, cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        D = c - (last == 0xFFFFFFFFu ? 1 : 0);
        gath.ensure((size_t)std::max<int64_t>(D, 1) * 4);
        CUDA_CHECK(cudaMemcpyAsync(gath.p, ru.p, (size_t)D * 4, cudaMemcpyDeviceToDevice, s));
        u = gath.as<uint32_t>();
        launch_edges(u, D, h->qlb.as<float>() + (size_t)f * kMaxBins,
                     h->qprevd.as<float>() + (size_t)f * kMaxBins, s);
        CUDA_CHECK(cudaStreamSynchronize(s));  // the local buffers die here
        continue;
      }
      launch_edges(u, D, h->qlb.as<float>() + (size_t)f * kMaxBins,
                   h->qprevd.as<float>() + (size_t)f * kMaxBins, s);
    }
    h->qprev.assign((size_t)F * kMaxBins, 0.f);
    CUDA_CHECK(cudaMemcpyAsync(h->qprev.data(), h->qprevd.p, (size_t)F * kMaxBins * 4, cudaMemcpyDeviceToHost, s));
    h->qfeat.ensure((size_t)std::max<int64_t>(n, 1) * F * 4);
    {
      Phase ph("quantile", s, (double)n * 8.0 * F);
      launch_quantize(feat, n, F, qm, h->qlb.as<float>(), h->qfeat.as<float>(), s);
    }
    CUDA_CHECK(cudaStreamSynchronize(s));
    h->qmask = qm;
    feat = h->qfeat.as<float>();
  };
  const uint8_t *lk_tab = nullptr;  // the bin pass's value hashes (device)
  const uint32_t *lk_mul = nullptr, *lk_sk = nullptr;
  for (int attempt = 0;; attempt++) {
    CUDA_CHECK(cudaMemsetAsync(h->gkey.p, 0xFF, (size_t)F * kGSlots * 4, s));
    CUDA_CHECK(cudaMemsetAsync(h->gcount.p, 0, (size_t)F * 4, s));
    CUDA_CHECK(cudaMemsetAsync(h->flags.p, 0, 16, s));
    if (sampled && attempt == 0) {
      Phase ph("discover", s, (double)kSampleChunk * kSampleChunks * 4.0 * F);
      const int64_t gap = (n - kSampleChunk * kSampleChunks) / (kSampleChunks - 1);
      launch_discover(feat, kSampleChunk * kSampleChunks, F, h->gkey.as<uint32_t>(),
                      h->gcount.as<uint32_t>(), h->flags.as<uint32_t>(), kSampleChunk, gap, s);
    } else {
      Phase ph("discover", s, (double)n * 4.0 * F);
      launch_discover(feat, n, F, h->gkey.as<uint32_t>(), h->gcount.as<uint32_t>(),
                      h->flags.as<uint32_t>(), 0, 0, s);
    }
    CUDA_CHECK(cudaMemsetAsync(h->lvals.p, 0, (size_t)F * kMaxBins * 4, s));
    CUDA_CHECK(cudaMemsetAsync(h->dval.p, 0, (size_t)F * kMaxBins * 4, s));
    {
      Phase ph("values", s, 0);
      launch_collect_values(h->gkey.as<uint32_t>(), h->gcount.as<uint32_t>(), F,
                            h->lvals.as<float>(), h->lcnt.as<int32_t>(), s);
    }
    comm_allgather(h->lvals.p, h->avals.p, (size_t)F * kMaxBins * 4, s, "allgather values");
    comm_allgather(h->lcnt.p, h->acnt.p, (size_t)F * 4, s, "allgather counts");
    {
      Phase ph("merge", s, 0);
      launch_merge_values(h->avals.as<float>(), h->acnt.as<int32_t>(), world, F, h->dval.as<float>(),
                          h->dnval.as<int32_t>(), h->flags.as<uint32_t>(), s);
    }
    if (check_flags(h->quantile && h->qmask == 0) & kFlagTooMany) {
      quantize_features();
      attempt = -1;  // ingest the quantised table from the start (sampled discovery again)
      continue;
    }
    // value tables to the host; per-feature perfect hashes value -> rank for the bin pass
    h->val.assign((size_t)F * kMaxBins, 0.f);
    h->nval.assign(F, 0);
    CUDA_CHECK(cudaMemcpyAsync(h->val.data(), h->dval.p, (size_t)F * kMaxBins * 4, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaMemcpyAsync(h->nval.data(), h->dnval.p, (size_t)F * 4, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    const double t_hash = trace ? now_us() : 0;
    {
      // the GPU waits for these (host threads per feature measured slower:
      // spawning them costs more than the ~8 us per feature), then ONE pinned
      // upload of all three tables
      std::vector<uint8_t> tab((size_t)lookup_table_bytes(F));
      std::vector<uint32_t> mul((size_t)2 * F), skeys((size_t)F * lookup_slots());
      for (int f = 0; f < F; f++)
        if (!build_value_hash(&h->val[(size_t)f * kMaxBins], h->nval[f], &mul[2 * f],
                              &tab[(size_t)f * lookup_table_bytes(1)], &skeys[(size_t)f * lookup_slots()]))
          throw Error(ADAPT_E_CUDA, "cannot build the value hash of feature " + std::to_string(f));
      Arena &si = h->stage_i;
      si.reset();
      const size_t o_tab = si.put(tab), o_mul = si.put(mul), o_sk = si.put(skeys);
      si.flush(s);
      lk_tab = si.ptr<uint8_t>(o_tab);  // (valid until the next train's upload)
      lk_mul = si.ptr<uint32_t>(o_mul);
      lk_sk = si.ptr<uint32_t>(o_sk);
    }
    if (trace)
      fprintf(stderr, "[adapt] ingest attempt %d: discovery..tables %.0f us, perfect hashes %.0f us (GPU idle)\n",
              attempt, t_hash - tr[7], now_us() - t_hash);
    CUDA_CHECK(cudaMemsetAsync(h->flags.p, 0, 16, s));
    {
      Phase ph("ingest", s, (double)n * (4.0 * F + 4.0 * V + F + 1));  // algorithmic
      launch_label_bin(feat, times, n, F, V, BS, lk_tab, lk_mul, lk_sk, sampled && attempt == 0 ? 1 : 0,
                       h->flags.as<uint32_t>(),
                       h->bins.as<uint8_t>(), pstride, h->labels.as<uint8_t>(), s);
    }
    const uint32_t fl = check_flags();
    if (!(fl & kFlagUnseen)) break;
    if (attempt > 0) throw Error(ADAPT_E_CUDA, "bin pass met a value the full discovery missed");
  }

  // histogram layout: node -> [DS][kc] (rows cumD[f] + rank, compact class columns)
  std::vector<int32_t> cumD(F);
  int64_t DS = 0;
  for (int f = 0; f < F; f++) {
    cumD[f] = (int32_t)DS;
    DS += h->nval[f];
  }
  // shared-memory groups of the level pass: group = one 32-bit word of the
  // bins row (4 features) x a class slab [k0, k0+kw); feature f takes
  // D_f x kwp counters, kwp = kw padded to an odd stride.  A word whose 4
  // features x all classes exceed one CTA's budget is split into class slabs.
  const int cap = (kHistSmemBudget - F * kMaxBins) / 4;
  struct G {
    int k0, kw, kwp, word, counters;
    std::vector<int32_t> off;
  };
  std::vector<G> gl;
  for (int w = 0; 4 * w < F; w++) {
    int dsum = 0;
    for (int f = 4 * w; f < std::min(F, 4 * w + 4); f++) dsum += h->nval[f];
    int kwp = C | 1;
    if ((int64_t)dsum * kwp > cap) {
      kwp = cap / dsum;
      if (!(kwp & 1)) kwp--;
    }
    for (int k0 = 0; k0 < C; k0 += kwp) {
      G t{k0, std::min(kwp, C - k0), 0, w, 0, std::vector<int32_t>(F, -1)};
      t.kwp = t.kw | 1;
      for (int f = 4 * w; f < std::min(F, 4 * w + 4); f++) {
        t.off[f] = t.counters;
        t.counters += h->nval[f] * t.kwp;
      }
      gl.push_back(t);
    }
  }
  const int ngroups = (int)gl.size();
  std::vector<HistGroupCost> gcost;  // the CTA planner's cost model per group
  for (auto &t : gl) {
    double u = 0;  // ns per row: its reductions, cheaper for features with few values
    for (int f = 4 * t.word; f < std::min(F, 4 * t.word + 4); f++)
      u += 0.0464 + 0.0218 * std::min(h->nval[f], 64) / 64.0;
    gcost.push_back(HistGroupCost{u, t.k0, t.kw, t.counters / t.kwp});
  }
  int max_group = 0;
  std::vector<int4> groups;
  std::vector<int32_t> gsoff;
  for (auto &t : gl) {
    groups.push_back(make_int4(t.k0, t.kw, t.kwp, t.word));
    gsoff.insert(gsoff.end(), t.off.begin(), t.off.end());
    max_group = std::max(max_group, t.counters);
  }
  h2d(h->hoff, cumD, s);
  h2d(h->grp, groups, s);
  h2d(h->gsoff, gsoff, s);

  // 2. level loop (a4-a8).  Per level: partition the previous level's split
  // parents (a7), histogram the smaller child of each (a4) — or the root —,
  // sum over ranks (a5), derive the siblings, search splits (a6), decide.
  // one tree (w_root: bootstrap weights or null), or with `mr` several trees
  // grown in ONE frontier (K-fold models): mr->R roots whose rows are pieces of
  // mr's planes; h->tree then holds all of them, roots first, level by level
  auto grow_tree = [&](const uint8_t *w_root, const MultiRoot *mr = nullptr) {
  h->tree.clear();
  h->stats.clear();
  const int R = mr ? mr->R : 1;
  const size_t ps = mr ? mr->pstride : pstride;
  const int64_t rows_out = mr ? mr->rows_out : n;  // plane capacity of the level passes
  adapt_node_t root{};
  root.feature = -1;
  root.left = root.right = -1;
  std::vector<FNode> frontier(R);
  for (int r = 0; r < R; r++) {
    h->tree.push_back(root);
    frontier[r].tree_idx = r;
    frontier[r].depth = 0;
    frontier[r].slot = r;
    frontier[r].direct = true;
    for (int k = 0; k < C; k++) frontier[r].cls.add(k);
  }
  // this rank's rows of frontier node j: pieces [pc_start[j], pc_start[j+1]) of
  // (offset, length) in the planes
  std::vector<std::pair<uint32_t, uint32_t>> pcs{{0u, (uint32_t)n}};
  std::vector<int32_t> pc_start{0, 1};
  if (mr) {
    pcs.clear();
    pc_start.assign(1, 0);
    for (int r = 0; r < R; r++) {
      for (const auto &pc : mr->pieces[r]) pcs.push_back(pc);
      pc_start.push_back((int32_t)pcs.size());
    }
  }
  std::vector<int2> pseg_children;  // per piece: frontier index of the left / right child
  int ndirect_slots = R;  // direct slots are 0..ndirect_slots-1, derived ones follow
  struct Derived {        // a derived node of the next level = parent - direct sibling
    int j, sib_j;         // frontier indices (next level)
    int64_t off_p;        // parent's histogram offset (this level; Hprev next level)
    ClassSet cls_p;       // parent's classes (its columns)
  };
  std::vector<Derived> derived;
  // planes: the root is histogrammed from the ingest output; pass d >= 1 moves
  // the parents' rows from one plane pair into the other
  const uint8_t *bins_in = mr ? mr->bins : h->bins.as<uint8_t>();
  const uint8_t *lab_in = mr ? mr->labs : h->labels.as<uint8_t>();
  const uint8_t *w_in = w_root;  // weight plane (forests), moved along with the rows
  if (w_root) {
    h->wA.ensure((size_t)std::max<int64_t>(n, 1) + 64);
    h->wB.ensure((size_t)std::max<int64_t>(n, 1) + 64);
  }
  h->binsA.ensure(ps * (BS < 4 ? 1 : BS / 4));
  h->binsB.ensure(ps * (BS < 4 ? 1 : BS / 4));
  h->labA.ensure((size_t)std::max<int64_t>(rows_out, 1) + 64);
  h->labB.ensure((size_t)std::max<int64_t>(rows_out, 1) + 64);
  int out_plane = 0;  // 0: A, 1: B
  int sms = 148;
  CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g_ctx.device));
  DevBuf *Hcur = &h->H0, *Hprev = &h->H1;
  // SURVEY §8(e) "the better option": per level, every rank keeps its LOCAL
  // histograms of all frontier nodes (derived siblings by local subtraction),
  // a reduce-scatter sums each node's histogram only at its owner rank (slot
  // ranges balanced by bytes), owners search the splits of their nodes, and an
  // all-gather of the winner records gives every rank the identical decisions.
  // Otherwise (default): all-reduce of the direct nodes, derived globally.
  const bool rs = hist_comm_rs();
  // two-level row moves: the rows move every other level (TAG
  // pass, then MOVE4 one level later); one rank, unweighted rows, one tree,
  // classes below 128 (label bit 7 carries the TAG pass's mark), and a table
  // large enough for the row passes to dominate (below it the per-level
  // schedule's device-built segments win: C3 1e6 rows 2.3 vs 3.9 ms).
  // ADAPT_TWO_LEVEL=1 / =0 forces it on / off (read per train), as does
  // ADAPT_ONE_LEVEL=1 (off)
  constexpr uint64_t kTwoLevelMinRows = 1ull << 24;
  const char *tl_env = getenv("ADAPT_TWO_LEVEL");
  const bool tl_off = getenv("ADAPT_ONE_LEVEL") != nullptr || (tl_env && atoi(tl_env) == 0);
  const bool tl_on = tl_env && atoi(tl_env) == 1;
  const bool two_level = !tl_off && (tl_on || n_total >= kTwoLevelMinRows) && !w_root && !mr && g_ctx.world == 1 &&
                         !rs && C <= 127;
  if (two_level) h->labT.ensure((size_t)std::max<int64_t>(rows_out, 1) + 64);
  std::vector<int4> pseg_gkids;  // per TAG segment: its parent's grandchildren (LL, LR, RL, RR)
  static const bool per_level = getenv("ADAPT_PROFILE_LEVELS") != nullptr;
  char nm[32];
  auto virtualize = [](std::vector<Seg> &v, bool by_slot) {  // row_base, node extents
    uint32_t total = 0;
    for (auto &sg : v) {
      sg.row_base = total;
      total += sg.len;
    }
    for (size_t i = 0; i < v.size();) {
      size_t k = i;
      uint32_t len = 0;
      const int key = by_slot ? v[i].hslot : v[i].direct;  // direct holds the parent id here
      while (k < v.size() && (by_slot ? v[k].hslot : v[k].direct) == key) len += v[k++].len;
      for (size_t t = i; t < k; t++) {
        v[t].node_base = v[i].row_base;
        v[t].node_len = len;
      }
      i = k;
    }
    return total;
  };

  if (trace) {
    const double t = now_us();
    CUDA_CHECK(cudaStreamSynchronize(s));
    fprintf(stderr, "[adapt] ingest: host %.0f us to the level loop, then %.0f us of queued work\n",
            t - tr[7], now_us() - t);
  }
  // a7 launch for level lvl over the split parents' pieces `segs` (virtualised
  // in place): input planes b_in/l_in/wi, output plane set oplane; the CTAs'
  // share reports come back asynchronously into h->hvis
  struct PartState {
    bool launched = false;
    int mode = 0;  // 0: partition (2-way move), 1: TAG pass, 2: MOVE4
    const int2 *kid_dev = nullptr;  // MOVE4: per segment, the parent's children (device)
    PartArgs pa{};
    int max_visits = 1;  // parents a partition range can touch
    size_t vbytes = 0;
    int64_t rows_part = 0;
    int32_t *hv = nullptr;
    int lvl = 0;
    // for segments built on the device: each partition segment's parent, each
    // parent's virtual span, rows per partition range
    std::vector<int32_t> seg_parent;
    std::vector<uint32_t> pbase, plen;
    uint32_t Rr = 1;
  };
  // the partition launch (and its share reports' D2H), on the stream
  auto launch_part = [&](PartState &st) {
    {
      const char *what = st.mode == 1 ? "tag" : "partition";
      snprintf(nm, sizeof nm, "%s_L%02d", what, st.lvl);
      // implementation bytes: a move reads and writes BS + 1 per row; TAG reads
      // one bins word and the label, writes the label
      Phase ph(per_level ? nm : what, s, (double)st.rows_part * (st.mode == 1 ? 6.0 : 2.0 * (BS + 1)));
      if (st.mode == 1) launch_tag(st.pa, s);
      else if (st.mode == 2) launch_partition4(st.pa, s);
      else launch_partition(st.pa, s);
    }
    st.launched = true;
    if (st.mode == 1) return;  // the TAG pass's reports stay on the device (MOVE4 reads them)
    h->hvis.grow(st.vbytes);
    st.hv = h->hvis.as<int32_t>();
    CUDA_CHECK(cudaMemcpyAsync(st.hv, st.pa.visits, st.vbytes, cudaMemcpyDeviceToHost, s));
    if (!h->vis_evt) CUDA_CHECK(cudaEventCreateWithFlags(&h->vis_evt, cudaEventDisableTiming));
    CUDA_CHECK(cudaEventRecord(h->vis_evt, s));
    st.launched = true;
  };
  // upload a partition's segments and size its share reports; `defer`: the
  // caller launches it (after the device has decided the segments' splits)
  auto start_part = [&](int lvl, std::vector<Seg> &segs, const uint8_t *b_in, const uint8_t *l_in,
                        const uint8_t *wi, int oplane, bool defer = false, int mode = 0) {
    PartState st;
    st.mode = mode;
    PartArgs &pa = st.pa;
    pa.lab_tag = h->labT.as<uint8_t>();
    const uint32_t total = virtualize(segs, false);
    st.rows_part = total;
    pa.nseg = (int)segs.size();
    pa.total_rows = total;
    pa.nranges = partition_ranges(sms, total);
    const uint32_t Rr = (total + pa.nranges - 1) / std::max(1, pa.nranges);
    st.Rr = std::max<uint32_t>(Rr, 1);
    st.seg_parent.resize(segs.size());
    for (size_t k = 0; k < segs.size(); k++) {
      const int p = segs[k].direct;
      st.seg_parent[k] = p;
      if ((int)st.pbase.size() <= p) st.pbase.resize(p + 1, 0), st.plen.resize(p + 1, 0);
      st.pbase[p] = segs[k].node_base;
      st.plen[p] = segs[k].node_len;
    }
    for (int r = 0, si = 0; r < pa.nranges && total; r++) {
      const uint32_t p0 = r * Rr, p1 = std::min<uint64_t>((uint64_t)p0 + Rr, total);
      while (si + 1 < pa.nseg && segs[si + 1].row_base <= p0) si++;
      int k = si, nodes = 0, last = -1;
      while (k < pa.nseg && segs[k].row_base < p1) {
        if (segs[k].direct != last) nodes++, last = segs[k].direct;
        k++;
      }
      st.max_visits = std::max(st.max_visits, nodes);
    }
    Arena &sp = h->stage_p;
    sp.reset();
    const size_t o_psegs = sp.put(segs);
    sp.flush(s);
    pa.segs = sp.ptr<Seg>(o_psegs);
    pa.bins_in = b_in;
    pa.lab_in = l_in;
    pa.bins_out = (oplane ? h->binsB : h->binsA).as<uint8_t>();
    pa.lab_out = (oplane ? h->labB : h->labA).as<uint8_t>();
    pa.w_in = wi;
    pa.w_out = w_root ? (oplane ? h->wB : h->wA).as<uint8_t>() : nullptr;
    pa.pstride = ps;
    pa.BS = BS;
    pa.F = F;
    pa.max_visits = st.max_visits;
    st.vbytes = (size_t)pa.nranges * st.max_visits * 6 * 4;
    h->visits.grow(st.vbytes);
    CUDA_CHECK(cudaMemsetAsync(h->visits.p, 0xFF, st.vbytes, s));
    pa.visits = h->visits.as<int32_t>();
    st.lvl = lvl;
    if (!defer) launch_part(st);
    return st;
  };
  // MOVE4 one level after the TAG pass `tg`: same segments (their splits decided
  // by the TAG pass's decide), same ranges; kid_j = each segment's two children
  auto start_move4 = [&](const PartState &tg, int lvl, const std::vector<int2> &kid_j, int oplane) {
    PartState st = tg;
    st.mode = 2;
    st.launched = false;
    st.lvl = lvl;
    PartArgs &pa = st.pa;
    pa.bins_out = (oplane ? h->binsB : h->binsA).as<uint8_t>();
    pa.lab_out = (oplane ? h->labB : h->labA).as<uint8_t>();
    pa.tag_visits = tg.pa.visits;
    st.vbytes = (size_t)pa.nranges * st.max_visits * 8 * 4;
    h->visits2.grow(st.vbytes);
    CUDA_CHECK(cudaMemsetAsync(h->visits2.p, 0xFF, st.vbytes, s));
    pa.visits = h->visits2.as<int32_t>();
    Arena &sk = h->stage_k;
    sk.reset();
    const size_t o_kid = sk.put(kid_j);
    sk.flush(s);
    st.kid_dev = sk.ptr<int2>(o_kid);
    h->kids.grow((size_t)std::max(pa.nseg, 1) * 2 * sizeof(int4));
    pa.kids = h->kids.as<int4>();
    return st;
  };
  PartState pending, tag_st;  // tag_st: the TAG pass behind the current tagged level
  static const bool trace2 = trace && atoi(getenv("ADAPT_TRACE_HOST")) >= 2;
  std::vector<std::pair<const char *, double>> ticks;  // (what, us) per level
  auto tick = [&](const char *what) {
    if (trace2) ticks.emplace_back(what, now_us());
  };
  for (int level = 0; !frontier.empty(); level++) {
    const int A = (int)frontier.size();
    if (trace) tr[0] = now_us();
    ticks.clear();
    tick("start");
    const uint8_t *hist_bins = bins_in, *hist_lab = lab_in, *hist_w = w_in;
    int64_t rows_part = 0;
    if (trace) tr[6] = now_us();
    // a7 of this level: normally launched already at the end of the previous
    // level's split decisions (overlapping the rest of its bookkeeping)
    PartState pst;
    if (level > 0) {
      if (!pending.launched) throw Error(ADAPT_E_CUDA, "internal: level without its partition");
      pst = pending;
    }
    pending = PartState{};
    PartArgs &pa = pst.pa;
    // tagged: this level's nodes are the TAG pass's children, their rows still
    // in the parents' pieces (pcs / pc_start), the direct ones marked in labT
    const bool tagged = level > 0 && pst.mode == 1, after4 = level > 0 && pst.mode == 2;
    if (tagged) tag_st = pst;
    const int max_visits = pst.max_visits;
    rows_part = pst.rows_part;
    int32_t *hv = pst.hv;
    double t_mv = trace ? now_us() : 0;
    // ---- uploads that do not depend on this level's partition: class maps
    // of the direct nodes, their slots, the subtraction triples, node slots ----
    // node histograms, class-compacted: slot offsets from the nodes' class counts
    const int nslots = A;  // every frontier node has a slot
    std::vector<int32_t> slot_kc(nslots, 0);
    for (const auto &fn : frontier) slot_kc[fn.slot] = fn.cls.count();
    std::vector<int64_t> soff(nslots + 1, 0);
    for (int k = 0; k < nslots; k++) soff[k + 1] = soff[k] + DS * slot_kc[k];
    const int64_t direct_bytes = soff[ndirect_slots] * 4;  // (direct slots first)
    tick("soff");
    // reduce-scatter mode: slot ranges [own[r], own[r+1]) owned by rank r,
    // balanced by histogram bytes, each padded to Q counters at offset r * Q
    const int NR = g_ctx.world, me = g_ctx.rank;
    std::vector<int32_t> own(NR + 1, nslots);
    int64_t Q = 0;
    if (rs) {
      const int64_t tot = soff[nslots];
      for (int r = 0; r < NR; r++)
        own[r] = (int32_t)(std::lower_bound(soff.begin(), soff.begin() + nslots, (tot * r + NR - 1) / NR) -
                           soff.begin());
      own[NR] = nslots;
      for (int r = 0; r < NR; r++) Q = std::max<int64_t>(Q, soff[own[r + 1]] - soff[own[r]]);
      Q = std::max<int64_t>(Q, 1);
      std::vector<int64_t> ps(nslots + 1);
      for (int r = 0; r < NR; r++)
        for (int k = own[r]; k < own[r + 1]; k++) ps[k] = r * Q + soff[k] - soff[own[r]];
      ps[nslots] = NR * Q;
      soff.swap(ps);
    }
    std::vector<uint8_t> cmaps;  // per direct node: class -> compact index (255: absent)
    cmaps.reserve((size_t)ndirect_slots * C);
    std::vector<int32_t> node_ci(A, -1), node_kc(A);
    std::vector<int64_t> node_off(A);
    for (int j = 0; j < A; j++) {
      const FNode &fn = frontier[j];
      node_off[j] = soff[fn.slot];
      node_kc[j] = fn.cls.count();
      if (!fn.direct) continue;
      const int ci = (int)(cmaps.size() / C);
      cmaps.resize(cmaps.size() + C, 255);
      uint8_t *m = &cmaps[(size_t)ci * C];
      fn.cls.each([&](int c, int k) { m[c] = (uint8_t)k; });
      node_ci[j] = ci;
    }
    tick("cmaps");
    std::vector<int64_t> res_off(A + 1, 0);  // winners: compact per-node records (D2H bytes)
    for (int j = 0; j < A; j++)
      res_off[j + 1] = res_off[j] + (int64_t)((sizeof(NodeRes) + 8 * (size_t)node_kc[j] + 7) / 8 * 8);
    std::vector<int32_t> big_nodes, small_nodes;  // split search: by class count
    for (int j = 0; j < A; j++)
      (node_kc[j] <= split_small_max_classes() ? small_nodes : big_nodes).push_back(j);
    tick("res_off+lists");
    std::vector<SubJob> jobs;
    std::vector<int16_t> maps;
    std::vector<int32_t> zstart(ndirect_slots), sstart;  // chunk prefixes (zero / subtract)
    jobs.reserve(derived.size());
    sstart.reserve(derived.size());
    maps.reserve(derived.size() * 2 * 16);
    int zblocks = 0, sblocks = 0;
    for (int k = 0; k < ndirect_slots; k++) {
      zstart[k] = zblocks;
      zblocks += chunk_count(DS * slot_kc[k]);
    }
    for (const auto &dv : derived) {
      SubJob jb{};
      jb.off_d = node_off[dv.j];
      jb.kc_d = node_kc[dv.j];
      jb.off_p = dv.off_p;
      jb.kc_p = dv.cls_p.count();
      jb.off_s = node_off[dv.sib_j];
      jb.kc_s = node_kc[dv.sib_j];
      jb.map = (int32_t)(maps.size() / 2);
      const ClassSet &cs = frontier[dv.sib_j].cls;
      frontier[dv.j].cls.each([&](int c, int) {  // derived column -> (parent, sibling or -1)
        maps.push_back((int16_t)dv.cls_p.rank(c));
        maps.push_back((int16_t)(cs.has(c) ? cs.rank(c) : -1));
      });
      jobs.push_back(jb);
      sstart.push_back(sblocks);
      sblocks += chunk_count(DS * jb.kc_d);
    }
    if (trace) tr[6] = now_us();
    tick("jobs");
    Arena &sa = h->stage_a;
    sa.reset();
    std::vector<int32_t> node_depth(A);
    for (int j = 0; j < A; j++) node_depth[j] = frontier[j].depth;
    const size_t o_cmaps = sa.put(cmaps), o_soff = sa.put(soff), o_skc = sa.put(slot_kc),
                 o_jobs = sa.put(jobs), o_maps = sa.put(maps), o_noff = sa.put(node_off),
                 o_nkc = sa.put(node_kc), o_zst = sa.put(zstart), o_sst = sa.put(sstart),
                 o_big = sa.put(big_nodes), o_small = sa.put(small_nodes), o_roff = sa.put(res_off),
                 o_ndep = sa.put(node_depth);
    sa.flush(s);
    Hcur->grow((size_t)soff[nslots] * 4 + 16);
    if (rs)  // padding after each owner's range: summed by the reduce-scatter, never read
      for (int r = 0; r < NR; r++) {
        const int64_t used = (own[r + 1] > own[r] ? soff[own[r + 1] - 1] + DS * slot_kc[own[r + 1] - 1]
                                                  : r * Q) - r * Q;
        if (used < Q)
          CUDA_CHECK(cudaMemsetAsync(Hcur->as<uint32_t>() + r * Q + used, 0, (size_t)(Q - used) * 4, s));
      }
    // the direct slots are zeroed right before the histogram pass, except the
    // ones its CTAs store whole (see "covered" below)
    static const bool zero_all = getenv("ADAPT_ZERO_ALL") != nullptr;
    auto zero_all_slots = [&]() {
      Phase ph("zero", s, 0);
      launch_zero_slots(Hcur->as<uint32_t>(), sa.ptr<int64_t>(o_soff), sa.ptr<int32_t>(o_skc), DS,
                        sa.ptr<int32_t>(o_zst), ndirect_slots, zblocks, s);
    };
    // histogram segments built on the device (single rank, unweighted: every
    // direct node's size is its parent's winner count, so the histogram pass
    // is queued behind the partition without waiting for its share reports)
    static const bool host_segs = getenv("ADAPT_HOST_SEGS") != nullptr;
    // (small levels: the host-built segments are cheaper than the builder
    // kernel's launch — C3's 1e6 rows: 2.17 vs 2.35 ms per train)
    const bool dev = level > 0 && pst.mode != 1 && !w_root && g_ctx.world == 1 && !rs && !host_segs &&
                     (pst.rows_part >= (1 << 22) || getenv("ADAPT_DEV_SEGS") != nullptr);
    if (tagged) {
      hist_bins = pa.bins_in;
      hist_lab = h->labT.as<uint8_t>();
      hist_w = nullptr;
    } else if (level > 0) {
      hist_bins = pa.bins_out;
      hist_lab = pa.lab_out;
      hist_w = pa.w_out;
    }
    if (trace) tr[1] = now_us();
    tick("tables_upload");
    // this level's pieces, from the partition's share reports: ranges visit a
    // parent at most once each and in range order, so every child's pieces come
    // out in offset order; a counting sort by child groups them (CSR)
    auto wait_pieces = [&]() {
      if (level == 0) return;
      if (tagged || after4) {  // single rank: the nodes' rows are their winner counts
        rows_part = 0;
        for (const auto &fn : frontier) rows_part += fn.rows;
      }
      if (tagged) return;  // nothing moved: the parents' pieces serve this level
      CUDA_CHECK(cudaEventSynchronize(h->vis_evt));
      if (trace) tr[2] = now_us();
      tick("wait_part");
      std::vector<int32_t> cnt(A + 1, 0);
      std::vector<std::array<uint32_t, 3>> flat;  // (child, offset, length)
      flat.reserve((size_t)2 * pa.nranges * max_visits);
      // on the last frontier level only the direct children's rows moved
      // (decide_segs_kernel); a derived child's rows are its share's rest
      const bool last = level == D - 1;
      int64_t skipped = 0;
      for (int b = 0; b < pa.nranges && after4; b++)  // MOVE4: four grandchildren per share
        for (int v = 0; v < max_visits; v++) {
          const int32_t *e = hv + ((size_t)b * max_visits + v) * 8;
          if (e[0] < 0) break;
          const int4 gk = pseg_gkids[e[0]];
          const uint32_t A = (uint32_t)e[1], B = (uint32_t)e[2], M = A + (uint32_t)e[3];
          // the four pieces must lie inside their regions [A, M) and [M, B)
          // (the TAG pass's count cL and MOVE4's placement agree)
          if (e[1] > e[2] || e[3] < 0 || e[3] > e[2] - e[1] || e[4] < 0 || e[5] < 0 || e[6] < 0 || e[7] < 0 ||
              (int64_t)e[4] + e[5] > e[3] || (int64_t)e[6] + e[7] > (int64_t)e[2] - e[1] - e[3])
            throw Error(ADAPT_E_CUDA, "internal: MOVE4 share report outside its parent's share");
          if (gk.x >= 0 && e[4] > 0) flat.push_back({(uint32_t)gk.x, A, (uint32_t)e[4]});
          if (gk.y >= 0 && e[5] > 0) flat.push_back({(uint32_t)gk.y, M - (uint32_t)e[5], (uint32_t)e[5]});
          if (gk.z >= 0 && e[6] > 0) flat.push_back({(uint32_t)gk.z, M, (uint32_t)e[6]});
          if (gk.w >= 0 && e[7] > 0) flat.push_back({(uint32_t)gk.w, B - (uint32_t)e[7], (uint32_t)e[7]});
        }
      for (int b = 0; b < pa.nranges && !after4; b++)
        for (int v = 0; v < max_visits; v++) {
          const int32_t *e = hv + ((size_t)b * max_visits + v) * 6;
          if (e[0] < 0) break;
          const int2 ch = pseg_children[e[0]];
          if (ch.x >= 0 && e[3] > 0) flat.push_back({(uint32_t)ch.x, (uint32_t)e[1], (uint32_t)e[3]});
          if (ch.y >= 0 && e[4] > 0)
            flat.push_back({(uint32_t)ch.y, (uint32_t)(e[2] - e[4]), (uint32_t)e[4]});
          if (last && ch.x >= 0 && ch.y >= 0 && (!frontier[ch.x].direct || !frontier[ch.y].direct))
            skipped += (int64_t)(e[2] - e[1]) - e[3] - e[4];
        }
      for (const auto &x : flat) cnt[x[0] + 1]++;
      for (int j = 0; j < A; j++) cnt[j + 1] += cnt[j];
      pc_start = cnt;
      pcs.assign(flat.size(), {0u, 0u});
      for (const auto &x : flat) pcs[cnt[x[0]]++] = {x[1], x[2]};
      // rows that reached this level's nodes (moved, or left in place on the last level)
      if (!after4) {
        rows_part = skipped;
        for (const auto &pc : pcs) rows_part += pc.second;
      }
      if (dev)  // the device built the histogram segments from the planned sizes
        for (int j = 0; j < A; j++) {
          if (!frontier[j].direct) continue;
          int64_t local = 0;
          for (int q = pc_start[j]; q < pc_start[j + 1]; q++) local += pcs[q].second;
          if (local != frontier[j].rows)
            throw Error(ADAPT_E_CUDA, "internal: a node's moved rows differ from its winner count");
        }
    };
    if (!dev) wait_pieces();
    if (trace) tr[3] = now_us();
    tick("pieces");
    // the next level's a7, prepared now and launched right behind this level's
    // winner kernel: its segments are every piece of every frontier node, and
    // the device fills in each parent's split and which children stay
    // (decide_segs_kernel) — no host round trip between the winners and the move
    PartState early;
    std::vector<Seg> esegs;
    const uint8_t *early_res = nullptr;  // winner records on the device, for decide_segs
    auto launch_early = [&](const uint8_t *res_dev) {
      if (early.pa.nseg == 0) return;
      {
        Phase ph("decide", s, 0);
        if (early.mode == 2)
          launch_decide_kids(early.kid_dev, early.pa.nseg, res_dev, sa.ptr<int64_t>(o_roff), sa.ptr<int32_t>(o_nkc),
                             sa.ptr<int32_t>(o_ndep), D, h->kids.as<int4>(), s);
        else
          launch_decide_segs(const_cast<Seg *>(early.pa.segs), early.pa.nseg, res_dev, sa.ptr<int64_t>(o_roff),
                             sa.ptr<int32_t>(o_nkc), sa.ptr<int32_t>(o_ndep), D, s, early.mode == 1);
      }
      launch_part(early);
    };
    // ---- a4: histograms of the direct nodes (the root, or the smaller children) ----
    std::vector<Seg> hsegs, fsegs;  // big nodes: smem-privatised pass; small: flat pass
    uint32_t htotal = 0, ftotal = 0;
    std::vector<PlanNode> pnodes;  // dev: the big nodes' planned layout
    std::vector<int4> bseg;        // dev: per partition segment, its parent's direct child's slots
    std::vector<double> cf_slot(tagged ? nslots : 0, 1.0);  // tagged: counted share of the rows read
    if (dev) {
      // slot templates: node j's slots are the partition ranges that visit its
      // parent (one piece each), in range order; sizes from the winner counts.
      // After MOVE4 the moved "parent" is j's GRANDparent (the TAG pass's
      // segment parent) and j is one of its four grandchildren (code LL, LR,
      // RL, RR); each of the grandparent's two children has at most one
      // direct child, so a segment carries two slot entries.
      const bool m4 = pst.mode == 2;
      std::vector<int> gp_of, code_of;
      if (m4) {
        gp_of.assign(A, -1);
        code_of.assign(A, -1);
        for (size_t k = 0; k < pseg_gkids.size(); k++) {
          const int4 gk = pseg_gkids[k];
          const int g[4] = {gk.x, gk.y, gk.z, gk.w};
          for (int c = 0; c < 4; c++)
            if (g[c] >= 0) gp_of[g[c]] = pst.seg_parent[k], code_of[g[c]] = c;
        }
      }
      std::vector<int4> pinfo((m4 ? 2 : 1) * pst.pbase.size(), make_int4(-1, 0, 0, 0));
      for (int j = 0; j < A; j++) {
        const FNode &fn = frontier[j];
        if (!fn.direct) continue;
        const bool small = fn.rows * 16 < DS * (node_kc[j] | 1);
        std::vector<Seg> &lst = small ? fsegs : hsegs;
        uint32_t &tot = small ? ftotal : htotal;
        const int p = m4 ? gp_of[j] : fn.par;
        if (p < 0 || p >= (int)pst.pbase.size() || pst.plen[p] == 0)
          throw Error(ADAPT_E_CUDA, "internal: a direct node without a partitioned parent");
        const int b0 = (int)(pst.pbase[p] / pst.Rr), b1 = (int)((pst.pbase[p] + pst.plen[p] - 1) / pst.Rr);
        if (m4)
          pinfo[2 * p + (code_of[j] >> 1)] = make_int4(code_of[j], small ? 1 : 0, (int)lst.size() - b0, 0);
        else
          pinfo[p] = make_int4(fn.side, small ? 1 : 0, (int)lst.size() - b0, 0);
        if (!small) pnodes.push_back(PlanNode{-1, -1, tot, (uint32_t)fn.rows, node_kc[j]});
        Seg sg{};
        sg.hslot = fn.slot;
        sg.cmap = node_ci[j];
        sg.ncls = node_kc[j];
        sg.node_base = tot;
        sg.node_len = (uint32_t)fn.rows;
        sg.row_base = tot;
        sg.feat = -1;
        for (int b = b0; b <= b1; b++) lst.push_back(sg);
        tot += (uint32_t)fn.rows;
      }
      if (m4) {
        bseg.resize(2 * pst.seg_parent.size());
        for (size_t k = 0; k < pst.seg_parent.size(); k++)
          for (int c = 0; c < 2; c++) bseg[2 * k + c] = pinfo[2 * pst.seg_parent[k] + c];
      } else {
        bseg.resize(pst.seg_parent.size());
        for (size_t k = 0; k < bseg.size(); k++) bseg[k] = pinfo[pst.seg_parent[k]];
      }
    } else {
      for (int j = 0; j < A; j++) {
        const FNode &fn = frontier[j];
        if (!fn.direct) continue;
        const int pj = tagged ? fn.par : j;  // tagged: the parent's pieces, marked rows count
        int64_t local = 0;
        for (int q = pc_start[pj]; q < pc_start[pj + 1]; q++) local += pcs[q].second;
        const bool small = local * 16 < DS * (node_kc[j] | 1);
        if (tagged) cf_slot[fn.slot] = local ? (double)fn.rows / (double)local : 1.0;
        for (int q = pc_start[pj]; q < pc_start[pj + 1]; q++) {
          const auto &pc = pcs[q];
          Seg sg{};
          sg.off = pc.first;
          sg.len = pc.second;
          sg.hslot = fn.slot;
          sg.cmap = node_ci[j];
          sg.ncls = node_kc[j];
          (small ? fsegs : hsegs).push_back(sg);
        }
      }
      ftotal = virtualize(fsegs, true);
      htotal = virtualize(hsegs, true);
    }
    tick("hsegs");
    if (htotal + ftotal > 0) {
      Arena &sb = h->stage_b;
      sb.reset();
      // one CTA per SM, each reading only its own group's word plane (the CTAs
      // of different groups share just the 1-byte labels and run unsynchronised)
      const int nranges = (int)std::max<int64_t>(1, std::min<int64_t>((htotal + 4095) / 4096,
                                                                      std::max(1, sms / ngroups)));
      tick("arena_reset");
      // small levels (C3's 1e6-row table: every level is launch/latency-bound)
      // take uniform row ranges per group, groups interleaved; the cost-balanced
      // plan pays from a few million rows on (C3: 3.5 vs 2.4 ms per train)
      constexpr uint32_t kPlanMinRows = 1u << 22;
      std::vector<HistCta> ctas;
      if (htotal >= kPlanMinRows) {
        ctas = dev ? plan_hist_ctas(pnodes, hsegs, htotal, gcost, nranges * ngroups)
                   : plan_hist_ctas(hsegs, htotal, gcost, nranges * ngroups, tagged ? &cf_slot : nullptr);
      } else {
        const uint32_t R = (htotal + nranges - 1) / nranges;
        for (int r = 0; r < nranges; r++)
          for (int g = 0; g < ngroups; g++)
            ctas.push_back(HistCta{g, std::min<uint32_t>(r * R, htotal), std::min<uint32_t>((r + 1) * R, htotal), -1});
      }
      tick("plan");
      // A direct slot needs no zeroing when, for every word group holding some
      // of its classes, one CTA sees the node's whole virtual range through the
      // shared-memory path: that CTA's flush STORES every counter of its block
      // (hist_kernel "sole"; a tiny portion counts into global memory instead,
      // a small node goes to the flat pass — both need the zeros)
      std::vector<char> covered(ndirect_slots, 0);
      if (!zero_all && !hsegs.empty()) {
        std::vector<std::vector<std::pair<uint32_t, uint32_t>>> rg(ngroups);  // CTA ranges per group
        for (const auto &ct : ctas) rg[ct.g].push_back({ct.p0, ct.p1});
        for (auto &v : rg) std::sort(v.begin(), v.end());
        for (size_t i = 0; i < hsegs.size();) {
          size_t k = i;
          while (k < hsegs.size() && hsegs[k].hslot == hsegs[i].hslot) k++;
          const Seg &sg = hsegs[i];
          const uint32_t nb = sg.node_base, ne = sg.node_base + sg.node_len;
          bool ok = sg.hslot >= 0 && sg.hslot < ndirect_slots && sg.node_len > 0;
          for (int g = 0; g < ngroups && ok; g++) {
            const int kn = std::min(gl[g].kw, sg.ncls - gl[g].k0);
            if (kn <= 0) continue;  // none of the node's classes in this group
            if ((int64_t)sg.node_len * 16 < (int64_t)gcost[g].dsw * (kn | 1)) {
              ok = false;  // a tiny portion: global atomics
              break;
            }
            const auto &v = rg[g];
            auto it = std::upper_bound(v.begin(), v.end(), std::make_pair(nb, UINT32_MAX));
            ok = it != v.begin() && std::prev(it)->first <= nb && std::prev(it)->second >= ne;
          }
          if (ok) covered[sg.hslot] = 1;
          i = k;
        }
      }
      std::vector<int32_t> zslot, zst2;
      int zb2 = 0;
      for (int k = 0; k < ndirect_slots; k++) {
        if (covered[k]) continue;
        zslot.push_back(k);
        zst2.push_back(zb2);
        zb2 += chunk_count(DS * slot_kc[k]);
      }
      const size_t o_hsegs = sb.put(hsegs), o_fsegs = sb.put(fsegs), o_ctas = sb.put(ctas),
                   o_bseg = sb.put(bseg), o_zslot = sb.put(zslot), o_zst2 = sb.put(zst2);
      sb.flush(s);
      {
        Phase ph("zero", s, 0);
        launch_zero_slots(Hcur->as<uint32_t>(), sa.ptr<int64_t>(o_soff), sa.ptr<int32_t>(o_skc), DS,
                          sb.ptr<int32_t>(o_zst2), (int)zslot.size(), zb2, s, sb.ptr<int32_t>(o_zslot));
      }
      tick("upload_b");
      Seg *d_hsegs = sb.ptr<Seg>(o_hsegs), *d_fsegs = sb.ptr<Seg>(o_fsegs);
      if (dev) {  // the templates are filled in place by the builder
        h->dseg_err.ensure(16);
        h->hseg_err.grow(16);
        CUDA_CHECK(cudaMemsetAsync(h->dseg_err.p, 0, 4, s));
        SegBuildArgs ba{};
        ba.mode4 = pst.mode == 2;
        ba.visits = pa.visits;  // the move's share reports (MOVE4: its own buffer)
        ba.nranges = pa.nranges;
        ba.max_visits = max_visits;
        ba.bseg = sb.ptr<int4>(o_bseg);
        ba.segs[0] = d_hsegs;
        ba.segs[1] = d_fsegs;
        ba.nslot[0] = (int)hsegs.size();
        ba.nslot[1] = (int)fsegs.size();
        ba.total[0] = htotal;
        ba.total[1] = ftotal;
        ba.err = h->dseg_err.as<int32_t>();
        {
          Phase ph("decide", s, 0);
          launch_build_hist_segs(ba, s);
        }
        CUDA_CHECK(cudaMemcpyAsync(h->hseg_err.p, h->dseg_err.p, 4, cudaMemcpyDeviceToHost, s));
      }
      HistArgs ha{};
      ha.segs = d_hsegs;
      ha.nseg = (int)hsegs.size();
      ha.total_rows = htotal;
      ha.bins_in = hist_bins;
      ha.lab_in = hist_lab;
      ha.w_in = hist_w;
      ha.pstride = ps;
      ha.BS = BS;
      ha.F = F;
      ha.C = C;
      ha.cumD = h->hoff.as<int32_t>();
      ha.nval = h->dnval.as<int32_t>();
      ha.groups = h->grp.as<int4>();
      ha.cmaps = sa.ptr<uint8_t>(o_cmaps);
      ha.ngroups = ngroups;
      ha.smem_counters = max_group;
      ha.H = Hcur->as<uint32_t>();
      ha.soff = sa.ptr<int64_t>(o_soff);
      ha.ctas = sb.ptr<HistCta>(o_ctas);
      ha.nctas = (int)ctas.size();
      ha.tagged = tagged ? 1 : 0;
      snprintf(nm, sizeof nm, "hist_L%02d", level);
      Phase ph(per_level ? nm : "hist", s, (double)(htotal + ftotal) * (F + 1));
      tick("hist_args");
      launch_hist(ha, s);
      tick("launch_hist");
      HistArgs fa = ha;  // the small nodes
      fa.segs = d_fsegs;
      fa.nseg = (int)fsegs.size();
      fa.total_rows = ftotal;
      launch_hist_flat(fa, s);
      tick("launch_flat");
    } else {
      zero_all_slots();  // no rows here: the (all-reduced) slots must still be zero
    }
    if (!rs && collectives_on() && ndirect_slots > 0)  // the direct slots are contiguous at the front
      comm_allreduce_sum(Hcur->p, (size_t)soff[ndirect_slots], false, s, "allreduce histograms");
    if (!jobs.empty()) {  // rs: local parent - local direct sibling = the sibling's local rows
      Phase ph("subtract", s, 0);
      launch_subtract(Hcur->as<uint32_t>(), Hprev->as<uint32_t>(), DS, sa.ptr<SubJob>(o_jobs),
                      sa.ptr<int16_t>(o_maps), sa.ptr<int32_t>(o_sst), (int)jobs.size(), sblocks, s);
    }
    h->hres.grow((size_t)res_off[A] + 16);
    uint8_t *hr = h->hres.as<uint8_t>();
    int64_t comm_bytes = collectives_on() ? (int64_t)soff[ndirect_slots] * 4 : 0;
    if (!rs) {
      h->cand.grow((size_t)A * F * sizeof(SplitCand));
      h->res.grow((size_t)res_off[A] + 16);
      {
        snprintf(nm, sizeof nm, "split_L%02d", level);
        Phase ph(per_level ? nm : "split", s, 0);
        launch_split(Hcur->as<uint32_t>(), sa.ptr<int64_t>(o_noff), sa.ptr<int32_t>(o_nkc),
                     sa.ptr<int32_t>(o_big), (int)big_nodes.size(), sa.ptr<int32_t>(o_small),
                     (int)small_nodes.size(), F, h->hoff.as<int32_t>(),
                     h->dnval.as<int32_t>(), h->cand.as<SplitCand>(), s);
      }
      {
        Phase ph("winner", s, 0);
        launch_winner(Hcur->as<uint32_t>(), sa.ptr<int64_t>(o_noff), sa.ptr<int32_t>(o_nkc), A, F, C,
                      h->hoff.as<int32_t>(), h->dnval.as<int32_t>(), h->cand.as<SplitCand>(),
                      h->res.as<uint8_t>(), sa.ptr<int64_t>(o_roff), s);
      }
      CUDA_CHECK(cudaMemcpyAsync(hr, h->res.p, (size_t)res_off[A], cudaMemcpyDeviceToHost, s));
      if (!h->win_evt) CUDA_CHECK(cudaEventCreateWithFlags(&h->win_evt, cudaEventDisableTiming));
      CUDA_CHECK(cudaEventRecord(h->win_evt, s));
      early_res = h->res.as<uint8_t>();
    } else {
      // a5 by ownership: this rank's slots summed over ranks into Hg
      h->Hg.grow((size_t)Q * 4 + 16);
      comm_reduce_scatter(Hcur->p, h->Hg.p, (size_t)Q, s, "reduce-scatter histograms");
      // a6 for the owned nodes only, in slot order: owned index i = slot own[r] + i
      std::vector<int32_t> slot_j(nslots);
      for (int j = 0; j < A; j++) slot_j[frontier[j].slot] = j;
      std::vector<int64_t> ooff;
      std::vector<int32_t> okc, obig, osmall;
      std::vector<std::vector<int64_t>> rb(NR);  // winner record offsets of every rank's owned nodes
      for (int r = 0; r < NR; r++) {
        rb[r].assign(1, 0);
        for (int k = own[r]; k < own[r + 1]; k++)
          rb[r].push_back(rb[r].back() + (res_off[slot_j[k] + 1] - res_off[slot_j[k]]));
      }
      int64_t RB = 16;
      for (int r = 0; r < NR; r++) RB = std::max(RB, rb[r].back());
      for (int k = own[me]; k < own[me + 1]; k++) {
        const int j = slot_j[k], i = (int)okc.size();
        ooff.push_back(soff[k] - me * Q);
        okc.push_back(node_kc[j]);
        (node_kc[j] <= split_small_max_classes() ? osmall : obig).push_back(i);
      }
      const int m = (int)okc.size();
      Arena &so = h->stage_r;
      so.reset();
      const size_t o_ooff = so.put(ooff), o_okc = so.put(okc), o_obig = so.put(obig),
                   o_osmall = so.put(osmall), o_orb = so.put(rb[me]);
      so.flush(s);
      h->cand.grow((size_t)std::max(m, 1) * F * sizeof(SplitCand));
      h->reso.grow((size_t)RB + 16);
      h->resall.grow((size_t)RB * NR + 16);
      {
        snprintf(nm, sizeof nm, "split_L%02d", level);
        Phase ph(per_level ? nm : "split", s, 0);
        launch_split(h->Hg.as<uint32_t>(), so.ptr<int64_t>(o_ooff), so.ptr<int32_t>(o_okc),
                     so.ptr<int32_t>(o_obig), (int)obig.size(), so.ptr<int32_t>(o_osmall),
                     (int)osmall.size(), F, h->hoff.as<int32_t>(), h->dnval.as<int32_t>(),
                     h->cand.as<SplitCand>(), s);
      }
      {
        Phase ph("winner", s, 0);
        launch_winner(h->Hg.as<uint32_t>(), so.ptr<int64_t>(o_ooff), so.ptr<int32_t>(o_okc), m, F, C,
                      h->hoff.as<int32_t>(), h->dnval.as<int32_t>(), h->cand.as<SplitCand>(),
                      h->reso.as<uint8_t>(), so.ptr<int64_t>(o_orb), s);
      }
      // every rank gets every owner's winner records (padded to RB bytes each)
      comm_allgather(h->reso.p, h->resall.p, (size_t)RB, s, "all-gather winners");
      h->hgat.grow((size_t)RB * NR + 16);
      uint8_t *ga = h->hgat.as<uint8_t>();
      CUDA_CHECK(cudaMemcpyAsync(ga, h->resall.p, (size_t)RB * NR, cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
      for (int r = 0; r < NR; r++)
        for (int k = own[r]; k < own[r + 1]; k++) {
          const int j = slot_j[k];
          memcpy(hr + res_off[j], ga + (size_t)r * RB + rb[r][k - own[r]], (size_t)(res_off[j + 1] - res_off[j]));
        }
      comm_bytes = NR * Q * 4 + RB * NR;
      if (!h->win_evt) CUDA_CHECK(cudaEventCreateWithFlags(&h->win_evt, cudaEventDisableTiming));
      CUDA_CHECK(cudaEventRecord(h->win_evt, s));
      if (level + 1 < D) {  // the records in node order on the device, for the early partition
        h->res.grow((size_t)res_off[A] + 16);
        CUDA_CHECK(cudaMemcpyAsync(h->res.p, hr, (size_t)res_off[A], cudaMemcpyHostToDevice, s));
        early_res = h->res.as<uint8_t>();
      }
    }
    if (dev) wait_pieces();  // (the histogram .. winner chain is queued already)
    // the next level's a7 (prepared after the winner launch: only needed behind it)
    if (level + 1 < D && tagged) {  // MOVE4 from the parents' planes (the TAG pass's segments)
      early = start_move4(tag_st, level + 1, pseg_children, out_plane);
    } else if (level + 1 < D) {
      esegs.reserve(pcs.size());
      for (int j = 0; j < A; j++)
        for (int q = pc_start[j]; q < pc_start[j + 1]; q++) {
          Seg sg{};
          sg.off = pcs[q].first;
          sg.len = pcs[q].second;
          sg.feat = -1;
          sg.direct = j;  // parent id (groups a parent's pieces); the decision fills the rest
          sg.hslot = -1;
          esegs.push_back(sg);
        }
      // two-level: the TAG pass instead of a move — except into the last frontier
      // level, where a partition moves only the direct children's rows (measured
      // cheaper than TAG + a histogram over the parents' rows)
      static const bool tag_last = getenv("ADAPT_TAG_LAST") != nullptr;
      const int mode = two_level && (level + 2 < D || tag_last) ? 1 : 0;
      early = level > 0
                  ? start_part(level + 1, esegs, (out_plane ? h->binsB : h->binsA).as<uint8_t>(),
                               (out_plane ? h->labB : h->labA).as<uint8_t>(),
                               w_root ? (out_plane ? h->wB : h->wA).as<uint8_t>() : nullptr, out_plane ^ 1, true,
                               mode)
                  : start_part(level + 1, esegs, bins_in, lab_in, w_in, out_plane, true, mode);
    }
    if (early_res) launch_early(early_res);
    if (trace) tr[4] = now_us();
    tick("launch_hist..winner");
    CUDA_CHECK(cudaEventSynchronize(h->win_evt));  // the winners (the early partition may still run)
    if (dev && htotal + ftotal > 0 && *h->hseg_err.as<int32_t>())
      throw Error(ADAPT_E_CUDA, "internal: device-built histogram segments disagree with the planned sizes");
    if (trace) tr[5] = now_us();
    tick("wait_winners");
    h->stats.push_back(A);
    h->stats.push_back(htotal + ftotal);
    h->stats.push_back(rows_part);
    h->stats.push_back((int64_t)soff[nslots] * 4);  // histogram bytes (direct + derived nodes)
    h->stats.push_back(comm_bytes);  // bytes through the per-level collectives
    h->stats.push_back(direct_bytes);  // the direct nodes' histograms

    // ---- decide every frontier node; build the next level ----
    std::vector<FNode> next;
    std::vector<int2> nchildren;
    std::vector<Derived> nderived;
    next.reserve((size_t)2 * A);
    nderived.reserve(A);
    nchildren.reserve((size_t)2 * A);
    h->tree.reserve(h->tree.size() + (size_t)2 * A);
    int ndirect = 0;
    // pass 1: what the next partition needs (split feature / rank, which
    // children stay in the frontier, the direct child's slot), then launch it;
    // pass 2 (the tree, the next frontier's class sets and subtraction jobs)
    // runs on the host while the GPU moves the rows
    struct Dec {
      bool inL, inR;
      int32_t hslot;
    };
    std::vector<Dec> dec(A, Dec{false, false, -1});
    // (the last frontier level's children are leaves: nothing to decide here)
    for (int j = 0; j < A && level + 1 < D; j++) {
      const NodeRes *nr = reinterpret_cast<const NodeRes *>(hr + res_off[j]);
      const uint32_t *Pd = reinterpret_cast<const uint32_t *>(nr + 1);
      const uint32_t *cLd = Pd + node_kc[j];
      const FNode &fn = frontier[j];
      const int kc = node_kc[j];
      int np = 0, npl = 0, npr = 0;
      for (int k = 0; k < kc; k++) {
        np += Pd[k] > 0;
        npl += cLd[k] > 0;
        npr += Pd[k] - cLd[k] > 0;
      }
      if (fn.depth >= D || np <= 1 || !nr->valid) continue;  // leaf (R10, R11)
      Dec &d = dec[j];
      d.inL = fn.depth + 1 < D && npl > 1;
      d.inR = fn.depth + 1 < D && npr > 1;
      if (!d.inL && !d.inR) continue;
      d.hslot = ndirect++;
    }
    tick("pass1");
    // the next level's a7 is already running (launched behind the winner kernel)
    if (ndirect > 0 && !early.launched)
      throw Error(ADAPT_E_CUDA, "internal: frontier continues without a partition");
    pending = early;
    // one pass over a node's compact classes: n, S = sum c^2 and the majority
    // class (ties -> lowest, R12) of the node, of its left part and of its
    // right part, and the children's class sets
    std::vector<uint64_t> P(C), PL(C), PR(C);
    std::vector<int2> kids(A, make_int2(-1, -1));  // frontier children of node j (-1: leaf / none)
    for (int j = 0; j < A; j++) {
      const NodeRes *nr = reinterpret_cast<const NodeRes *>(hr + res_off[j]);
      const uint32_t *Pd = reinterpret_cast<const uint32_t *>(nr + 1);  // compact columns
      const uint32_t *cLd = Pd + node_kc[j];
      const FNode &fn = frontier[j];
      // everything in the node's compact columns (class cl[k], ascending)
      const int kc = node_kc[j];
      int cl_of[kMaxC + 1];
      fn.cls.each([&](int c, int k) { cl_of[k] = c; });
      auto stats = [&](adapt_node_t &o, const uint64_t *cnt) {  // n, label, gini (fill_stats)
        uint64_t nn = 0;
        unsigned __int128 S = 0;
        int best = 0;
        for (int k = 0; k < kc; k++) {
          nn += cnt[k];
          S += (unsigned __int128)cnt[k] * cnt[k];
          if (cnt[k] > cnt[best]) best = k;  // ties -> lowest class (R12)
        }
        o.n = (int64_t)nn;
        o.label = kc ? cl_of[best] : 0;
        o.gini = nn ? 1.0 - (double)(uint64_t)S / ((double)nn * (double)nn) : 0.0;
      };
      auto npresent = [&](const uint64_t *cnt) {
        int z = 0;
        for (int k = 0; k < kc; k++) z += cnt[k] > 0;
        return z;
      };
      auto present = [&](const uint64_t *cnt) {
        ClassSet v;
        for (int k = 0; k < kc; k++)
          if (cnt[k]) v.add(cl_of[k]);
        return v;
      };
      for (int k = 0; k < kc; k++) {
        P[k] = Pd[k];
        PL[k] = cLd[k];
        PR[k] = P[k] - PL[k];
      }
      stats(h->tree[fn.tree_idx], P.data());
      h->tree[fn.tree_idx].depth = fn.depth;
      if (fn.depth >= D || npresent(P.data()) <= 1 || !nr->valid) continue;  // leaf (R10, R11)
      const int f = nr->feat;
      adapt_node_t &nd = h->tree[fn.tree_idx];
      nd.feature = f;
      if ((h->qmask >> f) & 1)  // R23: between the bins b_lo and b_lo + 1 of the quantiser
        nd.threshold = ((double)h->qprev[f * kMaxBins + nr->b_lo + 1] +
                        (double)h->val[f * kMaxBins + nr->b_lo + 1]) / 2;
      else
        nd.threshold = ((double)h->val[f * kMaxBins + nr->b_lo] +
                        (double)h->val[f * kMaxBins + nr->b_hi]) / 2;  // R7
      const int32_t li = (int32_t)h->tree.size();
      nd.left = li;
      nd.right = li + 1;
      adapt_node_t cl{}, cr{};
      cl.feature = cr.feature = -1;
      cl.left = cl.right = cr.left = cr.right = -1;
      cl.depth = cr.depth = fn.depth + 1;
      const bool inL = dec[j].inL, inR = dec[j].inR;
      // frontier children get their stats from their own class totals next level
      if (!inL) stats(cl, PL.data());
      if (!inR) stats(cr, PR.data());
      h->tree.push_back(cl);
      h->tree.push_back(cr);
      if (!inL && !inR) continue;
      const uint64_t nL = nr->nL, nR = nr->n - nr->nL;
      int dir;
      if (inL && inR) dir = nL <= nR ? 0 : 1;  // histogram the smaller child
      else dir = inL ? 0 : 1;
      const int32_t hslot = dec[j].hslot;
      int jl = -1, jr = -1;
      if (inL) {
        jl = (int)next.size();
        next.push_back(FNode{li, fn.depth + 1, dir == 0 ? hslot : -1, dir == 0, present(PL.data()),
                             (int64_t)nr->nL, j, 0});
      }
      if (inR) {
        jr = (int)next.size();
        next.push_back(FNode{li + 1, fn.depth + 1, dir == 1 ? hslot : -1, dir == 1, present(PR.data()),
                             (int64_t)(nr->n - nr->nL), j, 1});
      }
      if (inL && inR) {  // the other child by subtraction from this node's histogram
        Derived dv;
        dv.j = dir == 0 ? jr : jl;
        dv.sib_j = dir == 0 ? jl : jr;
        dv.off_p = node_off[j];
        dv.cls_p = fn.cls;
        nderived.push_back(dv);
      }
      kids[j] = make_int2(jl, jr);
    }
    if (tagged) {  // MOVE4's grandchildren per TAG segment (the next level's pieces)
      pseg_gkids.resize(pseg_children.size());
      for (size_t q = 0; q < pseg_children.size(); q++) {
        const int2 c = pseg_children[q];
        const int2 l = c.x >= 0 ? kids[c.x] : make_int2(-1, -1), r = c.y >= 0 ? kids[c.y] : make_int2(-1, -1);
        pseg_gkids[q] = make_int4(l.x, l.y, r.x, r.y);
      }
    } else {
      for (int j = 0; j < A; j++)  // the children of each early-partition segment (all pieces)
        for (int q = pc_start[j]; q < pc_start[j + 1]; q++) nchildren.push_back(kids[j]);
    }
    // derived slots follow the direct ones
    for (size_t i = 0; i < nderived.size(); i++) next[nderived[i].j].slot = ndirect + (int)i;
    tick("pass2");
    if (trace2) {
      fprintf(stderr, "[adapt] L%02d host:", level);
      for (size_t i = 1; i < ticks.size(); i++)
        fprintf(stderr, " %s %.0f", ticks[i].first, ticks[i].second - ticks[i - 1].second);
      fprintf(stderr, " us\n");
    }
    if (trace)
      fprintf(stderr, "[adapt] L%02d A=%d part-launch %.0f us (tables %.0f, ranges %.0f), wait %.0f, pieces %.0f, "
              "hist..winner launch %.0f, wait %.0f, decide %.0f us\n", level, A,
              level ? tr[1] - tr[0] : 0.0, tr[6] - tr[0], t_mv - tr[6], level ? tr[2] - tr[1] : 0.0, level ? tr[3] - tr[2] : 0.0,
              tr[4] - tr[3], tr[5] - tr[4], now_us() - tr[5]);
    frontier.swap(next);
    if (!tagged) pseg_children.swap(nchildren);
    ndirect_slots = ndirect;
    derived.swap(nderived);
    std::swap(Hcur, Hprev);
    // the planes just written are the input of the next partition; the root
    // level moved nothing, so level 1 still reads the ingest output
    if (level > 0 && !tagged) {  // (a tagged level moved nothing)
      bins_in = (out_plane ? h->binsB : h->binsA).as<uint8_t>();
      lab_in = (out_plane ? h->labB : h->labA).as<uint8_t>();
      if (w_root) w_in = (out_plane ? h->wB : h->wA).as<uint8_t>();
      out_plane ^= 1;
    }
  }
  };  // grow_tree

  auto shard_lo = [&]() {  // this rank's first global row
    uint64_t lo = 0;
    if (collectives_on()) {
      DevBuf nb, allb;
      nb.ensure(8);
      allb.ensure((size_t)world * 8);
      const uint64_t mine = (uint64_t)n;
      CUDA_CHECK(cudaMemcpyAsync(nb.p, &mine, 8, cudaMemcpyHostToDevice, s));
      comm_allgather(nb.p, allb.p, 8, s, "allgather row counts");
      std::vector<uint64_t> all(world);
      CUDA_CHECK(cudaMemcpyAsync(all.data(), allb.p, (size_t)world * 8, cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
      for (int r = 0; r < g_ctx.rank; r++) lo += all[r];
    }
    return lo;
  };

  if (h->multi_n) {  // adapt_train_many: k regions' trees in ONE multi-root frontier (C2, R15)
    const auto &mn = *h->multi_n;
    const int R = (int)mn.size();
    std::vector<uint64_t> tot(mn.begin(), mn.end());
    if (collectives_on()) {
      DevBuf t;
      t.ensure((size_t)R * 8);
      CUDA_CHECK(cudaMemcpyAsync(t.p, tot.data(), (size_t)R * 8, cudaMemcpyHostToDevice, s));
      comm_allreduce_sum(t.p, (size_t)R, true, s, "allreduce region rows");
      CUDA_CHECK(cudaMemcpyAsync(tot.data(), t.p, (size_t)R * 8, cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
    }
    for (int r = 0; r < R; r++)
      if (tot[r] == 0) throw Error(ADAPT_E_INSUFFICIENT_DATA, "a region has no rows");
    MultiRoot mr;
    mr.R = R;
    mr.bins = h->bins.as<uint8_t>();
    mr.labs = h->labels.as<uint8_t>();
    mr.pstride = pstride;
    mr.rows_out = n;
    mr.pieces.resize(R);
    int64_t off = 0;
    for (int r = 0; r < R; r++) {
      if (mn[r]) mr.pieces[r].push_back({(uint32_t)off, (uint32_t)mn[r]});
      off += mn[r];
    }
    grow_tree(nullptr, &mr);
    h->multi_trees.assign(R, {});
    for (int r = 0; r < R; r++) {  // canonical BFS per region (BFS from its root)
      auto &tr = h->multi_trees[r];
      std::vector<int32_t> q{r};
      for (size_t qi = 0; qi < q.size(); qi++) {
        adapt_node_t nd = h->tree[q[qi]];
        if (nd.feature >= 0) {
          q.push_back(nd.left);
          q.push_back(nd.right);
          nd.left = (int32_t)(q.size() - 2);
          nd.right = (int32_t)(q.size() - 1);
        }
        tr.push_back(nd);
      }
    }
    h->trained_n = n;
    return;
  }

  if (h->kfold) {  // K-fold harness (R22): all models of a batch of shuffles in ONE frontier
    const auto &kf = *h->kfold;
    const int K = kf.K, m = kf.m;
    if (n_total < (uint64_t)K) throw Error(ADAPT_E_INSUFFICIENT_DATA, "fewer rows than K groups");
    const uint64_t lo = shard_lo();
    std::vector<uint64_t> bnd(K + 1);
    for (int j = 0; j <= K; j++)  // ceil(j N / K): the first position of group j
      bnd[j] = (uint64_t)(((unsigned __int128)j * n_total + K - 1) / K);
    h2d(h->kbnd, bnd, s);
    // shuffles per batch: the models' rows (m copies of the table per shuffle)
    // must stay below 2^30 per rank (u32 positions, plane memory)
    const int64_t per_shuffle = std::max<int64_t>(1, (int64_t)m * n);
    const int Sb = (int)std::max<int64_t>(1, std::min<int64_t>(kf.shuffles, (1ll << 30) / per_shuffle));
    const int nb = kfold_eval_blocks();
    h->kfold_trees.clear();
    std::vector<int64_t> stats;
    for (int s0 = 0; s0 < kf.shuffles; s0 += Sb) {
      const int sb = std::min(Sb, kf.shuffles - s0), R = sb * K;
      const int64_t nn = std::max<int64_t>(n, 1);
      const size_t ps = bins_plane_stride(std::max<int64_t>((int64_t)sb * m * n, (int64_t)sb * n), BS);
      h->kgrp.ensure((size_t)sb * nn);
      h->kcnt.ensure((size_t)R * 8);
      CUDA_CHECK(cudaMemsetAsync(h->kcnt.p, 0, (size_t)R * 8, s));
      {
        Phase ph("kfold", s, (double)n * sb);
        for (int j = 0; j < sb; j++)
          launch_kfold_groups(kf.seed, s0 + j, n_total, h->kbnd.as<uint64_t>(), K, lo, n,
                              h->kgrp.as<uint8_t>() + (size_t)j * nn,
                              h->kcnt.as<unsigned long long>() + (size_t)j * K, s);
      }
      std::vector<unsigned long long> cnt(R);
      CUDA_CHECK(cudaMemcpyAsync(cnt.data(), h->kcnt.p, (size_t)R * 8, cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
      std::vector<uint32_t> cur(R);  // group (j, g) lands at [cur, cur + cnt) of the sorted planes
      uint32_t acc = 0;
      for (int r = 0; r < R; r++) {
        cur[r] = acc;
        acc += (uint32_t)cnt[r];
      }
      MultiRoot mr;
      mr.R = R;
      mr.pstride = ps;
      mr.rows_out = (int64_t)sb * m * n;
      mr.pieces.resize(R);
      for (int j = 0; j < sb; j++)
        for (int k = 0; k < K; k++)
          for (int t = 0; t < m; t++) {
            const int g = j * K + (k + t) % K;
            if (cnt[g]) mr.pieces[j * K + k].push_back({cur[g], (uint32_t)cnt[g]});
          }
      h2d(h->kcur, cur, s);
      h->ksb.ensure(ps * (BS < 4 ? 1 : BS / 4));
      h->klab.ensure((size_t)sb * nn + 64);
      {
        Phase ph("kfold", s, (double)n * sb * 2 * (BS + 1));
        launch_kfold_scatter(h->bins.as<uint8_t>(), pstride, h->labels.as<uint8_t>(), n, BS,
                             h->kgrp.as<uint8_t>(), sb, K, h->kcur.as<unsigned int>(), h->ksb.as<uint8_t>(), ps,
                             h->klab.as<uint8_t>(), s);
      }
      mr.bins = h->ksb.as<uint8_t>();
      mr.labs = h->klab.as<uint8_t>();
      grow_tree(nullptr, &mr);
      stats.insert(stats.end(), h->stats.begin(), h->stats.end());
      // the combined array -> one canonical BFS tree per model (BFS from its root)
      std::vector<std::vector<adapt_node_t>> batch(R);
      for (int r = 0; r < R; r++) {
        auto &tr = batch[r];
        std::vector<int32_t> q{r};
        for (size_t qi = 0; qi < q.size(); qi++) {
          adapt_node_t nd = h->tree[q[qi]];
          if (nd.feature >= 0) {
            q.push_back(nd.left);
            q.push_back(nd.right);
            nd.left = (int32_t)(q.size() - 2);
            nd.right = (int32_t)(q.size() - 1);
          }
          tr.push_back(nd);
        }
      }
      // held-out evaluation of the batch's models in one pass over the rows
      std::vector<DNode> d;
      std::vector<int32_t> roots;
      for (const auto &tr : batch) {
        const int32_t off = (int32_t)d.size();
        roots.push_back(off);
        for (const auto &nd : tr) {
          DNode x;
          x.thr = nd.feature >= 0 ? round_down_f32(nd.threshold) : 0.f;
          x.meta = nd.feature >= 0 ? ((nd.left + off) << 6) | nd.feature : -1 - nd.label;
          d.push_back(x);
        }
      }
      if (d.size() >= (1u << 25)) throw Error(ADAPT_E_INVALID_ARG, "K-fold models too large (2^25 nodes)");
      h2d(h->knodes, d, s);
      h2d(h->kroots, roots, s);
      h->kpart.ensure((size_t)nb * R * sizeof(KfoldPartial));
      std::vector<KfoldPartial> part((size_t)nb * R);
      if (n) {
        Phase ph("kfold", s, (double)n * (4.0 * F + 2 + sb));
        launch_kfold_eval_many(feat, n, F, V, times, h->labels.as<uint8_t>(), h->kgrp.as<uint8_t>(), sb, K, m,
                               h->knodes.as<DNode>(), h->kroots.as<int32_t>(), h->kpart.as<KfoldPartial>(), s);
        CUDA_CHECK(cudaMemcpyAsync(part.data(), h->kpart.p, part.size() * sizeof(KfoldPartial),
                                   cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
      }
      std::vector<KfoldPartial> mine(R, KfoldPartial{0, 0, 0.0, 0.0});
      if (n)
        for (int b = 0; b < nb; b++)  // block order
          for (int r = 0; r < R; r++) {
            const KfoldPartial &p = part[(size_t)b * R + r];
            mine[r].n_test += p.n_test;
            mine[r].n_correct += p.n_correct;
            mine[r].t_selected += p.t_selected;
            mine[r].t_best += p.t_best;
          }
      std::vector<KfoldPartial> tot = mine;
      if (collectives_on()) {  // every rank's partials, summed in rank order
        DevBuf sendb, allb;
        sendb.ensure((size_t)R * 32);
        allb.ensure((size_t)world * R * 32);
        CUDA_CHECK(cudaMemcpyAsync(sendb.p, mine.data(), (size_t)R * 32, cudaMemcpyHostToDevice, s));
        comm_allgather(sendb.p, allb.p, (size_t)R * 32, s, "allgather kfold results");
        std::vector<KfoldPartial> all((size_t)world * R);
        CUDA_CHECK(cudaMemcpyAsync(all.data(), allb.p, (size_t)world * R * 32, cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        for (int r = 0; r < R; r++) {
          tot[r] = all[r];
          for (int w = 1; w < world; w++) {
            const KfoldPartial &p = all[(size_t)w * R + r];
            tot[r].n_test += p.n_test;
            tot[r].n_correct += p.n_correct;
            tot[r].t_selected += p.t_selected;
            tot[r].t_best += p.t_best;
          }
        }
      }
      for (int r = 0; r < R; r++) {
        adapt_kfold_result_t &o = kf.out[(size_t)s0 * K + r];
        o.shuffle = s0 + r / K;
        o.fold = r % K;
        o.n_nodes = (int32_t)batch[r].size();
        o.pad_ = 0;
        o.n_test = (int64_t)tot[r].n_test;
        o.n_train = (int64_t)n_total - o.n_test;
        o.n_correct = (int64_t)tot[r].n_correct;
        o.t_selected = tot[r].t_selected;
        o.t_best = tot[r].t_best;
        h->kfold_trees.push_back(std::move(batch[r]));
      }
    }
    h->stats.swap(stats);
    return;  // the region's own model is restored by adapt_kfold
  }

  if (h->kind == 0) {
    grow_tree(nullptr);
    if (trace) tr[7] = now_us();
    h->forest.clear();
  } else {  // random forest: T trees on bootstrap resamples of the global table (R19)
    const uint64_t lo = shard_lo();
    h->wcnt.ensure(16);
    h->wplane.ensure((size_t)std::max<int64_t>(n, 1) + 64);
    std::vector<std::vector<adapt_node_t>> forest;
    std::vector<int64_t> stats;
    for (int t = 0; t < h->T; t++) {
      {
        Phase ph("bootstrap", s, 0);
        launch_bootstrap(h->seed, t, n_total, lo, n, h->wplane.as<uint8_t>(),
                         h->wcnt.as<unsigned long long>(), s);
      }
      uint64_t sums[2];
      CUDA_CHECK(cudaMemcpyAsync(sums, h->wcnt.p, 16, cudaMemcpyDeviceToHost, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
      if (sums[0] != sums[1])
        throw Error(ADAPT_E_INVALID_ARG, "bootstrap multiplicity above 255 (u8 weights)");
      grow_tree(h->wplane.as<uint8_t>());
      forest.push_back(h->tree);
      stats.insert(stats.end(), h->stats.begin(), h->stats.end());
    }
    h->forest.swap(forest);
    h->stats.swap(stats);
    h->tree = h->forest[0];
  }
  h->trained_n = n;
  h->trained = true;
  upload_tree(h, s);
  if (h->kind == 1) upload_forest(h, s);
  if (trace && h->kind == 0) fprintf(stderr, "[adapt] finalize: last level's decide -> upload_tree done %.0f us\n", now_us() - tr[7]);
}

int walk_tree(const std::vector<adapt_node_t> &tr, const float *x) {
  int k = 0;
  while (tr[k].feature >= 0) {
    const double v = (double)x[tr[k].feature];
    k = v <= tr[k].threshold ? tr[k].left : tr[k].right;  // NaN -> right (R8)
  }
  return tr[k].label;
}

// Table-1 get_policy on the host (one vector): the tree, or the forest's
// majority vote with ties -> lowest variant (R20)
int select_host_walk(adapt_region *h, const float *x) {
  if (h->forest.empty()) return walk_tree(h->tree, x);
  std::vector<int> votes(h->V, 0);
  for (const auto &tr : h->forest) votes[walk_tree(tr, x)]++;
  return (int)(std::max_element(votes.begin(), votes.end()) - votes.begin());  // first max
}

void select_device(adapt_region *h, const float *X, int64_t m, int32_t *out, cudaStream_t s) {
  if (h->forest.empty()) {
    SelTree t{h->d_tree.as<DNode>(), (int)h->tree.size(), h->d_blocks.as<uint4>(),
              h->heap_td ? h->d_heap.as<uint2>() : nullptr, h->heap_td ? h->d_exits.as<int32_t>() : nullptr,
              h->heap_td ? h->d_blocks2.as<uint4>() : nullptr, h->heap_td};
    launch_select(t, X, m, h->F, out, s);
  } else {
    launch_select_forest(h->d_forest.as<DNode>(), h->forest_nodes, h->d_roots.as<int32_t>(),
                         (int)h->forest.size(), X, m, h->F, out, s);
  }
  // the device tree may be replaced (retrain, set_tree, K-fold restore) on
  // another stream: upload_tree waits for this event before overwriting it
  if (!h->sel_evt) CUDA_CHECK(cudaEventCreateWithFlags(&h->sel_evt, cudaEventDisableTiming));
  CUDA_CHECK(cudaEventRecord(h->sel_evt, s));
}

// distinct (features, variant) pairs of the host records, kept
// incrementally by adapt_record: the shim asks after every end()
void add_pair(adapt_region *h, const float *x, int variant) {
  std::string key((size_t)h->F * 4 + 4, '\0');
  for (int f = 0; f < h->F; f++) {
    const float c = canon(x[f]);
    memcpy(&key[(size_t)f * 4], &c, 4);
  }
  memcpy(&key[(size_t)h->F * 4], &variant, 4);
  h->pair_set.insert(std::move(key));
}

int64_t distinct_pairs(adapt_region *h) { return (int64_t)h->pair_set.size(); }

template <class Fn>
int guarded(Fn &&fn) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  try {
    fn();
    return ADAPT_OK;
  } catch (const Error &e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception &e) {
    g_last_error = e.what();
    return ADAPT_E_CUDA;
  }
}

}  // namespace
}  // namespace adapt

using namespace adapt;

extern "C" {

const char *adapt_last_error(void) { return g_last_error.c_str(); }

const char *adapt_version(void) {
#ifndef ADAPT_GIT
#define ADAPT_GIT "dev"
#endif
  return "adapt sm_100a " ADAPT_GIT;
}

int adapt_nccl_unique_id(void *out128) {
  return guarded([&] {
    if (!out128) throw Error(ADAPT_E_INVALID_ARG, "null out");
    g_nccl.load();
    ncclUniqueId id;
    g_nccl.check(g_nccl.GetUniqueId(&id), "ncclGetUniqueId");
    memcpy(out128, &id, sizeof(id));
  });
}

int adapt_init(int device, int rank, int world, const void *nccl_unique_id) {
  return guarded([&] {
    if (world < 1 || rank < 0 || rank >= world || device < 0)
      throw Error(ADAPT_E_INVALID_ARG, "bad device/rank/world");
    if (g_ctx.inited) {
      if (g_ctx.device == device && g_ctx.rank == rank && g_ctx.world == world) return;
      if (g_ctx.world == 1 && world == 1 && g_regions.empty()) {
        g_ctx.inited = false;
      } else {
        throw Error(ADAPT_E_USAGE, "already initialised with a different device/rank/world");
      }
    }
    int n = 0;
    CUDA_CHECK(cudaGetDeviceCount(&n));
    if (device >= n) throw Error(ADAPT_E_INVALID_ARG, "no such device");
    CUDA_CHECK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) throw Error(ADAPT_E_CUDA, "libadapt is built for sm_100a (B200) only");
    if (world > 1) {
      if (!nccl_unique_id) throw Error(ADAPT_E_INVALID_ARG, "world > 1 needs an ncclUniqueId");
      g_nccl.load();
      ncclUniqueId id;
      memcpy(&id, nccl_unique_id, sizeof(id));
      g_nccl.check(g_nccl.CommInitRank(&g_ctx.comm, world, id, rank), "ncclCommInitRank");
    } else if (getenv("ADAPT_NCCL_SELF")) {  // testing: a 1-rank NCCL communicator
      g_nccl.load();
      ncclUniqueId id;
      g_nccl.check(g_nccl.GetUniqueId(&id), "ncclGetUniqueId");
      g_nccl.check(g_nccl.CommInitRank(&g_ctx.comm, 1, id, 0), "ncclCommInitRank");
    }
    g_ctx.device = device;
    g_ctx.rank = rank;
    g_ctx.world = world;
    g_ctx.inited = true;
  });
}

int adapt_init_host_comm(int device, int rank, int world, const adapt_host_comm_t *comm) {
  return guarded([&] {
    if (world < 1 || rank < 0 || rank >= world || device < 0)
      throw Error(ADAPT_E_INVALID_ARG, "bad device/rank/world");
    if (!comm || !comm->all_gather || !comm->all_reduce_u64)
      throw Error(ADAPT_E_INVALID_ARG, "null host collective hooks");
    if (g_ctx.inited) {
      if (g_ctx.world == 1 && g_regions.empty()) g_ctx.inited = false;
      else throw Error(ADAPT_E_USAGE, "already initialised; call adapt_finalize first");
    }
    int n = 0;
    CUDA_CHECK(cudaGetDeviceCount(&n));
    if (device >= n) throw Error(ADAPT_E_INVALID_ARG, "no such device");
    CUDA_CHECK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) throw Error(ADAPT_E_CUDA, "libadapt is built for sm_100a (B200) only");
    g_ctx.device = device;
    g_ctx.rank = rank;
    g_ctx.world = world;
    g_ctx.host_comm = true;
    g_ctx.hooks = *comm;
    g_ctx.inited = true;
  });
}

int adapt_finalize(void) {
  return guarded([&] {
    g_regions.clear();
    g_multi.reset();
    if (g_ctx.comm) g_nccl.CommDestroy(g_ctx.comm);
    g_ctx = Ctx{};
  });
}

int adapt_region_create(const char *id, int num_features, int num_variants,
                        const char *model_params, int min_train_data, adapt_region_t **out) {
  return guarded([&] {
    if (!id || !*id || !out) throw Error(ADAPT_E_INVALID_ARG, "null id or out");
    *out = nullptr;
    if (num_features < 1 || num_features > kMaxF)
      throw Error(ADAPT_E_INVALID_ARG, "num_features must be in [1,64]");
    if (num_variants < 1 || num_variants > kMaxC)
      throw Error(ADAPT_E_INVALID_ARG, "num_variants must be in [1,255]");
    int depth = 2;
    int kind = 0, trees = 1;
    uint64_t seed = 0;
    bool quantile = false;
    parse_params(model_params, &depth, &kind, &trees, &seed, &quantile);
    const int mtd = min_train_data > 0 ? min_train_data : num_variants;
    auto it = g_regions.find(id);
    if (it != g_regions.end()) {
      adapt_region *h = it->second.get();
      if (h->F != num_features || h->V != num_variants || h->D != depth || h->min_train != mtd ||
          h->kind != kind || h->T != trees || h->seed != seed || h->quantile != quantile)
        throw Error(ADAPT_E_SPEC_MISMATCH, std::string("region '") + id + "' exists with another spec");
      *out = h;
      return;
    }
    auto h = std::make_unique<adapt_region>();
    h->id = id;
    h->F = num_features;
    h->V = num_variants;
    h->D = depth;
    h->kind = kind;
    h->T = trees;
    h->seed = seed;
    h->quantile = quantile;
    h->min_train = mtd;
    *out = h.get();
    g_regions.emplace(id, std::move(h));
  });
}

int adapt_region_destroy(adapt_region_t *h) {
  return guarded([&] {
    checked(h);
    g_regions.erase(h->id);
  });
}

int adapt_region_info(adapt_region_t *h, int *F, int *V, int *D, int *mtd, int64_t *rows,
                      int *trained) {
  return guarded([&] {
    checked(h);
    if (F) *F = h->F;
    if (V) *V = h->V;
    if (D) *D = h->D;
    if (mtd) *mtd = h->min_train;
    if (rows) *rows = h->have_table ? h->n : (int64_t)h->rvar.size() + h->rec_n;
    if (trained) *trained = h->trained;
  });
}

int adapt_record(adapt_region_t *h, const float *features, int variant, uint64_t elapsed_ns) {
  return guarded([&] {
    checked(h);
    if (!features) throw Error(ADAPT_E_INVALID_ARG, "null features");
    if (variant < 0 || variant >= h->V) throw Error(ADAPT_E_BAD_VALUE, "variant out of range");
    for (int f = 0; f < h->F; f++)
      if (!std::isfinite(features[f])) throw Error(ADAPT_E_BAD_VALUE, "non-finite feature");
    h->rfeat.insert(h->rfeat.end(), features, features + h->F);
    h->rvar.push_back(variant);
    h->rns.push_back(elapsed_ns);
    add_pair(h, features, variant);
  });
}

int adapt_record_batch(adapt_region_t *h, const float *features, const int32_t *variants,
                       const uint64_t *elapsed_ns, int64_t m, int on_device, void *stream) {
  return guarded([&] {
    checked(h);
    ensure_init();
    if (m < 0 || (m > 0 && (!features || !variants || !elapsed_ns)))
      throw Error(ADAPT_E_INVALID_ARG, "bad record batch");
    if (m == 0) return;
    cudaStream_t s = (cudaStream_t)stream;
    if (h->rec_n + m + (int64_t)h->rvar.size() >= (int64_t)0xFFFFFFFFll)
      throw Error(ADAPT_E_INVALID_ARG, "more than 2^32-1 records");
    reserve_records(h, h->rec_n + m, s);
    const cudaMemcpyKind k = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CUDA_CHECK(cudaMemcpyAsync(h->rec_feat.as<float>() + h->rec_n * h->F, features,
                               (size_t)m * h->F * 4, k, s));
    CUDA_CHECK(cudaMemcpyAsync(h->rec_var.as<int32_t>() + h->rec_n, variants, (size_t)m * 4, k, s));
    CUDA_CHECK(cudaMemcpyAsync(h->rec_ns.as<uint64_t>() + h->rec_n, elapsed_ns, (size_t)m * 8, k, s));
    CUDA_CHECK(cudaStreamSynchronize(s));  // host sources may be reused after return
    h->rec_n += m;
  });
}

int adapt_get_wide_table(adapt_region_t *h, float *features, float *times, int64_t cap,
                         int64_t *n) {
  return guarded([&] {
    checked(h);
    if (!n) throw Error(ADAPT_E_INVALID_ARG, "null n");
    if (!h->trained) throw Error(ADAPT_E_NOT_TRAINED, "not trained");
    if (!h->aggregated) throw Error(ADAPT_E_USAGE, "the last train used a wide table, not records");
    *n = h->trained_n;
    if (cap < h->trained_n) return;  // size query
    if (h->trained_n && (!features || !times)) throw Error(ADAPT_E_INVALID_ARG, "null output");
    if (h->trained_n) {
      CUDA_CHECK(cudaMemcpy(features, h->agg_feat.p, (size_t)h->trained_n * h->F * 4,
                            cudaMemcpyDeviceToHost));
      CUDA_CHECK(cudaMemcpy(times, h->agg_times.p, (size_t)h->trained_n * h->V * 4,
                            cudaMemcpyDeviceToHost));
    }
  });
}

int adapt_record_table(adapt_region_t *h, const float *features, const float *times, int64_t n,
                       int on_device, void *stream) {
  return guarded([&] {
    checked(h);
    ensure_init();
    if (n < 0 || (n > 0 && (!features || !times))) throw Error(ADAPT_E_INVALID_ARG, "bad table");
    cudaStream_t s = (cudaStream_t)stream;
    h->n = n;
    h->have_table = true;
    if (on_device) {
      h->d_feat = features;
      h->d_times = times;
    } else {
      h->own_feat.ensure((size_t)n * h->F * 4 + 16);
      h->own_times.ensure((size_t)n * h->V * 4 + 16);
      Phase ph("h2d", s, (double)n * (h->F + h->V) * 4);
      if (n) {
        CUDA_CHECK(cudaMemcpyAsync(h->own_feat.p, features, (size_t)n * h->F * 4, cudaMemcpyHostToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(h->own_times.p, times, (size_t)n * h->V * 4, cudaMemcpyHostToDevice, s));
      }
      h->d_feat = h->own_feat.as<float>();
      h->d_times = h->own_times.as<float>();
    }
    if (!on_device) CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

int adapt_distinct_pairs(adapt_region_t *h, int64_t *count) {
  return guarded([&] {
    checked(h);
    if (!count) throw Error(ADAPT_E_INVALID_ARG, "null count");
    if (h->rec_n == 0) {
      *count = distinct_pairs(h);  // host records only: the shim's per-call bookkeeping
    } else {  // with device-batch records: measured cells of the GPU aggregation
      ensure_init();
      h->hsmall.ensure(1 << 16);
      gpu_aggregate(h, nullptr, count);
      h->aggregated = false;  // agg_feat/times now hold this count's aggregation
    }
  });
}

int adapt_train(adapt_region_t *h, void *stream) {
  return guarded([&] {
    checked(h);
    ensure_init();
    train_region(h, (cudaStream_t)stream);
    if (h->have_table && h->d_feat != h->own_feat.as<float>()) {
      h->d_feat = nullptr;  // borrowed pointers are released when train returns
      h->d_times = nullptr;
      h->have_table = false;
    }
  });
}

namespace adapt {
namespace {
// adapt_train_many for k >= 2 decision-tree regions with equal (F, V, D) and
// recorded wide tables: ONE ingest over the union of their tables and ONE
// level loop whose frontier starts with k roots (each region's rows).  The
// union's value tables only re-index the bins: thresholds are node-local
// midpoints of the values present (R7), so every region's tree is the one
// adapt_train would build.  Returns false (nothing changed) when the fused
// path does not apply; the caller then trains the regions one by one.

bool train_many_fused(adapt_region *const *hs, int k, cudaStream_t s) {
  if (k < 2) return false;
  const adapt_region *h0 = hs[0];
  for (int r = 0; r < k; r++) {
    const adapt_region *h = hs[r];
    if (h->kind != 0 || h->quantile || !h->have_table || h->F != h0->F || h->V != h0->V || h->D != h0->D)
      return false;
    for (int q = 0; q < r; q++)
      if (hs[q] == h) return false;
  }
  if (!g_multi) g_multi = std::make_unique<adapt_region>();
  adapt_region *u = g_multi.get();
  u->id = "__adapt_train_many";
  u->F = h0->F;
  u->V = h0->V;
  u->D = h0->D;
  u->kind = 0;
  std::vector<int64_t> mn(k);
  int64_t n = 0;
  for (int r = 0; r < k; r++) n += (mn[r] = hs[r]->n);
  const int F = u->F, V = u->V;
  u->own_feat.ensure((size_t)std::max<int64_t>(n, 1) * F * 4 + 16);
  u->own_times.ensure((size_t)std::max<int64_t>(n, 1) * V * 4 + 16);
  int64_t off = 0;
  for (int r = 0; r < k; r++) {
    if (mn[r]) {
      CUDA_CHECK(cudaMemcpyAsync(u->own_feat.as<float>() + off * F, hs[r]->d_feat, (size_t)mn[r] * F * 4,
                                 cudaMemcpyDeviceToDevice, s));
      CUDA_CHECK(cudaMemcpyAsync(u->own_times.as<float>() + off * V, hs[r]->d_times, (size_t)mn[r] * V * 4,
                                 cudaMemcpyDeviceToDevice, s));
    }
    off += mn[r];
  }
  u->n = n;
  u->have_table = true;
  u->d_feat = u->own_feat.as<float>();
  u->d_times = u->own_times.as<float>();
  u->multi_n = &mn;
  try {
    train_region(u, s);
  } catch (const Error &e) {
    u->multi_n = nullptr;
    if (e.code == ADAPT_E_TOO_MANY_DISTINCT || e.code == ADAPT_E_INSUFFICIENT_DATA)
      return false;  // the union overflows 256 values / an empty region: one by one
    throw;
  }
  u->multi_n = nullptr;
  // every region: its tree, and its slice of the union's labels and bins
  off = 0;
  for (int r = 0; r < k; r++) {
    adapt_region *h = hs[r];
    const int64_t nr = mn[r];
    h->BS = u->BS;
    h->pstride = bins_plane_stride(nr, u->BS);
    h->bins.ensure(bins_bytes(nr, u->BS));
    h->labels.ensure((size_t)std::max<int64_t>(nr, 1) + 64);
    const int planes = u->BS < 4 ? 1 : u->BS / 4, wb = u->BS < 4 ? u->BS : 4;
    if (nr) {
      for (int p = 0; p < planes; p++)
        CUDA_CHECK(cudaMemcpyAsync(h->bins.as<uint8_t>() + p * h->pstride,
                                   u->bins.as<uint8_t>() + p * u->pstride + off * wb, (size_t)nr * wb,
                                   cudaMemcpyDeviceToDevice, s));
      CUDA_CHECK(cudaMemcpyAsync(h->labels.p, u->labels.as<uint8_t>() + off, (size_t)nr,
                                 cudaMemcpyDeviceToDevice, s));
    }
    h->val = u->val;
    h->nval = u->nval;
    h->qmask = 0;
    h->tree = std::move(u->multi_trees[r]);
    h->forest.clear();
    h->stats = u->stats;
    h->aggregated = false;
    h->trained_n = nr;
    h->trained = true;
    upload_tree(h, s);
    off += nr;
  }
  return true;
}
}  // namespace
}  // namespace adapt

int adapt_train_many(adapt_region_t *const *hs, int k, void *stream) {
  if (!hs || k < 0) return guarded([&] { throw Error(ADAPT_E_INVALID_ARG, "bad region list"); });
  bool fused = false;
  const int rc = guarded([&] {
    for (int i = 0; i < k; i++) checked(hs[i]);
    ensure_init();
    fused = train_many_fused(hs, k, (cudaStream_t)stream);
    if (fused)
      for (int i = 0; i < k; i++) {
        adapt_region *h = hs[i];
        if (h->have_table && h->d_feat != h->own_feat.as<float>()) {
          h->d_feat = nullptr;  // borrowed pointers are released when train returns
          h->d_times = nullptr;
          h->have_table = false;
        }
      }
  });
  if (rc || fused) return rc;
  for (int i = 0; i < k; i++) {
    int rc = adapt_train(hs[i], stream);
    if (rc) return rc;
  }
  return ADAPT_OK;
}

int adapt_select(adapt_region_t *h, const float *features, int32_t *variant) {
  return guarded([&] {
    checked(h);
    if (!features || !variant) throw Error(ADAPT_E_INVALID_ARG, "null argument");
    if (!h->trained) throw Error(ADAPT_E_NOT_TRAINED, "region not trained");
    *variant = select_host_walk(h, features);
  });
}

int adapt_select_batch(adapt_region_t *h, const float *d_X, int64_t m, int32_t *d_out,
                       void *stream) {
  return guarded([&] {
    checked(h);
    ensure_init();
    if (m < 0 || (m > 0 && (!d_X || !d_out))) throw Error(ADAPT_E_INVALID_ARG, "bad batch");
    if (!h->trained) throw Error(ADAPT_E_NOT_TRAINED, "region not trained");
    cudaStream_t s = (cudaStream_t)stream;
    Phase ph("select", s, (double)m * (4.0 * h->F + 4));
    select_device(h, d_X, m, d_out, s);
  });
}

int adapt_select_table(adapt_region_t *h, int32_t *out, int out_on_device, void *stream) {
  return guarded([&] {
    checked(h);
    ensure_init();
    if (!out && h->n > 0) throw Error(ADAPT_E_INVALID_ARG, "null out");
    if (!h->trained) throw Error(ADAPT_E_NOT_TRAINED, "region not trained");
    if (!h->have_table || h->d_feat != h->own_feat.as<float>())
      throw Error(ADAPT_E_USAGE, "no host-recorded wide table on the device");
    cudaStream_t s = (cudaStream_t)stream;
    if (h->n == 0) return;
    if (out_on_device) {
      Phase ph("select", s, (double)h->n * (4.0 * h->F + 4));
      select_device(h, h->d_feat, h->n, out, s);
      return;
    }
    h->oa.ensure((size_t)h->n * 4);
    {
      Phase ph("select", s, (double)h->n * (4.0 * h->F + 4));
      select_device(h, h->d_feat, h->n, h->oa.as<int32_t>(), s);
    }
    CUDA_CHECK(cudaMemcpyAsync(out, h->oa.p, (size_t)h->n * 4, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

int adapt_select_batch_host(adapt_region_t *h, const float *X, int64_t m, int32_t *out,
                            void *stream) {
  return guarded([&] {
    checked(h);
    ensure_init();
    if (m < 0 || (m > 0 && (!X || !out))) throw Error(ADAPT_E_INVALID_ARG, "bad batch");
    if (!h->trained) throw Error(ADAPT_E_NOT_TRAINED, "region not trained");
    cudaStream_t s = (cudaStream_t)stream;
    const int F = h->F;
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(m, (256ll << 20) / (4 * F)));
    h->xa.ensure((size_t)chunk * F * 4);
    h->xb.ensure((size_t)chunk * F * 4);
    h->oa.ensure((size_t)chunk * 4);
    h->ob.ensure((size_t)chunk * 4);
    cudaStream_t st[2];
    cudaEvent_t ready;
    CUDA_CHECK(cudaStreamCreateWithFlags(&st[0], cudaStreamNonBlocking));
    CUDA_CHECK(cudaStreamCreateWithFlags(&st[1], cudaStreamNonBlocking));
    CUDA_CHECK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    CUDA_CHECK(cudaEventRecord(ready, s));  // order after prior work on the caller's stream
    CUDA_CHECK(cudaStreamWaitEvent(st[0], ready, 0));
    CUDA_CHECK(cudaStreamWaitEvent(st[1], ready, 0));
    for (int64_t c = 0, i = 0; c < m; c += chunk, i++) {
      const int64_t k = std::min(chunk, m - c);
      cudaStream_t q = st[i & 1];
      float *dx = (i & 1) ? h->xb.as<float>() : h->xa.as<float>();
      int32_t *dout = (i & 1) ? h->ob.as<int32_t>() : h->oa.as<int32_t>();
      CUDA_CHECK(cudaMemcpyAsync(dx, X + c * F, (size_t)k * F * 4, cudaMemcpyHostToDevice, q));
      {
        Phase ph("select", q, (double)k * (4.0 * F + 4));
        select_device(h, dx, k, dout, q);
      }
      CUDA_CHECK(cudaMemcpyAsync(out + c, dout, (size_t)k * 4, cudaMemcpyDeviceToHost, q));
    }
    CUDA_CHECK(cudaStreamSynchronize(st[0]));
    CUDA_CHECK(cudaStreamSynchronize(st[1]));
    cudaStreamDestroy(st[0]);
    cudaStreamDestroy(st[1]);
    cudaEventDestroy(ready);
  });
}

int adapt_get_tree(adapt_region_t *h, adapt_node_t *out, int32_t cap, int32_t *n_nodes) {
  return guarded([&] {
    checked(h);
    if (!n_nodes) throw Error(ADAPT_E_INVALID_ARG, "null n_nodes");
    if (!h->trained) throw Error(ADAPT_E_NOT_TRAINED, "region not trained");
    *n_nodes = (int32_t)h->tree.size();
    if (!out || cap < (int32_t)h->tree.size()) throw Error(ADAPT_E_INVALID_ARG, "capacity too small");
    memcpy(out, h->tree.data(), h->tree.size() * sizeof(adapt_node_t));
  });
}

int adapt_forest_size(adapt_region_t *h, int32_t *trees) {
  return guarded([&] {
    checked(h);
    if (!trees) throw Error(ADAPT_E_INVALID_ARG, "null trees");
    if (!h->trained) throw Error(ADAPT_E_NOT_TRAINED, "region not trained");
    *trees = h->forest.empty() ? 1 : (int32_t)h->forest.size();
  });
}

int adapt_kfold(adapt_region_t *h, int K, int train_groups, int shuffles, uint64_t seed,
                adapt_kfold_result_t *out, void *stream) {
  return guarded([&] {
    checked(h);
    ensure_init();
    if (K < 2 || K > kKfoldMaxK || train_groups < 1 || train_groups >= K || shuffles < 1 || !out)
      throw Error(ADAPT_E_INVALID_ARG, "bad K-fold spec");
    if (h->kind != 0) throw Error(ADAPT_E_USAGE, "adapt_kfold needs a dtree region");
    cudaStream_t s = (cudaStream_t)stream;
    // the region's own model survives the harness
    std::vector<adapt_node_t> prev_tree = h->tree;
    std::vector<int64_t> prev_stats = h->stats;
    const bool prev_trained = h->trained;
    const int64_t prev_n = h->trained_n;
    const adapt_region::KfoldSpec spec{K, train_groups, shuffles, seed, out};
    auto restore = [&]() {
      h->kfold = nullptr;
      h->tree.swap(prev_tree);
      h->stats.swap(prev_stats);
      h->trained = prev_trained;
      h->trained_n = prev_n;
      if (h->have_table && h->d_feat != h->own_feat.as<float>()) {
        h->d_feat = nullptr;  // borrowed pointers are released when the call returns
        h->d_times = nullptr;
        h->have_table = false;
      }
    };
    h->kfold = &spec;
    try {
      train_region(h, s);
    } catch (...) {
      restore();
      throw;
    }
    restore();
    if (h->trained && !h->tree.empty()) upload_tree(h, s);
  });
}

int adapt_get_kfold_tree(adapt_region_t *h, int32_t model, adapt_node_t *out, int32_t cap,
                         int32_t *n_nodes) {
  return guarded([&] {
    checked(h);
    if (!n_nodes) throw Error(ADAPT_E_INVALID_ARG, "null n_nodes");
    if (model < 0 || model >= (int32_t)h->kfold_trees.size())
      throw Error(ADAPT_E_INVALID_ARG, "no such K-fold model");
    const auto &tr = h->kfold_trees[model];
    *n_nodes = (int32_t)tr.size();
    if (!out || cap < (int32_t)tr.size()) throw Error(ADAPT_E_INVALID_ARG, "capacity too small");
    memcpy(out, tr.data(), tr.size() * sizeof(adapt_node_t));
  });
}

int adapt_get_forest_tree(adapt_region_t *h, int32_t t, adapt_node_t *out, int32_t cap,
                          int32_t *n_nodes) {
  return guarded([&] {
    checked(h);
    if (!n_nodes) throw Error(ADAPT_E_INVALID_ARG, "null n_nodes");
    if (!h->trained) throw Error(ADAPT_E_NOT_TRAINED, "region not trained");
    const int T = h->forest.empty() ? 1 : (int)h->forest.size();
    if (t < 0 || t >= T) throw Error(ADAPT_E_INVALID_ARG, "tree index out of range");
    const auto &tr = h->forest.empty() ? h->tree : h->forest[t];
    *n_nodes = (int32_t)tr.size();
    if (!out || cap < (int32_t)tr.size()) throw Error(ADAPT_E_INVALID_ARG, "capacity too small");
    memcpy(out, tr.data(), tr.size() * sizeof(adapt_node_t));
  });
}

int adapt_set_tree(adapt_region_t *h, const adapt_node_t *nodes, int32_t n_nodes) {
  return guarded([&] {
    checked(h);
    ensure_init();
    if (!nodes || n_nodes < 1) throw Error(ADAPT_E_INVALID_ARG, "empty tree");
    if (n_nodes >= (1 << 25)) throw Error(ADAPT_E_INVALID_ARG, "tree too large");
    std::vector<uint8_t> has_parent(n_nodes, 0);  // a tree: one parent per node
    for (int32_t k = 0; k < n_nodes; k++) {
      const adapt_node_t &nd = nodes[k];
      if (nd.feature >= 0 && nd.left > k && nd.right == nd.left + 1 && nd.right < n_nodes) {
        if (has_parent[nd.left] || has_parent[nd.right])
          throw Error(ADAPT_E_INVALID_ARG, "node with two parents at " + std::to_string(nd.left));
        has_parent[nd.left] = has_parent[nd.right] = 1;
      }
      if (nd.feature >= 0) {
        if (nd.feature >= h->F || nd.left <= k || nd.right != nd.left + 1 || nd.right >= n_nodes ||
            !std::isfinite(nd.threshold))
          throw Error(ADAPT_E_INVALID_ARG, "bad internal node " + std::to_string(k));
      } else if (nd.label < 0 || nd.label >= h->V) {
        throw Error(ADAPT_E_INVALID_ARG, "bad leaf label at node " + std::to_string(k));
      }
    }
    if (h->kind != 0) throw Error(ADAPT_E_USAGE, "adapt_set_tree on a forest region");
    h->tree.assign(nodes, nodes + n_nodes);
    h->forest.clear();
    h->trained = true;
    upload_tree(h, 0);
  });
}

int adapt_get_labels(adapt_region_t *h, uint8_t *out, int64_t n) {
  return guarded([&] {
    checked(h);
    if (!h->trained || !h->BS) throw Error(ADAPT_E_NOT_TRAINED, "region not trained");
    if (!out || n != h->trained_n) throw Error(ADAPT_E_INVALID_ARG, "n must equal the trained row count");
    if (n) CUDA_CHECK(cudaMemcpy(out, h->labels.p, (size_t)n, cudaMemcpyDeviceToHost));
  });
}

int adapt_get_value_table(adapt_region_t *h, int f, float *vals, int *count) {
  return guarded([&] {
    checked(h);
    if (!h->trained || h->nval.empty()) throw Error(ADAPT_E_NOT_TRAINED, "region not trained");
    if (f < 0 || f >= h->F || !vals || !count) throw Error(ADAPT_E_INVALID_ARG, "bad argument");
    *count = h->nval[f];
    memcpy(vals, &h->val[(size_t)f * kMaxBins], (size_t)h->nval[f] * 4);
  });
}

int adapt_get_bins(adapt_region_t *h, uint8_t *out, int64_t n) {
  return guarded([&] {
    checked(h);
    if (!h->trained || !h->BS) throw Error(ADAPT_E_NOT_TRAINED, "region not trained");
    if (!out || n != h->trained_n) throw Error(ADAPT_E_INVALID_ARG, "n must equal the trained row count");
    DevBuf tmp;
    tmp.ensure((size_t)n * h->F + 16);
    launch_bins_out(h->bins.as<uint8_t>(), h->pstride, n, h->F, h->BS, tmp.as<uint8_t>(), 0);
    CUDA_CHECK(cudaMemcpy(out, tmp.p, (size_t)n * h->F, cudaMemcpyDeviceToHost));
  });
}

int adapt_profile_enable(int enable) {
  return guarded([&] { g_prof.on = enable != 0; });
}

int adapt_profile_reset(void) {
  return guarded([&] {
    g_prof.drain();
    for (auto &a : g_prof.acc) a = Prof::Acc{};
  });
}

int adapt_profile_get(adapt_phase_t *out, int cap, int *n) {
  return guarded([&] {
    if (!n) throw Error(ADAPT_E_INVALID_ARG, "null n");
    g_prof.drain();
    *n = (int)g_prof.names.size();
    for (int i = 0; i < *n && i < cap && out; i++) {
      memset(&out[i], 0, sizeof(adapt_phase_t));
      snprintf(out[i].name, sizeof(out[i].name), "%s", g_prof.names[i].c_str());
      out[i].launches = g_prof.acc[i].launches;
      out[i].ms = g_prof.acc[i].ms;
      out[i].bytes = g_prof.acc[i].bytes;
    }
  });
}

constexpr size_t kStatsPerLevel = 6;
int adapt_train_stats(adapt_region_t *h, int64_t *out, int cap, int *levels) {
  return guarded([&] {
    checked(h);
    if (!levels) throw Error(ADAPT_E_INVALID_ARG, "null levels");
    *levels = (int)(h->stats.size() / kStatsPerLevel);
    for (size_t i = 0; i < h->stats.size() && (int)i < cap && out; i++) out[i] = h->stats[i];
  });
}

// ---------------------------------------------------- Apollo Table-1 shim --
void *__adapt_region_create(const char *id, int num_features, int num_policies,
                            const char *model_type_params, int min_train_data) {
  adapt_region_t *h = nullptr;
  if (adapt_region_create(id, num_features, num_policies, model_type_params, min_train_data, &h))
    return nullptr;
  return h;
}

void __adapt_region_begin(void *r) {
  guarded([&] {
    adapt_region *h = checked(static_cast<adapt_region *>(r));
    if (h->active) throw Error(ADAPT_E_USAGE, "begin while active (S:141)");
    h->active = true;
    h->ctx_feat.clear();
    h->ctx_policy = -1;
    clock_gettime(CLOCK_MONOTONIC, &h->t0);
  });
}

void __adapt_region_set_feature(void *r, float v) {
  guarded([&] {
    adapt_region *h = checked(static_cast<adapt_region *>(r));
    if (!h->active) throw Error(ADAPT_E_USAGE, "set_feature without begin (S:151)");
    if ((int)h->ctx_feat.size() >= h->F) throw Error(ADAPT_E_ARITY, "too many features (S:151)");
    h->ctx_feat.push_back(v);
  });
}

int __adapt_region_get_policy(void *r) {
  int policy = 0;
  int rc = guarded([&] {
    adapt_region *h = checked(static_cast<adapt_region *>(r));
    if (!h->active) throw Error(ADAPT_E_USAGE, "get_policy without begin");
    if ((int)h->ctx_feat.size() != h->F) throw Error(ADAPT_E_ARITY, "features incomplete (S:161)");
    if (h->trained) {
      policy = select_host_walk(h, h->ctx_feat.data());
    } else {  // round-robin exploration
      policy = h->cursor;
      h->cursor = (h->cursor + 1) % h->V;
    }
    h->ctx_policy = policy;
  });
  return rc ? 0 : policy;
}

void __adapt_region_end(void *r) {
  guarded([&] {
    adapt_region *h = checked(static_cast<adapt_region *>(r));
    if (!h->active) throw Error(ADAPT_E_USAGE, "end without begin (S:171)");
    timespec t1;
    clock_gettime(CLOCK_MONOTONIC, &t1);
    h->active = false;
    if (h->ctx_policy < 0 || (int)h->ctx_feat.size() != h->F) return;  // nothing to record
    int64_t ns = (int64_t)(t1.tv_sec - h->t0.tv_sec) * 1000000000ll + (t1.tv_nsec - h->t0.tv_nsec);
    if (ns < 0) ns = 0;
    int rc = adapt_record(h, h->ctx_feat.data(), h->ctx_policy, (uint64_t)ns);
    if (rc) throw Error(rc, g_last_error);
    const int64_t pairs = distinct_pairs(h);
    // P:569 auto-train; after a failed attempt, retry only once new distinct
    // pairs have arrived (the same records would fail the same way)
    if (!h->trained && !h->have_table && pairs >= h->min_train && pairs > h->autotrain_failed_at) {
      rc = adapt_train(h, nullptr);
      if (rc) {
        h->autotrain_failed_at = pairs;
        throw Error(rc, g_last_error);
      }
    }
  });
}

void __adapt_region_train(void *r) {
  guarded([&] {
    adapt_region *h = checked(static_cast<adapt_region *>(r));
    if (h->rvar.empty() && h->rec_n == 0 && !h->have_table)
      throw Error(ADAPT_E_INSUFFICIENT_DATA, "no records (S:181)");
    int rc = adapt_train(h, nullptr);
    if (rc) throw Error(rc, g_last_error);
  });
}

}  // extern "C"
