// dyna_kv.cu — host side of the C ABI declared in include/dyna_kv.h.
//
// Owns pool geometry and validation, peer mappings (P2P in-process, CUDA IPC
// across processes), the per-(sender, destination) signalling channels, the
// variant/engine choice, and the launch of the kernels in
// dyna_kv_kernels.cuh.  Paper mapping: PAPER.md §3.1 P:352 (instances
// exchange the required KV blocks) and §4.3 P:556 (chunk-granular push,
// placement steered on the receiver = the destination block table).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "dyna_kv.h"
#include "dyna_kv_kernels.cuh"

using namespace dynakv;

// ============================================================== errors
namespace {
thread_local std::string g_err;

dyna_status fail(dyna_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define CUDA_TRY(expr)                                                                         \
  do {                                                                                         \
    cudaError_t e_ = (expr);                                                                   \
    if (e_ != cudaSuccess) {                                                                   \
      return fail(DYNA_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                                   \
    }                                                                                          \
  } while (0)

struct DeviceGuard {  // restores the caller's current device
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

std::atomic<uint64_t> g_launches{0};
std::mutex g_mu;

// Process-wide deferred error word in mapped pinned host memory: kernels
// atomicOr ERR_* bits into it; dyna_kv_wait / dyna_kv_poll_error read it.
unsigned int* g_err_word = nullptr;

unsigned int* err_word() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_err_word) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, 64, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) return nullptr;
    std::memset(p, 0, 64);
    g_err_word = static_cast<unsigned int*>(p);
  }
  return g_err_word;
}

dyna_status take_device_error() {
  unsigned int* w = err_word();
  if (!w) return DYNA_OK;
  const unsigned int bits = __atomic_exchange_n(w, 0u, __ATOMIC_ACQ_REL);
  if (bits & ERR_BAD_BLOCK) return fail(DYNA_ERANGE, "device-side check: block id outside [0, num_blocks)");
  if (bits & ERR_TIMEOUT) return fail(DYNA_ETIMEDOUT, "device-side chunk wait timed out");
  return DYNA_OK;
}

struct DevInfo {
  int sms = 0;
  cudaStream_t aux = nullptr;  // library stream for destination-side kernels (staged, cross-device)
  unsigned long long* sched = nullptr;  // [kSchedSlots][2] dynamic-scheduling counters, zero at rest
  std::atomic<uint32_t> sched_seq{0};
};
std::map<int, DevInfo> g_dev;

constexpr int kVecU = 8;
constexpr int kVecThreads = 256;
constexpr int kVecPiece = 8192;
constexpr int kBulkPiece = 32768;
constexpr int kBulkStages = 6;
constexpr int64_t kStageSlotBytes = 64ll << 20;  // staged variant: bytes per staging slot
constexpr uint32_t kSchedSlots = 1u << 15;       // dynamic-scheduling counter slots per device

// CUDA loads kernels lazily by default, and loading one synchronises the
// context.  A producer-coupled migration is resident and waiting while the
// producer marks chunks; a first-ever launch of any kernel during that window
// would deadlock against it.  So every kernel of this library is loaded when a
// device is first used.
void preload_kernels() {
  cudaFuncAttributes a{};
  const void* ks[] = {
      (const void*)k_mark_ready, (const void*)k_wait_flag, (const void*)k_fill, (const void*)k_release_sys,
      (const void*)k_copy_vec<4, false, SingleSource, false>, (const void*)k_copy_vec<4, true, SingleSource, false>,
      (const void*)k_copy_vec<8, false, SingleSource, false>, (const void*)k_copy_vec<8, true, SingleSource, false>,
      (const void*)k_copy_vec<16, false, SingleSource, false>, (const void*)k_copy_vec<16, true, SingleSource, false>,
      (const void*)k_copy_vec<8, false, SingleSource, true>, (const void*)k_copy_vec<8, true, SingleSource, true>,
      (const void*)k_copy_vec<4, false, BatchSource, false>, (const void*)k_copy_vec<8, false, BatchSource, false>,
      (const void*)k_copy_vec<16, false, BatchSource, false>,
      (const void*)k_copy_bulk<false, SingleSource>, (const void*)k_copy_bulk<true, SingleSource>,
      (const void*)k_copy_bulk<false, BatchSource>,
      (const void*)k_copy_bulk_ws<false, SingleSource>, (const void*)k_copy_bulk_ws<true, SingleSource>,
      (const void*)k_copy_bulk_ws<false, BatchSource>,
  };
  for (const void* k : ks) cudaFuncGetAttributes(&a, k);
}

DevInfo* dev_info(int dev) {
  std::lock_guard<std::mutex> lk(g_mu);
  DevInfo& d = g_dev[dev];
  if (d.sms == 0) {
    DeviceGuard g(dev);
    preload_kernels();
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    if (d.sms <= 0) d.sms = 1;
    if (cudaMalloc(&d.sched, sizeof(unsigned long long) * 2 * kSchedSlots) != cudaSuccess ||
        cudaMemset(d.sched, 0, sizeof(unsigned long long) * 2 * kSchedSlots) != cudaSuccess)
      d.sched = nullptr;  // dynamic scheduling unavailable: static round-robin
  }
  return &d;
}

}  // namespace

// ============================================================== objects
struct Channel {  // sender pool -> destination pool
  std::map<int, unsigned long long*> counters;  // per kernel device: [DYNA_MAX_CHUNKS], zero at rest
  char* sstage = nullptr;                      // staged variant: 2 slots on the source device
  char* dstage = nullptr;                      // staged variant: 2 slots on the destination device
  int64_t slot_bytes = 0;
  int sdev = -1, ddev = -1;
};

struct dyna_kv_pool {
  dyna_kv_pool_desc desc{};
  char* base = nullptr;
  int dev = 0;               // device on which `base` can be dereferenced
  bool imported = false;
  void* ipc_pool_map = nullptr;
  void* ipc_inbox_map = nullptr;
  unsigned long long* inbox = nullptr;  // [DYNA_MAX_INSTANCES][DYNA_MAX_CHUNKS]
  bool own_inbox = false;
  int64_t row = 0;
  std::mutex mu;
  std::map<const dyna_kv_pool*, Channel> channels;  // keyed by destination pool
};

struct dyna_kv_ready {
  int dev = 0;
  int32_t max_chunks = 0;
  unsigned long long timeout_ns = 10ull * 1000 * 1000 * 1000;  // per chunk wait
  unsigned long long* slots = nullptr;  // device, zero-initialised
  std::atomic<uint64_t> epoch{0};
};

struct dyna_kv_channel {
  int dev = 0;                 // device on which `base` can be dereferenced
  bool imported = false;
  char* base = nullptr;        // [slots][slot_bytes] | full[slots] | credit[slots]
  int32_t slots = 0;
  uint64_t slot_bytes = 0;
  int32_t sender = 0;
  dyna_kv_pool_desc desc{};    // the receiver pool's geometry
  dyna_kv_pool* dst = nullptr; // receiver side
  unsigned long long* full = nullptr;
  unsigned long long* credit = nullptr;
  uint64_t push_seq = 0, place_seq = 0;  // next sub-chunk number on each side
  unsigned long long* push_counters = nullptr;  // sender-device counters for the full-word release
  int push_counters_dev = -1;
  unsigned long long* place_counters = nullptr; // receiver-device counters for inbox chunk flags
  std::mutex mu;
};

struct dyna_kv_xfer {
  cudaEvent_t ev = nullptr;
  bool captured = false;  // enqueued during CUDA-graph capture: the work runs at replay
  int32_t variant = 0, engine = 0, piece = 0, stages = 0, unroll = 0, launches = 0;
  int dev = 0;
  bool empty = false;
  uint64_t epoch = 0;
  int32_t nchunks = 0;
  int32_t sender = 0;
};

namespace {

std::mutex g_ev_mu;
std::map<int, std::vector<cudaEvent_t>> g_ev_free;

cudaError_t get_event(int dev, cudaEvent_t* ev) {
  {
    std::lock_guard<std::mutex> lk(g_ev_mu);
    auto& v = g_ev_free[dev];
    if (!v.empty()) {
      *ev = v.back();
      v.pop_back();
      return cudaSuccess;
    }
  }
  return cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
}
void put_event(int dev, cudaEvent_t ev) {
  std::lock_guard<std::mutex> lk(g_ev_mu);
  g_ev_free[dev].push_back(ev);
}

constexpr size_t kInboxBytes = sizeof(unsigned long long) * DYNA_MAX_INSTANCES * DYNA_MAX_CHUNKS;

bool desc_valid(const dyna_kv_pool_desc* d) {
  return d && d->num_layers > 0 && d->num_kv_heads > 0 && d->head_dim > 0 && d->elem_bytes > 0 &&
         d->block_size > 0 && d->num_blocks > 0 && d->device >= 0 && d->instance >= 0 &&
         d->instance < DYNA_MAX_INSTANCES;
}

int64_t gcd64(int64_t a, int64_t b) {
  while (b) {
    int64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

// Build a launch plan for tokens [t0, t1) cut into chunks of c tokens.
// g: run grid in tokens (absolute token index; divides the paged block sizes).
Plan make_plan(const Side& s, const Side& d, int64_t row, int64_t t0, int64_t t1, int l0, int lm, int64_t c,
               int64_t g, int piece) {
  Plan p{};
  p.src = s;
  p.dst = d;
  p.row = row;
  p.t0 = t0;
  p.t1 = t1;
  p.l0 = l0;
  p.lm = lm;
  p.c = (int32_t)c;
  p.g = (int32_t)g;
  const bool aligned = (t0 % g == 0) && (c % g == 0);
  p.R = aligned ? (int32_t)(c / g) : (int32_t)((c - 1) / g + 2);
  const int64_t run_max = std::min(g, c) * row;
  p.piece = piece;
  p.P = (int32_t)((run_max + piece - 1) / piece);
  p.nchunks = (int32_t)((t1 - t0 + c - 1) / c);
  p.items_per_chunk = (int64_t)lm * 2 * p.R * p.P;
  p.n_items = p.items_per_chunk * p.nchunks;
  p.mig_t0 = t0;
  p.mig_t1 = t1;
  p.sig_c = (int32_t)c;
  p.err = g_err_word;
  return p;
}

// Programmatic dependent launch for the copy kernels (DYNA_KV_PDL=0 in the
// environment turns it off): consecutive migrations on a stream overlap launch
// + prologue with the previous kernel's drain.  Correct either way (see pdl_enter()).
bool pdl_enabled() {  // default on (measured: +5-16% on small calls, +0.3% on 512 MiB calls)
  static const bool on = [] {
    const char* e = std::getenv("DYNA_KV_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_kernel(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                          Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <int U, bool SIG, class Src>
int vec_occupancy() {
  static std::map<int, int> cache;  // per device
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_copy_vec<U, SIG, Src>, kVecThreads, 0);
  if (occ <= 0) occ = 1;
  cache[dev] = occ;
  return occ;
}

// Balanced persistent grid: the fewest workers (warps or CTAs) that still need
// only ceil(n / max_workers) rounds, so every worker gets the same number of
// items (+-1) and no partial last round leaves most of the chip idle.
int64_t balanced_workers(int64_t n_items, int64_t max_workers) {
  if (n_items <= max_workers) return n_items;
  const int64_t rounds = (n_items + max_workers - 1) / max_workers;
  return (n_items + rounds - 1) / rounds;
}

// Counter slot for one dynamically scheduled launch (nullptr: static round-robin).
unsigned long long* sched_slot(DevInfo* di, int schedule) {
  if (schedule != DYNA_SCHED_DYNAMIC || !di->sched) return nullptr;  // default: static
  const uint32_t k = di->sched_seq.fetch_add(1, std::memory_order_relaxed) % kSchedSlots;
  return di->sched + 2 * (size_t)k;
}

template <int U, bool SIG, class Src>
void launch_vec(const Src& src, int64_t n_items, int64_t max_grid, int sms, cudaStream_t st,
                unsigned long long* sched) {
  const int occ = vec_occupancy<U, SIG, Src>();
  constexpr int wpc = kVecThreads / 32;  // warps per CTA
  int64_t max_ctas = (int64_t)sms * occ;
  if (max_grid > 0) max_ctas = std::min<int64_t>(max_ctas, max_grid);
  const int64_t warps = balanced_workers(n_items, max_ctas * wpc);
  const int64_t grid = (warps + wpc - 1) / wpc;
  launch_kernel(k_copy_vec<U, SIG, Src, false>, (unsigned)grid, kVecThreads, 0, st, src, sched);
}

template <bool SIG, class Src>
dyna_status launch_bulk(const Src& src, int64_t n_items, int piece, int stages, int64_t max_grid, int sms,
                        cudaStream_t st, unsigned long long* sched, bool ws) {
  const size_t smem = (size_t)stages * piece;
  auto kern = ws ? k_copy_bulk_ws<SIG, Src> : k_copy_bulk<SIG, Src>;
  const int threads = ws ? 64 : 32;
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
  if (occ <= 0) return fail(DYNA_EINVAL, "BULK: %zu B of shared memory per CTA does not fit", smem);
  int64_t cap = (int64_t)sms * occ;
  if (max_grid > 0) cap = std::min<int64_t>(cap, max_grid);
  CUDA_TRY(launch_kernel(kern, (unsigned)balanced_workers(n_items, cap), threads, smem, st, src, stages, sched));
  return DYNA_OK;
}

// Launch one copy kernel over `src` (n_items items; piece bytes per item).
// engine: DYNA_ENGINE_VEC / BULK.  SIG: per-chunk signalling (single plan only).
template <class Src>
dyna_status launch_src(const Src& src, int64_t n_items, bool sig, int piece, int engine, int max_ctas, int stages,
                       int unroll, int dev, cudaStream_t st, int schedule) {
  if (n_items == 0) return DYNA_OK;
  if (n_items >= (int64_t(1) << 31))
    return fail(DYNA_ERANGE, "%lld work items in one launch (item math is 32-bit); use a larger piece or split the range",
                (long long)n_items);
  DevInfo* di = dev_info(dev);
  unsigned long long* sc = sched_slot(di, schedule);
  if (engine == DYNA_ENGINE_BULK || engine == DYNA_ENGINE_BULK_WS) {
    const bool ws = engine == DYNA_ENGINE_BULK_WS;
    dyna_status r = sig ? launch_bulk<true>(src, n_items, piece, stages, max_ctas, di->sms, st, sc, ws)
                        : launch_bulk<false>(src, n_items, piece, stages, max_ctas, di->sms, st, sc, ws);
    if (r) return r;
  } else if (unroll == 4) {
    sig ? launch_vec<4, true>(src, n_items, max_ctas, di->sms, st, sc)
        : launch_vec<4, false>(src, n_items, max_ctas, di->sms, st, sc);
  } else if (unroll == 16) {
    sig ? launch_vec<16, true>(src, n_items, max_ctas, di->sms, st, sc)
        : launch_vec<16, false>(src, n_items, max_ctas, di->sms, st, sc);
  } else {
    sig ? launch_vec<8, true>(src, n_items, max_ctas, di->sms, st, sc)
        : launch_vec<8, false>(src, n_items, max_ctas, di->sms, st, sc);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  CUDA_TRY(cudaGetLastError());
  return DYNA_OK;
}

// Producer-coupled launch: VEC engine, coherent loads, per-warp ready waits.
dyna_status launch_ready(const Plan& p, int max_ctas, int dev, cudaStream_t st, int schedule) {
  DevInfo* di = dev_info(dev);
  SingleSource src{p};
  const bool sig = p.counters != nullptr;
  int occ = 0;
  if (sig)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_copy_vec<8, true, SingleSource, true>, kVecThreads, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_copy_vec<8, false, SingleSource, true>, kVecThreads, 0);
  // never more than half the SMs' worth of CTAs: the producer must be able to run beside us
  int64_t cap = std::max(1, di->sms / 2);
  if (max_ctas > 0) cap = std::min<int64_t>(cap, max_ctas);
  cap = std::min<int64_t>(cap, (int64_t)di->sms * std::max(occ, 1));
  constexpr int wpc = kVecThreads / 32;
  const int64_t warps = balanced_workers(p.n_items, cap * wpc);
  const unsigned grid = (unsigned)((warps + wpc - 1) / wpc);
  unsigned long long* sc = sched_slot(di, schedule);
  if (sig)
    k_copy_vec<8, true, SingleSource, true><<<grid, kVecThreads, 0, st>>>(src, sc);
  else
    k_copy_vec<8, false, SingleSource, true><<<grid, kVecThreads, 0, st>>>(src, sc);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  CUDA_TRY(cudaGetLastError());
  return DYNA_OK;
}

dyna_status launch_copy(const Plan& p, int engine, int max_ctas, int stages, int unroll, int dev,
                        cudaStream_t st, int schedule) {
  SingleSource src{p};
  return launch_src(src, p.n_items, p.counters != nullptr, p.piece, engine, max_ctas, stages, unroll, dev, st,
                    schedule);
}

// ------------------------------------------------------------------ calibration (a6)
const dyna_kv_calib_entry kCalibDefault[] = {
#include "calib_default.inc"
    {0, -1, 0, 0, 0, 0, 0, 0}  // sentinel (never matches: peer = -1)
};
std::mutex g_calib_mu;
std::vector<dyna_kv_calib_entry> g_calib(std::begin(kCalibDefault), std::end(kCalibDefault) - 1);

// Best calibrated entry for (row bytes, locality, call tokens): entries for this
// exact row size first, generic (row_bytes == 0) ones only if none matches;
// within a class the smallest max_chunk_tokens that covers the call wins.
bool calib_lookup(int64_t row, int peer, int64_t c, dyna_kv_calib_entry* out) {
  std::lock_guard<std::mutex> lk(g_calib_mu);
  for (int pass = 0; pass < 2; ++pass) {
    const dyna_kv_calib_entry* best = nullptr;
    for (const auto& e : g_calib) {
      const bool row_ok = pass == 0 ? e.row_bytes == row : e.row_bytes == 0;
      if (!row_ok || e.peer != peer || c > e.max_chunk_tokens) continue;
      if (!best || e.max_chunk_tokens < best->max_chunk_tokens) best = &e;
    }
    if (best) {
      *out = *best;
      return true;
    }
  }
  return false;
}

Side paged(const dyna_kv_pool* pool, const int32_t* ids) {
  Side s{};
  s.base = pool->base;
  s.table = ids;
  s.nb = pool->desc.num_blocks;
  s.bs = pool->desc.block_size;
  s.linear = 0;
  return s;
}
Side linear(char* base) {
  Side s{};
  s.base = base;
  s.linear = 1;
  return s;
}

// Synchronous checks that need the host copies of the tables.
dyna_status check_host_tables(const dyna_block_table& src, const dyna_block_table& dst, int64_t t0, int64_t t1) {
  struct Span {
    int32_t id;
    int64_t lo, hi;  // slot range [lo, hi) inside block id
  };
  auto spans = [&](const dyna_block_table& t, std::vector<Span>& out) -> dyna_status {
    const int64_t bs = t.pool->desc.block_size, nb = t.pool->desc.num_blocks;
    for (int64_t j = t0 / bs; j <= (t1 - 1) / bs; ++j) {
      const int32_t id = t.host_block_ids[j];
      if (id < 0 || id >= nb) return fail(DYNA_ERANGE, "block_ids[%lld] = %d outside [0, %lld)", (long long)j, id, (long long)nb);
      const int64_t lo = std::max(t0, j * bs) - j * bs, hi = std::min(t1, (j + 1) * bs) - j * bs;
      out.push_back({id, lo, hi});
    }
    return DYNA_OK;
  };
  std::vector<Span> s, d;
  if (src.host_block_ids) {
    dyna_status r = spans(src, s);
    if (r) return r;
  }
  if (dst.host_block_ids) {
    dyna_status r = spans(dst, d);
    if (r) return r;
    auto by_id = [](const Span& a, const Span& b) { return a.id != b.id ? a.id < b.id : a.lo < b.lo; };
    std::vector<Span> ds = d;
    std::sort(ds.begin(), ds.end(), by_id);
    for (size_t i = 1; i < ds.size(); ++i)
      if (ds[i].id == ds[i - 1].id && ds[i].lo < ds[i - 1].hi)
        return fail(DYNA_EALIAS, "destination block %d is reached twice by the token range", ds[i].id);
    if (src.host_block_ids && src.pool->base == dst.pool->base) {
      std::vector<Span> ss = s;
      std::sort(ss.begin(), ss.end(), by_id);
      size_t i = 0;
      for (const Span& x : ds) {
        while (i < ss.size() && ss[i].id < x.id) ++i;
        for (size_t k = i; k < ss.size() && ss[k].id == x.id; ++k)
          if (ss[k].lo < x.hi && x.lo < ss[k].hi)
            return fail(DYNA_EALIAS, "same pool: destination rows of block %d overlap source rows", x.id);
      }
    }
  }
  return DYNA_OK;
}

dyna_status ensure_peer(int dev, int peer) {
  if (dev == peer) return DYNA_OK;
  int can = 0;
  if (cudaDeviceCanAccessPeer(&can, dev, peer) != cudaSuccess || !can)
    return fail(DYNA_EPEER, "device %d cannot access device %d (no P2P)", dev, peer);
  DeviceGuard g(dev);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return DYNA_OK;
  }
  if (e != cudaSuccess) return fail(DYNA_EPEER, "cudaDeviceEnablePeerAccess(%d->%d): %s", dev, peer, cudaGetErrorString(e));
  return DYNA_OK;
}

// Epochs are monotone per (sender instance, destination pool), whatever the
// variant or the source pool object, so a flag never moves backwards.
std::map<std::pair<int, const dyna_kv_pool*>, uint64_t> g_epochs;

uint64_t next_epoch(int sender, const dyna_kv_pool* dst) {
  std::lock_guard<std::mutex> lk(g_mu);
  return ++g_epochs[{sender, dst}];
}

// Self-resetting per-chunk byte counters of channel src -> dst on device kdev.
dyna_status channel_counters(dyna_kv_pool* src, const dyna_kv_pool* dst, int kdev, unsigned long long** out) {
  std::lock_guard<std::mutex> lk(src->mu);
  Channel& ch = src->channels[dst];
  unsigned long long*& c = ch.counters[kdev];
  if (!c) {
    DeviceGuard g(kdev);
    CUDA_TRY(cudaMalloc(&c, sizeof(unsigned long long) * DYNA_MAX_CHUNKS));
    CUDA_TRY(cudaMemset(c, 0, sizeof(unsigned long long) * DYNA_MAX_CHUNKS));
  }
  *out = c;
  return DYNA_OK;
}

// Staging slots of channel src -> dst (staged variant): 2 x slot on each side.
dyna_status channel_staging(dyna_kv_pool* src, const dyna_kv_pool* dst, int64_t slot, char** sbuf, char** dbuf) {
  std::lock_guard<std::mutex> lk(src->mu);
  Channel& ch = src->channels[dst];
  if (ch.slot_bytes < slot) {
    if (ch.sstage) {  // grow: the previous migration on this channel must be done with them
      DeviceGuard g(ch.sdev);
      cudaDeviceSynchronize();
      cudaFree(ch.sstage);
      ch.sstage = nullptr;
    }
    if (ch.dstage) {
      DeviceGuard g(ch.ddev);
      cudaDeviceSynchronize();
      cudaFree(ch.dstage);
      ch.dstage = nullptr;
    }
    ch.slot_bytes = 0;
    {
      DeviceGuard g(src->dev);
      if (cudaMalloc(&ch.sstage, 2 * slot) != cudaSuccess) return fail(DYNA_ENOMEM, "staging (source side)");
      ch.sdev = src->dev;
    }
    {
      DeviceGuard g(dst->dev);
      if (cudaMalloc(&ch.dstage, 2 * slot) != cudaSuccess) return fail(DYNA_ENOMEM, "staging (destination side)");
      ch.ddev = dst->dev;
    }
    ch.slot_bytes = slot;
  }
  *sbuf = ch.sstage;
  *dbuf = ch.dstage;
  return DYNA_OK;
}

// ------------------------------------------------------------------ staged variant (a2, a3, a4)
// K1 gather -> source staging slot, K2 slot -> destination-side slot, K3 scatter
// slot -> destination rows (+ per-chunk flag).  Chunks are cut into sub-chunks
// that fit one staging slot; two slots per side alternate.  Same device:
// everything in stream order.  Two devices of one process: K3 runs on a
// library stream of the destination device, ordered with events.
dyna_status run_staged(dyna_kv_pool* S, dyna_kv_pool* D, const int32_t* sids, const int32_t* dids, dyna_range tr,
                       int l0, int lm, int64_t c, bool signal, int engine, int piece, int stages, int unroll,
                       int max_ctas, cudaStream_t stream, dyna_kv_xfer* x, int schedule) {
  if (D->imported)
    return fail(DYNA_ENOTSUP, "STAGED variant into an imported (cross-process) pool is not supported; use FUSED");
  const int64_t row = S->row;
  const bool cross = D->dev != S->dev;
  const int64_t nchunks = (tr.end - tr.begin + c - 1) / c;
  DevInfo* ddi = dev_info(D->dev);
  cudaStream_t dstream = stream;
  if (cross) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!ddi->aux) {
      DeviceGuard g(D->dev);
      CUDA_TRY(cudaStreamCreateWithFlags(&ddi->aux, cudaStreamNonBlocking));
    }
    dstream = ddi->aux;
  }
  const int64_t tok_bytes = row * lm * 2;
  const int64_t sc = std::max<int64_t>(1, std::min<int64_t>(c, kStageSlotBytes / tok_bytes));
  const int64_t slot = sc * tok_bytes;
  char *sbuf = nullptr, *dbuf = nullptr;
  dyna_status r = channel_staging(S, D, slot, &sbuf, &dbuf);
  if (r) return r;
  unsigned long long* counters = nullptr;
  if (signal) {
    if ((r = channel_counters(S, D, D->dev, &counters))) return r;
    x->epoch = next_epoch(S->desc.instance, D);
  }
  cudaEvent_t done_src[2] = {nullptr, nullptr};  // K2 of slot i finished (cross-device)
  cudaEvent_t done_dst[2] = {nullptr, nullptr};  // K3 of slot i finished (cross-device)
  if (cross)
    for (int i = 0; i < 2; ++i) {
      CUDA_TRY(get_event(S->dev, &done_src[i]));
      DeviceGuard g(D->dev);
      CUDA_TRY(get_event(D->dev, &done_dst[i]));
    }
  int64_t sub = 0;
  for (int64_t k = 0; k < nchunks && !r; ++k) {
    const int64_t a = tr.begin + k * c, b = std::min(a + c, tr.end);
    for (int64_t sa = a; sa < b && !r; sa += sc, ++sub) {
      const int64_t sb = std::min(sa + sc, b);
      const int si = (int)(sub & 1);
      char* sslot = sbuf + si * slot;
      char* dslot = dbuf + si * slot;
      if (cross && sub >= 2) CUDA_TRY(cudaStreamWaitEvent(stream, done_dst[si], 0));
      Plan k1 = make_plan(paged(S, sids), linear(sslot), row, sa, sb, l0, lm, sb - sa, S->desc.block_size, piece);
      if ((r = launch_copy(k1, engine, max_ctas, stages, unroll, S->dev, stream, schedule))) break;
      // K2: the sub-chunk slot is [lm][2][n][row] = two contiguous halves
      // (K and V of all layers): a flat plan with one token of `half` bytes.
      Plan k2 = make_plan(linear(sslot), linear(dslot), (sb - sa) * row * lm, 0, 1, 0, 1, 1, 1, piece);
      if ((r = launch_copy(k2, engine, max_ctas, stages, unroll, S->dev, stream, schedule))) break;
      Plan k3 = make_plan(linear(dslot), paged(D, dids), row, sa, sb, l0, lm, sb - sa, D->desc.block_size, piece);
      k3.mig_t0 = tr.begin;
      k3.mig_t1 = tr.end;
      k3.sig_c = (int32_t)c;
      if (signal) {
        k3.counters = counters;
        k3.flags = D->inbox + (size_t)S->desc.instance * DYNA_MAX_CHUNKS;
        k3.epoch = x->epoch;
      }
      if (cross) {
        CUDA_TRY(cudaEventRecord(done_src[si], stream));
        DeviceGuard g(D->dev);
        CUDA_TRY(cudaStreamWaitEvent(dstream, done_src[si], 0));
        if ((r = launch_copy(k3, engine, max_ctas, stages, unroll, D->dev, dstream, schedule))) break;
        CUDA_TRY(cudaEventRecord(done_dst[si], dstream));
      } else {
        if ((r = launch_copy(k3, engine, max_ctas, stages, unroll, S->dev, stream, schedule))) break;
      }
    }
  }
  if (cross) {  // the migration completes on `stream` once the last scatters are done
    const int last = (int)((sub - 1) & 1);
    CUDA_TRY(cudaStreamWaitEvent(stream, done_dst[last], 0));
    if (sub >= 2) CUDA_TRY(cudaStreamWaitEvent(stream, done_dst[last ^ 1], 0));
    for (int i = 0; i < 2; ++i) {
      put_event(S->dev, done_src[i]);
      put_event(D->dev, done_dst[i]);
    }
  }
  return r;
}

// Completion event of a migration (none while the stream is being captured
// into a CUDA graph: the captured work only runs at replay).
dyna_status record_completion(dyna_kv_xfer* x, int dev, cudaStream_t stream) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone) {
    x->captured = true;
    return DYNA_OK;
  }
  cudaError_t e = get_event(dev, &x->ev);
  if (e == cudaSuccess) e = cudaEventRecord(x->ev, stream);
  if (e != cudaSuccess) return fail(DYNA_ECUDA, "event record: %s", cudaGetErrorString(e));
  return DYNA_OK;
}

// ------------------------------------------------------------------ upload ring
// Host-resident inputs (block tables passed only as host_block_ids, batch
// descriptors) travel to the device through a per-device ring: pinned host
// staging -> one cudaMemcpyAsync on the caller's stream -> device buffer read
// by the kernel that follows on the same stream.  A span is reused only after
// the event recorded behind its consumer kernel has completed.
constexpr size_t kRingBytes = 8u << 20;

struct UploadRing {
  char* host = nullptr;
  char* dev = nullptr;
  size_t head = 0;
  struct Span {
    size_t b, e;
    cudaEvent_t ev;
  };
  std::deque<Span> live;
  std::vector<cudaEvent_t> free_ev;
  std::mutex mu;
};
std::mutex g_rings_mu;
std::map<int, UploadRing*> g_rings;

// Holds the ring's lock from upload() until finish() records the release event.
class RingLease {
 public:
  explicit RingLease(int dev) : dev_(dev) {}
  ~RingLease() {
    if (ring_) ring_->mu.unlock();
  }

  // Reserve `bytes` of the ring: *hptr (pinned host) is filled by the caller,
  // then copy() moves it to *dptr on the stream.  At most once per lease.
  dyna_status reserve(size_t bytes, char** dptr, char** hptr, cudaStream_t st) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone)
      return fail(DYNA_ENOTSUP, "host-resident inputs cannot be captured in a CUDA graph "
                                "(a replay would read recycled staging); pass device block_ids");
    {
      std::lock_guard<std::mutex> lk(g_rings_mu);
      UploadRing*& r = g_rings[dev_];
      if (!r) r = new UploadRing();
      ring_ = r;
    }
    ring_->mu.lock();  // held until the lease is destroyed (after finish())
    UploadRing& R = *ring_;
    if (!R.host) {
      DeviceGuard g(dev_);
      if (cudaHostAlloc(&R.host, kRingBytes, cudaHostAllocPortable) != cudaSuccess ||
          cudaMalloc(&R.dev, kRingBytes) != cudaSuccess)
        return fail(DYNA_ENOMEM, "upload ring (%zu B pinned + device)", kRingBytes);
    }
    bytes = (bytes + 255) & ~size_t(255);
    if (bytes > kRingBytes) return fail(DYNA_ENOMEM, "host-resident inputs of %zu B exceed the upload ring", bytes);
    size_t b = R.head;
    if (b + bytes > kRingBytes) b = 0;
    const size_t e = b + bytes;
    // free every live span that overlaps [b, e) (spans sit in allocation order)
    while (!R.live.empty() && R.live.front().b < e && b < R.live.front().e) {
      cudaEventSynchronize(R.live.front().ev);
      R.free_ev.push_back(R.live.front().ev);
      R.live.pop_front();
    }
    R.head = e;
    span_b_ = b;
    span_e_ = e;
    *dptr = R.dev + b;
    *hptr = R.host + b;
    return DYNA_OK;
  }

  dyna_status copy(cudaStream_t st) {
    UploadRing& R = *ring_;
    CUDA_TRY(cudaMemcpyAsync(R.dev + span_b_, R.host + span_b_, span_e_ - span_b_, cudaMemcpyHostToDevice, st));
    return DYNA_OK;
  }

  // After the consumer kernel(s) are enqueued on `st`.
  dyna_status finish(cudaStream_t st) {
    if (!ring_ || span_e_ == 0) return DYNA_OK;
    UploadRing& R = *ring_;
    cudaEvent_t ev = nullptr;
    if (!R.free_ev.empty()) {
      ev = R.free_ev.back();
      R.free_ev.pop_back();
    } else {
      DeviceGuard g(dev_);
      CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    CUDA_TRY(cudaEventRecord(ev, st));
    R.live.push_back({span_b_, span_e_, ev});
    span_e_ = 0;
    return DYNA_OK;
  }

 private:
  int dev_;
  UploadRing* ring_ = nullptr;
  size_t span_b_ = 0, span_e_ = 0;
};

// ------------------------------------------------------------------ shared validation
dyna_status check_opts(const dyna_kv_opts* opts, dyna_kv_opts* o) {
  *o = dyna_kv_opts{};
  if (opts) *o = *opts;
  if (o->variant < 0 || o->variant > 2 || o->engine < 0 || o->engine > 3 || o->max_ctas < 0 || o->piece_bytes < 0 ||
      o->piece_bytes % 16 || o->stages < 0 || o->stages == 1 || o->stages > kMaxStages ||
      (o->unroll != 0 && o->unroll != 4 && o->unroll != 8 && o->unroll != 16) || o->schedule < 0 ||
      o->schedule > DYNA_SCHED_DYNAMIC)
    return fail(DYNA_EINVAL, "invalid dyna_kv_opts");
  return DYNA_OK;
}

// Geometry, ranges, table presence and (with host ids) ids / aliasing.  *empty: nothing to move.
dyna_status validate_pair(const dyna_block_table& src, const dyna_block_table& dst, dyna_range tr, dyna_range lr,
                          int32_t chunk_tokens, bool* empty) {
  if (!src.pool || !dst.pool) return fail(DYNA_EINVAL, "NULL pool in a block table");
  const dyna_kv_pool_desc &gs = src.pool->desc, &gd = dst.pool->desc;
  if (gs.num_layers != gd.num_layers || gs.num_kv_heads != gd.num_kv_heads || gs.head_dim != gd.head_dim ||
      gs.elem_bytes != gd.elem_bytes)
    return fail(DYNA_EGEOM, "source and destination geometry differ (L, H, d, e)");
  if (lr.begin < 0 || lr.begin > lr.end || lr.end > gs.num_layers)
    return fail(DYNA_ERANGE, "layer range [%lld, %lld) outside [0, %d)", (long long)lr.begin, (long long)lr.end,
                gs.num_layers);
  if (tr.begin < 0 || tr.begin > tr.end) return fail(DYNA_ERANGE, "bad token range");
  if (tr.end >= (int64_t(1) << 31)) return fail(DYNA_ERANGE, "token indices must be < 2^31");
  *empty = tr.begin == tr.end || lr.begin == lr.end;
  if (*empty) return DYNA_OK;
  if (chunk_tokens <= 0) return fail(DYNA_ERANGE, "chunk_tokens must be > 0");
  if (src.len < 0 || dst.len < 0 || tr.end > src.len * gs.block_size || tr.end > dst.len * gd.block_size)
    return fail(DYNA_ERANGE, "token range end %lld exceeds a block table (src %lld, dst %lld tokens)",
                (long long)tr.end, (long long)(src.len * gs.block_size), (long long)(dst.len * gd.block_size));
  if ((!src.block_ids && !src.host_block_ids) || (!dst.block_ids && !dst.host_block_ids))
    return fail(DYNA_EINVAL, "a block table has neither device nor host block ids");
  return check_host_tables(src, dst, tr.begin, tr.end);
}

// The destination must be addressable from the source (launching) device.
dyna_status check_reach(const dyna_kv_pool* S, const dyna_kv_pool* D) {
  if (D->imported) {
    if (D->dev != S->dev)
      return fail(DYNA_EPEER, "imported destination is mapped on device %d, source is on %d", D->dev, S->dev);
    return DYNA_OK;
  }
  return D->dev == S->dev ? DYNA_OK : ensure_peer(S->dev, D->dev);
}

struct Choice {
  int variant, engine, piece, stages, unroll;
};

// a6: unset choices come from the calibration table (measured GB/s per row
// bytes, locality and call size), else FUSED + VEC.
Choice choose(const dyna_kv_opts& o, int64_t row, int peer, int64_t ntok) {
  dyna_kv_calib_entry ce{};
  const bool calibrated =
      (o.variant == DYNA_VARIANT_AUTO || o.engine == DYNA_ENGINE_AUTO) && calib_lookup(row, peer, ntok, &ce);
  Choice c{};
  c.variant = o.variant ? o.variant : (calibrated && ce.variant ? ce.variant : DYNA_VARIANT_FUSED);
  c.engine = o.engine ? o.engine : (calibrated && ce.engine ? ce.engine : DYNA_ENGINE_VEC);
  const bool use_ce = calibrated && (!o.engine || o.engine == ce.engine);
  c.piece = o.piece_bytes ? o.piece_bytes
                          : (use_ce && ce.piece_bytes ? ce.piece_bytes
                                                     : (c.engine == DYNA_ENGINE_VEC ? kVecPiece : kBulkPiece));
  c.stages = o.stages ? o.stages : (use_ce && ce.stages ? ce.stages : kBulkStages);
  c.unroll = o.unroll ? o.unroll : (use_ce && ce.unroll ? ce.unroll : kVecU);
  return c;
}

// Entries [0, last touched] of a table's host ids (what the kernel may read).
size_t table_upload_bytes(const dyna_block_table& t, int64_t t1) {
  return (size_t)((t1 - 1) / t.pool->desc.block_size + 1) * sizeof(int32_t);
}

}  // namespace

// ============================================================== API
extern "C" {

const char* dyna_kv_last_error(void) { return g_err.c_str(); }

dyna_status dyna_kv_calib_set(const dyna_kv_calib_entry* entries, int32_t n) {
  if (n < 0 || n > 256 || (n > 0 && !entries)) return fail(DYNA_EINVAL, "calibration: 0 <= n <= 256");
  for (int32_t i = 0; i < n; ++i) {
    const auto& e = entries[i];
    if (e.row_bytes < 0 || e.peer < 0 || e.peer > 1 || e.max_chunk_tokens <= 0 || e.variant < 0 || e.variant > 2 ||
        e.engine < 0 || e.engine > 3 || e.piece_bytes < 0 || e.piece_bytes % 16 || e.stages < 0 || e.stages == 1 ||
        e.stages > kMaxStages || (e.unroll != 0 && e.unroll != 4 && e.unroll != 8 && e.unroll != 16))
      return fail(DYNA_EINVAL, "calibration entry %d invalid", i);
  }
  std::lock_guard<std::mutex> lk(g_calib_mu);
  if (n == 0)
    g_calib.assign(std::begin(kCalibDefault), std::end(kCalibDefault) - 1);
  else
    g_calib.assign(entries, entries + n);
  return DYNA_OK;
}

int32_t dyna_kv_calib_get(dyna_kv_calib_entry* out, int32_t cap) {
  std::lock_guard<std::mutex> lk(g_calib_mu);
  for (int32_t i = 0; i < cap && i < (int32_t)g_calib.size(); ++i) out[i] = g_calib[i];
  return (int32_t)g_calib.size();
}
uint64_t dyna_kv_launch_count(void) { return g_launches.load(); }
dyna_status dyna_kv_poll_error(void) { return take_device_error(); }

size_t dyna_kv_pool_bytes(const dyna_kv_pool_desc* d) {
  if (!desc_valid(d)) return 0;
  return (size_t)d->num_layers * 2 * (size_t)d->num_blocks * d->block_size * (size_t)d->num_kv_heads *
         d->head_dim * d->elem_bytes;
}

dyna_status dyna_kv_pool_create(const dyna_kv_pool_desc* desc, void* device_base, dyna_kv_pool_t* out) {
  if (!out || !desc || !device_base) return fail(DYNA_EINVAL, "NULL argument");
  *out = nullptr;
  if (!desc_valid(desc)) return fail(DYNA_EINVAL, "invalid pool descriptor");
  const int64_t row = (int64_t)desc->num_kv_heads * desc->head_dim * desc->elem_bytes;
  if (row % 16) return fail(DYNA_EGEOM, "row bytes H*d*e = %lld is not a multiple of 16", (long long)row);
  if (reinterpret_cast<uintptr_t>(device_base) % 256) return fail(DYNA_EINVAL, "device_base not 256-B aligned");
  if (!err_word()) return fail(DYNA_ECUDA, "cannot allocate mapped error word");
  cudaPointerAttributes attr{};
  CUDA_TRY(cudaPointerGetAttributes(&attr, device_base));
  if (attr.type != cudaMemoryTypeDevice || attr.device != desc->device)
    return fail(DYNA_EINVAL, "device_base is not device memory of device %d", desc->device);
  auto* p = new dyna_kv_pool();
  p->desc = *desc;
  p->base = static_cast<char*>(device_base);
  p->dev = desc->device;
  p->row = row;
  {
    DeviceGuard g(desc->device);
    if (cudaMalloc(&p->inbox, kInboxBytes) != cudaSuccess || cudaMemset(p->inbox, 0, kInboxBytes) != cudaSuccess) {
      delete p;
      return fail(DYNA_ENOMEM, "cannot allocate the %zu B chunk-flag inbox", kInboxBytes);
    }
  }
  p->own_inbox = true;
  dev_info(desc->device);
  *out = p;
  return DYNA_OK;
}

dyna_status dyna_kv_pool_destroy(dyna_kv_pool_t p) {
  if (!p) return fail(DYNA_EINVAL, "NULL pool");
  {
    DeviceGuard g(p->dev);
    for (auto& kv : p->channels) {
      for (auto& c : kv.second.counters) {
        DeviceGuard g2(c.first);
        cudaFree(c.second);
      }
      if (kv.second.sstage) {
        DeviceGuard g2(kv.second.sdev);
        cudaFree(kv.second.sstage);
      }
      if (kv.second.dstage) {
        DeviceGuard g2(kv.second.ddev);
        cudaFree(kv.second.dstage);
      }
    }
    if (p->own_inbox) cudaFree(p->inbox);
    if (p->imported) {
      if (p->ipc_pool_map) cudaIpcCloseMemHandle(p->ipc_pool_map);
      if (p->ipc_inbox_map) cudaIpcCloseMemHandle(p->ipc_inbox_map);
    }
  }
  delete p;
  return DYNA_OK;
}

dyna_status dyna_kv_enable_peer(int32_t device, int32_t peer) { return ensure_peer(device, peer); }

dyna_status dyna_kv_migrate(dyna_block_table src, dyna_block_table dst, dyna_range tr, dyna_range lr,
                            int32_t chunk_tokens, struct CUstream_st* stream, dyna_kv_xfer_t* out) {
  return dyna_kv_migrate_ex(src, dst, tr, lr, chunk_tokens, stream, nullptr, out);
}

static dyna_status migrate_impl(dyna_block_table src, dyna_block_table dst, dyna_range tr, dyna_range lr,
                                int32_t chunk_tokens, struct CUstream_st* stream_, const dyna_kv_opts* opts,
                                dyna_kv_ready* board, uint64_t ready_epoch, dyna_kv_xfer_t* out);

dyna_status dyna_kv_migrate_ex(dyna_block_table src, dyna_block_table dst, dyna_range tr, dyna_range lr,
                               int32_t chunk_tokens, struct CUstream_st* stream_, const dyna_kv_opts* opts,
                               dyna_kv_xfer_t* out) {
  return migrate_impl(src, dst, tr, lr, chunk_tokens, stream_, opts, nullptr, 0, out);
}

dyna_status dyna_kv_migrate_on_ready(dyna_block_table src, dyna_block_table dst, dyna_range tr, dyna_range lr,
                                     int32_t chunk_tokens, dyna_kv_ready_t board, uint64_t epoch,
                                     struct CUstream_st* stream_, const dyna_kv_opts* opts, dyna_kv_xfer_t* out) {
  if (!board) return fail(DYNA_EINVAL, "NULL ready board");
  return migrate_impl(src, dst, tr, lr, chunk_tokens, stream_, opts, board, epoch, out);
}

static dyna_status migrate_impl(dyna_block_table src, dyna_block_table dst, dyna_range tr, dyna_range lr,
                                int32_t chunk_tokens, struct CUstream_st* stream_, const dyna_kv_opts* opts,
                                dyna_kv_ready* board, uint64_t ready_epoch, dyna_kv_xfer_t* out) {
  if (!out) return fail(DYNA_EINVAL, "NULL out");
  *out = nullptr;
  dyna_kv_opts o{};
  dyna_status r = check_opts(opts, &o);
  if (r) return r;
  bool empty = false;
  if ((r = validate_pair(src, dst, tr, lr, chunk_tokens, &empty))) return r;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  dyna_kv_pool* S = src.pool;
  dyna_kv_pool* D = dst.pool;
  const dyna_kv_pool_desc &gs = S->desc, &gd = D->desc;
  const int64_t ntok = tr.end - tr.begin;
  const int64_t nchunks = empty ? 0 : (ntok + chunk_tokens - 1) / chunk_tokens;
  const bool signal = (o.flags & DYNA_MIGRATE_SIGNAL) != 0;
  if (signal && nchunks > DYNA_MAX_CHUNKS)
    return fail(DYNA_ERANGE, "%lld chunks > DYNA_MAX_CHUNKS (%d) with signalling", (long long)nchunks, DYNA_MAX_CHUNKS);
  if (board) {
    if (board->dev != src.pool->dev) return fail(DYNA_EINVAL, "ready board must live on the source device");
    if (nchunks > board->max_chunks)
      return fail(DYNA_ERANGE, "%lld chunks > the ready board's %d slots", (long long)nchunks, board->max_chunks);
    if (o.variant == DYNA_VARIANT_STAGED || (o.engine && o.engine != DYNA_ENGINE_VEC))
      return fail(DYNA_ENOTSUP, "producer-coupled migration: FUSED variant, VEC engine only");
  }
  if (empty) {  // s = 0 (or no layers) -> nothing to ship, nothing enqueued
    auto* x = new dyna_kv_xfer();
    x->dev = S->dev;
    x->sender = gs.instance;
    x->empty = true;
    *out = x;
    return DYNA_OK;
  }
  if ((r = check_reach(S, D))) return r;
  if (!err_word()) return fail(DYNA_ECUDA, "no error word");

  const int64_t row = S->row;
  const int l0 = (int)lr.begin, lm = (int)(lr.end - lr.begin);
  const int64_t c = chunk_tokens;
  const int peer_dst = (D->dev != S->dev || D->imported) ? 1 : 0;
  Choice ch = choose(o, row, peer_dst, ntok);
  if (signal && !o.engine && ch.engine != DYNA_ENGINE_VEC) {
    // measured (bench.py e2e, per-chunk flags on): the VEC engine's per-warp fences beat
    // draining bulk-store groups before each chunk's count (2720 vs 2540 GB/s)
    ch.engine = DYNA_ENGINE_VEC;
    ch.unroll = kVecU;
    if (!o.piece_bytes) ch.piece = kVecPiece;
  }
  if (board) {  // producer-coupled: the VEC engine (each warp waits on its own chunk's mark)
    ch.variant = DYNA_VARIANT_FUSED;
    ch.engine = DYNA_ENGINE_VEC;
    ch.unroll = 8;
    if (!o.piece_bytes) ch.piece = kVecPiece;
  }
  const int variant = ch.variant, engine = ch.engine, piece = ch.piece, stages = ch.stages, unroll = ch.unroll;

  DeviceGuard guard(S->dev);
  // Host-resident tables (block_ids == NULL): upload the entries the kernels may read.
  RingLease lease(S->dev);
  const int32_t* sids = src.block_ids;
  const int32_t* dids = dst.block_ids;
  if (!sids || !dids) {
    if (variant == DYNA_VARIANT_STAGED && D->dev != S->dev)
      return fail(DYNA_ENOTSUP, "cross-device STAGED needs device block_ids for the destination");
    const size_t sb = sids ? 0 : (table_upload_bytes(src, tr.end) + 15) & ~size_t(15);
    const size_t db = dids ? 0 : table_upload_bytes(dst, tr.end);
    char *base = nullptr, *h = nullptr;
    if ((r = lease.reserve(sb + db, &base, &h, stream))) return r;
    if (!sids) std::memcpy(h, src.host_block_ids, table_upload_bytes(src, tr.end));
    if (!dids) std::memcpy(h + sb, dst.host_block_ids, db);
    if ((r = lease.copy(stream))) return r;
    if (!sids) sids = reinterpret_cast<const int32_t*>(base);
    if (!dids) dids = reinterpret_cast<const int32_t*>(base + sb);
  }

  auto* x = new dyna_kv_xfer();
  x->dev = S->dev;
  x->sender = gs.instance;
  x->nchunks = (int32_t)nchunks;
  x->variant = variant;
  x->engine = engine;
  x->piece = piece;
  x->stages = engine != DYNA_ENGINE_VEC ? stages : 0;
  x->unroll = engine == DYNA_ENGINE_VEC ? unroll : 0;
  const uint64_t launches0 = g_launches.load();
  if (variant == DYNA_VARIANT_FUSED) {
    // K4 / K4-local: source rows -> destination rows, one launch for all chunks.
    const int64_t g = gcd64(gs.block_size, gd.block_size);
    Plan p = make_plan(paged(S, sids), paged(D, dids), row, tr.begin, tr.end, l0, lm, c, g, piece);
    if (signal) {
      if ((r = channel_counters(S, D, S->dev, &p.counters))) {
        delete x;
        return r;
      }
      p.flags = D->inbox + (size_t)gs.instance * DYNA_MAX_CHUNKS;
      p.epoch = x->epoch = next_epoch(gs.instance, D);
      p.sys_fence = peer_dst;
    }
    if (board) {
      p.ready = board->slots;
      p.ready_epoch = ready_epoch;
      p.ready_timeout_ns = board->timeout_ns;
      r = launch_ready(p, o.max_ctas, S->dev, stream, o.schedule);
    } else {
      r = launch_copy(p, engine, o.max_ctas, stages, unroll, S->dev, stream, o.schedule);
    }
  } else {
    r = run_staged(S, D, sids, dids, tr, l0, lm, c, signal, engine, piece, stages, unroll, o.max_ctas, stream, x,
                   o.schedule);
  }
  if (!r) r = lease.finish(stream);
  if (r) {
    delete x;
    return r;
  }
  x->launches = (int32_t)(g_launches.load() - launches0);
  if ((r = record_completion(x, S->dev, stream))) {
    delete x;
    return r;
  }
  *out = x;
  return DYNA_OK;
}

dyna_status dyna_kv_migrate_batch(const dyna_kv_migration* migs, int32_t n, dyna_range lr, int32_t chunk_tokens,
                                  struct CUstream_st* stream_, const dyna_kv_opts* opts, dyna_kv_xfer_t* out) {
  if (!out) return fail(DYNA_EINVAL, "NULL out");
  *out = nullptr;
  if (n < 0 || (n > 0 && !migs) || n > DYNA_MAX_BATCH) return fail(DYNA_EINVAL, "0 <= n <= DYNA_MAX_BATCH");
  dyna_kv_opts o{};
  dyna_status r = check_opts(opts, &o);
  if (r) return r;
  if (o.variant == DYNA_VARIANT_STAGED) return fail(DYNA_ENOTSUP, "batch: FUSED variant only");
  if (o.flags & DYNA_MIGRATE_SIGNAL) return fail(DYNA_ENOTSUP, "batch: no per-chunk signalling (use dyna_kv_migrate_ex)");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  std::vector<int32_t> live;
  int64_t total_tok = 0;
  dyna_kv_pool* S0 = nullptr;
  int peer = 0;
  for (int32_t i = 0; i < n; ++i) {
    bool empty = false;
    if ((r = validate_pair(migs[i].src, migs[i].dst, migs[i].token_range, lr, chunk_tokens, &empty))) {
      g_err = "migration " + std::to_string(i) + ": " + g_err;
      return r;
    }
    if (empty) continue;
    dyna_kv_pool *S = migs[i].src.pool, *D = migs[i].dst.pool;
    if (!S0) S0 = S;
    if (S->dev != S0->dev || S->row != S0->row)
      return fail(DYNA_EINVAL, "batch: all sources on one device with one row size");
    if ((r = check_reach(S, D))) return r;
    peer |= (D->dev != S->dev || D->imported) ? 1 : 0;
    total_tok += migs[i].token_range.end - migs[i].token_range.begin;
    live.push_back(i);
  }
  auto* x = new dyna_kv_xfer();
  if (live.empty()) {
    x->empty = true;
    *out = x;
    return DYNA_OK;
  }
  if (!err_word()) {
    delete x;
    return fail(DYNA_ECUDA, "no error word");
  }
  x->dev = S0->dev;
  x->sender = S0->desc.instance;
  Choice ch = choose(o, S0->row, peer, total_tok);
  if (!o.engine && ch.engine != DYNA_ENGINE_VEC) {
    // measured (scripts/batch_probe.py): with many plans the BULK engine's single issuing
    // thread is latency-bound on per-item plan lookups; the warp-parallel VEC engine is not
    ch.engine = DYNA_ENGINE_VEC;
    ch.unroll = kVecU;
    if (!o.piece_bytes) ch.piece = kVecPiece;
  }
  const int l0 = (int)lr.begin, lm = (int)(lr.end - lr.begin);
  DeviceGuard guard(S0->dev);
  // One upload: [plans][item bases][host-resident tables].
  const size_t m = live.size();
  const size_t plans_b = ((m * sizeof(Plan)) + 15) & ~size_t(15);
  const size_t bases_b = ((m * sizeof(int64_t)) + 15) & ~size_t(15);
  std::vector<size_t> soff(m, 0), doff(m, 0);
  size_t tab_b = 0;
  for (size_t k = 0; k < m; ++k) {
    const dyna_kv_migration& mg = migs[live[k]];
    if (!mg.src.block_ids) {
      soff[k] = plans_b + bases_b + tab_b;
      tab_b += (table_upload_bytes(mg.src, mg.token_range.end) + 15) & ~size_t(15);
    }
    if (!mg.dst.block_ids) {
      doff[k] = plans_b + bases_b + tab_b;
      tab_b += (table_upload_bytes(mg.dst, mg.token_range.end) + 15) & ~size_t(15);
    }
  }
  RingLease lease(S0->dev);
  int64_t total_items = 0;
  char *dbase = nullptr, *h = nullptr;
  if ((r = lease.reserve(plans_b + bases_b + tab_b, &dbase, &h, stream))) {
    delete x;
    return r;
  }
  std::vector<Plan> plans(m);
  std::vector<int64_t> bases(m);
  for (size_t k = 0; k < m; ++k) {
    const dyna_kv_migration& mg = migs[live[k]];
    dyna_kv_pool *S = mg.src.pool, *D = mg.dst.pool;
    const int32_t* sids = mg.src.block_ids ? mg.src.block_ids : reinterpret_cast<const int32_t*>(dbase + soff[k]);
    const int32_t* dids = mg.dst.block_ids ? mg.dst.block_ids : reinterpret_cast<const int32_t*>(dbase + doff[k]);
    const int64_t g = gcd64(S->desc.block_size, D->desc.block_size);
    plans[k] = make_plan(paged(S, sids), paged(D, dids), S->row, mg.token_range.begin, mg.token_range.end, l0, lm,
                         chunk_tokens, g, ch.piece);
    bases[k] = total_items;
    total_items += plans[k].n_items;
  }
  // fill the pinned staging now that the device pointers are known, then one copy
  std::memcpy(h, plans.data(), m * sizeof(Plan));
  std::memcpy(h + plans_b, bases.data(), m * sizeof(int64_t));
  for (size_t k = 0; k < m; ++k) {
    const dyna_kv_migration& mg = migs[live[k]];
    if (!mg.src.block_ids)
      std::memcpy(h + soff[k], mg.src.host_block_ids, table_upload_bytes(mg.src, mg.token_range.end));
    if (!mg.dst.block_ids)
      std::memcpy(h + doff[k], mg.dst.host_block_ids, table_upload_bytes(mg.dst, mg.token_range.end));
  }
  if ((r = lease.copy(stream))) {
    delete x;
    return r;
  }
  BatchSource bsrc{reinterpret_cast<const Plan*>(dbase), reinterpret_cast<const int64_t*>(dbase + plans_b),
                   (int32_t)m, total_items};
  x->variant = DYNA_VARIANT_FUSED;
  x->engine = ch.engine;
  x->piece = ch.piece;
  x->stages = ch.engine != DYNA_ENGINE_VEC ? ch.stages : 0;
  x->unroll = ch.engine == DYNA_ENGINE_VEC ? ch.unroll : 0;
  x->launches = 1;
  r = launch_src(bsrc, total_items, false, ch.piece, ch.engine, o.max_ctas, ch.stages, ch.unroll, S0->dev, stream,
                 o.schedule);
  if (!r) r = lease.finish(stream);
  if (r) {
    delete x;
    return r;
  }
  if ((r = record_completion(x, S0->dev, stream))) {
    delete x;
    return r;
  }
  *out = x;
  return DYNA_OK;
}

dyna_status dyna_kv_ready_create(int32_t device, int32_t max_chunks, dyna_kv_ready_t* out) {
  if (!out || device < 0 || max_chunks <= 0 || max_chunks > (1 << 24)) return fail(DYNA_EINVAL, "bad argument");
  *out = nullptr;
  auto* b = new dyna_kv_ready();
  b->dev = device;
  b->max_chunks = max_chunks;
  DeviceGuard g(device);
  if (cudaMalloc(&b->slots, sizeof(unsigned long long) * max_chunks) != cudaSuccess ||
      cudaMemset(b->slots, 0, sizeof(unsigned long long) * max_chunks) != cudaSuccess) {
    delete b;
    return fail(DYNA_ENOMEM, "ready board of %d slots", max_chunks);
  }
  dev_info(device);
  *out = b;
  return DYNA_OK;
}

dyna_status dyna_kv_ready_destroy(dyna_kv_ready_t b) {
  if (!b) return fail(DYNA_EINVAL, "NULL board");
  {
    DeviceGuard g(b->dev);
    cudaFree(b->slots);
  }
  delete b;
  return DYNA_OK;
}

dyna_status dyna_kv_ready_set_timeout(dyna_kv_ready_t b, uint64_t timeout_ns) {
  if (!b || timeout_ns == 0) return fail(DYNA_EINVAL, "bad argument");
  b->timeout_ns = timeout_ns;
  return DYNA_OK;
}

dyna_status dyna_kv_ready_begin(dyna_kv_ready_t b, uint64_t* epoch) {
  if (!b || !epoch) return fail(DYNA_EINVAL, "NULL argument");
  *epoch = ++b->epoch;
  return DYNA_OK;
}

dyna_status dyna_kv_ready_mark(dyna_kv_ready_t b, int32_t chunk, uint64_t epoch, struct CUstream_st* stream) {
  if (!b) return fail(DYNA_EINVAL, "NULL board");
  if (chunk < 0 || chunk >= b->max_chunks) return fail(DYNA_ERANGE, "chunk %d outside the board", chunk);
  DeviceGuard g(b->dev);
  k_mark_ready<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(b->slots + chunk, epoch);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  CUDA_TRY(cudaGetLastError());
  return DYNA_OK;
}

// ---------------------------------------------------------------- receiver-steered placement channel
static constexpr unsigned long long kChanWaitNs = 10ull * 1000 * 1000 * 1000;

static int64_t chan_subchunk(const dyna_kv_channel* ch, int64_t row, int lm, int64_t c) {
  const int64_t tok = row * lm * 2;
  return std::min<int64_t>(c, (int64_t)ch->slot_bytes / tok);
}

dyna_status dyna_kv_channel_create(dyna_kv_pool_t dst, int32_t sender, int32_t slots, uint64_t slot_bytes,
                                   dyna_kv_channel_t* out) {
  if (!out || !dst) return fail(DYNA_EINVAL, "NULL argument");
  *out = nullptr;
  if (dst->imported) return fail(DYNA_EINVAL, "create the channel on the destination pool's owner");
  if (slots < 2 || slots > 1024 || slot_bytes == 0 || slot_bytes % 16 || sender < 0 || sender >= DYNA_MAX_INSTANCES)
    return fail(DYNA_EINVAL, "channel: 2 <= slots <= 1024, slot_bytes a positive multiple of 16, valid sender");
  auto* ch = new dyna_kv_channel();
  ch->dev = dst->dev;
  ch->slots = slots;
  ch->slot_bytes = slot_bytes;
  ch->sender = sender;
  ch->desc = dst->desc;
  ch->dst = dst;
  const size_t data = (size_t)slots * slot_bytes;
  const size_t total = data + 2 * sizeof(unsigned long long) * slots;
  DeviceGuard g(dst->dev);
  if (cudaMalloc(&ch->base, total) != cudaSuccess) {
    delete ch;
    return fail(DYNA_ENOMEM, "channel of %zu B", total);
  }
  ch->full = reinterpret_cast<unsigned long long*>(ch->base + data);
  ch->credit = ch->full + slots;
  if (cudaMemset(ch->full, 0, 2 * sizeof(unsigned long long) * slots) != cudaSuccess) {
    cudaFree(ch->base);
    delete ch;
    return fail(DYNA_ECUDA, "channel init");
  }
  dev_info(dst->dev);
  *out = ch;
  return DYNA_OK;
}

dyna_status dyna_kv_channel_export(dyna_kv_channel_t ch, dyna_kv_channel_handle* out) {
  if (!ch || !out) return fail(DYNA_EINVAL, "NULL argument");
  if (ch->imported) return fail(DYNA_EINVAL, "cannot re-export an imported channel");
  std::memset(out, 0, sizeof *out);
  DeviceGuard g(ch->dev);
  cudaIpcMemHandle_t h{};
  CUDA_TRY(cudaIpcGetMemHandle(&h, ch->base));
  std::memcpy(out->mem, &h, sizeof h);
  out->slot_bytes = ch->slot_bytes;
  out->slots = ch->slots;
  out->sender = ch->sender;
  out->desc = ch->desc;
  return DYNA_OK;
}

dyna_status dyna_kv_channel_import(const dyna_kv_channel_handle* h, int32_t local_device, dyna_kv_channel_t* out) {
  if (!h || !out) return fail(DYNA_EINVAL, "NULL argument");
  *out = nullptr;
  if (h->slots < 2 || h->slot_bytes == 0 || !desc_valid(&h->desc)) return fail(DYNA_EINVAL, "invalid channel handle");
  DeviceGuard g(local_device);
  cudaIpcMemHandle_t mh{};
  std::memcpy(&mh, h->mem, sizeof mh);
  void* m = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&m, mh, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(DYNA_EPEER, "cudaIpcOpenMemHandle(channel): %s", cudaGetErrorString(e));
  auto* ch = new dyna_kv_channel();
  ch->dev = local_device;
  ch->imported = true;
  ch->base = static_cast<char*>(m);
  ch->slots = h->slots;
  ch->slot_bytes = h->slot_bytes;
  ch->sender = h->sender;
  ch->desc = h->desc;
  ch->full = reinterpret_cast<unsigned long long*>(ch->base + (size_t)h->slots * h->slot_bytes);
  ch->credit = ch->full + h->slots;
  if (!err_word()) {
    cudaIpcCloseMemHandle(m);
    delete ch;
    return fail(DYNA_ECUDA, "no error word");
  }
  dev_info(local_device);
  *out = ch;
  return DYNA_OK;
}

dyna_status dyna_kv_channel_destroy(dyna_kv_channel_t ch) {
  if (!ch) return fail(DYNA_EINVAL, "NULL channel");
  if (ch->push_counters) {
    DeviceGuard g(ch->push_counters_dev);
    cudaFree(ch->push_counters);
  }
  {
    DeviceGuard g(ch->dev);
    if (ch->place_counters) cudaFree(ch->place_counters);
    if (ch->imported)
      cudaIpcCloseMemHandle(ch->base);
    else
      cudaFree(ch->base);
  }
  delete ch;
  return DYNA_OK;
}

// Shared checks of push / place: geometry against the channel, ranges, a device table.
static dyna_status chan_check(const dyna_kv_channel* ch, const dyna_block_table& t, dyna_range tr, dyna_range lr,
                              int32_t c, bool* empty) {
  if (!ch || !t.pool) return fail(DYNA_EINVAL, "NULL channel or pool");
  const dyna_kv_pool_desc &g = t.pool->desc, &cg = ch->desc;
  if (g.num_layers != cg.num_layers || g.num_kv_heads != cg.num_kv_heads || g.head_dim != cg.head_dim ||
      g.elem_bytes != cg.elem_bytes)
    return fail(DYNA_EGEOM, "pool geometry differs from the channel's");
  if (lr.begin < 0 || lr.begin > lr.end || lr.end > g.num_layers) return fail(DYNA_ERANGE, "bad layer range");
  if (tr.begin < 0 || tr.begin > tr.end || tr.end >= (int64_t(1) << 31)) return fail(DYNA_ERANGE, "bad token range");
  *empty = tr.begin == tr.end || lr.begin == lr.end;
  if (*empty) return DYNA_OK;
  if (c <= 0) return fail(DYNA_ERANGE, "chunk_tokens must be > 0");
  if (tr.end > t.len * g.block_size) return fail(DYNA_ERANGE, "token range exceeds the block table");
  if (!t.block_ids) return fail(DYNA_EINVAL, "push/place need device block_ids");
  if (chan_subchunk(ch, t.pool->row, (int)(lr.end - lr.begin), c) < 1)
    return fail(DYNA_EINVAL, "a channel slot of %llu B cannot hold one token of this layer range",
                (unsigned long long)ch->slot_bytes);
  if (t.host_block_ids) {
    const int64_t bs = g.block_size;
    for (int64_t j = tr.begin / bs; j <= (tr.end - 1) / bs; ++j)
      if (t.host_block_ids[j] < 0 || t.host_block_ids[j] >= g.num_blocks)
        return fail(DYNA_ERANGE, "block_ids[%lld] = %d outside [0, %d)", (long long)j, t.host_block_ids[j],
                    g.num_blocks);
  }
  return DYNA_OK;
}

static dyna_status chan_counters(unsigned long long** c, int dev) {
  if (*c) return DYNA_OK;
  DeviceGuard g(dev);
  CUDA_TRY(cudaMalloc(c, sizeof(unsigned long long) * DYNA_MAX_CHUNKS));
  CUDA_TRY(cudaMemset(*c, 0, sizeof(unsigned long long) * DYNA_MAX_CHUNKS));
  return DYNA_OK;
}

dyna_status dyna_kv_push(dyna_block_table src, dyna_range tr, dyna_range lr, int32_t c, dyna_kv_channel_t ch,
                         struct CUstream_st* stream_, dyna_kv_xfer_t* out) {
  if (!out) return fail(DYNA_EINVAL, "NULL out");
  *out = nullptr;
  bool empty = false;
  dyna_status r = chan_check(ch, src, tr, lr, c, &empty);
  if (r) return r;
  dyna_kv_pool* S = src.pool;
  auto* x = new dyna_kv_xfer();
  x->dev = S->dev;
  x->sender = ch->sender;
  if (empty) {
    x->empty = true;
    *out = x;
    return DYNA_OK;
  }
  if (ch->imported ? ch->dev != S->dev : (ch->dev != S->dev && (r = ensure_peer(S->dev, ch->dev)) != DYNA_OK)) {
    delete x;
    return r ? r : fail(DYNA_EPEER, "channel mapped on device %d, source on %d", ch->dev, S->dev);
  }
  std::lock_guard<std::mutex> lk(ch->mu);
  if ((r = chan_counters(&ch->push_counters, S->dev))) {
    delete x;
    return r;
  }
  ch->push_counters_dev = S->dev;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  DeviceGuard guard(S->dev);
  const int l0 = (int)lr.begin, lm = (int)(lr.end - lr.begin);
  const int64_t sc = chan_subchunk(ch, S->row, lm, c);
  const uint64_t seq0 = ch->push_seq;
  const uint64_t launches0 = g_launches.load();
  for (int64_t a = tr.begin; a < tr.end && !r; a += c) {
    const int64_t b = std::min<int64_t>(a + c, tr.end);
    for (int64_t sa = a; sa < b && !r; sa += sc) {
      const int64_t sb = std::min(sa + sc, b);
      const uint64_t q = ch->push_seq++;
      const int slot = (int)(q % ch->slots);
      if (q >= (uint64_t)ch->slots) {  // wait for the receiver's credit on this slot
        k_wait_flag<<<1, 1, 0, stream>>>(ch->credit + slot, q - ch->slots + 1, kChanWaitNs, g_err_word);
        g_launches.fetch_add(1, std::memory_order_relaxed);
      }
      // gather straight into the receiver's slot; the last writer releases full[slot] = q + 1
      Plan p = make_plan(paged(S, src.block_ids), linear(ch->base + (size_t)slot * ch->slot_bytes), S->row, sa,
                         sb, l0, lm, sb - sa, S->desc.block_size, kVecPiece);
      p.counters = ch->push_counters;
      p.flags = ch->full + slot;
      p.epoch = q + 1;
      p.sys_fence = 1;
      r = launch_copy(p, DYNA_ENGINE_VEC, 0, kBulkStages, kVecU, S->dev, stream, 0);
    }
  }
  if (!r) {
    CUDA_TRY(cudaGetLastError());
    r = record_completion(x, S->dev, stream);
  }
  if (r) {
    delete x;
    return r;
  }
  x->variant = DYNA_VARIANT_STAGED;
  x->engine = DYNA_ENGINE_VEC;
  x->nchunks = (int32_t)(ch->push_seq - seq0);
  x->launches = (int32_t)(g_launches.load() - launches0);
  *out = x;
  return DYNA_OK;
}

dyna_status dyna_kv_place(dyna_kv_channel_t ch, dyna_block_table dst, dyna_range tr, dyna_range lr, int32_t c,
                          struct CUstream_st* stream_, const dyna_kv_opts* opts, dyna_kv_xfer_t* out) {
  if (!out) return fail(DYNA_EINVAL, "NULL out");
  *out = nullptr;
  bool empty = false;
  dyna_status r = chan_check(ch, dst, tr, lr, c, &empty);
  if (r) return r;
  if (ch->imported || dst.pool != ch->dst) return fail(DYNA_EINVAL, "place on the channel's owner, into its pool");
  dyna_kv_opts o{};
  if ((r = check_opts(opts, &o))) return r;
  const bool signal = (o.flags & DYNA_MIGRATE_SIGNAL) != 0;
  dyna_kv_pool* D = dst.pool;
  const int64_t nchunks = empty ? 0 : (tr.end - tr.begin + c - 1) / c;
  if (signal && nchunks > DYNA_MAX_CHUNKS) return fail(DYNA_ERANGE, "too many chunks for signalling");
  auto* x = new dyna_kv_xfer();
  x->dev = D->dev;
  x->sender = ch->sender;
  x->nchunks = (int32_t)nchunks;
  if (empty) {
    x->empty = true;
    *out = x;
    return DYNA_OK;
  }
  std::lock_guard<std::mutex> lk(ch->mu);
  if (signal) {
    if ((r = chan_counters(&ch->place_counters, D->dev))) {
      delete x;
      return r;
    }
    x->epoch = next_epoch(ch->sender, D);
  }
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  DeviceGuard guard(D->dev);
  const int l0 = (int)lr.begin, lm = (int)(lr.end - lr.begin);
  const int64_t sc = chan_subchunk(ch, D->row, lm, c);
  const uint64_t launches0 = g_launches.load();
  for (int64_t a = tr.begin; a < tr.end && !r; a += c) {
    const int64_t b = std::min<int64_t>(a + c, tr.end);
    for (int64_t sa = a; sa < b && !r; sa += sc) {
      const int64_t sb = std::min(sa + sc, b);
      const uint64_t q = ch->place_seq++;
      const int slot = (int)(q % ch->slots);
      k_wait_flag<<<1, 1, 0, stream>>>(ch->full + slot, q + 1, kChanWaitNs, g_err_word);
      Plan p = make_plan(linear(ch->base + (size_t)slot * ch->slot_bytes), paged(D, dst.block_ids), D->row, sa, sb,
                         l0, lm, sb - sa, D->desc.block_size, kVecPiece);
      p.mig_t0 = tr.begin;
      p.mig_t1 = tr.end;
      p.sig_c = c;
      if (signal) {
        p.counters = ch->place_counters;
        p.flags = D->inbox + (size_t)ch->sender * DYNA_MAX_CHUNKS;
        p.epoch = x->epoch;
      }
      r = launch_copy(p, DYNA_ENGINE_VEC, o.max_ctas, kBulkStages, kVecU, D->dev, stream, 0);
      k_release_sys<<<1, 1, 0, stream>>>(ch->credit + slot, q + 1);  // the slot may be refilled
      g_launches.fetch_add(2, std::memory_order_relaxed);
    }
  }
  if (!r) {
    CUDA_TRY(cudaGetLastError());
    r = record_completion(x, D->dev, stream);
  }
  if (r) {
    delete x;
    return r;
  }
  x->variant = DYNA_VARIANT_STAGED;
  x->engine = DYNA_ENGINE_VEC;
  x->launches = (int32_t)(g_launches.load() - launches0);
  *out = x;
  return DYNA_OK;
}

dyna_status dyna_kv_query(dyna_kv_xfer_t x) {
  if (!x) return fail(DYNA_EINVAL, "NULL xfer");
  if (x->empty || x->captured) return DYNA_OK;
  cudaError_t e = cudaEventQuery(x->ev);
  if (e == cudaSuccess) return DYNA_OK;
  if (e == cudaErrorNotReady) return DYNA_EAGAIN;
  return fail(DYNA_ECUDA, "%s", cudaGetErrorString(e));
}

dyna_status dyna_kv_wait(dyna_kv_xfer_t x) {
  if (!x) return fail(DYNA_EINVAL, "NULL xfer");
  dyna_status r = DYNA_OK;
  if (!x->empty && !x->captured) {
    cudaError_t e = cudaEventSynchronize(x->ev);
    if (e != cudaSuccess) r = fail(DYNA_ECUDA, "migration failed: %s", cudaGetErrorString(e));
    put_event(x->dev, x->ev);
    if (!r) r = take_device_error();
  }
  delete x;
  return r;
}

dyna_status dyna_kv_stream_wait(dyna_kv_xfer_t x, struct CUstream_st* stream) {
  if (!x) return fail(DYNA_EINVAL, "NULL xfer");
  if (x->empty) return DYNA_OK;
  if (x->captured) return fail(DYNA_ENOTSUP, "captured migration: order on the graph instead");
  CUDA_TRY(cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), x->ev, 0));
  return DYNA_OK;
}

dyna_status dyna_kv_xfer_info(dyna_kv_xfer_t x, uint64_t* epoch, int32_t* num_chunks, int32_t* sender) {
  if (!x) return fail(DYNA_EINVAL, "NULL xfer");
  if (epoch) *epoch = x->epoch;
  if (num_chunks) *num_chunks = x->nchunks;
  if (sender) *sender = x->sender;
  return DYNA_OK;
}

dyna_status dyna_kv_xfer_plan(dyna_kv_xfer_t x, int32_t* variant, int32_t* engine, int32_t* piece, int32_t* stages,
                              int32_t* unroll, int32_t* launches) {
  if (!x) return fail(DYNA_EINVAL, "NULL xfer");
  if (variant) *variant = x->variant;
  if (engine) *engine = x->engine;
  if (piece) *piece = x->piece;
  if (stages) *stages = x->stages;
  if (unroll) *unroll = x->unroll;
  if (launches) *launches = x->launches;
  return DYNA_OK;
}

dyna_status dyna_kv_stream_wait_chunk(dyna_kv_pool_t dst, int32_t sender, int32_t chunk, uint64_t epoch,
                                      uint64_t timeout_ns, struct CUstream_st* stream) {
  if (!dst) return fail(DYNA_EINVAL, "NULL pool");
  if (dst->imported) return fail(DYNA_EINVAL, "wait on the owner's side: this pool is an imported mapping");
  if (sender < 0 || sender >= DYNA_MAX_INSTANCES || chunk < 0 || chunk >= DYNA_MAX_CHUNKS)
    return fail(DYNA_ERANGE, "sender/chunk out of range");
  if (!err_word()) return fail(DYNA_ECUDA, "no error word");
  DeviceGuard g(dst->dev);
  k_wait_flag<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      dst->inbox + (size_t)sender * DYNA_MAX_CHUNKS + chunk, epoch, timeout_ns, g_err_word);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  CUDA_TRY(cudaGetLastError());
  return DYNA_OK;
}

dyna_status dyna_kv_copy_flags(dyna_kv_pool_t dst, int32_t sender, int32_t first, int32_t n, uint64_t* host_out,
                               struct CUstream_st* stream) {
  if (!dst || !host_out) return fail(DYNA_EINVAL, "NULL argument");
  if (sender < 0 || sender >= DYNA_MAX_INSTANCES || first < 0 || n < 0 || first + n > DYNA_MAX_CHUNKS)
    return fail(DYNA_ERANGE, "sender/chunk range out of range");
  if (n == 0) return DYNA_OK;
  DeviceGuard g(dst->dev);
  CUDA_TRY(cudaMemcpyAsync(host_out, dst->inbox + (size_t)sender * DYNA_MAX_CHUNKS + first,
                           sizeof(uint64_t) * (size_t)n, cudaMemcpyDeviceToHost,
                           reinterpret_cast<cudaStream_t>(stream)));
  return DYNA_OK;
}

// ---------------------------------------------------------------- IPC
typedef int (*PFN_cuMemGetAddressRange)(unsigned long long*, size_t*, unsigned long long);

dyna_status dyna_kv_pool_export(dyna_kv_pool_t p, dyna_kv_ipc_handle* out) {
  if (!p || !out) return fail(DYNA_EINVAL, "NULL argument");
  if (p->imported) return fail(DYNA_EINVAL, "cannot re-export an imported pool");
  std::memset(out, 0, sizeof *out);
  DeviceGuard g(p->dev);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  CUDA_TRY(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
  if (!fn) return fail(DYNA_ENOTSUP, "cuMemGetAddressRange unavailable");
  unsigned long long alloc_base = 0;
  size_t alloc_size = 0;
  if (reinterpret_cast<PFN_cuMemGetAddressRange>(fn)(&alloc_base, &alloc_size,
                                                    reinterpret_cast<unsigned long long>(p->base)) != 0)
    return fail(DYNA_ECUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h{};
  CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(alloc_base)));
  static_assert(sizeof(h) <= 64, "ipc handle size");
  std::memcpy(out->pool_mem, &h, sizeof h);
  out->pool_offset = reinterpret_cast<unsigned long long>(p->base) - alloc_base;
  cudaIpcMemHandle_t hi{};
  CUDA_TRY(cudaIpcGetMemHandle(&hi, p->inbox));
  std::memcpy(out->inbox_mem, &hi, sizeof hi);
  out->desc = p->desc;
  return DYNA_OK;
}

dyna_status dyna_kv_pool_import(const dyna_kv_ipc_handle* h, int32_t local_device, dyna_kv_pool_t* out) {
  if (!h || !out) return fail(DYNA_EINVAL, "NULL argument");
  *out = nullptr;
  if (!desc_valid(&h->desc)) return fail(DYNA_EINVAL, "invalid descriptor in handle");
  DeviceGuard g(local_device);
  cudaIpcMemHandle_t hp{}, hi{};
  std::memcpy(&hp, h->pool_mem, sizeof hp);
  std::memcpy(&hi, h->inbox_mem, sizeof hi);
  void *mp = nullptr, *mi = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&mp, hp, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(DYNA_EPEER, "cudaIpcOpenMemHandle(pool): %s", cudaGetErrorString(e));
  e = cudaIpcOpenMemHandle(&mi, hi, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    cudaIpcCloseMemHandle(mp);
    return fail(DYNA_EPEER, "cudaIpcOpenMemHandle(inbox): %s", cudaGetErrorString(e));
  }
  auto* p = new dyna_kv_pool();
  p->desc = h->desc;
  p->base = static_cast<char*>(mp) + h->pool_offset;
  p->dev = local_device;
  p->imported = true;
  p->ipc_pool_map = mp;
  p->ipc_inbox_map = mi;
  p->inbox = static_cast<unsigned long long*>(mi);
  p->row = (int64_t)h->desc.num_kv_heads * h->desc.head_dim * h->desc.elem_bytes;
  if (!err_word()) {
    dyna_kv_pool_destroy(p);
    return fail(DYNA_ECUDA, "no error word");
  }
  dev_info(local_device);
  *out = p;
  return DYNA_OK;
}

// ---------------------------------------------------------------- test-input generator
dyna_status dyna_kv_debug_fill(void* dst, uint64_t bytes, uint64_t seed, uint64_t byte_offset,
                               struct CUstream_st* stream) {
  if (!dst || bytes % 16 || byte_offset % 8 || reinterpret_cast<uintptr_t>(dst) % 16)
    return fail(DYNA_EINVAL, "fill: dst 16-B aligned, bytes multiple of 16, offset multiple of 8");
  if (bytes == 0) return DYNA_OK;
  cudaPointerAttributes attr{};
  CUDA_TRY(cudaPointerGetAttributes(&attr, dst));
  const int dev = attr.device;
  DevInfo* di = dev_info(dev);
  DeviceGuard g(dev);
  const unsigned long long key = [](unsigned long long z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }(seed);
  const uint64_t n16 = bytes / 16;
  const unsigned grid = (unsigned)std::min<uint64_t>((n16 + 255) / 256, (uint64_t)di->sms * 8);
  k_fill<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(static_cast<ulonglong2*>(dst), n16, key,
                                                                   byte_offset / 8);
  CUDA_TRY(cudaGetLastError());
  return DYNA_OK;
}

}  // extern "C"
