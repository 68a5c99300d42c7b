// runtime.cu — devices, errors, events, pools and their IPC export/import, peer
// access, the calibration table, signalling channels' counters and
// staging, and the test-input fill.  Paper mapping: PAPER.md §3.1 P:352 (instances
// exchange the required KV blocks).
#include <chrono>
#include <deque>
#include <random>

#include "runtime.cuh"

using namespace dynakv;
using namespace dynakv::rt;

namespace dynakv {
namespace rt {

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

dyna_status err_take(unsigned int* w) {
  if (!w) return DYNA_OK;
  const unsigned int bits = __atomic_exchange_n(w, 0u, __ATOMIC_ACQ_REL);
  if (bits & ERR_BAD_BLOCK) return fail(DYNA_ERANGE, "device-side check: block id outside [0, num_blocks)");
  if (bits & ERR_TIMEOUT) return fail(DYNA_ETIMEDOUT, "device-side chunk wait timed out");
  return DYNA_OK;
}

dyna_status take_device_error() { return err_take(err_word()); }

// Per-migration words: slabs of mapped pinned host memory, never freed, words recycled.
static std::mutex g_errpool_mu;
static std::vector<unsigned int*> g_err_free;
constexpr int kErrSlabWords = 4096;

unsigned int* err_acquire() {
  std::lock_guard<std::mutex> lk(g_errpool_mu);
  if (g_err_free.empty()) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, sizeof(unsigned int) * kErrSlabWords, cudaHostAllocMapped | cudaHostAllocPortable) !=
        cudaSuccess)
      return nullptr;
    std::memset(p, 0, sizeof(unsigned int) * kErrSlabWords);
    unsigned int* w = static_cast<unsigned int*>(p);
    for (int i = kErrSlabWords - 1; i >= 0; --i) g_err_free.push_back(w + i);
  }
  unsigned int* w = g_err_free.back();
  g_err_free.pop_back();
  __atomic_store_n(w, 0u, __ATOMIC_RELEASE);
  return w;
}

void err_release(unsigned int* w) {
  if (!w) return;
  std::lock_guard<std::mutex> lk(g_errpool_mu);
  g_err_free.push_back(w);
}

std::map<int, DevInfo> g_dev;

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
bool calib_lookup(int64_t row, int peer, int64_t c, dyna_kv_calib_entry* out, bool* exact) {
  std::lock_guard<std::mutex> lk(g_calib_mu);
  for (int pass = 0; pass < 2; ++pass) {
    if (exact) *exact = pass == 0;
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

// Replace the entries of one (row bytes, locality) class by measured ones (dyna_kv_calibrate).
void calib_install(int64_t row, int peer, const std::vector<dyna_kv_calib_entry>& es) {
  std::lock_guard<std::mutex> lk(g_calib_mu);
  std::vector<dyna_kv_calib_entry> keep;
  for (const auto& e : g_calib)
    if (!(e.row_bytes == row && e.peer == peer)) keep.push_back(e);
  keep.insert(keep.end(), es.begin(), es.end());
  g_calib.swap(keep);
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

// Rows a table reaches for tokens [t0, t1), as (pool uid, block id, slot range) spans; ids
// are range-checked on the way (DYNA_ERANGE).  Needs the host copy of the ids.
dyna_status table_spans(const dyna_block_table& t, int64_t t0, int64_t t1, std::vector<Span>& out, int32_t who,
                        int32_t h0, int32_t h1) {
  const int64_t bs = t.pool->desc.block_size, nb = t.pool->desc.num_blocks;
  for (int64_t j = t0 / bs; j <= (t1 - 1) / bs; ++j) {
    const int32_t id = t.host_block_ids[j];
    if (id < 0 || id >= nb) return fail(DYNA_ERANGE, "block_ids[%lld] = %d outside [0, %lld)", (long long)j, id, (long long)nb);
    const int64_t lo = std::max(t0, j * bs) - j * bs, hi = std::min(t1, (j + 1) * bs) - j * bs;
    out.push_back({t.pool->uid, id, lo, hi, who, h0, h1});
  }
  return DYNA_OK;
}

// Reading R7: destination rows (heads) must be distinct (no two writes of one byte) and, where
// a source pool is a destination pool, disjoint from the source rows (heads) being read.
// Source rows may repeat (shared prefix blocks).  All spans of one call or one batch together.
// O(spans): per destination pool (few per call) a block-indexed table, valid for this call only
// through a per-thread generation stamp, chains the spans of each block; a new span is compared
// with the spans already chained on its block (few: one per head range / row range of the block).
dyna_status check_alias(std::vector<Span>& dst, std::vector<Span>& src) {
  if (dst.empty()) return DYNA_OK;
  struct Index {
    std::vector<uint32_t> stamp;  // == gen: head[] is valid for this call
    std::vector<int32_t> head;    // last span chained on the block
  };
  thread_local std::vector<Index> tables;
  thread_local uint32_t gen = 0;
  if (++gen == 0) {  // wrapped: forget every stamp
    for (Index& x : tables) std::fill(x.stamp.begin(), x.stamp.end(), 0u);
    gen = 1;
  }
  std::vector<uint64_t> uids;  // destination pools of this call -> tables[k]
  auto slot = [&](uint64_t u) -> int {
    for (size_t k = 0; k < uids.size(); ++k)
      if (uids[k] == u) return (int)k;
    return -1;
  };
  auto overlap = [](const Span& a, const Span& b) {
    return a.uid == b.uid && a.id == b.id && a.lo < b.hi && b.lo < a.hi && a.h0 < b.h1 && b.h0 < a.h1;
  };
  auto named = [](const Span& a, const Span& b, const char* what) {
    if (a.who < 0) return fail(DYNA_EALIAS, "%s block %d", what, a.id);
    return fail(DYNA_EALIAS, "migration %d: %s block %d (also migration %d)", std::max(a.who, b.who), what, a.id,
                std::min(a.who, b.who));
  };
  std::vector<int32_t> next(dst.size());
  for (size_t i = 0; i < dst.size(); ++i) {
    const Span& d = dst[i];
    int k = slot(d.uid);
    if (k < 0) {
      k = (int)uids.size();
      uids.push_back(d.uid);
      if (tables.size() <= (size_t)k) tables.resize(k + 1);
    }
    Index& t = tables[k];
    const size_t id = (size_t)(uint32_t)d.id;
    if (t.stamp.size() <= id) {
      t.stamp.resize(id + 1, 0u);
      t.head.resize(id + 1, -1);
    }
    if (t.stamp[id] != gen) {
      t.stamp[id] = gen;
      t.head[id] = -1;
    }
    for (int32_t j = t.head[id]; j >= 0; j = next[j])
      if (overlap(d, dst[j])) return named(d, dst[j], "destination rows written twice in");
    next[i] = t.head[id];
    t.head[id] = (int32_t)i;
  }
  for (const Span& s : src) {  // only source rows of pools this call writes matter
    const int k = slot(s.uid);
    if (k < 0) continue;
    const Index& t = tables[k];
    const size_t id = (size_t)(uint32_t)s.id;
    if (id >= t.stamp.size() || t.stamp[id] != gen) continue;
    for (int32_t j = t.head[id]; j >= 0; j = next[j])
      if (overlap(s, dst[j])) return named(dst[j], s, "destination rows that are also source rows in");
  }
  return DYNA_OK;
}

// Two pool objects over the same memory: one uid (an imported mapping carries its owner's), or
// local pools whose byte ranges overlap.  *same: identical layout (rows can be compared by id).
bool pools_overlap(const dyna_kv_pool* a, const dyna_kv_pool* b, bool* same) {
  *same = a->uid == b->uid || a->base == b->base;
  if (*same) return true;
  if (a->imported || b->imported || a->dev != b->dev) return false;
  const char *a0 = a->base, *a1 = a0 + dyna_kv_pool_bytes(&a->desc);
  const char *b0 = b->base, *b1 = b0 + dyna_kv_pool_bytes(&b->desc);
  return a0 < b1 && b0 < a1;
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

// Flag rows: per (sender instance, destination inbox uid), the next epoch and the next free
// slot.  Slots are handed out in consecutive ranges and recycle after DYNA_MAX_CHUNKS chunks;
// flags are raised with an atomic max, so a late writer never moves a flag backwards.
// DYNA_MIGRATE_OVERLAP_PREV: a launch that may still be running holds its slots' counters.  At most 128
// kernels run at once on a device, so only reservations made during the library's last
// kWindowLaunches launches can belong to a running kernel; if those reservations (with the ring's
// wrap waste) fit in DYNA_MAX_CHUNKS slots, none of them reuses another's slots.
constexpr uint64_t kWindowLaunches = 128;
struct FlagRow {
  uint64_t epoch = 0;
  int64_t cursor = 0;
  std::deque<std::pair<uint64_t, int64_t>> recent;  // (library launch count at reservation, slots consumed)
  int64_t window_slots = 0;                          // sum of `recent`'s slots
};
static std::map<std::pair<int, uint64_t>, FlagRow> g_flag_rows;

dyna_status flag_reserve(int sender, const dyna_kv_pool* dst, int64_t nchunks, uint64_t* epoch, int32_t* first_slot) {
  if (sender < 0 || sender >= DYNA_MAX_INSTANCES) return fail(DYNA_EINVAL, "sender %d", sender);
  if (nchunks > DYNA_MAX_CHUNKS)
    return fail(DYNA_ERANGE, "%lld chunks > DYNA_MAX_CHUNKS (%d) with signalling", (long long)nchunks, DYNA_MAX_CHUNKS);
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_pair(sender, dst->uid);
  auto it = g_flag_rows.find(key);
  if (it == g_flag_rows.end()) {  // first use in this process: start above every flag already in the row
    std::vector<unsigned long long> row(DYNA_MAX_CHUNKS);
    DeviceGuard g(dst->dev);
    cudaStream_t s = nullptr;
    CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaError_t e = cudaMemcpyAsync(row.data(), dst->inbox + (size_t)sender * DYNA_MAX_CHUNKS,
                                    sizeof(unsigned long long) * DYNA_MAX_CHUNKS, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (e != cudaSuccess) return fail(DYNA_ECUDA, "reading the inbox row: %s", cudaGetErrorString(e));
    FlagRow fr;
    for (unsigned long long v : row) fr.epoch = std::max<uint64_t>(fr.epoch, v);
    it = g_flag_rows.emplace(key, fr).first;
  }
  FlagRow& fr = it->second;
  int64_t consumed = nchunks;
  if (fr.cursor + nchunks > DYNA_MAX_CHUNKS) {
    consumed += DYNA_MAX_CHUNKS - fr.cursor;  // the skipped tail of the ring counts as used this lap
    fr.cursor = 0;
  }
  *first_slot = (int32_t)fr.cursor;
  const uint64_t now = g_launches.load();
  while (!fr.recent.empty() && fr.recent.front().first + kWindowLaunches < now) {
    fr.window_slots -= fr.recent.front().second;
    fr.recent.pop_front();
  }
  fr.recent.emplace_back(now, consumed);
  fr.window_slots += consumed;
  fr.cursor += nchunks;
  *epoch = ++fr.epoch;
  return DYNA_OK;
}

bool flag_slots_shared_recently(int sender, const dyna_kv_pool* dst, int32_t first, int64_t n) {
  (void)first;
  (void)n;
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_flag_rows.find(std::make_pair(sender, dst->uid));
  if (it == g_flag_rows.end()) return true;
  return it->second.window_slots > DYNA_MAX_CHUNKS;  // the recent reservations wrapped onto each other
}

// Zeroed device memory allocated during a call: zeroed on a non-blocking library stream, waited
// for on the host.  (A plain cudaMemset runs on the legacy stream, which would wait for a
// producer-coupled migration still waiting for its marks on a blocking stream.)
dyna_status zeroed_alloc(void** p, size_t bytes, int dev) {
  DeviceGuard g(dev);
  DevInfo* di = dev_info(dev);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!di->maps) CUDA_TRY(cudaStreamCreateWithFlags(&di->maps, cudaStreamNonBlocking));
  }
  CUDA_TRY(cudaMalloc(p, bytes));
  CUDA_TRY(cudaMemsetAsync(*p, 0, bytes, di->maps));
  CUDA_TRY(cudaStreamSynchronize(di->maps));
  return DYNA_OK;
}

// A host image copied to device memory and waited for on the host, on a non-blocking library stream.
dyna_status upload_sync(int dev, void* dst, const void* src, size_t bytes) {
  DeviceGuard g(dev);
  DevInfo* di = dev_info(dev);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!di->maps) CUDA_TRY(cudaStreamCreateWithFlags(&di->maps, cudaStreamNonBlocking));
  }
  CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, di->maps));
  CUDA_TRY(cudaStreamSynchronize(di->maps));
  return DYNA_OK;
}

// Self-resetting per-chunk byte counters of channel src -> dst on device kdev.
dyna_status channel_counters(dyna_kv_pool* src, const dyna_kv_pool* dst, int kdev, unsigned long long** out) {
  std::lock_guard<std::mutex> lk(src->mu);
  Channel& ch = src->channels[dst];
  unsigned long long*& c = ch.counters[kdev];
  if (!c) {
    dyna_status r = zeroed_alloc(reinterpret_cast<void**>(&c), sizeof(unsigned long long) * DYNA_MAX_CHUNKS, kdev);
    if (r) return r;
  }
  *out = c;
  return DYNA_OK;
}

dyna_status channel_tile_maps(dyna_kv_pool* S, const dyna_kv_pool* D, const Plan& p, int kdev, cudaStream_t st,
                              const char** out) {
  *out = nullptr;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  const bool capturing = cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone;
  const TileKey key{D->uid, D->base, p.row, p.spitch, p.dpitch, p.scol, p.dcol, p.l0, p.lm, p.tile_rows, p.lkb};
  constexpr size_t set_b = (size_t)kTileMaps * kTileMapBytes;
  std::lock_guard<std::mutex> lk(S->mu);
  if (!S->tmaps || kdev != S->dev) return DYNA_OK;
  for (size_t i = 0; i < S->tkeys.size(); ++i)
    if (S->tkeys[i] == key) {
      *out = S->tmaps + i * set_b;
      return DYNA_OK;
    }
  // a miss: fill the next set (not under capture: the fill synchronises with the host)
  if (capturing || S->tkeys.size() >= (size_t)kTileCacheSets) return DYNA_OK;
  DevInfo* di = dev_info(kdev);
  DeviceGuard g(kdev);
  {
    std::lock_guard<std::mutex> lk2(g_mu);
    if (!di->maps) CUDA_TRY(cudaStreamCreateWithFlags(&di->maps, cudaStreamNonBlocking));
  }
  const size_t i = S->tkeys.size();
  if (!tile_encode(p, S->tmaps_host + i * set_b)) return DYNA_OK;
  // its own non-blocking stream, waited for on the host: the set is complete before any kernel can
  // name it, whatever stream that kernel runs on (no device-wide synchronisation involved)
  CUDA_TRY(cudaMemcpyAsync(S->tmaps + i * set_b, S->tmaps_host + i * set_b, set_b, cudaMemcpyHostToDevice, di->maps));
  CUDA_TRY(cudaStreamSynchronize(di->maps));
  S->tkeys.push_back(key);
  *out = S->tmaps + i * set_b;
  return DYNA_OK;
}

// Staging slots of channel src -> dst (staged variant): 2 x slot on each side.  *prev_done:
// the end of the previous STAGED migration on this channel (its stream may differ), which
// the caller orders its kernels after; growing the slots waits for it on the host first.
dyna_status channel_staging(dyna_kv_pool* src, const dyna_kv_pool* dst, int64_t slot, char** sbuf, char** dbuf,
                            cudaEvent_t* prev_done) {
  std::lock_guard<std::mutex> lk(src->mu);
  Channel& ch = src->channels[dst];
  if (ch.slot_bytes < slot) {
    if (ch.staged_done) CUDA_TRY(cudaEventSynchronize(ch.staged_done));  // the old slots are no longer read
    retire(ch.sdev, ch.sstage, Mem::Device);
    retire(ch.ddev, ch.dstage, Mem::Device);
    ch.sstage = ch.dstage = nullptr;
    ch.slot_bytes = 0;
    flush_retired();
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
  *prev_done = ch.staged_done;
  return DYNA_OK;
}

// Record the end of a STAGED migration on `stream` (source device) as the channel's lease.
dyna_status channel_staging_done(dyna_kv_pool* src, const dyna_kv_pool* dst, cudaStream_t stream) {
  std::lock_guard<std::mutex> lk(src->mu);
  Channel& ch = src->channels[dst];
  if (!ch.staged_done) {
    DeviceGuard g(src->dev);
    CUDA_TRY(cudaEventCreateWithFlags(&ch.staged_done, cudaEventDisableTiming));
  }
  CUDA_TRY(cudaEventRecord(ch.staged_done, stream));
  return DYNA_OK;
}

std::mutex g_rings_mu;
std::map<int, UploadRing*> g_rings;

// The device's upload ring, allocated when its first pool is created rather than by the first
// migration with host tables (an allocation during a producer-coupled wait may synchronise).
dyna_status ensure_upload_ring(int dev) {
  UploadRing* r = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_rings_mu);
    UploadRing*& slot = g_rings[dev];
    if (!slot) slot = new UploadRing();
    r = slot;
  }
  std::lock_guard<std::mutex> lk(r->mu);
  if (r->host) return DYNA_OK;
  DeviceGuard g(dev);
  if (cudaHostAlloc(&r->host, kRingBytes, cudaHostAllocPortable) != cudaSuccess ||
      cudaMalloc(&r->dev, kRingBytes) != cudaSuccess)
    return fail(DYNA_ENOMEM, "upload ring (%zu B pinned + device)", kRingBytes);
  return DYNA_OK;
}

uint64_t new_uid() {
  static std::atomic<uint64_t> seq{0};
  static const uint64_t base = [] {
    std::random_device rd;
    return ((uint64_t)rd() << 32) ^ rd() ^ (uint64_t)std::chrono::steady_clock::now().time_since_epoch().count();
  }();
  uint64_t z = base + 0x9E3779B97F4A7C15ull * (seq.fetch_add(1) + 1);  // splitmix64 finaliser: distinct, well spread
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace rt
}  // namespace dynakv

namespace dynakv {
namespace rt {
struct Retired {
  int dev;
  void* ptr;
  Mem kind;
};
static std::mutex g_retired_mu;
static std::vector<Retired> g_retired;

void retire(int dev, void* ptr, Mem kind) {
  if (!ptr) return;
  std::lock_guard<std::mutex> lk(g_retired_mu);
  g_retired.push_back({dev, ptr, kind});
}

void flush_retired() {
  std::vector<Retired> v;
  {
    std::lock_guard<std::mutex> lk(g_retired_mu);
    v.swap(g_retired);
  }
  for (const Retired& r : v) {
    DeviceGuard g(r.dev);
    if (r.kind == Mem::Device) cudaFree(r.ptr);
    else if (r.kind == Mem::Host) cudaFreeHost(r.ptr);
    else cudaIpcCloseMemHandle(r.ptr);
  }
}
}  // namespace rt
}  // namespace dynakv

extern "C" {


const char* dyna_kv_last_error(void) { return g_err.c_str(); }

dyna_status dyna_kv_calib_set(const dyna_kv_calib_entry* entries, int32_t n) {
  if (n < 0 || n > 256 || (n > 0 && !entries)) return fail(DYNA_EINVAL, "calibration: 0 <= n <= 256");
  for (int32_t i = 0; i < n; ++i) {
    const auto& e = entries[i];
    if (e.row_bytes < 0 || e.peer < 0 || e.peer > 1 || e.max_chunk_tokens <= 0 || e.variant < 0 || e.variant > 2 ||
        e.engine < 0 || e.engine > DYNA_ENGINE_TILES || e.piece_bytes < 0 || e.piece_bytes % 16 || e.stages < 0 || e.stages == 1 ||
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
  flush_retired();
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
  p->uid = new_uid();
  p->base = static_cast<char*>(device_base);
  p->dev = desc->device;
  p->row = row;
  {
    DeviceGuard g(desc->device);
    if (cudaMalloc(&p->inbox, kInboxBytes) != cudaSuccess || cudaMemset(p->inbox, 0, kInboxBytes) != cudaSuccess) {
      delete p;
      return fail(DYNA_ENOMEM, "cannot allocate the %zu B chunk-flag inbox", kInboxBytes);
    }
    const size_t tb = (size_t)kTileCacheSets * kTileMaps * kTileMapBytes;
    if (cudaMalloc(&p->tmaps, tb) != cudaSuccess || cudaHostAlloc(&p->tmaps_host, tb, cudaHostAllocPortable) != cudaSuccess) {
      cudaFree(p->inbox);
      if (p->tmaps) cudaFree(p->tmaps);
      delete p;
      return fail(DYNA_ENOMEM, "cannot allocate the %zu B tile-map cache", tb);
    }
  }
  p->own_inbox = true;
  dev_info(desc->device);
  dyna_status r = ensure_upload_ring(desc->device);
  if (r) {
    dyna_kv_pool_destroy(p);
    return r;
  }
  *out = p;
  return DYNA_OK;
}

dyna_status dyna_kv_pool_destroy(dyna_kv_pool_t p) {
  if (!p) return fail(DYNA_EINVAL, "NULL pool");
  for (auto& kv : p->channels) {  // retired, not freed: a destroy never synchronises the device
    for (auto& c : kv.second.counters) retire(c.first, c.second, Mem::Device);
    retire(kv.second.sdev, kv.second.sstage, Mem::Device);
    retire(kv.second.ddev, kv.second.dstage, Mem::Device);
  }
  retire(p->dev, p->tmaps, Mem::Device);
  retire(p->dev, p->tmaps_host, Mem::Host);
  if (p->own_inbox) retire(p->dev, p->inbox, Mem::Device);
  if (p->imported) {
    retire(p->dev, p->ipc_pool_map, Mem::Ipc);
    retire(p->dev, p->ipc_inbox_map, Mem::Ipc);
  }
  delete p;
  return DYNA_OK;
}

dyna_status dyna_kv_enable_peer(int32_t device, int32_t peer) { return ensure_peer(device, peer); }

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
  out->uid = p->uid;
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
  flush_retired();
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
  p->uid = h->uid;
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
  DeviceGuard g(dev);
  const unsigned long long key = [](unsigned long long z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }(seed);
  return launch_fill(dst, bytes, key, byte_offset / 8, dev, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
