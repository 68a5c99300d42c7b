// runtime.cuh — internals of the host runtime behind include/dyna_kv.h, shared by
// runtime.cu (devices, pools, IPC, calibration, upload ring), launch.cu (plans and
// every kernel launch), migrate.cu (migrations, batches, completion) and
// coupling.cu (producer-coupled ready boards, receiver-steered channels).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <limits>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "dyna_kv.h"
#include "plan.cuh"

#define CUDA_TRY(expr)                                                                         \
  do {                                                                                         \
    cudaError_t e_ = (expr);                                                                   \
    if (e_ != cudaSuccess) {                                                                   \
      return fail(DYNA_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                                   \
    }                                                                                          \
  } while (0)

namespace dynakv {
namespace rt {

// ---------------------------------------------------------------- errors, globals
extern thread_local std::string g_err;
dyna_status fail(dyna_status s, const char* fmt, ...);
extern std::atomic<uint64_t> g_launches;
extern std::mutex g_mu;
// Deferred device-side errors.  Every migration handle owns one word of mapped pinned host
// memory that its kernels atomicOr ERR_* bits into; dyna_kv_wait reads and releases it, so a
// migration's wait reports that migration's errors only.  g_err_word is the process-wide word
// of work that has no handle of its own (dyna_kv_stream_wait_chunk) and of migrations captured
// into CUDA graphs (their kernels outlive the handle): dyna_kv_poll_error reads it.
extern unsigned int* g_err_word;
unsigned int* err_word();
unsigned int* err_acquire();  // a zeroed word (nullptr if none can be allocated)
void err_release(unsigned int* w);
dyna_status err_take(unsigned int* w);  // read-and-clear, as a status
dyna_status take_device_error();

// copy-engine defaults (the calibration table overrides them per call size)
constexpr int kVecU = 8;
constexpr int kVecThreads = 256;
constexpr int kVecPiece = 8192;
constexpr int kBulkPiece = 32768;
constexpr int kBulkStages = 4;
constexpr int64_t kMinBulkRun = 16384;  // AUTO never picks BULK below this contiguous run length
constexpr int64_t kTileRunMax = 32768;  // AUTO moves whole rows as TMA tiles below this contiguous run length
constexpr int64_t kTileMinTokens = 1024;  // ... in calls of at least this many tokens (below, VEC is faster:
                                          // profiles/r02_calib_native_full.json) when no exact-row entry decides
constexpr int64_t kStageSlotBytes = 64ll << 20;  // staged variant: bytes per staging slot
constexpr uint32_t kSchedSlots = 1u << 15;       // dynamic-scheduling counter slots per device
constexpr size_t kInboxBytes = sizeof(unsigned long long) * DYNA_MAX_INSTANCES * DYNA_MAX_CHUNKS;

// ------------------------------------------------------------------ upload ring
// Host-resident inputs (block tables passed only as host_block_ids, batch
// descriptors) travel to the device through a per-device ring: pinned host
// staging -> one cudaMemcpyAsync on the caller's stream -> device buffer read
// by the kernel that follows on the same stream.  A span is reused only after
// the event recorded behind its consumer kernel has completed.
constexpr size_t kRingBytes = 8u << 20;

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

struct DevInfo {
  int sms = 0;
  cudaStream_t aux = nullptr;  // library stream for destination-side kernels (staged, cross-device)
  cudaStream_t upload = nullptr;  // library stream for host-resident table uploads (overlap the previous kernel)
  cudaStream_t maps = nullptr;    // library stream for tile-map cache fills (host-synchronised, once per key)
  unsigned long long* sched = nullptr;  // [kSchedSlots][2] dynamic-scheduling counters, zero at rest
  std::atomic<uint32_t> sched_seq{0};
};

// ============================================================== objects

DevInfo* dev_info(int dev);
cudaError_t get_event(int dev, cudaEvent_t* ev);
void put_event(int dev, cudaEvent_t ev);
bool desc_valid(const dyna_kv_pool_desc* d);
int64_t gcd64(int64_t a, int64_t b);
bool calib_lookup(int64_t row, int peer, int64_t c, dyna_kv_calib_entry* out, bool* exact = nullptr);
void calib_install(int64_t row, int peer, const std::vector<dyna_kv_calib_entry>& es);
dyna_status zeroed_alloc(void** p, size_t bytes, int dev);  // no legacy-stream synchronisation
dyna_status upload_sync(int dev, void* dst, const void* src, size_t bytes);  // likewise
dyna_status ensure_peer(int dev, int peer);
// Per-chunk flags: each signalled logical migration gets a fresh epoch and its own range of
// consecutive inbox slots of (sender instance, destination inbox).  Keyed on the inbox's uid
// (carried in IPC handles, so every mapping of one pool shares it); on first use in a process
// the epoch is seeded from the largest value in that inbox row, so a restarted sender or a
// re-imported pool never hands out an epoch a stale flag already satisfies.
uint64_t new_uid();
dyna_status flag_reserve(int sender, const dyna_kv_pool* dst, int64_t nchunks, uint64_t* epoch, int32_t* first_slot);
// DYNA_MIGRATE_OVERLAP_PREV with flags: whether the slots [first, first + n) (a reservation just
// made) may be shared with a launch that is still running — conservatively, whether the row's
// reservations of the library's last 128 launches (at most 128 kernels run at once on a device;
// one batch launch may hold many reservations) wrapped the ring onto each other — so the overlapped
// launch must wait for its predecessor before it touches those slots' counters.
bool flag_slots_shared_recently(int sender, const dyna_kv_pool* dst, int32_t first, int64_t n);
struct Span {  // the rows [lo, hi) of block `id` of the pool with this uid, heads [h0, h1) of them
  uint64_t uid;
  int32_t id;
  int64_t lo, hi;
  int32_t who;   // batch entry (-1: a single call)
  int32_t h0, h1;
};
dyna_status table_spans(const dyna_block_table& t, int64_t t0, int64_t t1, std::vector<Span>& out, int32_t who,
                        int32_t h0 = 0, int32_t h1 = std::numeric_limits<int32_t>::max());
dyna_status check_alias(std::vector<Span>& dst, std::vector<Span>& src);
bool pools_overlap(const dyna_kv_pool* a, const dyna_kv_pool* b, bool* same);

// Deferred release.  cudaFree / cudaFreeHost / cudaIpcCloseMemHandle may synchronise the
// device, which deadlocks against a producer-coupled migration that is waiting for marks
// (and a binding object's garbage collection can destroy a pool at any moment).  So the
// destroy calls only retire their allocations; they are released by the next call that
// allocates anyway (pool / board / channel create or import), or at process exit.
enum class Mem { Device, Host, Ipc };
void retire(int dev, void* ptr, Mem kind);
void flush_retired();

}  // namespace rt
}  // namespace dynakv

// ---------------------------------------------------------------- objects behind the opaque handles
// Tile-map cache key: everything the four maps of a tile plan encode besides the channel's own
// source pool (the destination's identity and base too: a channel outlives a destroyed destination).
struct TileKey {
  uint64_t duid;
  const char* dbase;
  int64_t slice, spitch, dpitch;
  int32_t scol, dcol, l0, lm, g, lkb;  // g: rows of a full box (tile_rows)
  bool operator==(const TileKey& o) const {
    return duid == o.duid && dbase == o.dbase && slice == o.slice && spitch == o.spitch && dpitch == o.dpitch &&
           scol == o.scol && dcol == o.dcol && l0 == o.l0 && lm == o.lm && g == o.g && lkb == o.lkb;
  }
};
constexpr int kTileCacheSets = 128;  // map sets cached per source pool (then calls upload their maps)

struct Channel {  // sender pool -> destination pool
  std::map<int, unsigned long long*> counters;  // per kernel device: [DYNA_MAX_CHUNKS], zero at rest
  char* sstage = nullptr;                      // staged variant: 2 slots on the source device
  char* dstage = nullptr;                      // staged variant: 2 slots on the destination device
  int64_t slot_bytes = 0;
  int sdev = -1, ddev = -1;
  cudaEvent_t staged_done = nullptr;           // end of the last STAGED migration on this channel (source device)
};

struct dyna_kv_pool {
  dyna_kv_pool_desc desc{};
  uint64_t uid = 0;          // identity of the pool's memory and inbox (random at create, carried by export)
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
  // tile maps of migrations from this pool, allocated at create (a migration never allocates them:
  // an allocation may synchronise the device), written once per key, never changed
  char* tmaps = nullptr;       // device, kTileCacheSets x kTileMaps x kTileMapBytes (nullptr: imported)
  char* tmaps_host = nullptr;  // their pinned source
  std::vector<TileKey> tkeys;  // set i is complete on the device once listed here
};

struct dyna_kv_ready {
  int dev = 0;
  int32_t max_chunks = 0;
  unsigned long long timeout_ns = 10ull * 1000 * 1000 * 1000;  // per chunk wait
  unsigned long long* slots = nullptr;  // device, zero-initialised
  std::atomic<uint64_t> epoch{0};
  // Cancellation: migrations with epoch <= the cancel epoch stop waiting.  The kernels poll a
  // DEVICE word (written by a DMA on the board's control stream): polling mapped host memory
  // from the waiting warps was measured to slow a concurrent cuBLAS producer by 20-100%.
  std::atomic<uint64_t> cancel_epoch{0};      // host copy (dyna_kv_wait reads it)
  unsigned long long* cancel_dev = nullptr;   // device word the kernels poll
  unsigned long long* cancel_stage = nullptr; // pinned staging of the DMA
  cudaStream_t ctrl = nullptr;                // non-blocking control stream of the board
  std::mutex cancel_mu;
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
  unsigned long long timeout_ns = 10ull * 1000 * 1000 * 1000;  // device-side waits
  unsigned long long* push_counters = nullptr;  // sender-device counters for the full-word release
  int push_counters_dev = -1;
  unsigned long long* place_counters = nullptr; // receiver-device counters for inbox chunk flags
  std::mutex mu;
};

struct dyna_kv_xfer {
  ~dyna_kv_xfer() {
    if (err && own_err && err != dynakv::rt::g_err_word) dynakv::rt::err_release(err);
  }
  unsigned int* err = nullptr;  // this migration's deferred-error word (g_err_word when captured)
  bool own_err = true;          // false: the word belongs to a prepared migration (dyna_kv_prepared)
  cudaEvent_t ev = nullptr;
  bool captured = false;  // enqueued during CUDA-graph capture: the work runs at replay
  int32_t variant = 0, engine = 0, piece = 0, stages = 0, unroll = 0, launches = 0;
  int dev = 0;
  bool empty = false;
  uint64_t epoch = 0;
  int32_t nchunks = 0;
  int32_t sender = 0;
  dyna_kv_ready* board = nullptr;  // producer-coupled: the board (for cancellation at dyna_kv_wait)
  uint64_t ready_epoch = 0;
  struct BatchEntry {              // signalled batches: where each entry's chunk flags live
    uint64_t epoch = 0;
    int32_t first_slot = 0, nchunks = 0, sender = 0;
  };
  std::vector<BatchEntry> batch;
  int32_t first_slot = 0;          // signalled: chunk k's flag is inbox slot [sender][first_slot + k]
};


// A batch planned and uploaded once (dyna_kv_prepare_batch): device memory with its plans, item
// bases, tile maps and host-resident tables, launched any number of times.
struct dyna_kv_prepared {
  bool empty = false;
  int dev = 0, sender = 0;
  char* mem = nullptr;             // device: [tile maps][plans][item bases][tables]
  unsigned int* err = nullptr;     // the deferred-error word its kernels write (shared by its launches)
  bool reshard = false;            // dyna_kv_prepare_reshard: isrc, else src
  dynakv::BatchSource src{};
  dynakv::InterleavedSource isrc{};
  bool tiles = false;
  int32_t engine = 0, piece = 0, stages = 0, unroll = 0, max_ctas = 0, schedule = 0;
};

namespace dynakv {
namespace rt {

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


extern std::mutex g_rings_mu;
extern std::map<int, UploadRing*> g_rings;
dyna_status ensure_upload_ring(int dev);

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
    if (b + bytes > kRingBytes) b = 0;  // wrap: the tail [head, end) is left unused this lap
    const size_t e = b + bytes;
    // Recycle finished spans from the front (oldest first), then wait for EVERY live span
    // that overlaps [b, e), wherever it sits in the queue: after a wrap the front may hold an
    // older span of the skipped tail while newer overlapping spans follow it, and spans of
    // different streams need not complete in allocation order.
    while (!R.live.empty() && cudaEventQuery(R.live.front().ev) == cudaSuccess) {
      R.free_ev.push_back(R.live.front().ev);
      R.live.pop_front();
    }
    for (auto it = R.live.begin(); it != R.live.end();) {
      if (it->b < e && b < it->e) {
        cudaEventSynchronize(it->ev);
        R.free_ev.push_back(it->ev);
        it = R.live.erase(it);
      } else {
        ++it;
      }
    }
    R.head = e;
    span_b_ = b;
    span_e_ = e;
    *dptr = R.dev + b;
    *hptr = R.host + b;
    return DYNA_OK;
  }

  // The copy runs on the device's upload stream and `st` waits for it: the upload
  // of call k+1 overlaps call k's kernel instead of sitting between the two on
  // `st` (DYNA_KV_UPLOAD_STREAM=0: copy on `st` itself).  The span cannot still be
  // read by an older kernel: reserve() waited for its release event.
  dyna_status copy(cudaStream_t st) {
    UploadRing& R = *ring_;
    cudaStream_t up = upload_stream();
    if (!up) {
      CUDA_TRY(cudaMemcpyAsync(R.dev + span_b_, R.host + span_b_, span_e_ - span_b_, cudaMemcpyHostToDevice, st));
      return DYNA_OK;
    }
    cudaEvent_t ev = nullptr;
    CUDA_TRY(get_event(dev_, &ev));
    CUDA_TRY(cudaMemcpyAsync(R.dev + span_b_, R.host + span_b_, span_e_ - span_b_, cudaMemcpyHostToDevice, up));
    CUDA_TRY(cudaEventRecord(ev, up));
    CUDA_TRY(cudaStreamWaitEvent(st, ev, 0));
    put_event(dev_, ev);  // the wait above already captured this record
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

  cudaStream_t upload_stream() {
    static const bool on = [] {
      const char* e = std::getenv("DYNA_KV_UPLOAD_STREAM");
      return !(e && e[0] == '0');
    }();
    if (!on) return nullptr;
    DevInfo* di = dev_info(dev_);
    std::lock_guard<std::mutex> lk(g_mu);
    if (!di->upload) {
      DeviceGuard g(dev_);
      if (cudaStreamCreateWithFlags(&di->upload, cudaStreamNonBlocking) != cudaSuccess) di->upload = nullptr;
    }
    return di->upload;
  }
};

struct Choice {
  int variant, engine, piece, stages, unroll;
  bool exact;  // chosen by a calibration entry for this exact row size (not a generic one)
};

Side paged(const dyna_kv_pool* pool, const int32_t* ids);
Side linear(char* base);
dyna_status channel_counters(dyna_kv_pool* src, const dyna_kv_pool* dst, int kdev, unsigned long long** out);
dyna_status channel_staging(dyna_kv_pool* src, const dyna_kv_pool* dst, int64_t slot, char** sbuf, char** dbuf,
                            cudaEvent_t* prev_done);
dyna_status channel_staging_done(dyna_kv_pool* src, const dyna_kv_pool* dst, cudaStream_t stream);

// launch.cu — the only translation unit that instantiates and launches kernels
void preload_kernels();
Plan make_plan(const Side& s, const Side& d, int64_t row, int64_t t0, int64_t t1, int l0, int lm, int64_t c,
               int64_t g, int piece);
void set_chunking(Plan& p, int64_t mig_t0, int64_t mig_t1, int64_t sig_c);
void set_run_groups(Plan& p, int J);
dyna_status launch_copy(const Plan& p, int engine, int max_ctas, int stages, int unroll, int dev, cudaStream_t st,
                        int schedule);
dyna_status launch_batch(const BatchSource& src, int64_t n_items, bool sig, int piece, int engine, int max_ctas,
                         int stages, int unroll, int dev, cudaStream_t st, int schedule);
dyna_status launch_ready(const Plan& p, int max_ctas, int dev, cudaStream_t st, int schedule);
Plan make_plan_sliced(const Side& s, const Side& d, int64_t slice, int64_t spitch, int64_t scol, int64_t dpitch,
                      int64_t dcol, int64_t t0, int64_t t1, int l0, int lm, int64_t c, int64_t g, int piece);
dyna_status launch_rows(const Plan& p, int max_ctas, int dev, cudaStream_t st);
dyna_status launch_rows_interleaved(const InterleavedSource& src, bool sig, int max_ctas, int dev, cudaStream_t st);
// head slices as TMA tensor tiles (k_copy_tiles)
bool tiles_enabled();
bool tile_shape(Plan& p);                    // box geometry + item counts (false: not a tile geometry)
bool tile_encode(const Plan& p, void* maps);  // maps: kTileMaps x kTileMapBytes of host memory
bool tile_plan(Plan& p, void* maps);          // both
// The device copy of a tile plan's maps from pool S to D, cached with S (kernel device kdev) and
// written at first use by a host-synchronised copy on a library stream; *out = nullptr when not
// available (a miss under capture, the cache is full, or S has none): the caller then uploads the
// maps with the call's tables, or does not tile.
dyna_status channel_tile_maps(dyna_kv_pool* S, const dyna_kv_pool* D, const Plan& p, int kdev, cudaStream_t st,
                              const char** out);
dyna_status launch_tiles_batch(const BatchSource& src, bool sig, int tile_bytes, int stages, int max_ctas, int dev,
                               cudaStream_t st);
dyna_status launch_tiles(const Plan& p, int stages, int max_ctas, int dev, cudaStream_t st);
dyna_status launch_tiles_interleaved(const InterleavedSource& src, bool sig, int tile_bytes, int stages, int max_ctas,
                                     int dev, cudaStream_t st);
dyna_status run_staged(dyna_kv_pool* S, dyna_kv_pool* D, const int32_t* sids, const int32_t* dids, dyna_range tr,
                       int l0, int lm, int64_t c, bool signal, int engine, int piece, int stages, int unroll,
                       int max_ctas, cudaStream_t stream, dyna_kv_xfer* x, int schedule);
void launch_wait_flag(const unsigned long long* flag, unsigned long long epoch, unsigned long long timeout_ns,
                      cudaStream_t st, unsigned int* err);
void launch_release_sys(unsigned long long* slot, unsigned long long v, cudaStream_t st);
void launch_mark_ready(unsigned long long* slot, unsigned long long v, cudaStream_t st);
dyna_status launch_fill(void* dst, uint64_t bytes, unsigned long long key, uint64_t first_word, int dev,
                        cudaStream_t st);

// migrate.cu
dyna_status new_xfer(int dev, int sender, cudaStream_t stream, dyna_kv_xfer** out);
dyna_status record_completion(dyna_kv_xfer* x, int dev, cudaStream_t stream);
dyna_status check_opts(const dyna_kv_opts* opts, dyna_kv_opts* o);
dyna_status validate_pair(const dyna_block_table& src, const dyna_block_table& dst, dyna_range tr, dyna_range lr,
                          int32_t chunk_tokens, bool unchecked, bool* empty, std::vector<Span>& dsp,
                          std::vector<Span>& ssp, int src_spans, bool heads_may_differ, int32_t who = -1);
dyna_status check_reach(const dyna_kv_pool* S, const dyna_kv_pool* D);
Choice choose(const dyna_kv_opts& o, int64_t row, int peer, int64_t ntok, int64_t run_bytes);
size_t table_upload_bytes(const dyna_block_table& t, int64_t t1);

}  // namespace rt
}  // namespace dynakv
