// launch.cu — launch plans and every kernel launch of the library: the copy
// engines (VEC, BULK, BULK_WS; balanced persistent grids, programmatic dependent
// launch), the staged variant (K1 gather, K2 transfer, K3 scatter; SURVEY §8
// a2-a4), producer-coupled launches, and the small flag / fill kernels.  The only
// translation unit that includes the kernels.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <type_traits>

#include "dyna_kv_kernels.cuh"
#include "runtime.cuh"

using namespace dynakv;
using namespace dynakv::rt;

namespace dynakv {
namespace rt {

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
      (const void*)k_copy_vec<4, true, BatchSource, false>, (const void*)k_copy_vec<8, true, BatchSource, false>,
      (const void*)k_copy_vec<16, true, BatchSource, false>,
      (const void*)k_copy_vec<16, false, BatchSource, false>,
      (const void*)k_copy_rows<8, false, SingleSource>, (const void*)k_copy_rows<8, true, SingleSource>,
      (const void*)k_copy_rows<8, false, InterleavedSource>, (const void*)k_copy_rows<8, true, InterleavedSource>,
      (const void*)k_copy_rows<8, false, BatchSource>, (const void*)k_copy_rows<8, true, BatchSource>,
      (const void*)k_copy_ring<false, SingleSource>, (const void*)k_copy_ring<true, SingleSource>,
      (const void*)k_copy_ring<true, SingleSource, true>, (const void*)k_copy_ring<false, BatchSource>,
      (const void*)k_copy_ring<true, BatchSource>, (const void*)k_copy_ring<true, BatchSource, true>,
      (const void*)k_copy_lanes<4, false, SingleSource>, (const void*)k_copy_lanes<4, true, SingleSource>,
      (const void*)k_copy_lanes<8, false, SingleSource>, (const void*)k_copy_lanes<8, true, SingleSource>,
      (const void*)k_copy_lanes<16, false, SingleSource>, (const void*)k_copy_lanes<16, true, SingleSource>,
      (const void*)k_copy_lanes<4, false, BatchSource>, (const void*)k_copy_lanes<4, true, BatchSource>,
      (const void*)k_copy_lanes<8, false, BatchSource>, (const void*)k_copy_lanes<8, true, BatchSource>,
      (const void*)k_copy_lanes<16, false, BatchSource>, (const void*)k_copy_lanes<16, true, BatchSource>,
      (const void*)k_copy_tiles<false, SingleSource>, (const void*)k_copy_tiles<true, SingleSource, true>,
      (const void*)k_copy_tiles<false, InterleavedSource>, (const void*)k_copy_tiles<true, InterleavedSource, true>,
      (const void*)k_copy_tiles<false, BatchSource>, (const void*)k_copy_tiles<true, BatchSource, true>,
  };
  for (const void* k : ks) cudaFuncGetAttributes(&a, k);
  // Allow the BULK rings any dynamic shared memory the device offers, once, here: a
  // cudaFuncSetAttribute per launch is one more driver call that may synchronise while a
  // producer-coupled migration waits.
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const void* bulk[] = {
      (const void*)k_copy_ring<false, SingleSource>, (const void*)k_copy_ring<true, SingleSource>,
      (const void*)k_copy_ring<true, SingleSource, true>, (const void*)k_copy_ring<false, BatchSource>,
      (const void*)k_copy_ring<true, BatchSource>, (const void*)k_copy_ring<true, BatchSource, true>,
      (const void*)k_copy_tiles<false, SingleSource>, (const void*)k_copy_tiles<true, SingleSource, true>,
      (const void*)k_copy_tiles<false, InterleavedSource>, (const void*)k_copy_tiles<true, InterleavedSource, true>,
      (const void*)k_copy_tiles<false, BatchSource>, (const void*)k_copy_tiles<true, BatchSource, true>,
  };
  for (const void* k : bulk) {
    cudaFuncGetAttributes(&a, k);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)a.sharedSizeBytes);
  }
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
  // runs per chunk: sized by the chunk length, or by the range when the whole range is one shorter chunk
  // (a 141-token request in 1024-token chunks would otherwise leave ~86% of its item slots empty)
  const int64_t ce = std::max<int64_t>(1, std::min<int64_t>(c, t1 - t0));
  const bool aligned = (t0 % g == 0) && (ce % g == 0);
  p.R = aligned ? (int32_t)(ce / g) : (int32_t)((ce - 1) / g + 2);
  const int64_t run_max = std::min(g, c) * row;
  p.piece = piece;
  p.P = (int32_t)((run_max + piece - 1) / piece);
  p.nchunks = (int32_t)((t1 - t0 + c - 1) / c);
  p.items_per_chunk = (int64_t)lm * 2 * p.R * p.P;
  p.n_items = p.items_per_chunk * p.nchunks;
  set_chunking(p, t0, t1, c);
  static const int jgroup = [] {  // experiment switch
    const char* e = std::getenv("DYNA_KV_JGROUP");
    return e ? std::atoi(e) : 0;
  }();
  set_run_groups(p, jgroup);
  p.err = g_err_word;
  return p;
}

// Item order inside a chunk: groups of J runs, each group visiting every (layer, K|V)
// slab before the next group (J <= 0 or J >= R: the plain layer-major order).  The run
// count is padded to a multiple of J; padding items are empty.
void set_run_groups(Plan& p, int J) {
  const int32_t R = p.R;
  p.J = (J <= 0 || J >= R) ? R : J;
  const int64_t rpad = (R + p.J - 1) / p.J * p.J;
  p.items_per_chunk = (int64_t)p.lm * 2 * rpad * p.P;
  p.n_items = p.items_per_chunk * p.nchunks;
}

// The migration's own chunking for a launch that may cover a sub-range of it.
// When the launch's chunks coincide with the migration's (same size, aligned
// start), the kernels take the chunk index without a 64-bit division.
void set_chunking(Plan& p, int64_t mig_t0, int64_t mig_t1, int64_t sig_c) {
  p.mig_t0 = mig_t0;
  p.mig_t1 = mig_t1;
  p.sig_c = (int32_t)sig_c;
  p.k_direct = (p.c == sig_c && (p.t0 - mig_t0) % sig_c == 0) ? 1 : 0;
  p.k_base = p.k_direct ? (int32_t)((p.t0 - mig_t0) / sig_c) : 0;
}

// Plan of a head-sliced migration: `slice` bytes per token at byte scol of a
// spitch-byte source row -> byte dcol of a dpitch-byte destination row.  Runs
// follow the same token grid g as make_plan; an item is up to `tpp` tokens of a run.
Plan make_plan_sliced(const Side& s, const Side& d, int64_t slice, int64_t spitch, int64_t scol, int64_t dpitch,
                      int64_t dcol, int64_t t0, int64_t t1, int l0, int lm, int64_t c, int64_t g, int piece) {
  Plan p = make_plan(s, d, slice, t0, t1, l0, lm, c, g, piece);
  p.spitch = spitch;
  p.dpitch = dpitch;
  p.scol = (int32_t)scol;
  p.dcol = (int32_t)dcol;
  p.tpp = (int32_t)std::max<int64_t>(1, piece / slice);
  p.P = (int32_t)((std::min(g, c) + p.tpp - 1) / p.tpp);
  p.J = p.R;  // the sliced decode uses the layer-major order
  p.items_per_chunk = (int64_t)lm * 2 * p.R * p.P;
  p.n_items = p.items_per_chunk * p.nchunks;
  p.vps = (int32_t)(slice / 16);
  p.vps_shift = (p.vps & (p.vps - 1)) == 0 ? __builtin_ctz((unsigned)p.vps) : -1;
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

// Resident 256-thread CTAs per SM of a VEC-family kernel (cached per device and kernel).
int vec_occupancy(const void* kern) {
  static std::map<std::pair<int, const void*>, int> cache;
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({dev, kern});
  if (it != cache.end()) return it->second;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kVecThreads, 0);
  if (occ <= 0) occ = 1;
  cache[{dev, kern}] = occ;
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

// VEC launches: the warp-cooperative-decode kernel (k_copy_lanes) for the default static
// schedule; k_copy_vec for dynamic scheduling (DYNA_KV_LANES=0 restores it for static too).
bool lanes_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DYNA_KV_LANES");
    return !(e && e[0] == '0');
  }();
  return on;
}

// sched: a dynamic-scheduling counter slot (DYNA_SCHED_DYNAMIC) or nullptr.  k_copy_lanes grabs up to 32
// consecutive items per warp and atomic (guided, like the ring's decoder: one 4-GiB call 0.93 -> 1.01 of
// the copy peak; it loses on short and on overlapped calls, so it is an option, not a default:
// profiles/r02_lanes_dynamic.jsonl); k_copy_vec (DYNA_KV_LANES=0) grabs one item at a time.
template <int U, bool SIG, class Src>
void launch_vec(const Src& src, int64_t n_items, int64_t max_grid, int sms, cudaStream_t st,
                unsigned long long* sched) {
  const bool lanes = lanes_enabled();
  const int occ = vec_occupancy(lanes ? (const void*)k_copy_lanes<U, SIG, Src>
                                      : (const void*)k_copy_vec<U, SIG, Src, false>);
  constexpr int wpc = kVecThreads / 32;  // warps per CTA
  int64_t max_ctas = (int64_t)sms * occ;
  if (max_grid > 0) max_ctas = std::min<int64_t>(max_ctas, max_grid);
  const int64_t warps = balanced_workers(n_items, max_ctas * wpc);
  const int64_t grid = (warps + wpc - 1) / wpc;
  if (lanes)
    launch_kernel(k_copy_lanes<U, SIG, Src>, (unsigned)grid, kVecThreads, 0, st, src, sched);
  else
    launch_kernel(k_copy_vec<U, SIG, Src, false>, (unsigned)grid, kVecThreads, 0, st, src, sched);
}

// Dynamic shared memory a kernel may use: the opt-in maximum minus the kernel's own
// static shared memory (per kernel: the accountant variants carry a mailbox).
int smem_avail(const void* kern) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({dev, kern});
  if (it != cache.end()) return it->second;
  int optin = 0;
  cudaFuncAttributes fa{};
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncGetAttributes(&fa, kern);
  const int v = optin - (int)fa.sharedSizeBytes;
  cache[{dev, kern}] = v;
  return v;
}

// The BULK engine: the decoder-fed TMA ring (k_copy_ring).  With per-chunk signalling a third
// warp is the accountant (the issuer posts finished chunks to it instead of fencing itself;
// measured); DYNA_KV_ACCOUNTANT=0 makes the issuer count with a release RMW.
template <bool SIG, class Src>
dyna_status launch_bulk(const Src& src, int64_t n_items, int piece, int stages, int64_t max_grid, int sms,
                        cudaStream_t st, unsigned long long* sched) {
  static const bool acc_on = [] {
    const char* e = std::getenv("DYNA_KV_ACCOUNTANT");
    return !(e && e[0] == '0');
  }();
  static const int lag_env = [] {  // experiment switch: slots refilled `lag` stores late (0 = by depth)
    const char* e = std::getenv("DYNA_KV_LAG");
    return e ? std::atoi(e) : 0;
  }();
  const bool acc = SIG && acc_on;
  void (*kring)(const Src, int, int, unsigned long long*) = acc ? k_copy_ring<SIG, Src, true> : k_copy_ring<SIG, Src>;
  const int threads = acc ? 96 : 64;
  // a ring deeper than the shared memory holds is cut to the stages that fit (at least 2)
  const int avail = smem_avail((const void*)kring);
  if ((int64_t)stages * piece > avail) stages = avail / piece;
  if (stages < 2) return fail(DYNA_EINVAL, "BULK: two %d-B pieces do not fit in shared memory", piece);
  const size_t smem = (size_t)stages * piece;
  int occ = 0;  // (the dynamic shared memory limit was raised once in preload_kernels)
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kring, threads, smem));
  if (occ <= 0) return fail(DYNA_EINVAL, "BULK: %zu B of shared memory per CTA does not fit", smem);
  int64_t cap = (int64_t)sms * occ;
  if (max_grid > 0) cap = std::min<int64_t>(cap, max_grid);
  const unsigned grid = (unsigned)balanced_workers(n_items, cap);
  const int lag = lag_env > 0 ? std::min(lag_env, std::max(1, stages - 2)) : (stages >= 4 ? 2 : 1);
  CUDA_TRY(launch_kernel(kring, grid, threads, smem, st, src, stages, lag, sched));
  return DYNA_OK;
}

constexpr int64_t kRingDynMinItemsPerSm = 24;
// bytes a launch moves: the item space is sized per chunk (runs x pieces of a full chunk), so short
// ranges leave most items empty — the dynamic-grab threshold counts real bytes
static int64_t payload_of(const SingleSource& s) { return (s.p.t1 - s.p.t0) * s.p.lm * 2 * s.p.row; }
static int64_t payload_of(const BatchSource& s) { return s.payload; }
static int64_t payload_of(const InterleavedSource& s) { return s.payload; }

// Guided dynamic grabs for a TMA-issuer launch (ring or tiles): from kRingDynMinItemsPerSm pieces per
// SM of real bytes, when at most a fifth of the item slots are empty, outside graph capture.
static unsigned long long* ring_dyn_slot(DevInfo* di, int64_t payload, int64_t n_items, int64_t piece,
                                         cudaStream_t st) {
  static const int64_t dyn_min = [] {  // experiment switch DYNA_KV_RING_DYN: pieces per SM (0 = never dynamic)
    const char* e = std::getenv("DYNA_KV_RING_DYN");
    return e ? (int64_t)std::atoll(e) : kRingDynMinItemsPerSm;
  }();
  if (dyn_min <= 0 || payload < dyn_min * (int64_t)di->sms * piece || n_items * piece > payload + payload / 4)
    return nullptr;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) return nullptr;
  return sched_slot(di, DYNA_SCHED_DYNAMIC);
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
  const bool ring = engine == DYNA_ENGINE_BULK || engine == DYNA_ENGINE_BULK_WS;
  // The ring takes guided dynamic grabs by default from ~24 pieces per SM: static round-robin gives
  // every CTA the same bytes, so SMs that run slower finish last (measured: dynamic +1-3% from 4096
  // items, e.g. the configs[2] batch 1.006 -> 1.019 of the copy peak; below, the first atomic's latency
  // costs more than the tail it saves: profiles/r02_dyn_threshold.jsonl).  Not when more than a
  // fifth of the item slots are empty (a short last chunk: grabs would walk empty slots at the end,
  // where the tail is decided), nor under graph capture (a captured slot would be shared by
  // concurrent replays).
  unsigned long long* dyn = ring && schedule == 0 ? ring_dyn_slot(di, payload_of(src), n_items, piece, st) : nullptr;
  unsigned long long* sc = dyn ? dyn : sched_slot(di, schedule);
  if (ring) {
    dyna_status r = sig ? launch_bulk<true>(src, n_items, piece, stages, max_ctas, di->sms, st, sc)
                        : launch_bulk<false>(src, n_items, piece, stages, max_ctas, di->sms, st, sc);
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

// Head-sliced fused copy: warp-per-item VEC engine over a balanced persistent grid.
template <class Src>
dyna_status launch_rows_src(const Src& src, int64_t n_items, bool sig, int max_ctas, int dev, cudaStream_t st) {
  if (n_items == 0) return DYNA_OK;
  if (n_items >= (int64_t(1) << 31)) return fail(DYNA_ERANGE, "too many work items in one launch");
  DevInfo* di = dev_info(dev);
  constexpr int threads = 32 * (kCopiers + 1);  // a decoder warp + the copier warps
  int o = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &o, sig ? (const void*)k_copy_rows<8, true, Src> : (const void*)k_copy_rows<8, false, Src>, threads, 0);
  int64_t cap = (int64_t)di->sms * std::max(o, 1);
  if (max_ctas > 0) cap = std::min<int64_t>(cap, max_ctas);
  // items go to CTAs round-robin (the decoder decodes 32 of its CTA's items at a time)
  const unsigned grid = (unsigned)balanced_workers((n_items + kCopiers - 1) / kCopiers, cap);
  if (sig) CUDA_TRY(launch_kernel(k_copy_rows<8, true, Src>, grid, threads, 0, st, src));
  else CUDA_TRY(launch_kernel(k_copy_rows<8, false, Src>, grid, threads, 0, st, src));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return DYNA_OK;
}

dyna_status launch_rows(const Plan& p, int max_ctas, int dev, cudaStream_t st) {
  return launch_rows_src(SingleSource{p}, p.n_items, p.counters != nullptr, max_ctas, dev, st);
}

dyna_status launch_rows_interleaved(const InterleavedSource& src, bool sig, int max_ctas, int dev, cudaStream_t st) {
  return launch_rows_src(src, src.total_items, sig, max_ctas, dev, st);
}


// ------------------------------------------------------------------ head slices as TMA tensor tiles
// cuTensorMapEncodeTiled through the runtime's driver entry point (no link against libcuda).
static PFN_cuTensorMapEncodeTiled_v12000 encode_tiled() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

bool tiles_enabled() {  // DYNA_KV_TILES=0: head slices on the VEC row kernel even when AUTO
  static const bool on = [] {
    const char* e = std::getenv("DYNA_KV_TILES");
    return !(e && e[0] == '0');
  }();
  return on;
}

static int tile_l2_promotion() {  // experiment switch DYNA_KV_TILE_L2 (0 none, 1 64B, 2 128B (default), 3 256B)
  static const int v = [] {
    const char* e = std::getenv("DYNA_KV_TILE_L2");
    return e ? std::atoi(e) : 2;
  }();
  return v;
}

static int tile_target_bytes() {  // experiment switch DYNA_KV_TILE_BYTES (default 32 KiB per box)
  static const int v = [] {
    const char* e = std::getenv("DYNA_KV_TILE_BYTES");
    const int x = e ? std::atoi(e) : 0;
    return x > 0 ? x : 32768;
  }();
  return v;
}

// One side's map: 4-D (e0 x 8-B elements, e1, row in slab, slab) over the slabs [2*l0, 2*(l0+lm)) of a
// paged pool, starting at byte `col` of each row; box (e0, e1, rows, lkb).
// A linear side (one packed chunk [l - l0][kv][t - a][slice], dyna_kv_pack / unpack) is the same
// lattice with `clen` rows per slab, starting at its base.
static bool encode_side(CUtensorMap* m, const Side& s, int64_t pitch, int64_t col, int l0, int lm, int64_t slice,
                        int64_t e0, int64_t rows, int64_t lkb, int64_t clen) {
  const int64_t slab_rows = s.linear ? clen : s.nb * (int64_t)s.bs;
  if (s.linear) pitch = slice, col = 0;
  char* base = s.linear ? s.base : s.base + (int64_t)2 * l0 * slab_rows * pitch + col;
  const cuuint64_t dims[4] = {(cuuint64_t)e0, (cuuint64_t)(slice / (e0 * 8)), (cuuint64_t)slab_rows,
                              (cuuint64_t)(2 * (int64_t)lm)};
  const cuuint64_t strides[3] = {(cuuint64_t)(e0 * 8), (cuuint64_t)pitch, (cuuint64_t)(slab_rows * pitch)};
  const cuuint32_t box[4] = {(cuuint32_t)e0, (cuuint32_t)(slice / (e0 * 8)), (cuuint32_t)rows, (cuuint32_t)lkb};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return encode_tiled()(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, base, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        (CUtensorMapL2promotion)tile_l2_promotion(),
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Turn a head-sliced plan (make_plan_sliced, paged -> paged) into a tile plan: slabs per box, ring
// slot, item counts.  False when the geometry does not fit a tensor map or shared memory (the caller
// then uses the VEC row kernel).
bool tile_shape(Plan& p) {
  // a linear side holds exactly one chunk (pack / unpack): its rows are chunk-relative
  if ((p.src.linear && p.dst.linear) || ((p.src.linear || p.dst.linear) && p.nchunks != 1) || !encode_tiled())
    return false;
  const int64_t slice = p.row, g = p.g;
  if (slice % 16 || p.scol % 16 || p.dcol % 16 || p.spitch % 16 || p.dpitch % 16) return false;
  const int64_t e0 = slice <= 2048 ? slice / 8 : 256;
  if (slice % (e0 * 8) || slice / (e0 * 8) > 256 || g < 1 || g > 256) return false;
  const int64_t lim = int64_t(1) << 31;
  if ((!p.src.linear && p.src.nb * (int64_t)p.src.bs >= lim) || (!p.dst.linear && p.dst.nb * (int64_t)p.dst.bs >= lim) ||
      p.t1 - p.t0 >= lim)
    return false;
  const int avail = smem_avail((const void*)k_copy_tiles<true, InterleavedSource, true>);
  // box rows: all g rows of a run when they fit the box target (or at least two ring slots), else the
  // largest divisor of g that does (a run is then several items of `rows` rows each)
  int64_t rows = 1;
  for (int64_t d = 1; d <= g; ++d)
    if (g % d == 0 && (d == 1 || d * slice <= std::max<int64_t>(tile_target_bytes(), g * slice)) &&
        2 * (d * slice + 1024) <= avail)
      rows = d;
  if (rows < g && rows * slice * 2 < tile_target_bytes()) {  // g rows did not fit: aim at the box target
    rows = 1;
    for (int64_t d = 1; d <= g; ++d)
      if (g % d == 0 && (d == 1 || d * slice <= tile_target_bytes())) rows = d;
  }
  const int64_t run = rows * slice;
  if (2 * (run + 1024) > avail) return false;
  const int64_t nlk = 2 * (int64_t)p.lm;
  int64_t lkb = 1;
  for (int64_t d = 1; d <= std::min<int64_t>(nlk, 256); ++d)
    if (nlk % d == 0 && (d == 1 || run * d <= tile_target_bytes()) && 2 * (run * d + 1024) <= avail) lkb = d;
  p.lkb = (int32_t)lkb;
  p.tile_rows = (int32_t)rows;
  p.tile_rstride = (int32_t)((slice * lkb + 127) / 128 * 128);
  p.tile_bytes = (int32_t)((std::max<int64_t>(run * lkb, (rows - 1) * p.tile_rstride) + 1023) / 1024 * 1024);
  p.P = (int32_t)(g / rows);  // pieces of a run
  p.items_per_chunk = (nlk / lkb) * p.R * p.P;
  p.n_items = p.items_per_chunk * p.nchunks;
  return true;
}

// The four maps of a tile plan (after tile_shape) into `maps` (host memory, 4 x 128 B; the caller
// copies them to 64-B-aligned device memory and sets p.tmaps).
bool tile_encode(const Plan& p, void* maps) {
  const int64_t slice = p.row, e0 = slice <= 2048 ? slice / 8 : 256;
  CUtensorMap* m = static_cast<CUtensorMap*>(maps);
  const int64_t clen = p.t1 - p.t0;  // linear sides: one chunk
  return encode_side(&m[0], p.src, p.spitch, p.scol, p.l0, p.lm, slice, e0, p.tile_rows, p.lkb, clen) &&
         encode_side(&m[1], p.dst, p.dpitch, p.dcol, p.l0, p.lm, slice, e0, p.tile_rows, p.lkb, clen) &&
         encode_side(&m[2], p.src, p.spitch, p.scol, p.l0, p.lm, slice, e0, 1, p.lkb, clen) &&
         encode_side(&m[3], p.dst, p.dpitch, p.dcol, p.l0, p.lm, slice, e0, 1, p.lkb, clen);
}

bool tile_plan(Plan& p, void* maps) { return tile_shape(p) && tile_encode(p, maps); }

template <bool SIG, class Src>
dyna_status launch_tiles_t(const Src& src, int64_t n_items, int tile_bytes, int stages, int max_ctas, int dev,
                           cudaStream_t st) {
  DevInfo* di = dev_info(dev);
  void (*kern)(const Src, int, int, unsigned long long*) = SIG ? k_copy_tiles<SIG, Src, true>
                                                               : k_copy_tiles<SIG, Src, false>;
  const int threads = SIG ? 96 : 64;
  if (stages <= 0) stages = 4;
  stages = std::min(stages, kMaxStages);
  const int avail = smem_avail((const void*)kern);
  if ((int64_t)stages * tile_bytes > avail) stages = avail / tile_bytes;
  if (stages < 2) return fail(DYNA_EINVAL, "tiles: two %d-B boxes do not fit in shared memory", tile_bytes);
  const size_t smem = (size_t)stages * tile_bytes;
  int occ = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
  if (occ <= 0) return fail(DYNA_EINVAL, "tiles: %zu B of shared memory per CTA does not fit", smem);
  int64_t cap = (int64_t)di->sms * occ;
  if (max_ctas > 0) cap = std::min<int64_t>(cap, max_ctas);
  const unsigned grid = (unsigned)balanced_workers(n_items, cap);
  const int lag = stages >= 4 ? 2 : 1;
  unsigned long long* dyn = ring_dyn_slot(di, payload_of(src), n_items, tile_bytes, st);  // (as the ring)
  CUDA_TRY(launch_kernel(kern, grid, threads, smem, st, src, stages, lag, dyn));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return DYNA_OK;
}

template <class Src>
dyna_status launch_tiles_src(const Src& src, int64_t n_items, bool sig, int tile_bytes, int stages, int max_ctas,
                             int dev, cudaStream_t st) {
  if (n_items == 0) return DYNA_OK;
  if (n_items >= (int64_t(1) << 31)) return fail(DYNA_ERANGE, "too many work items in one launch");
  return sig ? launch_tiles_t<true>(src, n_items, tile_bytes, stages, max_ctas, dev, st)
             : launch_tiles_t<false>(src, n_items, tile_bytes, stages, max_ctas, dev, st);
}

dyna_status launch_tiles(const Plan& p, int stages, int max_ctas, int dev, cudaStream_t st) {
  return launch_tiles_src(SingleSource{p}, p.n_items, p.counters != nullptr, p.tile_bytes, stages, max_ctas, dev, st);
}

dyna_status launch_tiles_batch(const BatchSource& src, bool sig, int tile_bytes, int stages, int max_ctas, int dev,
                               cudaStream_t st) {
  return launch_tiles_src(src, src.total_items, sig, tile_bytes, stages, max_ctas, dev, st);
}

dyna_status launch_tiles_interleaved(const InterleavedSource& src, bool sig, int tile_bytes, int stages, int max_ctas,
                                     int dev, cudaStream_t st) {
  return launch_tiles_src(src, src.total_items, sig, tile_bytes, stages, max_ctas, dev, st);
}

dyna_status launch_copy(const Plan& p, int engine, int max_ctas, int stages, int unroll, int dev,
                        cudaStream_t st, int schedule) {
  SingleSource src{p};
  return launch_src(src, p.n_items, p.counters != nullptr, p.piece, engine, max_ctas, stages, unroll, dev, st,
                    schedule);
}

// ------------------------------------------------------------------ staged variant (a2, a3, a4)
static bool k2_dma() {
  static const bool on = [] {
    const char* e = std::getenv("DYNA_KV_K2_KERNEL");
    return !(e && e[0] == '1');
  }();
  return on;
}

// K1 gather -> source staging slot, K2 slot -> destination-side slot, K3 scatter
// slot -> destination rows (+ per-chunk flag).  Chunks are cut into sub-chunks
// that fit one staging slot; two slots per side alternate.  Same device:
// everything in stream order.  Two devices of one process: K3 runs on a
// library stream of the destination device, ordered with events.
dyna_status run_staged(dyna_kv_pool* S, dyna_kv_pool* D, const int32_t* sids, const int32_t* dids, dyna_range tr,
                       int l0, int lm, int64_t c, bool signal, int engine, int piece, int stages, int unroll,
                       int max_ctas, cudaStream_t stream, dyna_kv_xfer* x, int schedule) {
  if (D->imported)
    return fail(DYNA_ENOTSUP, "STAGED variant into an imported (cross-process) pool: use the receiver-steered "
                              "channel (dyna_kv_push / dyna_kv_place) or FUSED");
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
  cudaEvent_t prev_done = nullptr;
  dyna_status r = channel_staging(S, D, slot, &sbuf, &dbuf, &prev_done);
  if (r) return r;
  // The staging slots belong to the (source, destination) pair: a STAGED migration on another
  // stream of the same pair must finish with them first (device-side order, no host wait).
  if (prev_done) CUDA_TRY(cudaStreamWaitEvent(stream, prev_done, 0));
  unsigned long long* counters = nullptr;
  unsigned long long* flags = nullptr;
  if (signal) {
    uint64_t epoch = 0;
    int32_t first = 0;
    if ((r = flag_reserve(S->desc.instance, D, nchunks, &epoch, &first))) return r;
    if ((r = channel_counters(S, D, D->dev, &counters))) return r;
    counters += first;
    flags = D->inbox + (size_t)S->desc.instance * DYNA_MAX_CHUNKS + first;
    x->epoch = epoch;
    x->first_slot = first;
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
      k1.err = x->err;
      if ((r = launch_copy(k1, engine, max_ctas, stages, unroll, S->dev, stream, schedule))) break;
      // K2: the sub-chunk slot [lm][2][n][row] is one contiguous range.  By default ONE copy-engine
      // transfer moves it (across devices a peer copy over NVLink: the paper's "DMA-pushed"),
      // which occupies no SM beside the producer; DYNA_KV_K2_KERNEL=1 moves it with the copy kernel
      // (a flat plan: two halves, K and V of all layers, of one `half`-byte token each).
      if (k2_dma()) {
        CUDA_TRY(cudaMemcpyAsync(dslot, sslot, (size_t)(2 * (sb - sa) * row * lm), cudaMemcpyDeviceToDevice, stream));
      } else {
        Plan k2 = make_plan(linear(sslot), linear(dslot), (sb - sa) * row * lm, 0, 1, 0, 1, 1, 1, piece);
        k2.err = x->err;
        if ((r = launch_copy(k2, engine, max_ctas, stages, unroll, S->dev, stream, schedule))) break;
      }
      Plan k3 = make_plan(linear(dslot), paged(D, dids), row, sa, sb, l0, lm, sb - sa, D->desc.block_size, piece);
      set_chunking(k3, tr.begin, tr.end, c);
      k3.err = x->err;
      if (signal) {
        k3.counters = counters;
        k3.flags = flags;
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
  if (!r) r = channel_staging_done(S, D, stream);
  return r;
}

dyna_status launch_batch(const BatchSource& src, int64_t n_items, bool sig, int piece, int engine, int max_ctas,
                         int stages, int unroll, int dev, cudaStream_t st, int schedule) {
  return launch_src(src, n_items, sig, piece, engine, max_ctas, stages, unroll, dev, st, schedule);
}

void launch_wait_flag(const unsigned long long* flag, unsigned long long epoch, unsigned long long timeout_ns,
                      cudaStream_t st, unsigned int* err) {
  k_wait_flag<<<1, 1, 0, st>>>(flag, epoch, timeout_ns, err);
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_release_sys(unsigned long long* slot, unsigned long long v, cudaStream_t st) {
  k_release_sys<<<1, 1, 0, st>>>(slot, v);
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_mark_ready(unsigned long long* slot, unsigned long long v, cudaStream_t st) {
  k_mark_ready<<<1, 1, 0, st>>>(slot, v);
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

dyna_status launch_fill(void* dst, uint64_t bytes, unsigned long long key, uint64_t first_word, int dev,
                        cudaStream_t st) {
  DevInfo* di = dev_info(dev);
  const uint64_t n16 = bytes / 16;
  const unsigned grid = (unsigned)std::min<uint64_t>((n16 + 255) / 256, (uint64_t)di->sms * 8);
  k_fill<<<grid, 256, 0, st>>>(static_cast<ulonglong2*>(dst), n16, key, first_word);
  CUDA_TRY(cudaGetLastError());
  return DYNA_OK;
}

}  // namespace rt
}  // namespace dynakv

