// dyna_kv_kernels.cuh — sm_100a kernels of the chunked KV-cache migration.
//
// One templated copy-kernel family covers the paper's push (§4.3,
// P:556) in all its shapes:
//   K4 / K4-local  paged src  -> paged dst   (fused; dst local or NVLink peer)
//   K1 gather      paged src  -> linear staging slot
//   K2 transfer    linear     -> linear (peer staging)
//   K3 scatter     linear     -> paged dst
// Two copy engines share one work decomposition:
//   VEC   one warp per work item; 16-B vector loads (ld.global.nc) issued in
//         an unrolled batch, then 16-B stores.
//   BULK  one elected thread per CTA drives TMA bulk copies
//         (cp.async.bulk global->smem completing on an mbarrier, then
//         smem->global as a bulk group) through a multi-stage smem ring.
// The payload is never interpreted: every byte is copied untouched (DESIGN.md
// reading R8), so there is no arithmetic and no tensor-core work.
//
// Work decomposition (step a1, computed on the device from the item index;
// no host-side descriptor list):
//   chunk k   = tokens [t0 + k*c, min(t0 + (k+1)*c, t1))               (R5)
//   run j     = chunk ∩ [G*g, (G+1)*g), G = floor(a_k / g) + j.  g divides
//               both block sizes, so a run is one contiguous byte range in
//               the source AND in the destination.
//   piece p   = bytes [p*piece, (p+1)*piece) of the run
//   item      = (k, l, kv, j, p), chunk-major so chunk 0 completes first.
#pragma once
#include <cstdint>
#include <type_traits>

#include "plan.cuh"

#ifndef DYNA_VEC_MINB
#define DYNA_VEC_MINB 3  // resident 256-thread CTAs per SM the VEC engine (U <= 8) is compiled for
#endif

#ifndef DYNA_LANES_MINB
#define DYNA_LANES_MINB 2  // resident 256-thread CTAs per SM of k_copy_lanes (2: up to 128 registers, no spills;
                           // precomputed-item micro-benchmark: 2 CTAs/SM 3100 vs 3 CTAs/SM 2900 GB/s)
#endif

#ifndef DYNA_MAIL_SLEEP
#define DYNA_MAIL_SLEEP 0  // accountant poll back-off (ns); 0 = spin
#endif

#ifndef DYNA_BULK_DEFER
#define DYNA_BULK_DEFER 4  // stores committed after a chunk switch before its bytes are counted
#endif

namespace dynakv {

struct Item {
  const char* src;
  char* dst;
  uint32_t n;    // bytes to copy (multiple of 16); 0 = nothing to copy
  uint32_t acc;  // bytes this item accounts for in its chunk (== n unless skipped)
  int32_t k;     // chunk index within the migration
  int32_t l;     // layer
};

__device__ __forceinline__ int64_t side_row(const Side& s, const Plan& p, int l, int kv, int64_t t,
                                            int64_t a, int64_t clen, bool& bad) {
  if (s.linear) return (((int64_t)(l - p.l0) * 2 + kv) * clen + (t - a)) * p.row;
  const int64_t jb = t / s.bs;
  const int32_t b = __ldg(s.table + jb);
  if (b < 0 || (int64_t)b >= s.nb) { bad = true; return 0; }
  return ((((int64_t)l * 2 + kv) * s.nb + b) * s.bs + (t - jb * s.bs)) * p.row;
}

__device__ __forceinline__ Item decode_item(const Plan& p, int64_t item) {
  Item it{nullptr, nullptr, 0u, 0u, 0, 0};
  const int64_t k = item / p.items_per_chunk;
  int64_t i = item - k * p.items_per_chunk;
  const int32_t pp = (int32_t)(i % p.P); i /= p.P;
  int32_t j;
  int kv, l;
  if (p.J == p.R) {  // (layer, K|V) slowest: concurrent items walk the runs of one slab
    j = (int32_t)(i % p.R);  i /= p.R;
    kv = (int)(i & 1);
    l = p.l0 + (int)(i >> 1);
  } else {           // groups of J runs, each group over every (layer, K|V) slab
    const int32_t jj = (int32_t)(i % p.J);  i /= p.J;
    const int32_t lk = (int32_t)(i % (2 * p.lm));
    j = (int32_t)(i / (2 * p.lm)) * p.J + jj;  // j >= runs of the chunk: an empty item
    kv = lk & 1;
    l = p.l0 + (lk >> 1);
  }
  const int64_t a = p.t0 + k * p.c;
  const int64_t b = min(a + (int64_t)p.c, p.t1);
  const int64_t G = a / p.g + j;
  const int64_t ta = max(a, G * p.g);
  const int64_t tb = min(b, (G + 1) * p.g);
  it.k = p.k_direct ? (int32_t)k + p.k_base : (int32_t)((a - p.mig_t0) / p.sig_c);
  it.l = l;
  if (ta >= tb) return it;
  const int64_t run = (tb - ta) * p.row;
  const int64_t off = (int64_t)pp * p.piece;
  if (off >= run) return it;
  const uint32_t n = (uint32_t)min((int64_t)p.piece, run - off);
  it.acc = n;
  bool bad = false;
  const int64_t so = side_row(p.src, p, l, kv, ta, a, b - a, bad);
  const int64_t dO = side_row(p.dst, p, l, kv, ta, a, b - a, bad);
  if (bad) {  // out-of-range block id: skip these rows, report at dyna_kv_wait
    if (p.err) atomicOr(p.err, ERR_BAD_BLOCK);
    return it;
  }
  it.src = p.src.base + so + off;
  it.dst = p.dst.base + dO + off;
  it.n = n;
  return it;
}

// Head-sliced decode (dyna_kv_migrate_heads): the same chunk / run grid as
// decode_item, but a token's bytes are a slice of `p.row` bytes at byte col of a
// row of pitch bytes, so a run is `rows` slices at a stride, not one contiguous
// range.  piece p = tokens [ta + p*tpp, ...) of the run.
struct SItem {
  const char* src;
  char* dst;
  uint32_t rows;  // slices to copy; 0 = nothing
  uint32_t acc;   // bytes this item accounts for in its chunk
  int32_t k;
  int32_t l;
};

__device__ __forceinline__ int64_t side_slice(const Side& s, const Plan& p, int l, int kv, int64_t t, int64_t a,
                                              int64_t clen, int64_t pitch, int32_t col, bool& bad) {
  if (s.linear) return (((int64_t)(l - p.l0) * 2 + kv) * clen + (t - a)) * p.row;  // packed slices
  const int64_t jb = t / s.bs;
  const int32_t b = __ldg(s.table + jb);
  if (b < 0 || (int64_t)b >= s.nb) { bad = true; return 0; }
  return ((((int64_t)l * 2 + kv) * s.nb + b) * s.bs + (t - jb * s.bs)) * pitch + col;
}

__device__ __forceinline__ SItem decode_item_sliced(const Plan& p, int64_t item) {
  SItem it{nullptr, nullptr, 0u, 0u, 0, 0};
  const int64_t k = item / p.items_per_chunk;
  int64_t i = item - k * p.items_per_chunk;
  const int32_t pp = (int32_t)(i % p.P); i /= p.P;
  const int32_t j = (int32_t)(i % p.R);  i /= p.R;
  const int kv = (int)(i & 1);
  const int l = p.l0 + (int)(i >> 1);
  const int64_t a = p.t0 + k * p.c;
  const int64_t b = min(a + (int64_t)p.c, p.t1);
  const int64_t G = a / p.g + j;
  const int64_t ta = max(a, G * p.g);
  const int64_t tb = min(b, (G + 1) * p.g);
  it.k = p.k_direct ? (int32_t)k + p.k_base : (int32_t)((a - p.mig_t0) / p.sig_c);
  it.l = l;
  const int64_t ra = ta + (int64_t)pp * p.tpp;
  if (ra >= tb) return it;
  const uint32_t rows = (uint32_t)min((int64_t)p.tpp, tb - ra);
  it.acc = rows * (uint32_t)p.row;
  bool bad = false;
  const int64_t so = side_slice(p.src, p, l, kv, ra, a, b - a, p.spitch, p.scol, bad);
  const int64_t dO = side_slice(p.dst, p, l, kv, ra, a, b - a, p.dpitch, p.dcol, bad);
  if (bad) {
    if (p.err) atomicOr(p.err, ERR_BAD_BLOCK);
    return it;
  }
  it.src = p.src.base + so;
  it.dst = p.dst.base + dO;
  it.rows = rows;
  return it;
}

// A chunk flag is raised, never lowered: max with release semantics at system scope (the
// receiver may be another GPU).  Slot ranges recycle after DYNA_MAX_CHUNKS chunks; a late
// writer of an older epoch then cannot move a newer flag backwards.
__device__ __forceinline__ void raise_flag(unsigned long long* ptr, unsigned long long v) {
  asm volatile("red.release.sys.global.max.u64 [%0], %1;" ::"l"(ptr), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* ptr) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(ptr) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* ptr) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ptr) : "memory");
  return v;
}

// Producer coupling (§4.3, "once chunk k completes, its KV block
// is immediately DMA-pushed"): block until the producer marked ready slot `slot`
// (chunk k, or (chunk k, layer l) when marks are per layer).  Returns false when
// the migration was cancelled before the mark became visible: the caller skips
// the slot's items.  A visible mark always wins, so a marked slot is copied by
// every warp that owns part of it.  A wait that times out is treated like a cancel
// (ERR_TIMEOUT recorded): the slot's rows were never marked, so its chunk gets no flag.
__device__ __forceinline__ bool wait_ready(const Plan& p, int32_t slot) {
  if (ld_acquire_gpu(p.ready + slot) >= p.ready_epoch) return true;
  unsigned long long t0, now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (uint32_t polls = 0; ld_acquire_gpu(p.ready + slot) < p.ready_epoch; ++polls) {
    // the cancel word: read on the first poll and then every 32nd (~16 us)
    if (p.cancel && (polls & 31) == 0 && *p.cancel >= p.ready_epoch) return false;
    __nanosleep(500);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now - t0 > p.ready_timeout_ns) {  // never hang the device: report at dyna_kv_wait
      if (p.err) atomicOr(p.err, ERR_TIMEOUT);
      return false;
    }
  }
  return true;
}

// Bytes of global chunk k of the whole migration.
__device__ __forceinline__ unsigned long long chunk_bytes(const Plan& p, int32_t k) {
  const int64_t a = p.mig_t0 + (int64_t)k * p.sig_c;
  const int64_t b = min(a + (int64_t)p.sig_c, p.mig_t1);
  return (unsigned long long)((b - a) * p.row * p.lm * 2);
}

__device__ __forceinline__ void fence_for(const Plan& p) {
  if (p.sys_fence) __threadfence_system(); else __threadfence();
}

// Called by ONE thread once an item's bytes are complete and visible at
// the destination's scope (the caller fenced).  The thread that closes chunk k resets
// the counter (self-cleaning channel) and releases the flag.
// wait for the previous grid on the stream to complete, its memory visible (PdlScope below)
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void account_chunk(const Plan& p, int32_t k, unsigned long long n) {
  if (n == 0) return;
  if (p.overlap_prev & kOverlapCounters) griddep_wait();  // slots still counted by an earlier launch (PdlScope)
  unsigned long long* ctr = p.counters + k;
  const unsigned long long total = chunk_bytes(p, k);
  const unsigned long long now = atomicAdd(ctr, n) + n;
  if ((now & kCountMask) == total) {
    *ctr = 0ull;
    if (now >= kPoison) return;  // a part of the chunk was skipped (cancelled): no flag
    __threadfence_system();
    raise_flag(p.flags + k, p.epoch);
  }
}

// ------------------------------------------------------------------ programmatic dependent launch
// Launched with programmatic stream serialization, a copy kernel may start
// while the previous kernel on the stream drains.  It lets its own dependents
// start launching at once, then waits for the previous grid to complete (and
// its memory to be visible) before touching any global memory.  Without the
// launch attribute both instructions are no-ops.
//
// DYNA_MIGRATE_OVERLAP_PREV (the caller's promise that this launch neither reads nor writes what
// the previous kernel on the stream writes, nor writes what it reads): the copies start without
// that wait, so back-to-back independent migrations do not drain and refill the memory pipeline
// between launches (measured: the ~4-5 us bubble per launch).  The wait still
// happens (a) before the first touch of the library's chunk counters and flags when the host saw
// the launch's slots reserved recently by another launch that may still count them
// (kOverlapCounters, griddep_wait in account_chunk*), and (b) in CTA 0 before it exits
// (PdlScope's destructor), so the grid never completes before the previous kernel: work after it
// on the stream, events and dyna_kv_wait keep plain stream order.  Only CTA 0 holds its SM for
// that: the other CTAs exit when their copies are done, so the next launch's CTAs take their SMs
// at once (a per-thread exit wait measured most of the gain away: profiles/r02_overlap_prev_probe).

struct PdlScope {  // no state: CTA 0's exit wait is unconditional (a no-op once the entry wait has run)
  template <class Src>
  __device__ __forceinline__ explicit PdlScope(const Src& src) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifndef DYNA_DIAG_PDL_NOWAIT  // diagnostic builds only (A/B of the launch bubble): every launch overlaps
    if (!src.overlap()) griddep_wait();
#endif
  }
  __device__ __forceinline__ ~PdlScope() {
    if (blockIdx.x == 0) griddep_wait();
  }
};

// ------------------------------------------------------------------ work distribution
// Static round-robin (ctr == nullptr) or dynamic: workers grab the next item
// index from a per-launch counter ctr[0], prefetched one grab ahead so the
// atomic's latency overlaps the current item.  ctr[1] counts finished
// workers; the last one resets the slot for the launch that reuses it.
struct Sched {
  unsigned long long* ctr;
  int64_t next, stride;
  unsigned long long pre;
  __device__ __forceinline__ void init(unsigned long long* c, int64_t first, int64_t stride_) {
    ctr = c;
    next = first;
    stride = stride_;
    if (ctr) pre = atomicAdd(ctr, 1ull);
  }
  __device__ __forceinline__ int64_t get() {
    if (!ctr) {
      const int64_t r = next;
      next += stride;
      return r;
    }
    const int64_t r = (int64_t)pre;
    pre = atomicAdd(ctr, 1ull);
    return r;
  }
  __device__ __forceinline__ void finish(unsigned long long n_workers) {
    if (!ctr) return;
    __threadfence();  // this worker's grabs are performed before it counts itself done
    if (atomicAdd(ctr + 1, 1ull) == n_workers - 1) {
      __threadfence();
      ctr[0] = 0ull;
      ctr[1] = 0ull;
    }
  }
};

// Same as account_chunk, for a thread whose counted writes are already complete
// and proxy-fenced: the count itself is a release RMW at the destination's scope,
// instead of a full fence followed by a relaxed add.
__device__ __forceinline__ void account_chunk_release(const Plan& p, int32_t k, uint32_t n) {
  if (n == 0) return;
  if (p.overlap_prev & kOverlapCounters) griddep_wait();  // (as account_chunk)
  unsigned long long* ctr = p.counters + k;
  const unsigned long long total = chunk_bytes(p, k);
  unsigned long long old;
  if (p.sys_fence)
    asm volatile("atom.add.release.sys.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(ctr), "l"((unsigned long long)n) : "memory");
  else
    asm volatile("atom.add.release.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(ctr), "l"((unsigned long long)n) : "memory");
  if (old + n == total) {
    __threadfence_system();  // acquire the other contributors' releases before publishing
    *ctr = 0ull;
    raise_flag(p.flags + k, p.epoch);
  }
}

// ------------------------------------------------------------------ VEC engine
__device__ __forceinline__ int4 ld_nc_v4(const int4* ptr) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(ptr));
  return r;
}
__device__ __forceinline__ int4 ld_v4(const int4* ptr) {  // coherent: source may be written during the kernel
  int4 r;
  asm volatile("ld.global.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(ptr)
               : "memory");
  return r;
}
__device__ __forceinline__ void st_v4(int4* ptr, const int4& v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(ptr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

// A warp copies n bytes (multiple of 16): U 16-B loads per lane in flight.
template <int U, bool NC = true>
__device__ __forceinline__ void warp_copy(const char* __restrict__ src, char* __restrict__ dst, uint32_t n,
                                          int lane) {
  const int4* s = reinterpret_cast<const int4*>(src);
  int4* d = reinterpret_cast<int4*>(dst);
  const uint32_t nv = n >> 4;
  uint32_t base = 0;
  for (; base + 32 * U <= nv; base += 32 * U) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = NC ? ld_nc_v4(s + base + u * 32 + lane) : ld_v4(s + base + u * 32 + lane);
#pragma unroll
    for (int u = 0; u < U; ++u) st_v4(d + base + u * 32 + lane, v[u]);
  }
  if (base < nv) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t idx = base + u * 32 + lane;
      if (idx < nv) v[u] = NC ? ld_nc_v4(s + idx) : ld_v4(s + idx);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t idx = base + u * 32 + lane;
      if (idx < nv) st_v4(d + idx, v[u]);
    }
  }
}

// A warp copies `rows` slices of vps 16-B vectors, source rows spitch bytes apart, destination
// rows dpitch apart: lane-major over the flattened vector index, U loads in flight per lane.
// The geometry comes in by value: read through a Plan in global memory (batches), every field
// would be reloaded after each store (the stores' asm clobbers memory).
template <int U>
__device__ __forceinline__ void warp_copy_rows(const char* __restrict__ src, char* __restrict__ dst, uint32_t rows,
                                               uint32_t vps, int sh, int64_t spitch, int64_t dpitch, int lane) {
  const uint32_t nv = rows * vps;
  for (uint32_t base = 0; base < nv; base += 32 * U) {
    int4 v[U];
    uint32_t r[U], c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t idx = base + u * 32 + lane;
      r[u] = sh >= 0 ? (idx >> sh) : idx / vps;
      c[u] = idx - r[u] * vps;
      if (idx < nv)
        v[u] = ld_nc_v4(reinterpret_cast<const int4*>(src + (int64_t)r[u] * spitch + (int64_t)c[u] * 16));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t idx = base + u * 32 + lane;
      if (idx < nv) st_v4(reinterpret_cast<int4*>(dst + (int64_t)r[u] * dpitch + (int64_t)c[u] * 16), v[u]);
    }
  }
}

// VEC engine with warp-cooperative decode (static round-robin schedule, no ready board):
// the warp's next 32 items are decoded at once, one per lane, then copied one after the
// other with the fields broadcast by shuffles.  Same per-(warp, chunk) signalling as
// k_copy_vec; batches carry each item's plan (per-request flags).
template <int U, bool SIGNAL, class Src>
__global__ void __launch_bounds__(256, DYNA_LANES_MINB) k_copy_lanes(const Src src, unsigned long long* sched) {
  PdlScope pdl(src);
  constexpr bool kBatch = std::is_same<Src, BatchSource>::value;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_items = src.total();
  int32_t cur_k = -1;
  const Plan* cur_p = nullptr;
  unsigned long long cur_acc = 0;
  int64_t m = 0, seen = 0, dbase = 0;
  for (;;) {
    // this round's items: static = every nwarps-th item from warp + m*nwarps; dynamic (sched, a
    // per-launch counter slot) = a guided grab of up to 32 consecutive items by lane 0
    int64_t gi;
    int cnt;
    if (sched) {
      unsigned long long b = 0, grab = 0;
      if (lane == 0) {
        grab = (unsigned long long)max((int64_t)1, min((int64_t)32, (n_items - seen) / (4 * nwarps)));
        b = atomicAdd(sched, grab);
      }
      b = __shfl_sync(0xffffffffu, b, 0);
      grab = __shfl_sync(0xffffffffu, grab, 0);
      seen = (int64_t)(b + grab);
      if ((int64_t)b >= n_items) break;
      dbase = (int64_t)b;
      cnt = (int)min((int64_t)grab, n_items - dbase);
      gi = lane < cnt ? dbase + lane : n_items;
    } else {
      if (warp + m * nwarps >= n_items) break;
      cnt = (int)min((int64_t)32, (n_items - 1 - warp) / nwarps - m + 1);
      gi = warp + (m + lane) * nwarps;
      m += 32;
    }
    Item mine{nullptr, nullptr, 0u, 0u, 0, 0};
    const Plan* mp = nullptr;
    if (gi < n_items) {
      int64_t item = gi;
      const Plan& ip = src.locate(item);
      if (kBatch) mp = &ip;
      mine = decode_item(ip, item);
    }
    for (int j = 0; j < cnt; ++j) {
      const char* isrc = reinterpret_cast<const char*>(__shfl_sync(0xffffffffu, (unsigned long long)mine.src, j));
      char* idst = reinterpret_cast<char*>(__shfl_sync(0xffffffffu, (unsigned long long)mine.dst, j));
      const uint32_t n = __shfl_sync(0xffffffffu, mine.n, j);
      const uint32_t acc = __shfl_sync(0xffffffffu, mine.acc, j);
      const int32_t k = __shfl_sync(0xffffffffu, mine.k, j);
      const Plan* pj = kBatch ? reinterpret_cast<const Plan*>(__shfl_sync(0xffffffffu, (unsigned long long)mp, j))
                              : nullptr;
      if (SIGNAL && acc && (k != cur_k || (kBatch && pj != cur_p))) {
        if (cur_acc) {
          const Plan& cp = kBatch ? *cur_p : src.locate_signal();
          fence_for(cp);
          __syncwarp();
          if (lane == 0) account_chunk(cp, cur_k, cur_acc);
        }
        cur_k = k;
        if (kBatch) cur_p = pj;
        cur_acc = 0;
      }
      if (n) warp_copy<U>(isrc, idst, n, lane);
      if (SIGNAL) cur_acc += acc;
    }
  }
  if (SIGNAL && cur_acc) {
    const Plan& cp = kBatch ? *cur_p : src.locate_signal();
    fence_for(cp);
    __syncwarp();
    if (lane == 0) account_chunk(cp, cur_k, cur_acc);
  }
  // dynamic: the last warp past the end resets the launch's counter slot
  if (sched && lane == 0 && atomicAdd(sched + 1, 1ull) == (unsigned long long)nwarps - 1) {
    sched[0] = 0ull;
    sched[1] = 0ull;
  }
}

template <int U, bool SIGNAL, class Src, bool READY = false>
__global__ void __launch_bounds__(256, (U >= 16 || READY) ? 2 : DYNA_VEC_MINB) k_copy_vec(const Src src, unsigned long long* sched_ctr) {
  PdlScope pdl(src);
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  Sched sched;  // lane 0 grabs, the warp follows
  if (lane == 0) sched.init(sched_ctr, warp, nwarps);
  // Signalling: a warp's consecutive items mostly share a chunk (chunk-major
  // order), so bytes are accumulated per chunk and fenced + counted once when
  // the warp moves on to another chunk — one fence per (warp, chunk), not per item.
  constexpr bool kBatch = std::is_same<Src, BatchSource>::value;
  int32_t cur_k = -1;
  const Plan* cur_p = nullptr;     // batches: the plan (request) chunk cur_k belongs to (flags are per request)
  unsigned long long cur_acc = 0;  // bytes of chunk cur_k, plus kPoison once if any of them was skipped
  int32_t ready_slot = -1;
  bool skip = false;      // READY: the current ready slot was cancelled
  const int64_t n_items = src.total();
  for (;;) {
    long long gi = 0;
    if (lane == 0) gi = sched.get();
    const int64_t gitem = __shfl_sync(0xffffffffu, gi, 0);
    if (gitem >= n_items) break;
    int64_t item = gitem;
    const Plan& p = src.locate(item);
    const Item it = decode_item(p, item);
    if (SIGNAL && it.acc && (it.k != cur_k || (kBatch && &p != cur_p))) {
      if (cur_acc) {
        const Plan& cp = kBatch ? *cur_p : p;  // (single plan: always the same)
        fence_for(cp);  // every lane's stores of chunk cur_k are performed ...
        __syncwarp();   // ... before lane 0 counts them
        if (lane == 0) account_chunk(cp, cur_k, cur_acc);
      }
      cur_k = it.k;
      if (kBatch) cur_p = &p;
      cur_acc = 0;
    }
    if (READY && it.acc) {
      const int32_t slot = p.ready_layers ? it.k * p.lm + (it.l - p.l0) : it.k;
      if (slot != ready_slot) {  // warp-uniform
        int go = 1;
        if (lane == 0) go = wait_ready(p, slot) ? 1 : 0;
        skip = __shfl_sync(0xffffffffu, go, 0) == 0;
        ready_slot = slot;
      }
    }
    if (READY && skip) {  // cancelled before this slot was marked: count it poisoned, copy nothing
      if (SIGNAL) cur_acc = (cur_acc | kPoison) + it.acc;  // poison at most once per (warp, chunk)
      continue;
    }
    if (it.n) warp_copy<U, !READY>(it.src, it.dst, it.n, lane);
    if (SIGNAL) cur_acc += it.acc;
  }
  if (SIGNAL && cur_acc) {
    const Plan& cp = kBatch ? *cur_p : src.locate_signal();
    fence_for(cp);
    __syncwarp();
    if (lane == 0) account_chunk(cp, cur_k, cur_acc);
  }
  if (lane == 0) sched.finish((unsigned long long)nwarps);
}

// ------------------------------------------------------------------ BULK engine
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}


__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Accountant hand-off (signalling, ACC kernels): the copying thread posts (chunk, bytes)
// after its bulk groups completed and a proxy fence; mbarrier arrive = release at CTA scope,
// wait = acquire, so the accountant's GPU-scope fence + count covers the poster's writes.
constexpr int kMail = 16;
struct Mailbox {
  uint64_t full[kMail], empty[kMail];
  const Plan* pl[kMail];  // batches: the plan (request) the chunk belongs to; nullptr = the launch's plan
  int32_t k[kMail];
  uint32_t acc[kMail];
  __device__ __forceinline__ void init() {
    for (int m = 0; m < kMail; ++m) {
      mbar_init(&full[m], 1);
      mbar_init(&empty[m], 1);
    }
  }
  __device__ __forceinline__ void post(int64_t& n, int32_t kk, uint32_t a, const Plan* plan = nullptr) {
    const int m = (int)(n % kMail);
    if (n >= kMail) mbar_wait(&empty[m], (uint32_t)(((n / kMail) - 1) & 1));
    pl[m] = plan;
    k[m] = kk;
    acc[m] = a;
    mbar_arrive(&full[m]);
    ++n;
  }
  // the accountant's loop, until the poster's sentinel (chunk -1).  It takes every entry that
  // has already arrived, then fences ONCE for all of them and counts them: the GPU-scope fence
  // (which must cover the poster's bulk stores) is the expensive step, so under load one fence
  // serves many chunks (measured: DESIGN.md §6b, r02 signalling rows).
  __device__ __forceinline__ bool ready(int64_t i) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred P1;\n"
        " mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        " selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(done)
        : "r"(smem_u32(&full[i % kMail])), "r"((uint32_t)((i / kMail) & 1))
        : "memory");
    return done != 0;
  }
  __device__ __forceinline__ void serve(const Plan& p) {
    for (int64_t i = 0;;) {
#if DYNA_MAIL_SLEEP > 0
      while (!ready(i)) __nanosleep(DYNA_MAIL_SLEEP);
#else
      mbar_wait(&full[i % kMail], (uint32_t)((i / kMail) & 1));
#endif
      int n = 1;
      while (n < kMail && ready(i + n)) ++n;
      int32_t kk[kMail];
      uint32_t aa[kMail];
      const Plan* pp[kMail];
      bool last = false;
      int m = 0;
      for (; m < n; ++m) {
        const int s = (int)((i + m) % kMail);
        kk[m] = k[s];
        aa[m] = acc[s];
        pp[m] = pl[s];
        mbar_arrive(&empty[s]);
        if (kk[m] < 0) {
          last = true;
          break;
        }
      }
      if (m > 0) {
        bool sys = false;
        for (int j = 0; j < m; ++j) sys |= (pp[j] ? pp[j]->sys_fence : p.sys_fence) != 0;
        if (sys) __threadfence_system(); else __threadfence();
        for (int j = 0; j < m; ++j) account_chunk(pp[j] ? *pp[j] : p, kk[j], aa[j]);
      }
      if (last) return;
      i += n;
    }
  }
};

// ------------------------------------------------------------------ BULK engine, decoder-fed ring
// One thread (warp 0, lane 0) drives a ring of `stages` shared-memory slots of p.piece bytes:
// loads (cp.async.bulk, completing on the slot's mbarrier) land ahead of the store front, and a
// slot is reloaded once the bulk store issued from it has read it out.  It never decodes
// (round 1's kernels did, on the same thread): warp 1 decodes the CTA's items 32 at a time (one per lane: the divisions and the
// two block-table loads of decode_item, and the batch's plan lookup) into a shared-memory
// queue of descriptors, NQ batches ahead.  The issuer's loop is then: wait for a landed
// slot, issue its store, wait for an older store to have read its slot, read the next
// descriptor from shared memory, issue its load.  Measured with precomputed items
// (scripts/native/copy_micro.cu, profiles/r02_copy_micro.jsonl): this loop moves random
// 32-KiB blocks at 3120 GB/s payload, where the same loop with the decode inline reached
// 2746 (r01_l3_probe.json).
struct Desc {
  const char* src;
  char* dst;
  const Plan* pl;  // batches: the item's plan (per-request chunk flags); unused for one plan
  uint32_t n;
  int32_t k;
};
constexpr int kQ = 4;  // descriptor batches in flight (32 items each)

// The decoder warp's next 32 item indices (gi per lane; n_items = none).  Static: round-robin over the
// grid.  Dynamic (sched != nullptr, a per-launch counter slot): guided grabs — lane 0 takes up to 32
// consecutive items per atomic while plenty remain, fewer towards the end, so the CTAs finish together
// even when SMs run at different rates.  Returns true once this CTA has no items left (warp-uniform).
__device__ __forceinline__ bool next_items(unsigned long long* sched, int64_t n_items, int64_t& m, int64_t& seen,
                                           int lane, int64_t& gi) {
  if (sched) {
    unsigned long long base = 0, grab = 0;
    if (lane == 0) {
      const int64_t rem = n_items - seen;
      grab = (unsigned long long)max((int64_t)1, min((int64_t)32, rem / (4 * (int64_t)gridDim.x)));
      base = atomicAdd(sched, grab);
    }
    base = __shfl_sync(0xffffffffu, base, 0);
    grab = __shfl_sync(0xffffffffu, grab, 0);
    seen = (int64_t)(base + grab);
    gi = (unsigned long long)lane < grab ? (int64_t)base + lane : n_items;
    return seen >= n_items;  // the counter has passed the end: every later grab is empty
  }
  gi = blockIdx.x + (m + lane) * (int64_t)gridDim.x;
  m += 32;
  return blockIdx.x + m * (int64_t)gridDim.x >= n_items;
}

// A decoder done with its grabs counts its CTA out; the last CTA past the end resets the launch's
// counter slot (every grab of the launch has returned by then: a CTA counts itself only after its
// final grab).
__device__ __forceinline__ void release_grabs(unsigned long long* sched, int lane) {
  if (sched && lane == 0 && atomicAdd(sched + 1, 1ull) == gridDim.x - 1) {
    sched[0] = 0ull;
    sched[1] = 0ull;
  }
}


template <bool SIGNAL, class Src, bool ACC = false>
__global__ void __launch_bounds__(ACC ? 96 : 64) k_copy_ring(const Src src, int stages, int lag,
                                                              unsigned long long* sched) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[kMaxStages];
  __shared__ __align__(8) uint64_t qfull[kQ], qempty[kQ];
  __shared__ __align__(8) Desc q[kQ][32];
  __shared__ int32_t qcount[kQ], qlast[kQ];
  __shared__ char* pend_dst[kMaxStages];
  __shared__ const Plan* pend_pl[kMaxStages];
  __shared__ uint32_t pend_n[kMaxStages];
  __shared__ int32_t pend_k[kMaxStages];
  __shared__ __align__(8) Mailbox mail[1];  // (ACC only)
  constexpr bool kBatch = std::is_same<Src, BatchSource>::value;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    for (int b = 0; b < kQ; ++b) {
      mbar_init(&qfull[b], 32);  // one arrive per decoder lane
      mbar_init(&qempty[b], 1);
    }
    if (ACC) mail[0].init();
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  PdlScope pdl(src);
  const Plan& p = src.locate_signal();  // per-launch fields (piece, signalling)
  const int64_t n_items = src.total();
  if (warp == 1) {  // ---------------- decoder
    int64_t m = 0;
    int64_t seen = 0;  // dynamic: the counter as last observed (guides the grab size)
    for (int64_t b = 0;; ++b) {
      const int qb = (int)(b % kQ);
      if (b >= kQ) mbar_wait(&qempty[qb], (uint32_t)(((b / kQ) - 1) & 1));
      int64_t gi;
      const bool last = next_items(sched, n_items, m, seen, lane, gi);
      Item it{nullptr, nullptr, 0u, 0u, 0, 0};
      const Plan* ipl = nullptr;
      if (gi < n_items) {
        int64_t item = gi;
        const Plan& ip = src.locate(item);
        ipl = kBatch ? &ip : nullptr;
        it = decode_item(ip, item);
        if (SIGNAL && it.n == 0 && it.acc) account_chunk(ip, it.k, it.acc);  // skipped (bad id): still closes the chunk
      }
      const unsigned mask = __ballot_sync(0xffffffffu, it.n != 0);
      if (it.n) q[qb][__popc(mask & ((1u << lane) - 1u))] = Desc{it.src, it.dst, ipl, it.n, it.k};
      if (lane == 0) {
        qcount[qb] = __popc(mask);
        qlast[qb] = last ? 1 : 0;
      }
      mbar_arrive(&qfull[qb]);  // every lane releases its own descriptor write (CTA scope)
      if (last) {
        release_grabs(sched, lane);
        return;
      }
    }
  }
  if (ACC && warp == 2) {  // ---------------- accountant
    if (lane == 0) mail[0].serve(p);
    return;
  }
  if (lane != 0) return;
  // ---------------- issuer (warp 0, lane 0)
  const int64_t piece = p.piece;
  int64_t qb = -1;
  int pos = 0, cnt = 0;
  bool qdone = false;
  int64_t posted = 0;
  auto refill = [&](int s) {
    while (pos == cnt) {
      if (qdone) {
        pend_n[s] = 0;
        return;
      }
      if (qb >= 0) mbar_arrive(&qempty[qb % kQ]);
      ++qb;
      const int qi = (int)(qb % kQ);
      mbar_wait(&qfull[qi], (uint32_t)((qb / kQ) & 1));
      cnt = qcount[qi];
      qdone = qlast[qi] != 0;
      pos = 0;
    }
    const Desc d = q[qb % kQ][pos++];
    mbar_expect_tx(&full[s], d.n);
    bulk_load(ring + s * piece, d.src, d.n, &full[s]);
    pend_dst[s] = d.dst;
    pend_n[s] = d.n;
    pend_k[s] = d.k;
    if (kBatch) pend_pl[s] = d.pl;
  };
  for (int s = 0; s < stages; ++s) refill(s);

  // Signalling: stores are counted per chunk (per (plan, chunk) in a batch).  When the next
  // store belongs to another chunk, the finished chunk's bytes are parked and counted once
  // kDefer more stores were committed after them, behind a wait_group kDefer.
  constexpr int kDefer = DYNA_BULK_DEFER;
  int32_t cur_k = -1, park_k = -1;
  const Plan *cur_pl = nullptr, *park_pl = nullptr;
  uint32_t cur_acc = 0, park_acc = 0;
  int since_park = 0;
  auto flush_park = [&](bool all) {
#ifndef DYNA_DIAG_NO_WAIT  // (DYNA_DIAG_*: unsafe diagnostic builds that drop one step each)
    if (all) bulk_wait_all<0>(); else bulk_wait_all<kDefer>();
#endif
#ifndef DYNA_DIAG_NO_PROXY
    asm volatile("fence.proxy.async.global;" ::: "memory");
#endif
#ifndef DYNA_DIAG_NO_COUNT
    if (ACC) mail[0].post(posted, park_k, park_acc, park_pl);
    else account_chunk_release(kBatch ? *park_pl : p, park_k, park_acc);
#endif
    park_k = -1;
    park_acc = 0;
  };
  for (int64_t iter = 0;; ++iter) {
    const int s = (int)(iter % stages);
    if (pend_n[s] == 0) break;
    if (SIGNAL && (pend_k[s] != cur_k || (kBatch && pend_pl[s] != cur_pl))) {
      if (park_acc) flush_park(true);
      park_k = cur_k;
      park_pl = cur_pl;
      park_acc = cur_acc;
      since_park = 0;
      cur_k = pend_k[s];
      if (kBatch) cur_pl = pend_pl[s];
      cur_acc = 0;
    }
    mbar_wait(&full[s], (uint32_t)((iter / stages) & 1));
    bulk_store(pend_dst[s], ring + s * piece, pend_n[s]);
    bulk_commit();
    if (SIGNAL) {
      cur_acc += pend_n[s];
      if (park_acc && ++since_park == kDefer) flush_park(false);
    }
    if (iter >= lag) {
      if (lag == 2) bulk_wait_read<2>(); else bulk_wait_read<1>();  // store iter-lag done reading smem
      refill((int)((iter - lag) % stages));
    }
  }
  bulk_wait_all<0>();
  if (SIGNAL) {
    if (park_acc) flush_park(true);
    if (cur_acc) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      if (ACC) {
        mail[0].post(posted, cur_k, cur_acc, cur_pl);
      } else {
        const Plan& P = kBatch ? *cur_pl : p;
        fence_for(P);
        account_chunk(P, cur_k, cur_acc);
      }
    }
  }
  if (ACC) mail[0].post(posted, -1, 0);  // the accountant may leave
}

// ------------------------------------------------------------------ head-sliced rows, decoder-fed
// dyna_kv_migrate_heads / dyna_kv_reshard: a token's bytes are a slice of a row, so an item is
// `rows` slices at a stride (4 KiB for 16 tokens x 256 B) — small items, where the per-item
// decode (five 64-bit divisions, two dependent block-table loads; for a reshard also the plan
// lookup) used to sit between a warp's copies.  Warp 0 of each CTA decodes the CTA's items 32
// at a time (one per lane) into a shared-memory queue, kQ batches ahead; the other kCopiers
// warps take descriptors round-robin and only copy (lane-major over 16-B vectors, U loads in
// flight per lane).  A micro-benchmark of the same access pattern with precomputed items moves
// 256-B slices of 2-KiB rows at 2790-2880 GB/s payload (profiles/r02_copy_micro_rows.jsonl).
struct SDesc {
  const char* src;
  char* dst;
  const Plan* pl;    // multi-plan launches: the item's plan (per-entry chunk flags)
  int64_t spitch, dpitch;
  uint32_t rows, acc;
  int32_t k;
  uint16_t vps;
  int16_t sh;
};
constexpr int kCopiers = 7;

template <int U, bool SIGNAL, class Src>
__global__ void __launch_bounds__(32 * (kCopiers + 1), 3) k_copy_rows(const Src src) {
  constexpr bool kMulti = !std::is_same<Src, SingleSource>::value;
  __shared__ __align__(16) SDesc q[kQ][32];
  __shared__ int32_t qcount[kQ], qlast[kQ];
  __shared__ __align__(8) uint64_t qfull[kQ], qempty[kQ];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int b = 0; b < kQ; ++b) {
      mbar_init(&qfull[b], 32);  // one arrive per decoder lane
      mbar_init(&qempty[b], 32 * kCopiers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  PdlScope pdl(src);
  const int64_t n_items = src.total();
  if (warp == 0) {  // ---------------- decoder
    int64_t m = 0;
    for (int64_t b = 0;; ++b) {
      const int qb = (int)(b % kQ);
      if (b >= kQ) mbar_wait(&qempty[qb], (uint32_t)(((b / kQ) - 1) & 1));
      const int64_t gi = blockIdx.x + (m + lane) * (int64_t)gridDim.x;
      m += 32;
      SItem it{nullptr, nullptr, 0u, 0u, 0, 0};
      const Plan* ipl = nullptr;
      if (gi < n_items) {
        int64_t item = gi;
        const Plan& ip = src.locate(item);
        ipl = &ip;
        it = decode_item_sliced(ip, item);
        if (SIGNAL && it.rows == 0 && it.acc) account_chunk(ip, it.k, it.acc);  // skipped (bad id)
      }
      const unsigned mask = __ballot_sync(0xffffffffu, it.rows != 0);
      if (it.rows) {
        SDesc d;
        d.src = it.src;
        d.dst = it.dst;
        d.pl = kMulti ? ipl : nullptr;
        d.spitch = ipl->spitch;
        d.dpitch = ipl->dpitch;
        d.rows = it.rows;
        d.acc = it.acc;
        d.k = it.k;
        d.vps = (uint16_t)ipl->vps;
        d.sh = (int16_t)ipl->vps_shift;
        q[qb][__popc(mask & ((1u << lane) - 1u))] = d;
      }
      const bool last = blockIdx.x + m * (int64_t)gridDim.x >= n_items;
      if (lane == 0) {
        qcount[qb] = __popc(mask);
        qlast[qb] = last ? 1 : 0;
      }
      mbar_arrive(&qfull[qb]);  // every lane releases its own descriptor write (CTA scope)
      if (last) return;
    }
  }
  // ---------------- copiers: descriptor i of each batch goes to copier i % kCopiers
  const int cw = warp - 1;
  int32_t cur_k = -1;
  const Plan* cur_p = nullptr;
  uint32_t cur_acc = 0;
  const Plan* single = kMulti ? nullptr : &src.locate_signal();
  for (int64_t b = 0;; ++b) {
    const int qb = (int)(b % kQ);
    mbar_wait(&qfull[qb], (uint32_t)((b / kQ) & 1));
    const int cnt = qcount[qb];
    const bool last = qlast[qb] != 0;
    for (int i = cw; i < cnt; i += kCopiers) {
      const SDesc d = q[qb][i];
      const Plan* dp = kMulti ? d.pl : single;
      if (SIGNAL && d.acc && (d.k != cur_k || (kMulti && dp != cur_p))) {
        if (cur_acc) {
          fence_for(*cur_p);
          __syncwarp();
          if (lane == 0) account_chunk(*cur_p, cur_k, cur_acc);
        }
        cur_k = d.k;
        cur_p = dp;
        cur_acc = 0;
      }
      warp_copy_rows<U>(d.src, d.dst, d.rows, d.vps, d.sh, d.spitch, d.dpitch, lane);
      if (SIGNAL) cur_acc += d.acc;
    }
    mbar_arrive(&qempty[qb]);  // every copier lane releases its own descriptor reads
    if (last) break;
  }
  if (SIGNAL && cur_acc) {
    fence_for(*cur_p);
    __syncwarp();
    if (lane == 0) account_chunk(*cur_p, cur_k, cur_acc);
  }
}

// ------------------------------------------------------------------ head slices as TMA tensor tiles
// The BULK engine for head slices (dyna_kv_migrate_heads / dyna_kv_reshard).  A 256-B slice of
// a 2-KiB row is too small for one bulk op, and k_copy_rows' 16-B loads stop at ~0.88 of the
// copy peak even with precomputed items (profiles/r02_copy_micro_rows.jsonl).  But the slices a
// run needs form a regular lattice in both pools: `rows` slices at the row pitch, and the same
// rows of every (layer, K|V) slab at the slab pitch (NB*bs*pitch; the layout is
// [l][kv][block][token][row]).  A 4-D tensor map per side
// (slice elements, -, row in slab, slab) turns one run across `lkb` slabs into ONE tensor load
// (strided global -> dense shared memory) and ONE tensor store (dense shared -> strided global),
// e.g. 16 rows x 256 B x 8 slabs = 32 KiB per op, with the TMA unit doing the striding.
// A run shorter than the box (ragged chunk boundary or range end) is moved as one single-row
// box per row (maps 2 and 3).  lkb divides 2*lm, so no box is ever clipped.
// Decode, queue, issuer loop and signalling are k_copy_ring's.
struct TDesc {
  const char* tm;   // the item's TileMaps
  const Plan* pl;   // multi-plan launches: the item's plan (per-entry chunk flags)
  int32_t ys, yd;   // row coordinates (within a slab) in the source / destination maps
  int32_t lk;       // first slab of the box (relative to 2*l0)
  uint32_t rows;    // == g: one run box; < g: one row box per row
  uint32_t acc;     // bytes counted for the item's chunk
  int32_t k;
};

__device__ __forceinline__ void tma_load_4d(void* sdst, const char* tmap, int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5}], [%6];" ::"r"(smem_u32(sdst)),
      "l"(tmap), "r"(0), "r"(0), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const char* tmap, const void* ssrc, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(tmap),
               "r"(0), "r"(0), "r"(c2), "r"(c3), "r"(smem_u32(ssrc))
               : "memory");
}

// Item = (chunk k, slab group, run j, piece pp), pieces fastest; a piece is tile_rows rows of the run
// (all of it unless a run's rows do not fit one box).  Paged sides only (tile plans are never linear).
__device__ __forceinline__ TDesc decode_item_tile(const Plan& p, int64_t item, bool& skipped) {
  TDesc d{p.tmaps, nullptr, 0, 0, 0, 0u, 0u, 0};
  skipped = false;
  const int64_t k = item / p.items_per_chunk;
  int64_t i = item - k * p.items_per_chunk;
  const int32_t pp = (int32_t)(i % p.P);
  i /= p.P;
  const int32_t j = (int32_t)(i % p.R);
  const int32_t lkg = (int32_t)(i / p.R);
  const int64_t a = p.t0 + k * p.c;
  const int64_t b = min(a + (int64_t)p.c, p.t1);
  const int64_t G = a / p.g + j;
  const int64_t ra = max(a, G * p.g) + (int64_t)pp * p.tile_rows;
  const int64_t ta = ra, tb = min(min(b, (G + 1) * p.g), ra + p.tile_rows);
  d.k = p.k_direct ? (int32_t)k + p.k_base : (int32_t)((a - p.mig_t0) / p.sig_c);
  if (ta >= tb) return d;
  d.lk = lkg * p.lkb;
  d.acc = (uint32_t)((tb - ta) * p.row * p.lkb);
  // row coordinate in a side's map: the paged row through the block table, or the chunk-relative
  // row of a linear side (a tile plan with a linear side has one chunk: a = t0)
  bool bad = false;
  auto row_of = [&](const Side& sd) -> int32_t {
    if (sd.linear) return (int32_t)(ta - a);
    const int64_t jb = ta / sd.bs;
    const int32_t blk = __ldg(sd.table + jb);
    if (blk < 0 || (int64_t)blk >= sd.nb) {
      bad = true;
      return 0;
    }
    return (int32_t)((int64_t)blk * sd.bs + (ta - jb * sd.bs));
  };
  d.ys = row_of(p.src);
  d.yd = row_of(p.dst);
  if (bad) {
    if (p.err) atomicOr(p.err, ERR_BAD_BLOCK);
    skipped = true;
    return d;
  }
  d.rows = (uint32_t)(tb - ta);
  return d;
}

template <bool SIGNAL, class Src, bool ACC = false>
__global__ void __launch_bounds__(ACC ? 96 : 64) k_copy_tiles(const Src src, int stages, int lag,
                                                               unsigned long long* sched) {
  extern __shared__ __align__(1024) unsigned char tile_ring[];
  __shared__ __align__(8) uint64_t full[kMaxStages];
  __shared__ __align__(8) uint64_t qfull[kQ], qempty[kQ];
  __shared__ __align__(8) TDesc q[kQ][32];
  __shared__ int32_t qcount[kQ], qlast[kQ];
  __shared__ TDesc pend[kMaxStages];
  __shared__ __align__(8) Mailbox mail[1];  // (ACC only)
  constexpr bool kMulti = !std::is_same<Src, SingleSource>::value;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    for (int b = 0; b < kQ; ++b) {
      mbar_init(&qfull[b], 32);  // one arrive per decoder lane
      mbar_init(&qempty[b], 1);
    }
    if (ACC) mail[0].init();
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  PdlScope pdl(src);
  const Plan& p = src.locate_signal();  // per-launch fields (box geometry, signalling)
  const int64_t n_items = src.total();
  if (warp == 1) {  // ---------------- decoder
    int64_t m = 0, seen = 0;
    for (int64_t b = 0;; ++b) {
      const int qb = (int)(b % kQ);
      if (b >= kQ) mbar_wait(&qempty[qb], (uint32_t)(((b / kQ) - 1) & 1));
      int64_t gi;
      const bool last = next_items(sched, n_items, m, seen, lane, gi);
      TDesc d{nullptr, nullptr, 0, 0, 0, 0u, 0u, 0};
      if (gi < n_items) {
        int64_t item = gi;
        const Plan& ip = src.locate(item);
        bool skipped = false;
        d = decode_item_tile(ip, item, skipped);
        d.pl = kMulti ? &ip : nullptr;
        if (SIGNAL && skipped) account_chunk(ip, d.k, d.acc);  // bad id: still closes the chunk
      }
      const unsigned mask = __ballot_sync(0xffffffffu, d.rows != 0);
      if (d.rows) q[qb][__popc(mask & ((1u << lane) - 1u))] = d;
      if (lane == 0) {
        qcount[qb] = __popc(mask);
        qlast[qb] = last ? 1 : 0;
      }
      mbar_arrive(&qfull[qb]);  // every lane releases its own descriptor write (CTA scope)
      if (last) {
        release_grabs(sched, lane);
        return;
      }
    }
  }
  if (ACC && warp == 2) {  // ---------------- accountant
    if (lane == 0) mail[0].serve(p);
    return;
  }
  if (lane != 0) return;
  // ---------------- issuer (warp 0, lane 0); the box geometry is the launch's (every plan of a
  // multi-plan tile launch has the same g, row, lkb and slot: checked on the host)
  const int32_t slot = p.tile_bytes;
  const uint32_t g = (uint32_t)p.tile_rows;  // rows of a full box
  const uint32_t row_box = (uint32_t)(p.row * p.lkb);  // bytes of one single-row box
  const uint32_t rstride = (uint32_t)p.tile_rstride;   // its smem stride (128-B aligned)
  // Maps were written by a host copy: acquire them for the tensormap proxy before first use.  Up to
  // 64 plans all at once here (round-robin launches change plans every item), else lazily.
  const char* fenced = nullptr;
  bool all_fenced = false;
  if constexpr (kMulti) {
    if (src.n <= 64) {
      for (int r = 0; r < src.n; ++r)
        for (int t = 0; t < kTileMaps; ++t)
          asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(src.plans[r].tmaps +
                                                                                      t * kTileMapBytes)
                       : "memory");
      all_fenced = true;
    }
  }
  int64_t qb = -1;
  int pos = 0, cnt = 0;
  bool qdone = false;
  int64_t posted = 0;
  auto refill = [&](int s) {
    while (pos == cnt) {
      if (qdone) {
        pend[s].rows = 0;
        return;
      }
      if (qb >= 0) mbar_arrive(&qempty[qb % kQ]);
      ++qb;
      const int qi = (int)(qb % kQ);
      mbar_wait(&qfull[qi], (uint32_t)((qb / kQ) & 1));
      cnt = qcount[qi];
      qdone = qlast[qi] != 0;
      pos = 0;
    }
    const TDesc d = q[qb % kQ][pos++];
    if (!all_fenced && d.tm != fenced) {
      for (int t = 0; t < kTileMaps; ++t)
        asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(d.tm + t * kTileMapBytes)
                     : "memory");
      fenced = d.tm;
    }
    unsigned char* sl = tile_ring + (size_t)s * slot;
    mbar_expect_tx(&full[s], d.rows * row_box);
    if (d.rows == g) {
      tma_load_4d(sl, d.tm, d.ys, d.lk, &full[s]);
    } else {
      for (uint32_t r = 0; r < d.rows; ++r) tma_load_4d(sl + r * rstride, d.tm + 2 * kTileMapBytes, d.ys + r, d.lk, &full[s]);
    }
    pend[s] = d;
  };
  for (int s = 0; s < stages; ++s) refill(s);

  constexpr int kDefer = DYNA_BULK_DEFER;
  int32_t cur_k = -1, park_k = -1;
  const Plan *cur_pl = nullptr, *park_pl = nullptr;
  uint32_t cur_acc = 0, park_acc = 0;
  int since_park = 0;
  auto flush_park = [&](bool all) {
    if (all) bulk_wait_all<0>(); else bulk_wait_all<kDefer>();
    asm volatile("fence.proxy.async.global;" ::: "memory");
    if (ACC) mail[0].post(posted, park_k, park_acc, park_pl);
    else account_chunk_release(kMulti ? *park_pl : p, park_k, park_acc);
    park_k = -1;
    park_acc = 0;
  };
  for (int64_t iter = 0;; ++iter) {
    const int s = (int)(iter % stages);
    const TDesc d = pend[s];
    if (d.rows == 0) break;
    if (SIGNAL && (d.k != cur_k || (kMulti && d.pl != cur_pl))) {
      if (park_acc) flush_park(true);
      park_k = cur_k;
      park_pl = cur_pl;
      park_acc = cur_acc;
      since_park = 0;
      cur_k = d.k;
      if (kMulti) cur_pl = d.pl;
      cur_acc = 0;
    }
    mbar_wait(&full[s], (uint32_t)((iter / stages) & 1));
    const unsigned char* sl = tile_ring + (size_t)s * slot;
    if (d.rows == g) {
      tma_store_4d(d.tm + kTileMapBytes, sl, d.yd, d.lk);
    } else {
      for (uint32_t r = 0; r < d.rows; ++r) tma_store_4d(d.tm + 3 * kTileMapBytes, sl + r * rstride, d.yd + r, d.lk);
    }
    bulk_commit();
    if (SIGNAL) {
      cur_acc += d.acc;
      if (park_acc && ++since_park == kDefer) flush_park(false);
    }
    if (iter >= lag) {
      if (lag == 2) bulk_wait_read<2>(); else bulk_wait_read<1>();  // store iter-lag done reading smem
      refill((int)((iter - lag) % stages));
    }
  }
  bulk_wait_all<0>();
  if (SIGNAL) {
    if (park_acc) flush_park(true);
    if (cur_acc) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      if (ACC) {
        mail[0].post(posted, cur_k, cur_acc, cur_pl);
      } else {
        const Plan& P = kMulti ? *cur_pl : p;
        fence_for(P);
        account_chunk(P, cur_k, cur_acc);
      }
    }
  }
  if (ACC) mail[0].post(posted, -1, 0);  // the accountant may leave
}

// ------------------------------------------------------------------ consumer-side chunk wait
__global__ void k_wait_flag(const unsigned long long* flag, unsigned long long epoch,
                            unsigned long long timeout_ns, unsigned int* err) {
  unsigned long long t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  while (ld_acquire_sys(flag) < epoch) {
    if (timeout_ns) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t_start > timeout_ns) {
        if (err) atomicOr(err, ERR_TIMEOUT);
        return;
      }
    }
    __nanosleep(256);
  }
}

// ------------------------------------------------------------------ producer side of the ready board
__global__ void k_mark_ready(unsigned long long* slot, unsigned long long epoch) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(slot), "l"(epoch) : "memory");
}

// Credit return of a placement channel: the slot may be overwritten once this
// runs (stream-ordered after the scatter that read it); system scope, the
// sender polls it from another GPU.
__global__ void k_release_sys(unsigned long long* slot, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(slot), "l"(v) : "memory");
}

// ------------------------------------------------------------------ test-input generator (not the method)
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void k_fill(ulonglong2* dst, uint64_t n16, unsigned long long key, uint64_t first_word) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
    const uint64_t w = first_word + 2 * i;
    ulonglong2 v;
    v.x = splitmix64(key ^ (w * 0xD1B54A32D192ED03ull));
    v.y = splitmix64(key ^ ((w + 1) * 0xD1B54A32D192ED03ull));
    dst[i] = v;
  }
}

}  // namespace dynakv
