// plan.cuh — the work description shared by the host runtime and the kernels
// (dyna_kv_kernels.cuh).  One Plan describes one launch of the copy kernels:
// which rows (a paged pool through a block table, or a linear staging slot)
// go where, in which chunking, and how completion is signalled.
#pragma once
#include <cstdint>

namespace dynakv {

struct Side {
  char* base;            // pool base, or staging base for a linear side
  const int32_t* table;  // block table (paged side); nullptr for a linear side
  int64_t nb;            // blocks in the pool (paged side)
  int32_t bs;            // tokens per block (paged side)
  int32_t linear;        // 1: staging layout [l-l0][kv][t-a][row] of one chunk
};

struct Plan {
  Side src, dst;
  int64_t row;              // bytes of one token's K or V in one layer (multiple of 16)
  int64_t t0, t1;           // token range of this launch
  int32_t l0, lm;           // first layer, number of layers
  int32_t c;                // chunk tokens
  int32_t g;                // run grid in tokens
  int32_t R;                // max runs per chunk
  int32_t P;                // pieces per run
  int32_t piece;            // bytes per piece (multiple of 16)
  int32_t nchunks;
  int64_t items_per_chunk;  // lm * 2 * R * P
  int64_t n_items;          // nchunks * items_per_chunk
  // The migration's own chunking (a launch may cover a sub-range of it,
  // e.g. one staging sub-chunk): flags and counters are per migration chunk.
  int64_t mig_t0, mig_t1;   // the whole migration's token range
  int32_t sig_c;            // the migration's chunk tokens
  int32_t J;                // runs per group: item order inside a chunk is (run group, l, kv, run, piece); J == R: (l, kv, run, piece)
  int32_t k_direct;         // 1: launch chunk k is migration chunk k + k_base (no division in the decode)
  int32_t k_base;
  // per-chunk completion signal (counters == nullptr: none)
  unsigned long long* counters;  // on the launching device, self-resetting
  unsigned long long* flags;     // destination inbox row of this sender
  unsigned long long epoch;
  int32_t sys_fence;             // 1: destination on another GPU (fence at system scope)
  unsigned int* err;             // deferred error word (mapped host memory)
  // producer coupling (nullptr: none): chunk k may be read only once ready[k] >= ready_epoch
  const unsigned long long* ready;
  unsigned long long ready_epoch;
  unsigned long long ready_timeout_ns;  // give up (ERR_TIMEOUT) after this long without the mark
  int32_t ready_layers;     // 0: one mark per chunk (slot k); 1: one per (chunk, layer) (slot k*lm + l-l0)
  // cancellation of a producer-coupled migration (nullptr: none): once *cancel >= ready_epoch,
  // chunks whose mark is not visible are skipped (device word, DMA-written by dyna_kv_ready_cancel)
  const volatile unsigned long long* cancel;
  // head-sliced rows (dyna_kv_migrate_heads; k_copy_vec<..., SLICED>): `row` is then the
  // slice of n_heads*d*e bytes moved per token, found at byte `col` of a pitch-byte row
  int64_t spitch, dpitch;   // bytes between consecutive tokens' rows (paged side: H*d*e of that pool)
  int32_t scol, dcol;       // byte offset of the slice inside a row
  int32_t tpp;              // tokens per work item
  int32_t vps, vps_shift;   // 16-B vectors per slice; log2(vps) or -1
  // TMA tensor tiles (k_copy_tiles: head slices on the BULK engine).  An item is one run of a
  // chunk across `lkb` consecutive (layer, K|V) slabs: a box of slice x rows x lkb, moved by
  // one tensor load and one tensor store through the maps at `tmaps` (global memory, 64-B
  // aligned: source run box, destination run box, source row box, destination row box).
  const char* tmaps;        // nullptr: not a tile plan
  int32_t lkb;              // slabs per box (divides 2*lm)
  int32_t tile_bytes;       // shared-memory ring slot: a full-run box (g * row * lkb B), or the single-row
                            // boxes of a shorter run at tile_rstride apart, rounded up to 1 KiB
  int32_t tile_rstride;     // smem stride of single-row boxes: row * lkb rounded up to 128 B (TMA alignment)
  int32_t tile_rows;        // rows of a full box: g, or a divisor of g when g rows do not fit (pieces of a run)
  // DYNA_MIGRATE_OVERLAP_PREV: kOverlapCopy = the launch does not wait for the previous kernel on
  // its stream before copying (CTA 0 waits before it exits: see PdlScope); kOverlapCounters = its
  // flag slots were reserved recently by another launch, so it also waits before it touches them
  int32_t overlap_prev;
};
constexpr int32_t kOverlapCopy = 1, kOverlapCounters = 2;
constexpr int kTileMapBytes = 128;  // sizeof(CUtensorMap)
constexpr int kTileMaps = 4;        // per plan

enum : unsigned { ERR_BAD_BLOCK = 1u, ERR_TIMEOUT = 2u };

// A skipped (cancelled) item adds its bytes plus this poison to its chunk's
// counter: the counter still completes and self-resets, but no flag is raised.
constexpr unsigned long long kPoison = 1ull << 48;
constexpr unsigned long long kCountMask = kPoison - 1;

constexpr int kMaxStages = 16;  // BULK ring depth limit

// Where a kernel's items come from: one plan (by value, in the constant bank),
// or a batch of plans in global memory with an exclusive prefix of item counts
// (dyna_kv_migrate_batch: many requests, one launch).
struct SingleSource {
  Plan p;
  __device__ __forceinline__ int64_t total() const { return p.n_items; }
  __device__ __forceinline__ const Plan& locate(int64_t& item) const { return p; }
  __device__ __forceinline__ const Plan& locate_signal() const { return p; }
  __device__ __forceinline__ bool overlap() const { return p.overlap_prev != 0; }
};
struct BatchSource {
  const Plan* plans;
  const int64_t* base;  // base[r] = first global item of plan r; nondecreasing
  int32_t n;
  int64_t total_items;
  int64_t payload;      // bytes the batch moves (host-side launch decisions; item slots can be empty)
  __device__ __forceinline__ int64_t total() const { return total_items; }
  __device__ __forceinline__ const Plan& locate(int64_t& item) const {
    int lo = 0, hi = n - 1;  // the last r with base[r] <= item
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (__ldg(base + mid) <= item) lo = mid; else hi = mid - 1;
    }
    item -= __ldg(base + lo);
    return plans[lo];
  }
  __device__ __forceinline__ const Plan& locate_signal() const { return plans[0]; }
  // plans live in library memory written by a copy the launch fully depends on: readable before the
  // grid-dependency wait
  __device__ __forceinline__ bool overlap() const { return plans[0].overlap_prev != 0; }
};
// n plans with identical item structure (dyna_kv_reshard: one request's head slices between
// TP ranks), one launch, items entry-major: global item g is item g % per of plan g / per.
// (Interleaving the plans item by item, so neighbouring warps move the slices of the same
// token rows together, measured 0.37-0.63 of the HBM peak vs 0.71-0.86 entry-major:
// profiles/r02_reshard_interleaved.json.)
struct InterleavedSource {
  const Plan* plans;
  int32_t n;
  int64_t total_items;
  int64_t payload;      // bytes the launch moves (host-side launch decisions)
  __device__ __forceinline__ int64_t total() const { return total_items; }
  __device__ __forceinline__ const Plan& locate(int64_t& item) const {
    const int64_t per = total_items / n;
    const int32_t r = (int32_t)(item / per);
    item -= (int64_t)r * per;
    return plans[r];
  }
  __device__ __forceinline__ const Plan& locate_signal() const { return plans[0]; }
  // plans live in library memory written by a copy the launch fully depends on: readable before the
  // grid-dependency wait
  __device__ __forceinline__ bool overlap() const { return plans[0].overlap_prev != 0; }
};

}  // namespace dynakv
