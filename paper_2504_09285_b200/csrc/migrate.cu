// migrate.cu — the push itself (§4.3): validation, variant /
// engine choice from the calibration table, host-resident tables through the
// upload ring, dyna_kv_migrate(_ex/_batch/_on_ready), and completion (wait, query,
// per-chunk flags on the receiver).
#include "runtime.cuh"

using namespace dynakv;
using namespace dynakv::rt;

namespace dynakv {
namespace rt {

static bool capturing(cudaStream_t stream) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(stream, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone;
}

// A migration handle with its own deferred-error word (the process-wide word when the
// stream is being captured: a graph's kernels keep writing after the handle is released).
dyna_status new_xfer(int dev, int sender, cudaStream_t stream, dyna_kv_xfer** out) {
  auto* x = new dyna_kv_xfer();
  x->dev = dev;
  x->sender = sender;
  x->err = capturing(stream) ? err_word() : err_acquire();
  if (!x->err) {
    delete x;
    return fail(DYNA_ENOMEM, "no deferred-error word");
  }
  *out = x;
  return DYNA_OK;
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

// ------------------------------------------------------------------ shared validation
dyna_status check_opts(const dyna_kv_opts* opts, dyna_kv_opts* o) {
  *o = dyna_kv_opts{};
  if (opts) *o = *opts;
  if ((o->flags & ~(DYNA_MIGRATE_SIGNAL | DYNA_READY_PER_LAYER | DYNA_MIGRATE_UNCHECKED | DYNA_MIGRATE_OVERLAP_PREV)) != 0 ||
      o->variant < 0 ||
      o->variant > 2 || o->engine < 0 || o->engine > DYNA_ENGINE_TILES || o->max_ctas < 0 || o->piece_bytes < 0 ||
      o->piece_bytes % 16 || o->stages < 0 || o->stages == 1 || o->stages > kMaxStages ||
      (o->unroll != 0 && o->unroll != 4 && o->unroll != 8 && o->unroll != 16) || o->schedule < 0 ||
      o->schedule > DYNA_SCHED_DYNAMIC)
    return fail(DYNA_EINVAL, "invalid dyna_kv_opts");
  return DYNA_OK;
}

// DYNA_MIGRATE_OVERLAP_PREV -> Plan::overlap_prev.  Not for dynamically scheduled launches (their
// per-launch counter slots are recycled by the previous launch's last CTA), producer-coupled ones
// (resident waiters) or the staged chain (its kernels depend on each other): those keep the wait.
static int32_t overlap_of(const dyna_kv_opts& o) {
  return (o.flags & DYNA_MIGRATE_OVERLAP_PREV) && o.schedule != DYNA_SCHED_DYNAMIC ? 1 : 0;
}

// Geometry, ranges and table presence; with host ids, the id range checks and the rows for the
// alias check of reading R7 (appended to dsp / ssp; the caller runs check_alias over a whole
// call or batch).  Without DYNA_MIGRATE_UNCHECKED the destination table must carry host ids
// (and so must the source table when it reads the destination pool), so that aliasing is
// always checked.  src_spans: 0 = source rows only when source and destination pool coincide,
// 1 = always (batches: another entry may write this source pool).  *empty: nothing to move.
dyna_status validate_pair(const dyna_block_table& src, const dyna_block_table& dst, dyna_range tr, dyna_range lr,
                          int32_t chunk_tokens, bool unchecked, bool* empty, std::vector<Span>& dsp,
                          std::vector<Span>& ssp, int src_spans, bool heads_may_differ, int32_t who) {
  if (!src.pool || !dst.pool) return fail(DYNA_EINVAL, "NULL pool in a block table");
  const dyna_kv_pool_desc &gs = src.pool->desc, &gd = dst.pool->desc;
  if (gs.num_layers != gd.num_layers || (!heads_may_differ && gs.num_kv_heads != gd.num_kv_heads) ||
      gs.head_dim != gd.head_dim || gs.elem_bytes != gd.elem_bytes)
    return fail(DYNA_EGEOM, heads_may_differ ? "source and destination geometry differ (L, d, e)"
                                             : "source and destination geometry differ (L, H, d, e)");
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
  bool same = false;
  if (pools_overlap(src.pool, dst.pool, &same) && !same)
    return fail(DYNA_EALIAS, "source and destination pools overlap in memory without being the same pool");
  if (!unchecked && !dst.host_block_ids)
    return fail(DYNA_EINVAL, "destination aliasing (reading R7) is checked on the host: give the destination "
                             "table's host_block_ids, or pass DYNA_MIGRATE_UNCHECKED");
  if (!unchecked && same && !src.host_block_ids)
    return fail(DYNA_EINVAL, "source and destination are one pool: give the source table's host_block_ids "
                             "too, or pass DYNA_MIGRATE_UNCHECKED");
  dyna_status r;
  if (dst.host_block_ids && (r = table_spans(dst, tr.begin, tr.end, dsp, who))) return r;
  if (src.host_block_ids) {
    if (src_spans || same) {
      if ((r = table_spans(src, tr.begin, tr.end, ssp, who))) return r;
    } else {  // range check only
      const int64_t bs = gs.block_size;
      for (int64_t j = tr.begin / bs; j <= (tr.end - 1) / bs; ++j) {
        const int32_t id = src.host_block_ids[j];
        if (id < 0 || id >= gs.num_blocks)
          return fail(DYNA_ERANGE, "block_ids[%lld] = %d outside [0, %lld)", (long long)j, id,
                      (long long)gs.num_blocks);
      }
    }
  }
  return DYNA_OK;
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

// a6: unset choices come from the calibration table (measured GB/s per row
// bytes, locality and call size), else FUSED + VEC.
Choice choose(const dyna_kv_opts& o, int64_t row, int peer, int64_t ntok, int64_t run_bytes) {
  dyna_kv_calib_entry ce{};
  bool exact = false;
  const bool calibrated =
      (o.variant == DYNA_VARIANT_AUTO || o.engine == DYNA_ENGINE_AUTO) && calib_lookup(row, peer, ntok, &ce, &exact);
  Choice c{};
  c.exact = calibrated && exact;
  c.variant = o.variant ? o.variant : (calibrated && ce.variant ? ce.variant : DYNA_VARIANT_FUSED);
  c.engine = o.engine ? o.engine : (calibrated && ce.engine ? ce.engine : DYNA_ENGINE_VEC);
  const bool use_ce = calibrated && (!o.engine || o.engine == ce.engine);
  c.piece = o.piece_bytes ? o.piece_bytes
                          : (use_ce && ce.piece_bytes ? ce.piece_bytes
                                                     : (c.engine == DYNA_ENGINE_VEC ? kVecPiece : kBulkPiece));
  c.stages = o.stages ? o.stages : (use_ce && ce.stages ? ce.stages : kBulkStages);
  c.unroll = o.unroll ? o.unroll : (use_ce && ce.unroll ? ce.unroll : kVecU);
  if (c.engine == DYNA_ENGINE_TILES && c.variant == DYNA_VARIANT_STAGED) {  // tiles are a fused-variant engine
    c.engine = DYNA_ENGINE_VEC;
    c.unroll = kVecU;
    if (!o.piece_bytes) c.piece = kVecPiece;
  }
  if (!o.engine && c.engine != DYNA_ENGINE_VEC && c.engine != DYNA_ENGINE_TILES && run_bytes < kMinBulkRun) {
    // a BULK item never spans two blocks; with short contiguous runs (e.g. one KV
    // head per TP rank: 256-B rows, 4-KiB blocks) its single issuing thread is
    // bound by items, not bytes (measured: 341 GB/s) — many warps do better
    c.engine = DYNA_ENGINE_VEC;
    c.unroll = kVecU;
    if (!o.piece_bytes) c.piece = kVecPiece;
  }
  return c;
}

// Entries [0, last touched] of a table's host ids (what the kernel may read).
size_t table_upload_bytes(const dyna_block_table& t, int64_t t1) {
  return (size_t)((t1 - 1) / t.pool->desc.block_size + 1) * sizeof(int32_t);
}

}  // namespace rt
}  // namespace dynakv

extern "C" {

dyna_status dyna_kv_migrate(dyna_block_table src, dyna_block_table dst, dyna_range tr, dyna_range lr,
                            int32_t chunk_tokens, struct CUstream_st* stream, dyna_kv_xfer_t* out) {
  return dyna_kv_migrate_ex(src, dst, tr, lr, chunk_tokens, stream, nullptr, out);
}

// A chunk stream's call: one chunk of a logical migration that started at mig_t0; its flag
// goes to slot first_slot + (t0 - mig_t0) / c of the stream's reserved slots (nslots of them).
struct ChunkCtx {
  int64_t mig_t0;
  uint64_t epoch;
  int32_t first_slot, nslots;
};
static dyna_status migrate_impl(dyna_block_table src, dyna_block_table dst, dyna_range tr, dyna_range lr,
                                int32_t chunk_tokens, struct CUstream_st* stream_, const dyna_kv_opts* opts,
                                dyna_kv_ready* board, uint64_t ready_epoch, dyna_kv_xfer_t* out,
                                const ChunkCtx* ctx = nullptr);

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

static dyna_kv_xfer* empty_xfer(const dyna_kv_pool* S) {
  auto* x = new dyna_kv_xfer();
  x->dev = S->dev;
  x->sender = S->desc.instance;
  x->empty = true;
  return x;
}

// Host-resident tables (block_ids == NULL): upload the entries the kernels may read.
// Host-resident tables (and, for tile plans, `head_bytes` of tensor maps at the front, 256-B
// aligned on the device: *dhead) go up in one upload-ring span on the stream.
static dyna_status upload_tables(RingLease& lease, const dyna_block_table& src, const dyna_block_table& dst,
                                 int64_t t1, cudaStream_t stream, const int32_t** sids, const int32_t** dids,
                                 const void* head = nullptr, size_t head_bytes = 0, const char** dhead = nullptr) {
  *sids = src.block_ids;
  *dids = dst.block_ids;
  if (*sids && *dids && head_bytes == 0) return DYNA_OK;
  const size_t hb = (head_bytes + 255) & ~size_t(255);
  const size_t sb = *sids ? 0 : (table_upload_bytes(src, t1) + 15) & ~size_t(15);
  const size_t db = *dids ? 0 : table_upload_bytes(dst, t1);
  char *base = nullptr, *h = nullptr;
  dyna_status r = lease.reserve(hb + sb + db, &base, &h, stream);
  if (r) return r;
  if (head_bytes) std::memcpy(h, head, head_bytes);
  if (!*sids) std::memcpy(h + hb, src.host_block_ids, table_upload_bytes(src, t1));
  if (!*dids) std::memcpy(h + hb + sb, dst.host_block_ids, db);
  if ((r = lease.copy(stream))) return r;
  if (!*sids) *sids = reinterpret_cast<const int32_t*>(base + hb);
  if (!*dids) *dids = reinterpret_cast<const int32_t*>(base + hb + sb);
  if (dhead) *dhead = base;
  return DYNA_OK;
}

// Head slices: the TMA tile engine (k_copy_tiles) for DYNA_ENGINE_BULK / BULK_WS, and for AUTO
// when the geometry fits a tensor map; otherwise the VEC row kernel.
static bool stream_capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone;
}
// AUTO keeps peer destinations (another GPU, or an imported pool) on VEC: tensor stores into peer
// memory have not been measured on a multi-GPU box; explicit BULK allows them.
static bool want_tiles(const dyna_kv_opts& o, bool peer) {
  if (o.engine == DYNA_ENGINE_BULK || o.engine == DYNA_ENGINE_BULK_WS || o.engine == DYNA_ENGINE_TILES) return true;
  return o.engine == DYNA_ENGINE_AUTO && tiles_enabled() && !peer;
}

// Where a tile plan's maps come from: the channel's cached device copy (*cached), else the host
// copy in `maps`, uploaded with the call's tables (not under capture: a replay would read recycled
// upload-ring staging).  False: neither (the caller does not tile).
static dyna_status tile_maps(dyna_kv_pool* S, const dyna_kv_pool* D, const Plan& p, cudaStream_t st,
                             const char** cached, char* maps, bool* ok) {
  *ok = false;
  dyna_status r = channel_tile_maps(S, D, p, S->dev, st, cached);
  if (r) return r;
  *ok = *cached || (!stream_capturing(st) && tile_encode(p, maps));
  return DYNA_OK;
}

static dyna_status migrate_impl(dyna_block_table src, dyna_block_table dst, dyna_range tr, dyna_range lr,
                                int32_t chunk_tokens, struct CUstream_st* stream_, const dyna_kv_opts* opts,
                                dyna_kv_ready* board, uint64_t ready_epoch, dyna_kv_xfer_t* out,
                                const ChunkCtx* ctx) {
  if (!out) return fail(DYNA_EINVAL, "NULL out");
  *out = nullptr;
  dyna_kv_opts o{};
  dyna_status r = check_opts(opts, &o);
  if (r) return r;
  if (ctx) {  // chunk streams: one fused launch per chunk, flags in the stream's slots
    if (o.variant == DYNA_VARIANT_STAGED) return fail(DYNA_ENOTSUP, "chunk stream: FUSED variant only");
    o.variant = DYNA_VARIANT_FUSED;
  }
  bool empty = false;
  std::vector<Span> dsp, ssp;
  const bool unchecked = (o.flags & DYNA_MIGRATE_UNCHECKED) != 0;
  if ((r = validate_pair(src, dst, tr, lr, chunk_tokens, unchecked, &empty, dsp, ssp, 0, false))) return r;
  if (!empty && (r = check_alias(dsp, ssp))) return r;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  dyna_kv_pool* S = src.pool;
  dyna_kv_pool* D = dst.pool;
  const dyna_kv_pool_desc &gs = S->desc, &gd = D->desc;
  const int64_t ntok = tr.end - tr.begin;
  const int64_t nchunks = empty ? 0 : (ntok + chunk_tokens - 1) / chunk_tokens;
  const bool signal = (o.flags & DYNA_MIGRATE_SIGNAL) != 0;
  if (signal && nchunks > DYNA_MAX_CHUNKS)
    return fail(DYNA_ERANGE, "%lld chunks > DYNA_MAX_CHUNKS (%d) with signalling", (long long)nchunks,
                DYNA_MAX_CHUNKS);
  if (ctx && signal && (tr.begin - ctx->mig_t0) / chunk_tokens + nchunks > ctx->nslots)
    return fail(DYNA_ERANGE, "chunk stream: chunk beyond the %d flag slots reserved at open", ctx->nslots);
  if (board) {
    if (board->dev != src.pool->dev) return fail(DYNA_EINVAL, "ready board must live on the source device");
    const int64_t nslots = nchunks * ((o.flags & DYNA_READY_PER_LAYER) ? (lr.end - lr.begin) : 1);
    if (nslots > board->max_chunks)
      return fail(DYNA_ERANGE, "%lld ready slots (chunks%s) > the ready board's %d", (long long)nslots,
                  (o.flags & DYNA_READY_PER_LAYER) ? " x layers" : "", board->max_chunks);
    if (o.variant == DYNA_VARIANT_STAGED || (o.engine && o.engine != DYNA_ENGINE_VEC))
      return fail(DYNA_ENOTSUP, "producer-coupled migration: FUSED variant, VEC engine only");
  } else if (o.flags & DYNA_READY_PER_LAYER) {
    return fail(DYNA_EINVAL, "DYNA_READY_PER_LAYER needs a ready board (dyna_kv_migrate_on_ready)");
  }
  if (empty) {  // s = 0 (or no layers) -> nothing to ship, nothing enqueued
    *out = empty_xfer(S);
    return DYNA_OK;
  }
  if ((r = check_reach(S, D))) return r;
  if (!err_word()) return fail(DYNA_ECUDA, "no error word");

  const int64_t row = S->row;
  const int l0 = (int)lr.begin, lm = (int)(lr.end - lr.begin);
  const int64_t c = chunk_tokens;
  const int peer_dst = (D->dev != S->dev || D->imported) ? 1 : 0;
  Choice ch = choose(o, row, peer_dst, ntok, std::min<int64_t>(gcd64(gs.block_size, gd.block_size), c) * row);
  if ((o.flags & DYNA_MIGRATE_OVERLAP_PREV) && !o.engine && !o.max_ctas && !peer_dst && !board &&
      o.schedule != DYNA_SCHED_DYNAMIC && ch.variant == DYNA_VARIANT_FUSED && !(row >= 8192 && ntok >= 4096)) {
    // Overlapped calls: the VEC engine (two shared-memory-free CTAs per SM, so the next call's CTAs
    // share an SM with this call's tail; per-warp chunk counts) beats the ring / tiles, signalled or
    // not (profiles/r02_ov_shapes.jsonl: 2-KiB rows, 256-token signalled calls 0.67 -> 0.97 of the copy
    // peak); 8-KiB rows from 4096 tokens keep the table's ring (1.02 vs 0.96-1.00), and so do calls
    // under an SM budget (max_ctas: a few ring CTAs keep more bytes in flight than a few VEC CTAs,
    // profiles/r02_overlap_b.json)
    ch.engine = DYNA_ENGINE_VEC;
    ch.exact = true;  // a measured choice: no tile rule on top
    if (!o.piece_bytes) ch.piece = row < 2048 ? 4096 : 8192;
    if (!o.unroll) ch.unroll = row < 2048 ? 8 : 4;
  }
  if (board) {  // producer-coupled: the VEC engine (each warp waits on its own chunk's mark)
    ch.variant = DYNA_VARIANT_FUSED;
    ch.engine = DYNA_ENGINE_VEC;
    ch.unroll = 8;
    if (!o.piece_bytes) ch.piece = kVecPiece;
  }
  const int64_t g = gcd64(gs.block_size, gd.block_size);
  // Short contiguous runs (small rows: e.g. one KV head per TP rank, 256-B rows in 4-KiB blocks) on
  // the same device: AUTO moves whole rows as TMA tiles (a row is a slice of itself; one box spans
  // several (layer, K|V) slabs, so items are ~32 KiB whatever the block).
  alignas(64) char maps[kTileMaps * kTileMapBytes];
  Plan tp{};
  const char* cached = nullptr;
  // tiles: asked for (DYNA_ENGINE_TILES), chosen by the calibration table, or AUTO's rule for short
  // runs on one device
  const bool tiles_asked = o.engine == DYNA_ENGINE_TILES;
  const bool tiles_auto = !o.engine && (ch.engine == DYNA_ENGINE_TILES ||
                                        (!ch.exact && !peer_dst && ntok >= kTileMinTokens &&
                                         std::min<int64_t>(g, c) * row < kTileRunMax && tiles_enabled()));
  bool tiles = (tiles_asked || tiles_auto) && ch.variant == DYNA_VARIANT_FUSED && !board &&
               o.schedule != DYNA_SCHED_DYNAMIC &&
               tile_shape(tp = make_plan_sliced(paged(S, nullptr), paged(D, nullptr), row, row, 0, row, 0, tr.begin,
                                                tr.end, l0, lm, c, g, ch.piece));
  if (tiles && (r = tile_maps(S, D, tp, stream, &cached, maps, &tiles))) return r;
  if (tiles_asked && !tiles)
    return fail(DYNA_ENOTSUP, "DYNA_ENGINE_TILES: %s", ch.variant != DYNA_VARIANT_FUSED ? "fused variant only"
                                                       : board ? "not with a ready board"
                                                               : "rows no tensor map can describe (or capturing "
                                                                 "without cached maps)");
  if (!tiles && ch.engine == DYNA_ENGINE_TILES) {  // calibrated tiles that do not apply here: VEC
    ch.engine = DYNA_ENGINE_VEC;
    ch.unroll = kVecU;
    if (!o.piece_bytes) ch.piece = kVecPiece;
  }
  const bool up_maps = tiles && !cached;
  if (tiles) {
    ch.engine = DYNA_ENGINE_TILES;
    ch.piece = tp.tile_bytes;
    ch.stages = o.stages ? o.stages : 4;
  }
  const int variant = ch.variant, engine = ch.engine, piece = ch.piece, stages = ch.stages, unroll = ch.unroll;

  DeviceGuard guard(S->dev);
  if (variant == DYNA_VARIANT_STAGED && D->dev != S->dev && !dst.block_ids)
    return fail(DYNA_ENOTSUP, "cross-device STAGED needs device block_ids for the destination");
  RingLease lease(S->dev);
  const int32_t *sids = nullptr, *dids = nullptr;
  const char* dmaps = nullptr;
  if ((r = upload_tables(lease, src, dst, tr.end, stream, &sids, &dids, up_maps ? maps : nullptr,
                         up_maps ? sizeof(maps) : 0, &dmaps)))
    return r;

  dyna_kv_xfer* x = nullptr;
  if ((r = new_xfer(S->dev, gs.instance, stream, &x))) return r;
  x->nchunks = (int32_t)nchunks;
  x->variant = variant;
  x->engine = engine;
  x->piece = piece;
  x->stages = engine != DYNA_ENGINE_VEC ? stages : 0;
  x->unroll = engine == DYNA_ENGINE_VEC ? unroll : 0;
  const uint64_t launches0 = g_launches.load();
  if (variant == DYNA_VARIANT_FUSED) {
    // K4 / K4-local: source rows -> destination rows, one launch for all chunks.
    Plan p = tiles ? tp : make_plan(paged(S, sids), paged(D, dids), row, tr.begin, tr.end, l0, lm, c, g, piece);
    if (tiles) {
      p.src.table = sids;
      p.dst.table = dids;
      p.tmaps = cached ? cached : dmaps;
    }
    p.err = x->err;
    p.overlap_prev = board ? 0 : overlap_of(o);
    if (ctx) set_chunking(p, ctx->mig_t0, tr.end, c);
    if (signal) {
      uint64_t epoch = 0;
      int32_t first = 0;
      if (ctx) {
        epoch = ctx->epoch;
        first = ctx->first_slot;
      } else if ((r = flag_reserve(gs.instance, D, nchunks, &epoch, &first))) {
        delete x;
        return r;
      }
      if ((r = channel_counters(S, D, S->dev, &p.counters))) {
        delete x;
        return r;
      }
      p.counters += first;
      p.flags = D->inbox + (size_t)gs.instance * DYNA_MAX_CHUNKS + first;
      p.epoch = x->epoch = epoch;
      x->first_slot = first;
      p.sys_fence = peer_dst;
      if (p.overlap_prev && (ctx || flag_slots_shared_recently(gs.instance, D, first, nchunks)))
        p.overlap_prev |= kOverlapCounters;  // (a chunk stream's pushes share one reservation: always wait)
    }
    if (board) {
      p.ready = board->slots;
      p.ready_epoch = ready_epoch;
      p.ready_timeout_ns = board->timeout_ns;
      p.ready_layers = (o.flags & DYNA_READY_PER_LAYER) ? 1 : 0;
      p.cancel = board->cancel_dev;
      x->board = board;
      x->ready_epoch = ready_epoch;
      r = launch_ready(p, o.max_ctas, S->dev, stream, o.schedule);
    } else {
      r = tiles ? launch_tiles(p, stages, o.max_ctas, S->dev, stream)
                : launch_copy(p, engine, o.max_ctas, stages, unroll, S->dev, stream, o.schedule);
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

// ---------------------------------------------------------------- chunk streams
}  // extern "C"
struct dyna_kv_chunkstream {
  dyna_block_table src{}, dst{};
  int64_t begin = 0, produced_end = 0, pushed_end = 0;
  dyna_range layers{};
  int32_t c = 0;
  cudaStream_t stream = nullptr;
  dyna_kv_opts opts{};
  uint64_t epoch = 0;
  int32_t sender = 0, first_slot = 0, nslots = 0;
  bool closed = false;
  std::vector<dyna_kv_xfer_t> pushed;
};
extern "C" {

static dyna_status stream_push(dyna_kv_chunkstream* s, int64_t a, int64_t b) {
  ChunkCtx ctx{s->begin, s->epoch, s->first_slot, s->nslots};
  dyna_kv_xfer_t x = nullptr;
  dyna_status r = migrate_impl(s->src, s->dst, dyna_range{a, b}, s->layers, s->c,
                               reinterpret_cast<struct CUstream_st*>(s->stream), &s->opts, nullptr, 0, &x, &ctx);
  if (r) return r;
  s->pushed.push_back(x);
  s->pushed_end = b;
  return DYNA_OK;
}

dyna_status dyna_kv_chunkstream_open(dyna_block_table src, dyna_block_table dst, int64_t begin, dyna_range layer_range,
                                int32_t chunk_tokens, struct CUstream_st* stream, const dyna_kv_opts* opts,
                                dyna_kv_chunkstream_t* out) {
  if (!out) return fail(DYNA_EINVAL, "NULL out");
  *out = nullptr;
  if (!src.pool || !dst.pool) return fail(DYNA_EINVAL, "NULL pool in a block table");
  if (begin < 0 || chunk_tokens <= 0) return fail(DYNA_ERANGE, "begin >= 0 and chunk_tokens > 0");
  dyna_kv_opts o{};
  dyna_status r = check_opts(opts, &o);
  if (r) return r;
  if (o.variant == DYNA_VARIANT_STAGED || (o.flags & DYNA_READY_PER_LAYER))
    return fail(DYNA_ENOTSUP, "chunk stream: FUSED variant, SM engines, no ready board");
  auto* s = new dyna_kv_chunkstream();
  s->src = src;
  s->dst = dst;
  s->begin = s->produced_end = s->pushed_end = begin;
  s->layers = layer_range;
  s->c = chunk_tokens;
  s->stream = reinterpret_cast<cudaStream_t>(stream);
  s->opts = o;
  s->sender = src.pool->desc.instance;
  if (o.flags & DYNA_MIGRATE_SIGNAL) {
    // the destination table bounds the tokens the stream can ever push: reserve that many slots
    const int64_t cap_tok = std::max<int64_t>(0, dst.len * dst.pool->desc.block_size - begin);
    s->nslots = (int32_t)std::min<int64_t>(DYNA_MAX_CHUNKS, (cap_tok + chunk_tokens - 1) / chunk_tokens);
    if ((r = flag_reserve(s->sender, dst.pool, s->nslots, &s->epoch, &s->first_slot))) {
      delete s;
      return r;
    }
  }
  *out = s;
  return DYNA_OK;
}

dyna_status dyna_kv_chunkstream_produced(dyna_kv_chunkstream_t s, int64_t n_tokens, int32_t* pushed) {
  if (!s) return fail(DYNA_EINVAL, "NULL stream");
  if (pushed) *pushed = 0;
  if (s->closed) return fail(DYNA_EINVAL, "stream closed");
  if (n_tokens < 0) return fail(DYNA_EINVAL, "n_tokens >= 0");
  s->produced_end += n_tokens;
  int32_t n = 0;
  while (s->pushed_end + s->c <= s->produced_end) {  // every chunk that became full goes now
    dyna_status r = stream_push(s, s->pushed_end, s->pushed_end + s->c);
    if (r) return r;
    ++n;
  }
  if (pushed) *pushed = n;
  return DYNA_OK;
}

dyna_status dyna_kv_chunkstream_close(dyna_kv_chunkstream_t s, int32_t* pushed) {
  if (!s) return fail(DYNA_EINVAL, "NULL stream");
  if (pushed) *pushed = 0;
  if (s->closed) return DYNA_OK;
  s->closed = true;
  if (s->produced_end > s->pushed_end) {  // alpha ended: the open partial chunk goes now
    dyna_status r = stream_push(s, s->pushed_end, s->produced_end);
    if (r) return r;
    if (pushed) *pushed = 1;
  }
  return DYNA_OK;
}

dyna_status dyna_kv_chunkstream_info(dyna_kv_chunkstream_t s, uint64_t* epoch, int32_t* sender, int32_t* first_slot,
                                     int64_t* produced_end, int64_t* pushed_end, int32_t* num_pushed) {
  if (!s) return fail(DYNA_EINVAL, "NULL stream");
  if (epoch) *epoch = s->epoch;
  if (sender) *sender = s->sender;
  if (first_slot) *first_slot = s->first_slot;
  if (produced_end) *produced_end = s->produced_end;
  if (pushed_end) *pushed_end = s->pushed_end;
  if (num_pushed) *num_pushed = (int32_t)s->pushed.size();
  return DYNA_OK;
}

dyna_status dyna_kv_chunkstream_finish(dyna_kv_chunkstream_t s) {
  if (!s) return fail(DYNA_EINVAL, "NULL stream");
  dyna_status first = DYNA_OK;
  std::string msg;
  for (dyna_kv_xfer_t x : s->pushed) {
    dyna_status r = dyna_kv_wait(x);
    if (r && !first) {
      first = r;
      msg = g_err;
    }
  }
  delete s;
  if (first) return fail(first, "%s", msg.c_str());
  return DYNA_OK;
}

dyna_status dyna_kv_migrate_heads(dyna_block_table src, dyna_block_table dst, dyna_range tr, dyna_range lr,
                                  dyna_range src_heads, int32_t dst_head_begin, int32_t chunk_tokens,
                                  struct CUstream_st* stream_, const dyna_kv_opts* opts, dyna_kv_xfer_t* out) {
  if (!out) return fail(DYNA_EINVAL, "NULL out");
  *out = nullptr;
  dyna_kv_opts o{};
  dyna_status r = check_opts(opts, &o);
  if (r) return r;
  if (o.flags & DYNA_READY_PER_LAYER) return fail(DYNA_EINVAL, "DYNA_READY_PER_LAYER needs a ready board");
  bool empty = false;
  std::vector<Span> dsp, ssp;
  if ((r = validate_pair(src, dst, tr, lr, chunk_tokens, (o.flags & DYNA_MIGRATE_UNCHECKED) != 0, &empty, dsp, ssp,
                         0, true)))
    return r;
  dyna_kv_pool* S = src.pool;
  dyna_kv_pool* D = dst.pool;
  const dyna_kv_pool_desc &gs = S->desc, &gd = D->desc;
  const int64_t nh = src_heads.end - src_heads.begin;
  if (src_heads.begin < 0 || nh < 0 || src_heads.end > gs.num_kv_heads || dst_head_begin < 0 ||
      dst_head_begin + nh > gd.num_kv_heads)
    return fail(DYNA_ERANGE, "heads [%lld, %lld) of %d -> [%d, %lld) of %d", (long long)src_heads.begin,
                (long long)src_heads.end, gs.num_kv_heads, dst_head_begin, (long long)(dst_head_begin + nh),
                gd.num_kv_heads);
  for (Span& x : dsp) x.h0 = dst_head_begin, x.h1 = (int32_t)(dst_head_begin + nh);  // only these heads change
  for (Span& x : ssp) x.h0 = (int32_t)src_heads.begin, x.h1 = (int32_t)src_heads.end;
  if (!empty && (r = check_alias(dsp, ssp))) return r;
  const int64_t head_bytes = (int64_t)gs.head_dim * gs.elem_bytes;
  if ((nh * head_bytes) % 16 || head_bytes % 16)
    return fail(DYNA_EGEOM, "head slices must be multiples of 16 bytes (d*e = %lld)", (long long)head_bytes);
  if (nh == gs.num_kv_heads && nh == gd.num_kv_heads)  // whole rows on both sides: the plain migration
    return migrate_impl(src, dst, tr, lr, chunk_tokens, stream_, opts, nullptr, 0, out);
  if (o.variant == DYNA_VARIANT_STAGED) return fail(DYNA_ENOTSUP, "head-sliced migration: FUSED variant only");
  const int64_t ntok = tr.end - tr.begin;
  const int64_t nchunks = (empty || nh == 0) ? 0 : (ntok + chunk_tokens - 1) / chunk_tokens;
  const bool signal = (o.flags & DYNA_MIGRATE_SIGNAL) != 0;
  if (signal && nchunks > DYNA_MAX_CHUNKS)
    return fail(DYNA_ERANGE, "%lld chunks > DYNA_MAX_CHUNKS (%d) with signalling", (long long)nchunks, DYNA_MAX_CHUNKS);
  if (nchunks == 0) {
    *out = empty_xfer(S);
    return DYNA_OK;
  }
  if ((r = check_reach(S, D))) return r;
  if (!err_word()) return fail(DYNA_ECUDA, "no error word");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const int peer_dst = (D->dev != S->dev || D->imported) ? 1 : 0;
  const int piece = o.piece_bytes ? o.piece_bytes : kVecPiece;

  DeviceGuard guard(S->dev);
  const int l0 = (int)lr.begin, lm = (int)(lr.end - lr.begin);
  Plan p = make_plan_sliced(paged(S, nullptr), paged(D, nullptr), nh * head_bytes, S->row,
                            src_heads.begin * head_bytes, D->row, (int64_t)dst_head_begin * head_bytes, tr.begin,
                            tr.end, l0, lm, chunk_tokens, gcd64(gs.block_size, gd.block_size), piece);
  alignas(64) char maps[kTileMaps * kTileMapBytes];
  const char* cached = nullptr;
  bool tiles = want_tiles(o, peer_dst != 0) && tile_shape(p);
  if (tiles && (r = tile_maps(S, D, p, stream, &cached, maps, &tiles))) return r;
  if (!tiles && o.engine != DYNA_ENGINE_AUTO && o.engine != DYNA_ENGINE_VEC)
    return fail(DYNA_ENOTSUP, "head slices of %lld B on the BULK engine: the geometry does not fit a TMA tensor map "
                              "(or the stream is capturing without cached maps); use DYNA_ENGINE_VEC",
                (long long)(nh * head_bytes));
  if (!tiles)  // tile_shape may have reshaped the plan: the row kernel's plan
    p = make_plan_sliced(paged(S, nullptr), paged(D, nullptr), nh * head_bytes, S->row, src_heads.begin * head_bytes,
                         D->row, (int64_t)dst_head_begin * head_bytes, tr.begin, tr.end, l0, lm, chunk_tokens,
                         gcd64(gs.block_size, gd.block_size), piece);
  const bool up_maps = tiles && !cached;
  RingLease lease(S->dev);
  const int32_t *sids = nullptr, *dids = nullptr;
  const char* dmaps = nullptr;
  if ((r = upload_tables(lease, src, dst, tr.end, stream, &sids, &dids, up_maps ? maps : nullptr,
                         up_maps ? sizeof(maps) : 0, &dmaps)))
    return r;
  p.src.table = sids;
  p.dst.table = dids;
  if (tiles) p.tmaps = cached ? cached : dmaps;
  dyna_kv_xfer* x = nullptr;
  if ((r = new_xfer(S->dev, gs.instance, stream, &x))) return r;
  x->nchunks = (int32_t)nchunks;
  x->variant = DYNA_VARIANT_FUSED;
  x->engine = tiles ? DYNA_ENGINE_TILES : DYNA_ENGINE_VEC;
  x->piece = tiles ? p.tile_bytes : piece;
  x->unroll = tiles ? 0 : 8;
  x->stages = tiles ? (o.stages ? o.stages : 4) : 0;
  const uint64_t launches0 = g_launches.load();
  p.err = x->err;
  p.overlap_prev = overlap_of(o);
  if (signal) {
    uint64_t epoch = 0;
    int32_t first = 0;
    if ((r = flag_reserve(gs.instance, D, nchunks, &epoch, &first)) ||
        (r = channel_counters(S, D, S->dev, &p.counters))) {
      delete x;
      return r;
    }
    p.counters += first;
    p.flags = D->inbox + (size_t)gs.instance * DYNA_MAX_CHUNKS + first;
    p.epoch = x->epoch = epoch;
    x->first_slot = first;
    p.sys_fence = peer_dst;
    if (p.overlap_prev && flag_slots_shared_recently(gs.instance, D, first, nchunks))
      p.overlap_prev |= kOverlapCounters;
  }
  r = tiles ? launch_tiles(p, o.stages, o.max_ctas, S->dev, stream) : launch_rows(p, o.max_ctas, S->dev, stream);
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

// ---------------------------------------------------------------- pack / unpack (K1 / K3 as calls)
// One side of the push against a caller's contiguous buffer [l - l0][kv][t - t0][row]:
// pack = paged source rows -> buffer (the staged variant's K1 gather), unpack = buffer ->
// paged destination rows (K3 scatter).  Same kernels and engine choice as a migration.
static dyna_status pack_impl(bool to_buf, dyna_block_table t, dyna_range tr, dyna_range lr, char* buf,
                             uint64_t buf_bytes, struct CUstream_st* stream_, const dyna_kv_opts* opts,
                             dyna_kv_xfer_t* out) {
  if (!out) return fail(DYNA_EINVAL, "NULL out");
  *out = nullptr;
  dyna_kv_opts o{};
  dyna_status r = check_opts(opts, &o);
  if (r) return r;
  if (o.flags & (DYNA_MIGRATE_SIGNAL | DYNA_READY_PER_LAYER))
    return fail(DYNA_EINVAL, "pack / unpack: no per-chunk flags or ready boards");
  if (o.variant == DYNA_VARIANT_STAGED) return fail(DYNA_ENOTSUP, "pack / unpack: one kernel, no staged variant");
  if (!t.pool) return fail(DYNA_EINVAL, "NULL pool");
  dyna_kv_pool* P = t.pool;
  const dyna_kv_pool_desc& g = P->desc;
  if (lr.begin < 0 || lr.begin > lr.end || lr.end > g.num_layers) return fail(DYNA_ERANGE, "bad layer range");
  if (tr.begin < 0 || tr.begin > tr.end || tr.end >= (int64_t(1) << 31)) return fail(DYNA_ERANGE, "bad token range");
  const int64_t n = tr.end - tr.begin, lm = lr.end - lr.begin;
  if (n == 0 || lm == 0) {
    *out = empty_xfer(P);
    return DYNA_OK;
  }
  const uint64_t need = (uint64_t)lm * 2 * n * P->row;
  if (!buf || buf_bytes < need)
    return fail(DYNA_EINVAL, "buffer of %llu B < the %llu B the range needs", (unsigned long long)buf_bytes,
                (unsigned long long)need);
  if (reinterpret_cast<uintptr_t>(buf) % 16) return fail(DYNA_EINVAL, "buffer not 16-B aligned");
  if (tr.end > t.len * g.block_size) return fail(DYNA_ERANGE, "token range exceeds the block table");
  if (!t.block_ids && !t.host_block_ids) return fail(DYNA_EINVAL, "a block table has neither device nor host block ids");
  if (!to_buf && !(o.flags & DYNA_MIGRATE_UNCHECKED) && !t.host_block_ids)
    return fail(DYNA_EINVAL, "destination aliasing (reading R7) is checked on the host: give the destination "
                             "table's host_block_ids, or pass DYNA_MIGRATE_UNCHECKED");
  if (t.host_block_ids) {
    std::vector<Span> sp, none;
    if ((r = table_spans(t, tr.begin, tr.end, sp, -1))) return r;
    if (!to_buf && (r = check_alias(sp, none))) return r;
  }
  if (!err_word()) return fail(DYNA_ECUDA, "no error word");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  Choice ch = choose(o, P->row, 0, n, std::min<int64_t>(g.block_size, n) * P->row);
  DeviceGuard guard(P->dev);
  // Short runs as TMA tiles (the packed side is one chunk: a linear map of its own), as migrations
  // do; the maps travel with the call (the buffer is the caller's), so not under capture.
  const int l0 = (int)lr.begin;
  alignas(64) char maps[kTileMaps * kTileMapBytes];
  Plan tp{};
  const bool tiles_asked = o.engine == DYNA_ENGINE_TILES;
  bool tiles = (tiles_asked || (!o.engine && (ch.engine == DYNA_ENGINE_TILES ||
                                              (!ch.exact && n >= kTileMinTokens &&
                                               std::min<int64_t>(g.block_size, n) * P->row < kTileRunMax &&
                                               tiles_enabled())))) &&
               o.schedule != DYNA_SCHED_DYNAMIC && !stream_capturing(stream);
  if (tiles) {
    tp = to_buf ? make_plan_sliced(paged(P, nullptr), linear(buf), P->row, P->row, 0, P->row, 0, tr.begin, tr.end, l0,
                                   (int)lm, n, g.block_size, ch.piece)
                : make_plan_sliced(linear(buf), paged(P, nullptr), P->row, P->row, 0, P->row, 0, tr.begin, tr.end, l0,
                                   (int)lm, n, g.block_size, ch.piece);
    tiles = tile_shape(tp) && tile_encode(tp, maps);
  }
  if (tiles_asked && !tiles)
    return fail(DYNA_ENOTSUP, "DYNA_ENGINE_TILES: rows no tensor map can describe (or the stream is capturing)");
  if (tiles) {
    ch.engine = DYNA_ENGINE_TILES;
    ch.piece = tp.tile_bytes;
    ch.stages = o.stages ? o.stages : 4;
  } else if (ch.engine == DYNA_ENGINE_TILES) {
    ch.engine = DYNA_ENGINE_VEC;
    ch.unroll = kVecU;
    if (!o.piece_bytes) ch.piece = kVecPiece;
  }
  RingLease lease(P->dev);
  const int32_t* ids = t.block_ids;
  const char* dmaps = nullptr;
  if (!ids || tiles) {
    char *base = nullptr, *h = nullptr;
    const size_t hb = tiles ? sizeof(maps) : 0;  // 512: keeps the table 16-B aligned
    const size_t tb = ids ? 0 : table_upload_bytes(t, tr.end);
    if ((r = lease.reserve(hb + tb, &base, &h, stream))) return r;
    if (tiles) std::memcpy(h, maps, hb);
    if (!ids) std::memcpy(h + hb, t.host_block_ids, tb);
    if ((r = lease.copy(stream))) return r;
    if (!ids) ids = reinterpret_cast<const int32_t*>(base + hb);
    dmaps = base;
  }
  dyna_kv_xfer* x = nullptr;
  if ((r = new_xfer(P->dev, g.instance, stream, &x))) return r;
  x->variant = DYNA_VARIANT_FUSED;
  x->engine = ch.engine;
  x->piece = ch.piece;
  x->stages = ch.engine != DYNA_ENGINE_VEC ? ch.stages : 0;
  x->unroll = ch.engine == DYNA_ENGINE_VEC ? ch.unroll : 0;
  const uint64_t launches0 = g_launches.load();
  // one chunk of n tokens: the linear side's layout is [l - l0][kv][t - t0][row]
  Plan p = tiles ? tp
           : to_buf ? make_plan(paged(P, ids), linear(buf), P->row, tr.begin, tr.end, (int)lr.begin, (int)lm, n,
                                g.block_size, ch.piece)
                    : make_plan(linear(buf), paged(P, ids), P->row, tr.begin, tr.end, (int)lr.begin, (int)lm, n,
                                g.block_size, ch.piece);
  if (tiles) {
    (to_buf ? p.src : p.dst).table = ids;
    p.tmaps = dmaps;
  }
  p.err = x->err;
  p.overlap_prev = overlap_of(o);
  r = tiles ? launch_tiles(p, ch.stages, o.max_ctas, P->dev, stream)
            : launch_copy(p, ch.engine, o.max_ctas, ch.stages, ch.unroll, P->dev, stream, o.schedule);
  if (!r) r = lease.finish(stream);
  if (r) {
    delete x;
    return r;
  }
  x->launches = (int32_t)(g_launches.load() - launches0);
  if ((r = record_completion(x, P->dev, stream))) {
    delete x;
    return r;
  }
  *out = x;
  return DYNA_OK;
}

dyna_status dyna_kv_pack(dyna_block_table src, dyna_range tr, dyna_range lr, void* buf, uint64_t buf_bytes,
                         struct CUstream_st* stream, const dyna_kv_opts* opts, dyna_kv_xfer_t* out) {
  return pack_impl(true, src, tr, lr, static_cast<char*>(buf), buf_bytes, stream, opts, out);
}

dyna_status dyna_kv_unpack(const void* buf, uint64_t buf_bytes, dyna_block_table dst, dyna_range tr, dyna_range lr,
                           struct CUstream_st* stream, const dyna_kv_opts* opts, dyna_kv_xfer_t* out) {
  return pack_impl(false, dst, tr, lr, const_cast<char*>(static_cast<const char*>(buf)), buf_bytes, stream, opts,
                   out);
}

// ---------------------------------------------------------------- reshard: one request's head slices, one launch
// Every entry moves heads [src_heads) of its source rows into heads [dst_head_begin, ...) of its
// destination rows, for the same tokens, layers and chunking; all entries' slices have one size,
// so their work items line up: one launch (InterleavedSource, entries one after the other).
}  // extern "C"

// A reshard, launched now (prep == nullptr) or planned and uploaded into *prep for later launches.
static dyna_status reshard_impl(const dyna_kv_head_migration* migs, int32_t n, dyna_range tr, dyna_range lr,
                                int32_t chunk_tokens, struct CUstream_st* stream_, const dyna_kv_opts* opts,
                                dyna_kv_xfer_t* out, dyna_kv_prepared* prep) {
  if (n < 0 || (n > 0 && !migs) || n > DYNA_MAX_BATCH) return fail(DYNA_EINVAL, "0 <= n <= DYNA_MAX_BATCH");
  dyna_kv_opts o{};
  dyna_status r = check_opts(opts, &o);
  if (r) return r;
  if (o.flags & DYNA_READY_PER_LAYER) return fail(DYNA_EINVAL, "DYNA_READY_PER_LAYER needs a ready board");
  if (o.variant == DYNA_VARIANT_STAGED) return fail(DYNA_ENOTSUP, "reshard: FUSED variant only");
  const bool signal = (o.flags & DYNA_MIGRATE_SIGNAL) != 0;
  if (prep && signal)
    return fail(DYNA_EINVAL, "prepared reshard: no per-chunk flags (every launch would need fresh epochs and slots)");
  const bool unchecked = (o.flags & DYNA_MIGRATE_UNCHECKED) != 0;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  std::vector<Span> dsp, ssp;
  std::vector<uint64_t> dst_uids;  // a source pool that some entry writes needs its rows checked too
  for (int32_t i = 0; i < n; ++i)
    if (migs[i].dst.pool) dst_uids.push_back(migs[i].dst.pool->uid);
  std::sort(dst_uids.begin(), dst_uids.end());
  dyna_kv_pool* S0 = nullptr;
  int64_t slice = -1, g = -1;
  bool empty = true;
  for (int32_t i = 0; i < n; ++i) {
    const dyna_kv_head_migration& m = migs[i];
    bool e = false;
    const size_t d0 = dsp.size(), s0 = ssp.size();
    const bool src_is_dst = m.src.pool && std::binary_search(dst_uids.begin(), dst_uids.end(), m.src.pool->uid);
    if ((r = validate_pair(m.src, m.dst, tr, lr, chunk_tokens, unchecked, &e, dsp, ssp, src_is_dst ? 1 : 0, true,
                           i))) {
      g_err = "migration " + std::to_string(i) + ": " + g_err;
      return r;
    }
    const dyna_kv_pool_desc &gs = m.src.pool->desc, &gd = m.dst.pool->desc;
    const int64_t nh = m.src_heads.end - m.src_heads.begin;
    if (m.src_heads.begin < 0 || nh <= 0 || m.src_heads.end > gs.num_kv_heads || m.dst_head_begin < 0 ||
        m.dst_head_begin + nh > gd.num_kv_heads)
      return fail(DYNA_ERANGE, "migration %d: heads [%lld, %lld) of %d -> [%d, ...) of %d", i,
                  (long long)m.src_heads.begin, (long long)m.src_heads.end, gs.num_kv_heads, m.dst_head_begin,
                  gd.num_kv_heads);
    for (size_t k = d0; k < dsp.size(); ++k) dsp[k].h0 = m.dst_head_begin, dsp[k].h1 = (int32_t)(m.dst_head_begin + nh);
    for (size_t k = s0; k < ssp.size(); ++k) ssp[k].h0 = (int32_t)m.src_heads.begin, ssp[k].h1 = (int32_t)m.src_heads.end;
    const int64_t he = (int64_t)gs.head_dim * gs.elem_bytes;
    if (he % 16) return fail(DYNA_EGEOM, "head slices must be multiples of 16 bytes (d*e = %lld)", (long long)he);
    const int64_t sl = nh * he, gi = gcd64(gs.block_size, gd.block_size);
    if (slice < 0) slice = sl, g = gi;
    if (sl != slice || gi != g)
      return fail(DYNA_EINVAL, "reshard: every entry must move slices of one size over one block grid");
    if (!S0) S0 = m.src.pool;
    if (m.src.pool->dev != S0->dev) return fail(DYNA_EINVAL, "reshard: all sources on one device");
    if (!e && (r = check_reach(m.src.pool, m.dst.pool))) return r;
    empty &= e;
  }
  if ((r = check_alias(dsp, ssp))) return r;
  if (empty && prep) {
    prep->empty = true;
    return DYNA_OK;
  }
  if (empty) {
    auto* x = new dyna_kv_xfer();
    x->empty = true;
    if (signal) x->batch.assign(n, dyna_kv_xfer::BatchEntry{});
    *out = x;
    return DYNA_OK;
  }
  if (!err_word()) return fail(DYNA_ECUDA, "no error word");
  const int64_t ntok = tr.end - tr.begin;
  const int64_t nchunks = (ntok + chunk_tokens - 1) / chunk_tokens;
  if (signal) {
    if (nchunks > DYNA_MAX_CHUNKS) return fail(DYNA_ERANGE, "%lld chunks > DYNA_MAX_CHUNKS", (long long)nchunks);
    std::map<std::pair<int, uint64_t>, int64_t> per_row;
    for (int32_t i = 0; i < n; ++i)
      if ((per_row[{migs[i].src.pool->desc.instance, migs[i].dst.pool->uid}] += nchunks) > DYNA_MAX_CHUNKS)
        return fail(DYNA_ERANGE, "reshard: more than DYNA_MAX_CHUNKS signalled chunks into one destination pool");
  }
  DeviceGuard guard(S0->dev);
  dyna_kv_xfer* x = nullptr;
  if ((r = new_xfer(S0->dev, S0->desc.instance, stream, &x))) return r;
  if (prep) {  // the plans' error word belongs to the prepared handle
    prep->err = x->err;
    x->own_err = false;
  }
  if (signal) {
    x->batch.assign(n, dyna_kv_xfer::BatchEntry{});
    for (int32_t i = 0; i < n; ++i) {
      dyna_kv_xfer::BatchEntry& be = x->batch[i];
      if ((r = flag_reserve(migs[i].src.pool->desc.instance, migs[i].dst.pool, nchunks, &be.epoch, &be.first_slot))) {
        delete x;
        return r;
      }
      be.nchunks = (int32_t)nchunks;
      be.sender = migs[i].src.pool->desc.instance;
    }
  }
  const int piece = o.piece_bytes ? o.piece_bytes : kVecPiece;
  // Plans first (tables and maps patched in once the upload span is known): a tile launch needs
  // every entry's geometry to fit a tensor map.
  std::vector<Plan> plans(n);
  const int l0 = (int)lr.begin, lm = (int)(lr.end - lr.begin);
  std::vector<char> maps_h;
  std::vector<const char*> cached(n, nullptr);  // channel-cached device maps per entry (else uploaded)
  bool any_peer = false;
  for (int32_t i = 0; i < n; ++i)
    any_peer |= migs[i].dst.pool->dev != migs[i].src.pool->dev || migs[i].dst.pool->imported;
  bool tiles = want_tiles(o, any_peer);
  if (tiles) maps_h.resize((size_t)n * kTileMaps * kTileMapBytes + 64);
  char* maps = tiles ? reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(maps_h.data()) + 63) & ~uintptr_t(63))
                     : nullptr;
  for (int32_t i = 0; i < n; ++i) {
    const dyna_kv_head_migration& m = migs[i];
    dyna_kv_pool *S = m.src.pool, *D = m.dst.pool;
    const int64_t he = (int64_t)S->desc.head_dim * S->desc.elem_bytes;
    plans[i] = make_plan_sliced(paged(S, nullptr), paged(D, nullptr), slice, S->row, m.src_heads.begin * he, D->row,
                                (int64_t)m.dst_head_begin * he, tr.begin, tr.end, l0, lm, chunk_tokens, g, piece);
    if (tiles && (tiles = tile_shape(plans[i])) &&
        (r = tile_maps(S, D, plans[i], stream, &cached[i], maps + (size_t)i * kTileMaps * kTileMapBytes, &tiles))) {
      delete x;
      return r;
    }
  }
  if (!tiles && o.engine != DYNA_ENGINE_AUTO && o.engine != DYNA_ENGINE_VEC) {
    delete x;
    return fail(DYNA_ENOTSUP, "reshard slices of %lld B on the BULK engine: the geometry does not fit a TMA tensor "
                              "map (or the stream is capturing); use DYNA_ENGINE_VEC", (long long)slice);
  }
  if (!tiles)  // an entry that did not fit: every entry back on the row kernel's plan
    for (int32_t i = 0; i < n; ++i) {
      const dyna_kv_head_migration& m = migs[i];
      dyna_kv_pool *S = m.src.pool, *D = m.dst.pool;
      const int64_t he = (int64_t)S->desc.head_dim * S->desc.elem_bytes;
      plans[i] = make_plan_sliced(paged(S, nullptr), paged(D, nullptr), slice, S->row, m.src_heads.begin * he,
                                  D->row, (int64_t)m.dst_head_begin * he, tr.begin, tr.end, l0, lm, chunk_tokens, g,
                                  piece);
    }
  const size_t maps_b = tiles ? (size_t)n * kTileMaps * kTileMapBytes : 0;  // multiple of 256
  const size_t plans_b = maps_b + (((n * sizeof(Plan)) + 15) & ~size_t(15));
  std::vector<size_t> soff(n, 0), doff(n, 0);
  size_t tab_b = 0;
  for (int32_t i = 0; i < n; ++i) {
    if (!migs[i].src.block_ids) {
      soff[i] = plans_b + tab_b;
      tab_b += (table_upload_bytes(migs[i].src, tr.end) + 15) & ~size_t(15);
    }
    if (!migs[i].dst.block_ids) {
      doff[i] = plans_b + tab_b;
      tab_b += (table_upload_bytes(migs[i].dst, tr.end) + 15) & ~size_t(15);
    }
  }
  RingLease lease(S0->dev);
  char *dbase = nullptr, *h = nullptr;
  std::vector<char> prep_host;
  if (prep) {  // memory of its own, uploaded once below
    prep_host.assign(plans_b + tab_b, 0);
    h = prep_host.data();
    if (cudaMalloc(&prep->mem, prep_host.size()) != cudaSuccess) {
      delete x;
      return fail(DYNA_ENOMEM, "prepared reshard: %zu B of device memory", prep_host.size());
    }
    dbase = prep->mem;
  } else if ((r = lease.reserve(plans_b + tab_b, &dbase, &h, stream))) {
    delete x;
    return r;
  }
  for (int32_t i = 0; i < n; ++i) {
    const dyna_kv_head_migration& m = migs[i];
    dyna_kv_pool *S = m.src.pool, *D = m.dst.pool;
    plans[i].src.table = m.src.block_ids ? m.src.block_ids : reinterpret_cast<const int32_t*>(dbase + soff[i]);
    plans[i].dst.table = m.dst.block_ids ? m.dst.block_ids : reinterpret_cast<const int32_t*>(dbase + doff[i]);
    if (tiles) plans[i].tmaps = cached[i] ? cached[i] : dbase + (size_t)i * kTileMaps * kTileMapBytes;
    plans[i].err = x->err;
    plans[i].overlap_prev = overlap_of(o);
    if (signal) {
      const dyna_kv_xfer::BatchEntry& be = x->batch[i];
      unsigned long long* ctr = nullptr;
      if ((r = channel_counters(S, D, S0->dev, &ctr))) {
        delete x;
        return r;
      }
      plans[i].counters = ctr + be.first_slot;
      plans[i].flags = D->inbox + (size_t)S->desc.instance * DYNA_MAX_CHUNKS + be.first_slot;
      plans[i].epoch = be.epoch;
      plans[i].sys_fence = (D->dev != S->dev || D->imported) ? 1 : 0;
      if (plans[i].overlap_prev && flag_slots_shared_recently(S->desc.instance, D, be.first_slot, nchunks))
        plans[i].overlap_prev |= kOverlapCounters;
    }
  }
  if (tiles) std::memcpy(h, maps, maps_b);
  std::memcpy(h + maps_b, plans.data(), n * sizeof(Plan));
  for (int32_t i = 0; i < n; ++i) {
    if (!migs[i].src.block_ids) std::memcpy(h + soff[i], migs[i].src.host_block_ids, table_upload_bytes(migs[i].src, tr.end));
    if (!migs[i].dst.block_ids) std::memcpy(h + doff[i], migs[i].dst.host_block_ids, table_upload_bytes(migs[i].dst, tr.end));
  }
  if (prep) {
    if ((r = upload_sync(S0->dev, dbase, h, prep_host.size()))) {
      delete x;
      return r;
    }
  } else if ((r = lease.copy(stream))) {
    delete x;
    return r;
  }
  int64_t payload = 0;
  for (int32_t i = 0; i < n; ++i) payload += (plans[i].t1 - plans[i].t0) * plans[i].lm * 2 * plans[i].row;
  InterleavedSource isrc{reinterpret_cast<const Plan*>(dbase + maps_b), n, plans[0].n_items * n, payload};
  x->variant = DYNA_VARIANT_FUSED;
  x->engine = tiles ? DYNA_ENGINE_TILES : DYNA_ENGINE_VEC;
  x->piece = tiles ? plans[0].tile_bytes : piece;
  x->unroll = tiles ? 0 : 8;
  x->stages = tiles ? (o.stages ? o.stages : 4) : 0;
  x->nchunks = (int32_t)nchunks;
  if (prep) {
    prep->reshard = true;
    prep->dev = S0->dev;
    prep->sender = S0->desc.instance;
    prep->isrc = isrc;
    prep->tiles = tiles;
    prep->engine = x->engine;
    prep->piece = tiles ? plans[0].tile_bytes : piece;
    prep->stages = o.stages;
    prep->max_ctas = o.max_ctas;
    delete x;
    return DYNA_OK;
  }
  const uint64_t launches0 = g_launches.load();
  r = tiles ? launch_tiles_interleaved(isrc, signal, plans[0].tile_bytes, o.stages, o.max_ctas, S0->dev, stream)
            : launch_rows_interleaved(isrc, signal, o.max_ctas, S0->dev, stream);
  if (!r) r = lease.finish(stream);
  if (r) {
    delete x;
    return r;
  }
  x->launches = (int32_t)(g_launches.load() - launches0);
  if ((r = record_completion(x, S0->dev, stream))) {
    delete x;
    return r;
  }
  *out = x;
  return DYNA_OK;
}

extern "C" {

dyna_status dyna_kv_reshard(const dyna_kv_head_migration* migs, int32_t n, dyna_range tr, dyna_range lr,
                            int32_t chunk_tokens, struct CUstream_st* stream, const dyna_kv_opts* opts,
                            dyna_kv_xfer_t* out) {
  if (!out) return fail(DYNA_EINVAL, "NULL out");
  *out = nullptr;
  return reshard_impl(migs, n, tr, lr, chunk_tokens, stream, opts, out, nullptr);
}

dyna_status dyna_kv_prepare_reshard(const dyna_kv_head_migration* migs, int32_t n, dyna_range tr, dyna_range lr,
                                    int32_t chunk_tokens, const dyna_kv_opts* opts, dyna_kv_prepared_t* out) {
  if (!out) return fail(DYNA_EINVAL, "NULL out");
  *out = nullptr;
  auto* p = new dyna_kv_prepared();
  const dyna_status r = reshard_impl(migs, n, tr, lr, chunk_tokens, nullptr, opts, nullptr, p);
  if (r) {
    if (p->mem) retire(p->dev, p->mem, Mem::Device);
    if (p->err) err_release(p->err);
    delete p;
    return r;
  }
  *out = p;
  return DYNA_OK;
}

}  // extern "C"

// A batch, launched now (prep == nullptr: *out receives the migration) or planned and uploaded into
// memory owned by *prep for later launches (dyna_kv_prepare_batch; out unused).
static dyna_status batch_impl(const dyna_kv_migration* migs, int32_t n, dyna_range lr, int32_t chunk_tokens,
                              struct CUstream_st* stream_, const dyna_kv_opts* opts, dyna_kv_xfer_t* out,
                              dyna_kv_prepared* prep) {
  if (n < 0 || (n > 0 && !migs) || n > DYNA_MAX_BATCH) return fail(DYNA_EINVAL, "0 <= n <= DYNA_MAX_BATCH");
  dyna_kv_opts o{};
  dyna_status r = check_opts(opts, &o);
  if (r) return r;
  if (o.variant == DYNA_VARIANT_STAGED) return fail(DYNA_ENOTSUP, "batch: FUSED variant only");
  if (o.flags & DYNA_READY_PER_LAYER) return fail(DYNA_EINVAL, "DYNA_READY_PER_LAYER needs a ready board");
  const bool signal = (o.flags & DYNA_MIGRATE_SIGNAL) != 0;
  if (prep && signal)
    return fail(DYNA_EINVAL, "prepared batch: no per-chunk flags (every launch would need fresh epochs and slots)");
  const bool unchecked = (o.flags & DYNA_MIGRATE_UNCHECKED) != 0;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  // Reading R7 across entries: one entry's source rows may be another entry's destination rows.
  std::vector<uint64_t> dst_uids;
  for (int32_t i = 0; i < n; ++i)
    if (migs[i].dst.pool) dst_uids.push_back(migs[i].dst.pool->uid);
  std::sort(dst_uids.begin(), dst_uids.end());
  std::vector<Span> dsp, ssp;
  std::vector<int32_t> live;
  int64_t total_tok = 0;
  dyna_kv_pool* S0 = nullptr;
  int peer = 0;
  for (int32_t i = 0; i < n; ++i) {
    bool empty = false;
    const dyna_block_table &ms = migs[i].src, &md = migs[i].dst;
    const bool src_is_dst = ms.pool && std::binary_search(dst_uids.begin(), dst_uids.end(), ms.pool->uid);
    if ((r = validate_pair(ms, md, migs[i].token_range, lr, chunk_tokens, unchecked, &empty, dsp, ssp,
                           src_is_dst ? 1 : 0, false, i))) {
      g_err = "migration " + std::to_string(i) + ": " + g_err;
      return r;
    }
    if (empty) continue;
    if (src_is_dst && !unchecked && !ms.host_block_ids)
      return fail(DYNA_EINVAL, "migration %d: its source pool is written by this batch: give the source table's "
                               "host_block_ids, or pass DYNA_MIGRATE_UNCHECKED", i);
    dyna_kv_pool *S = ms.pool, *D = md.pool;
    if (!S0) S0 = S;
    if (S->dev != S0->dev || S->row != S0->row)
      return fail(DYNA_EINVAL, "batch: all sources on one device with one row size");
    if ((r = check_reach(S, D))) return r;
    peer |= (D->dev != S->dev || D->imported) ? 1 : 0;
    total_tok += migs[i].token_range.end - migs[i].token_range.begin;
    live.push_back(i);
  }
  if ((r = check_alias(dsp, ssp))) return r;
  if (live.empty()) {
    if (prep) {
      prep->empty = true;
      return DYNA_OK;
    }
    auto* x = new dyna_kv_xfer();
    x->empty = true;
    if (signal) x->batch.assign(n, dyna_kv_xfer::BatchEntry{});  // every entry: 0 chunks
    *out = x;
    return DYNA_OK;
  }
  if (!err_word()) return fail(DYNA_ECUDA, "no error word");
  int64_t run_min = std::numeric_limits<int64_t>::max();  // shortest contiguous run in the batch
  for (int32_t i : live)
    run_min = std::min<int64_t>(run_min, std::min<int64_t>(gcd64(migs[i].src.pool->desc.block_size,
                                                                  migs[i].dst.pool->desc.block_size),
                                                            chunk_tokens) * S0->row);
  Choice ch = choose(o, S0->row, peer, total_tok, run_min);
  DeviceGuard guard(S0->dev);
  dyna_kv_xfer* x = nullptr;
  if ((r = new_xfer(S0->dev, S0->desc.instance, stream, &x))) return r;
  if (prep) {  // the plans' error word belongs to the prepared handle
    prep->err = x->err;
    x->own_err = false;
  }
  const int l0 = (int)lr.begin, lm = (int)(lr.end - lr.begin);
  if (signal) {  // each entry: its own epoch and slot range of its (sender, destination pool)
    // the entries of one launch must not share slots (their counters live there): at most
    // DYNA_MAX_CHUNKS signalled chunks per (sender, destination pool) in one batch
    std::map<std::pair<int, uint64_t>, int64_t> per_row;
    for (int32_t i : live) {
      int64_t& tot = per_row[{migs[i].src.pool->desc.instance, migs[i].dst.pool->uid}];
      tot += (migs[i].token_range.end - migs[i].token_range.begin + chunk_tokens - 1) / chunk_tokens;
      if (tot > DYNA_MAX_CHUNKS) {
        delete x;
        return fail(DYNA_ERANGE, "batch: more than DYNA_MAX_CHUNKS (%d) signalled chunks from sender %d into one "
                                 "destination pool", DYNA_MAX_CHUNKS, migs[i].src.pool->desc.instance);
      }
    }
    x->batch.assign(n, dyna_kv_xfer::BatchEntry{});
    for (int32_t i : live) {
      dyna_kv_pool *S = migs[i].src.pool, *D = migs[i].dst.pool;
      const int64_t nck = (migs[i].token_range.end - migs[i].token_range.begin + chunk_tokens - 1) / chunk_tokens;
      dyna_kv_xfer::BatchEntry& be = x->batch[i];
      if ((r = flag_reserve(S->desc.instance, D, nck, &be.epoch, &be.first_slot))) {
        delete x;
        return r;
      }
      be.nchunks = (int32_t)nck;
      be.sender = S->desc.instance;
    }
  }
  const size_t m = live.size();
  // Short contiguous runs on the same device (AUTO): every entry as a tile plan, one map set per
  // distinct (source pool, destination pool), all entries with one ring slot.
  std::vector<Plan> tplans;
  std::vector<char> maps_h;
  std::vector<int32_t> map_of(m, 0);
  std::vector<size_t> pair_rep;               // a plan of each distinct (source, destination) pair
  std::vector<const char*> pair_cached;       // its channel-cached device maps (else uploaded)
  const bool tiles_asked = o.engine == DYNA_ENGINE_TILES;
  bool tiles = (tiles_asked || (!o.engine && (ch.engine == DYNA_ENGINE_TILES ||
                                              (!ch.exact && !peer && total_tok >= kTileMinTokens &&
                                               run_min < kTileRunMax && tiles_enabled())))) &&
               o.schedule != DYNA_SCHED_DYNAMIC;
  if (tiles) {
    std::map<std::pair<const dyna_kv_pool*, const dyna_kv_pool*>, int32_t> pair_idx;
    tplans.resize(m);
    for (size_t k = 0; k < m && tiles; ++k) {
      const dyna_kv_migration& mg = migs[live[k]];
      dyna_kv_pool *S = mg.src.pool, *D = mg.dst.pool;
      const int64_t g = gcd64(S->desc.block_size, D->desc.block_size);
      tplans[k] = make_plan_sliced(paged(S, nullptr), paged(D, nullptr), S->row, S->row, 0, D->row, 0,
                                   mg.token_range.begin, mg.token_range.end, l0, lm, chunk_tokens, g, ch.piece);
      // one box geometry for the whole launch (the kernel's issuer takes g, the slab count and the
      // slot from the launch's first plan): entries must agree on the run grid too
      tiles = tile_shape(tplans[k]) && tplans[k].tile_bytes == tplans[0].tile_bytes &&
              tplans[k].g == tplans[0].g && tplans[k].lkb == tplans[0].lkb &&
              tplans[k].tile_rows == tplans[0].tile_rows &&
              tplans[k].tile_rstride == tplans[0].tile_rstride;
      auto it = pair_idx.find({S, D});
      if (it == pair_idx.end()) {
        it = pair_idx.emplace(std::make_pair(S, D), (int32_t)pair_rep.size()).first;
        pair_rep.push_back(k);
      }
      map_of[k] = it->second;
    }
    if (tiles) {
      maps_h.resize(pair_rep.size() * kTileMaps * kTileMapBytes + 64);
      char* mp = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(maps_h.data()) + 63) & ~uintptr_t(63));
      pair_cached.assign(pair_rep.size(), nullptr);
      for (size_t q = 0; q < pair_rep.size() && tiles; ++q) {
        const dyna_kv_migration& mg = migs[live[pair_rep[q]]];
        if ((r = tile_maps(mg.src.pool, mg.dst.pool, tplans[pair_rep[q]], stream, &pair_cached[q],
                           mp + q * kTileMaps * kTileMapBytes, &tiles))) {
          delete x;
          return r;
        }
      }
    }
  }
  if (tiles_asked && !tiles) {
    delete x;
    return fail(DYNA_ENOTSUP, "DYNA_ENGINE_TILES: the batch's rows do not fit one tensor-map geometry (or capturing "
                              "without cached maps)");
  }
  if (!tiles && ch.engine == DYNA_ENGINE_TILES) {  // calibrated tiles that do not apply to this batch: VEC
    ch.engine = DYNA_ENGINE_VEC;
    ch.unroll = o.unroll ? o.unroll : kVecU;
    if (!o.piece_bytes) ch.piece = kVecPiece;
  }
  const size_t npairs = tiles ? pair_rep.size() : 0;
  const size_t maps_b = npairs * kTileMaps * kTileMapBytes;  // multiple of 256
  if (tiles) {
    ch.engine = DYNA_ENGINE_TILES;
    ch.piece = tplans[0].tile_bytes;
    ch.stages = o.stages ? o.stages : 4;
  }
  // One upload: [tile maps][plans][item bases][host-resident tables].
  const size_t plans_b = maps_b + (((m * sizeof(Plan)) + 15) & ~size_t(15));
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
  std::vector<char> prep_host;
  if (prep) {  // memory of its own, uploaded once below
    prep_host.assign(plans_b + bases_b + tab_b, 0);
    h = prep_host.data();
    if (cudaMalloc(&prep->mem, prep_host.size()) != cudaSuccess) {
      delete x;
      return fail(DYNA_ENOMEM, "prepared batch: %zu B of device memory", prep_host.size());
    }
    dbase = prep->mem;
  } else if ((r = lease.reserve(plans_b + bases_b + tab_b, &dbase, &h, stream))) {
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
    if (tiles) {
      plans[k] = tplans[k];
      plans[k].src.table = sids;
      plans[k].dst.table = dids;
      plans[k].tmaps = pair_cached[map_of[k]] ? pair_cached[map_of[k]]
                                              : dbase + (size_t)map_of[k] * kTileMaps * kTileMapBytes;
    } else {
      plans[k] = make_plan(paged(S, sids), paged(D, dids), S->row, mg.token_range.begin, mg.token_range.end, l0, lm,
                           chunk_tokens, g, ch.piece);
    }
    plans[k].err = x->err;
    plans[k].overlap_prev = overlap_of(o);
    if (signal) {  // entry k's chunk j: counter / inbox slot first_slot + j of its (sender, destination)
      dyna_kv_xfer::BatchEntry& be = x->batch[live[k]];
      unsigned long long* ctr = nullptr;
      if ((r = channel_counters(S, D, S0->dev, &ctr))) {
        delete x;
        return r;
      }
      plans[k].counters = ctr + be.first_slot;
      plans[k].flags = D->inbox + (size_t)S->desc.instance * DYNA_MAX_CHUNKS + be.first_slot;
      plans[k].epoch = be.epoch;
      plans[k].sys_fence = (D->dev != S->dev || D->imported) ? 1 : 0;
      if (plans[k].overlap_prev && flag_slots_shared_recently(S->desc.instance, D, be.first_slot, be.nchunks))
        plans[k].overlap_prev |= kOverlapCounters;
    }
    bases[k] = total_items;
    total_items += plans[k].n_items;
  }
  // fill the pinned staging now that the device pointers are known, then one copy
  if (tiles)
    std::memcpy(h, reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(maps_h.data()) + 63) & ~uintptr_t(63)),
                maps_b);
  std::memcpy(h + maps_b, plans.data(), m * sizeof(Plan));
  std::memcpy(h + plans_b, bases.data(), m * sizeof(int64_t));
  for (size_t k = 0; k < m; ++k) {
    const dyna_kv_migration& mg = migs[live[k]];
    if (!mg.src.block_ids)
      std::memcpy(h + soff[k], mg.src.host_block_ids, table_upload_bytes(mg.src, mg.token_range.end));
    if (!mg.dst.block_ids)
      std::memcpy(h + doff[k], mg.dst.host_block_ids, table_upload_bytes(mg.dst, mg.token_range.end));
  }
  if (prep) {
    if ((r = upload_sync(S0->dev, dbase, h, prep_host.size()))) {
      delete x;
      return r;
    }
  } else if ((r = lease.copy(stream))) {
    delete x;
    return r;
  }
  int64_t payload = 0;
  for (size_t k = 0; k < m; ++k) payload += (plans[k].t1 - plans[k].t0) * plans[k].lm * 2 * plans[k].row;
  BatchSource bsrc{reinterpret_cast<const Plan*>(dbase + maps_b), reinterpret_cast<const int64_t*>(dbase + plans_b),
                   (int32_t)m, total_items, payload};
  x->variant = DYNA_VARIANT_FUSED;
  x->engine = ch.engine;
  x->piece = ch.piece;
  x->stages = ch.engine != DYNA_ENGINE_VEC ? ch.stages : 0;
  x->unroll = ch.engine == DYNA_ENGINE_VEC ? ch.unroll : 0;
  x->launches = 1;
  if (prep) {
    prep->dev = S0->dev;
    prep->sender = S0->desc.instance;
    prep->src = bsrc;
    prep->tiles = tiles;
    prep->engine = ch.engine;
    prep->piece = ch.piece;
    prep->stages = ch.stages;
    prep->unroll = ch.unroll;
    prep->max_ctas = o.max_ctas;
    prep->schedule = o.schedule;
    delete x;
    return DYNA_OK;
  }
  r = tiles ? launch_tiles_batch(bsrc, signal, ch.piece, ch.stages, o.max_ctas, S0->dev, stream)
            : launch_batch(bsrc, total_items, signal, ch.piece, ch.engine, o.max_ctas, ch.stages, ch.unroll,
                           S0->dev, stream, o.schedule);
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

extern "C" {

dyna_status dyna_kv_migrate_batch(const dyna_kv_migration* migs, int32_t n, dyna_range lr, int32_t chunk_tokens,
                                  struct CUstream_st* stream, const dyna_kv_opts* opts, dyna_kv_xfer_t* out) {
  if (!out) return fail(DYNA_EINVAL, "NULL out");
  *out = nullptr;
  return batch_impl(migs, n, lr, chunk_tokens, stream, opts, out, nullptr);
}

// ---------------------------------------------------------------- prepared batches (plan once, launch many)
dyna_status dyna_kv_prepare_batch(const dyna_kv_migration* migs, int32_t n, dyna_range lr, int32_t chunk_tokens,
                                  const dyna_kv_opts* opts, dyna_kv_prepared_t* out) {
  if (!out) return fail(DYNA_EINVAL, "NULL out");
  *out = nullptr;
  auto* p = new dyna_kv_prepared();
  const dyna_status r = batch_impl(migs, n, lr, chunk_tokens, nullptr, opts, nullptr, p);
  if (r) {
    if (p->mem) retire(p->dev, p->mem, Mem::Device);
    if (p->err) err_release(p->err);
    delete p;
    return r;
  }
  *out = p;
  return DYNA_OK;
}

dyna_status dyna_kv_prepared_launch(dyna_kv_prepared_t p, struct CUstream_st* stream_, dyna_kv_xfer_t* out) {
  if (!p || !out) return fail(DYNA_EINVAL, "NULL argument");
  *out = nullptr;
  if (p->empty) {
    auto* x = new dyna_kv_xfer();
    x->empty = true;
    *out = x;
    return DYNA_OK;
  }
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  DeviceGuard guard(p->dev);
  dyna_kv_xfer* x = nullptr;
  dyna_status r = new_xfer(p->dev, p->sender, stream, &x);
  if (r) return r;
  if (x->err != g_err_word) err_release(x->err);
  x->err = p->err;  // its kernels report into the handle's word
  x->own_err = false;
  x->variant = DYNA_VARIANT_FUSED;
  x->engine = p->engine;
  x->piece = p->piece;
  x->stages = p->engine != DYNA_ENGINE_VEC ? p->stages : 0;
  x->unroll = p->engine == DYNA_ENGINE_VEC ? p->unroll : 0;
  x->launches = 1;
  if (p->reshard)
    r = p->tiles ? launch_tiles_interleaved(p->isrc, false, p->piece, p->stages, p->max_ctas, p->dev, stream)
                 : launch_rows_interleaved(p->isrc, false, p->max_ctas, p->dev, stream);
  else
    r = p->tiles ? launch_tiles_batch(p->src, false, p->piece, p->stages, p->max_ctas, p->dev, stream)
                 : launch_batch(p->src, p->src.total_items, false, p->piece, p->engine, p->max_ctas, p->stages,
                                p->unroll, p->dev, stream, p->schedule);
  if (!r) r = record_completion(x, p->dev, stream);
  if (r) {
    delete x;
    return r;
  }
  *out = x;
  return DYNA_OK;
}

dyna_status dyna_kv_prepared_destroy(dyna_kv_prepared_t p) {
  if (!p) return fail(DYNA_EINVAL, "NULL prepared");
  if (p->mem) retire(p->dev, p->mem, Mem::Device);  // never synchronises (see pool_destroy)
  if (p->err) err_release(p->err);
  delete p;
  return DYNA_OK;
}

// ---------------------------------------------------------------- a6: measure the AUTO table here
dyna_status dyna_kv_calibrate(dyna_block_table src, dyna_block_table dst, const int32_t* chunk_tokens, int32_t n,
                              int32_t reps, struct CUstream_st* stream_, dyna_kv_calib_entry* out, float* gbps) {
  if (n <= 0 || !chunk_tokens || !out || reps < 1) return fail(DYNA_EINVAL, "calibrate: n > 0, chunk sizes, out, reps >= 1");
  for (int32_t i = 0; i < n; ++i)
    if (chunk_tokens[i] <= 0 || (i && chunk_tokens[i] <= chunk_tokens[i - 1]))
      return fail(DYNA_EINVAL, "calibrate: chunk sizes must be positive and ascending");
  if (!src.pool || !dst.pool) return fail(DYNA_EINVAL, "NULL pool in a block table");
  dyna_kv_pool *S = src.pool, *D = dst.pool;
  const int64_t T = std::min<int64_t>(src.len * S->desc.block_size, dst.len * D->desc.block_size);
  if (chunk_tokens[n - 1] > T)
    return fail(DYNA_ERANGE, "calibrate: chunk of %d tokens > the tables' %lld tokens", chunk_tokens[n - 1],
                (long long)T);
  struct Cand { int32_t variant, engine, piece, stages, unroll; };
  static const Cand kCands[DYNA_CALIB_CANDIDATES] = {
      {DYNA_VARIANT_FUSED, DYNA_ENGINE_VEC, 4096, 0, 8},   {DYNA_VARIANT_FUSED, DYNA_ENGINE_VEC, 8192, 0, 4},
      {DYNA_VARIANT_FUSED, DYNA_ENGINE_VEC, 16384, 0, 16}, {DYNA_VARIANT_FUSED, DYNA_ENGINE_BULK, 32768, 4, 0},
      {DYNA_VARIANT_STAGED, DYNA_ENGINE_VEC, 8192, 0, 8},  {DYNA_VARIANT_STAGED, DYNA_ENGINE_BULK, 32768, 4, 0},
      {DYNA_VARIANT_FUSED, DYNA_ENGINE_TILES, 0, 4, 0}};
  const int peer = (D->dev != S->dev || D->imported) ? 1 : 0;
  const bool staged_ok = !D->imported && (D->dev == S->dev || dst.block_ids);
  const int64_t L = S->desc.num_layers;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  DeviceGuard guard(S->dev);
  // the gate: a one-thread kernel spinning on a mapped host word holds the stream while the host
  // enqueues a candidate's calls, so the events around them see device time only
  unsigned long long* gate = nullptr;
  CUDA_TRY(cudaHostAlloc(&gate, sizeof(unsigned long long), cudaHostAllocMapped | cudaHostAllocPortable));
  *gate = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  dyna_status r = DYNA_OK;
  std::vector<dyna_kv_calib_entry> chosen;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess)
    r = fail(DYNA_ECUDA, "calibrate: events");
  unsigned long long open = 0;
  for (int32_t i = 0; i < n && !r; ++i) {
    const int64_t c = chunk_tokens[i];
    float best_ms = 0.f;
    int best = -1;
    for (int k = 0; k < DYNA_CALIB_CANDIDATES && !r; ++k) {
      const Cand& cd = kCands[k];
      if (gbps) gbps[i * DYNA_CALIB_CANDIDATES + k] = 0.f;
      if (cd.variant == DYNA_VARIANT_STAGED && !staged_ok) continue;
      // tensor-map stores into peer memory are unmeasured: not a candidate across
      // GPUs, as AUTO never tiles there either (explicit DYNA_ENGINE_TILES still may)
      if (cd.engine == DYNA_ENGINE_TILES && peer) continue;
      dyna_kv_opts o{cd.variant, cd.engine, 0, 0, cd.piece, cd.stages, cd.unroll, 0};
      bool skip = false;
      for (int pass = 0; pass < 2 && !r; ++pass) {
        // pass 0, ungated, warms up whatever a first call allocates (staging, error words): an
        // allocation that synchronises the device must not meet a closed gate
        if (pass == 1) {
          ++open;
          launch_wait_flag(gate, open, 10ull * 1000 * 1000 * 1000, stream, nullptr);
          if (cudaEventRecord(e0, stream) != cudaSuccess) r = fail(DYNA_ECUDA, "calibrate: event");
        }
        std::vector<dyna_kv_xfer_t> xs;
        for (int32_t j = 0; j < (pass ? reps : 1) && !r; ++j) {
          const int64_t span = T - c + 1;
          const int64_t t0 = ((int64_t)j * c) % span;
          dyna_kv_xfer_t x = nullptr;
          r = dyna_kv_migrate_ex(src, dst, dyna_range{t0, t0 + c}, dyna_range{0, L}, (int32_t)c, stream_, &o, &x);
          if (!r) xs.push_back(x);
        }
        if (r == DYNA_ENOTSUP && pass == 0 && cd.engine == DYNA_ENGINE_TILES) {  // no tensor map fits: skip
          r = DYNA_OK;
          skip = true;
          break;
        }
        if (pass == 1 && !r && cudaEventRecord(e1, stream) != cudaSuccess) r = fail(DYNA_ECUDA, "calibrate: event");
        if (pass == 1) __atomic_store_n(gate, open, __ATOMIC_RELEASE);  // open: the queued calls run back to back
        for (dyna_kv_xfer_t x : xs) {
          const dyna_status w = dyna_kv_wait(x);
          if (!r) r = w;
        }
      }
      if (r) break;
      if (skip) continue;
      float ms = 0.f;
      cudaError_t ce = cudaEventSynchronize(e1);  // (no early return: the gate below must open)
      if (ce == cudaSuccess) ce = cudaEventElapsedTime(&ms, e0, e1);
      if (ce != cudaSuccess) {
        r = fail(DYNA_ECUDA, "calibrate: %s", cudaGetErrorString(ce));
        break;
      }
      ms /= (float)reps;
      const double bytes = (double)c * 2 * L * S->row;
      if (gbps) gbps[i * DYNA_CALIB_CANDIDATES + k] = (float)(bytes / (ms * 1e-3) / 1e9);
      if (best < 0 || ms < best_ms) best_ms = ms, best = k;
    }
    if (!r && best >= 0) {
      const Cand& cd = kCands[best];
      out[i] = dyna_kv_calib_entry{(int32_t)S->row, peer, i == n - 1 ? (int32_t)1073741824 : (int32_t)c,
                                   cd.variant, cd.engine, cd.piece, cd.stages, cd.unroll};
      chosen.push_back(out[i]);
    }
  }
  __atomic_store_n(gate, ~0ull, __ATOMIC_RELEASE);
  cudaStreamSynchronize(stream);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  cudaFreeHost(gate);
  if (r) return r;
  calib_install(S->row, peer, chosen);
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
    if (!r) r = err_take(x->err);  // this migration's own word
    if (!r && x->board && x->board->cancel_epoch.load() >= x->ready_epoch)
      r = fail(DYNA_ECANCELED, "migration cancelled (dyna_kv_ready_cancel)");
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

dyna_status dyna_kv_xfer_info(dyna_kv_xfer_t x, uint64_t* epoch, int32_t* num_chunks, int32_t* sender,
                              int32_t* first_slot) {
  if (!x) return fail(DYNA_EINVAL, "NULL xfer");
  if (first_slot) *first_slot = x->first_slot;
  if (epoch) *epoch = x->epoch;
  if (num_chunks) *num_chunks = x->nchunks;
  if (sender) *sender = x->sender;
  return DYNA_OK;
}

dyna_status dyna_kv_batch_info(dyna_kv_xfer_t x, int32_t index, uint64_t* epoch, int32_t* first_slot,
                               int32_t* num_chunks, int32_t* sender) {
  if (!x) return fail(DYNA_EINVAL, "NULL xfer");
  if (x->batch.empty()) return fail(DYNA_EINVAL, "not a signalled dyna_kv_migrate_batch");
  if (index < 0 || (size_t)index >= x->batch.size()) return fail(DYNA_ERANGE, "batch index %d", index);
  const dyna_kv_xfer::BatchEntry& be = x->batch[index];
  if (epoch) *epoch = be.epoch;
  if (first_slot) *first_slot = be.first_slot;
  if (num_chunks) *num_chunks = be.nchunks;
  if (sender) *sender = be.sender;
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
  launch_wait_flag(dst->inbox + (size_t)sender * DYNA_MAX_CHUNKS + chunk, epoch, timeout_ns,
                   reinterpret_cast<cudaStream_t>(stream), g_err_word);
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

}  // extern "C"
