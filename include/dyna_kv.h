/*
 * dyna_kv.h — C ABI of the B200-native chunked KV-cache migration library
 * (libdyna_kv.so, sources in paper_2504_09285_b200/csrc/).
 *
 * The operation (PAPER.md = arXiv 2504.09285, DynaServe):
 *   §3.1 P:306-308  a request of L = P + D tokens is split at s into the
 *                   micro-requests r^alpha (tokens 1..s) and r^beta
 *                   (tokens s+1..L); s = ceil(phi*L).
 *   §3.1 P:352      "When the micro-requests of an LLM request span two
 *                   execution instances, the instances exchange the required
 *                   KV cache blocks."
 *   §4.3 P:556      r^alpha is processed "in equal-sized chunks"; "once chunk
 *                   k completes, its KV block is immediately DMA-pushed" to
 *                   the other instance, and messages steer "placement on the
 *                   receiver side".
 * dyna_kv_migrate() is that push: for every layer l in layer_range, K and V,
 * every token t in token_range, all KV heads, the row of the source pool
 * reached through the source block table is copied, bit for bit, to the row
 * of the destination pool reached through the destination block table
 * (the receiver's placement).  Nothing else in either pool changes.  Token
 * indices are 0-based and ranges half-open (reading R1: paper token
 * i is index i-1, so r^alpha is [0, s)).
 *
 * Pool layout (reading R3; the paper does not fix one):
 *   element (l, kv, block b, slot j, head h, i) of e bytes lives at byte
 *   ((((l*2 + kv)*NB + b)*bs + j)*H + h)*d*e + i*e        kv: 0 = K, 1 = V
 * i.e. [L][2][NB][bs][H][d].  One token's K (or V) in one layer is one
 * contiguous "row" of H*d*e bytes; a block is bs consecutive rows.
 *
 * API map:
 *   pools            dyna_kv_pool_bytes / _create / _destroy, _export / _import (CUDA IPC)
 *   the push         dyna_kv_migrate / _ex (variant, engine, SM budget, per-chunk flags,
 *                    overlap with the previous independent call)
 *   completion       dyna_kv_wait / _query / _stream_wait, _xfer_info, _stream_wait_chunk,
 *                    _copy_flags, _xfer_plan, _poll_error
 *   many requests    dyna_kv_migrate_batch (+ _batch_info for per-request flags)
 *   producer-coupled dyna_kv_ready_* + dyna_kv_migrate_on_ready (per chunk or per layer,
 *                    cancellable)
 *   decode-side      dyna_kv_chunkstream_* (chunks pushed as the tokens are produced)
 *   receiver-steered dyna_kv_channel_* + dyna_kv_push / _place (and _heads forms)
 *   TP resharding    dyna_kv_migrate_heads, dyna_kv_reshard (all rank pairs, one launch),
 *                    dyna_kv_push_heads / _place_heads
 *   halves           dyna_kv_pack / _unpack (source rows -> contiguous buffer -> destination rows)
 *   selection        dyna_kv_calib_set / _get (the measured AUTO table), dyna_kv_calibrate (measure it here)
 *   plan once        dyna_kv_prepare_batch / _prepared_launch / _prepared_destroy (CUDA-graph friendly batches)
 *
 * Errors: every call returns a dyna_status; negative values are errors and
 * dyna_kv_last_error() returns a thread-local message.  No call throws.
 * Synchronous errors leave nothing enqueued.
 *
 * Threading: calls are thread-safe; a pool handle may be used from several
 * threads as long as it is not destroyed concurrently.
 */
#ifndef DYNA_KV_H
#define DYNA_KV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define DYNA_API __attribute__((visibility("default")))
#else
#define DYNA_API
#endif

struct CUstream_st; /* cudaStream_t == struct CUstream_st* ; NULL = legacy default stream */

typedef int32_t dyna_status;
#define DYNA_OK         0
#define DYNA_EINVAL    (-1)  /* NULL handle/pointer, bad option value, misaligned base, destination table
                                without host ids (aliasing unchecked) and no DYNA_MIGRATE_UNCHECKED */
#define DYNA_EGEOM     (-2)  /* geometry mismatch (L, H, d, e differ) or row bytes % 16 != 0 */
#define DYNA_ERANGE    (-3)  /* token/layer range outside the tables/pool, block id out of range,
                                chunk_tokens <= 0, too many chunks for signalling */
#define DYNA_EALIAS    (-4)  /* two destination rows coincide (within a call or a batch), dst rows overlap
                                src rows of the same pool, or two distinct pools overlap in memory */
#define DYNA_EPEER     (-5)  /* destination memory not reachable from the source device (no P2P / IPC) */
#define DYNA_ENOMEM    (-6)
#define DYNA_ECUDA     (-7)  /* a CUDA runtime error (message in dyna_kv_last_error) */
#define DYNA_ETIMEDOUT (-8)
#define DYNA_EAGAIN    (-9)  /* dyna_kv_query: still in flight */
#define DYNA_ENOTSUP   (-10)
#define DYNA_ECANCELED (-11) /* dyna_kv_wait: the producer-coupled migration was cancelled (dyna_kv_ready_cancel) */

/* Pool geometry.  All fields > 0 except device (a CUDA ordinal >= 0) and
 * instance (0 <= instance < DYNA_MAX_INSTANCES; the id this pool's owner uses
 * as a sender when signalling peers, e.g. its rank). */
typedef struct {
    int32_t num_layers;    /* L */
    int32_t num_kv_heads;  /* H */
    int32_t head_dim;      /* d */
    int32_t elem_bytes;    /* e: 2 for fp16/bf16.  The copy is bitwise, dtype-agnostic. */
    int32_t block_size;    /* bs: tokens per block (source and destination may differ) */
    int32_t num_blocks;    /* NB */
    int32_t device;        /* CUDA ordinal owning the memory */
    int32_t instance;      /* sender id for per-chunk flags */
} dyna_kv_pool_desc;

#define DYNA_MAX_INSTANCES 64
#define DYNA_MAX_CHUNKS    4096   /* inbox slots per (sender, destination pool): the most chunks one
                                     signalled migration may have; slot ranges recycle after this many */

typedef struct dyna_kv_pool* dyna_kv_pool_t;
typedef struct dyna_kv_xfer* dyna_kv_xfer_t;

/* A request's block table on one pool: logical token t lives in block
 * block_ids[t / bs] at slot t % bs.
 *   block_ids       DEVICE pointer, int32[len], readable from the source
 *                   device (device memory of the source GPU, or of a peer
 *                   with P2P enabled).  Caller-owned; must stay valid and
 *                   unmodified until dyna_kv_wait returns (like the source of
 *                   cudaMemcpyAsync).  May be NULL when host_block_ids is
 *                   given: the library then copies the entries the call needs
 *                   ([0, last touched block]) to the device itself, ordered on
 *                   `stream` (a scheduler's tables usually live on the host).
 *   host_block_ids  HOST copy of the same ids.  Where given, ids are
 *                   range-checked and destination aliasing (DESIGN.md reading
 *                   R7: two writes of one destination row, or a destination
 *                   row that is also read as a source row) is rejected
 *                   synchronously (DYNA_ERANGE / DYNA_EALIAS); the host array
 *                   may be reused as soon as the call returns.  The DESTINATION
 *                   table must carry host ids (and the source table too when
 *                   it reads the destination pool), else the call fails with
 *                   DYNA_EINVAL — unless opts->flags has DYNA_MIGRATE_UNCHECKED
 *                   (the caller guarantees fresh, distinct destination blocks,
 *                   e.g. from its allocator).  Ids without a host copy are
 *                   range-checked on the device: offending rows are skipped and
 *                   dyna_kv_wait returns DYNA_ERANGE. */
typedef struct {
    dyna_kv_pool_t pool;
    const int32_t* block_ids;
    const int32_t* host_block_ids;
    int64_t len;
} dyna_block_table;

typedef struct { int64_t begin, end; } dyna_range;  /* half-open [begin, end) */

/* Variant. */
#define DYNA_VARIANT_AUTO   0  /* calibrated choice per (row bytes, locality, call size) */
#define DYNA_VARIANT_FUSED  1  /* one kernel: source rows -> destination rows (K4 / K4-local) */
#define DYNA_VARIANT_STAGED 2  /* gather -> staging -> peer staging (+flag) -> scatter (K1, K2, K3) */
/* Copy engine inside the kernels. */
#define DYNA_ENGINE_AUTO 0
#define DYNA_ENGINE_VEC  1     /* warp-per-segment 16-B vector loads/stores (LDG.128 / STG.128) */
#define DYNA_ENGINE_BULK 2     /* TMA bulk copies through a shared-memory ring (UBLKCP): one issuing thread,
                                  fed item descriptors by a decoder warp */
#define DYNA_ENGINE_BULK_WS 3  /* alias of DYNA_ENGINE_BULK (kept for callers of the round-1 warp-specialised kernel) */
#define DYNA_ENGINE_TILES 4    /* TMA tensor tiles (UTMALDG / UTMASTG): a block's rows (or head slices) of several
                                  (layer, K|V) slabs per 4-D tensor load / store, one issuing thread fed by a decoder
                                  warp.  Fused variant only (the staged variant's K1 / K3 then use VEC); DYNA_ENOTSUP
                                  when no tensor map can describe the rows.  AUTO picks it for
                                  contiguous runs under 32 KiB on one device and for head slices. */
/* flags */
#define DYNA_MIGRATE_SIGNAL 1  /* write a per-chunk flag into the destination pool's inbox */
#define DYNA_READY_PER_LAYER 2 /* dyna_kv_migrate_on_ready: one ready mark per (chunk, layer), see below */
#define DYNA_MIGRATE_UNCHECKED 4 /* destination tables may come without host ids: the caller guarantees that
                                    no destination row is written twice or read as a source row (R7) */
#define DYNA_MIGRATE_OVERLAP_PREV 8 /* the caller guarantees that this call neither reads nor writes memory
                                    that the kernel enqueued immediately before it on `stream` writes, nor
                                    writes memory that kernel reads — nor, when that kernel was itself a call
                                    with this flag, the kernel before it, and so on (a run of flagged calls
                                    may execute concurrently: it must be mutually independent).  E.g. chunk
                                    k+1 of a request pushed after chunk k, or another request's migration:
                                    disjoint destination rows, tables and sources not produced by those
                                    kernels.  The copy kernel then starts moving
                                    bytes while that kernel drains (programmatic dependent launch without the
                                    grid-dependency wait) instead of after it: the ~4-5 us bubble between
                                    back-to-back migrations disappears.  Stream order is
                                    otherwise kept: one CTA of the kernel waits for its predecessor before
                                    the grid can complete (and every thread does before touching chunk
                                    counters whose slots another launch reserved recently), so work
                                    enqueued after it, events, dyna_kv_wait and flags still imply the
                                    predecessor's completion.
                                    Work before the predecessor is ordered as usual (an event the stream waits
                                    for, e.g. the producer's, is a full dependency).  Applies to FUSED
                                    migrations, batches, head migrations, reshards, pack / unpack and
                                    prepared launches; ignored (the launch waits) for the STAGED chain,
                                    producer-coupled launches and an explicit DYNA_SCHED_DYNAMIC.  With the AUTO
                                    engine a same-device migration with this flag and no max_ctas runs
                                    on the VEC engine (measured best for overlapped calls; 8-KiB rows from
                                    4096 tokens keep the table's ring).  Violating the promise
                                    gives unspecified destination bytes, as a data race would. */

typedef struct {
    int32_t variant;    /* DYNA_VARIANT_*  (0 = auto) */
    int32_t engine;     /* DYNA_ENGINE_*   (0 = auto) */
    int32_t max_ctas;   /* cap on CTAs per kernel (SM budget for overlap with a producer); 0 = no cap */
    int32_t flags;      /* DYNA_MIGRATE_* */
    int32_t piece_bytes;/* bytes per work item; 0 = engine default.  Multiple of 16. */
    int32_t stages;     /* BULK: shared-memory ring depth (2..16); 0 = default.  Cut to the depth that
                           fits in one CTA's shared memory (DYNA_EINVAL if two pieces do not fit) */
    int32_t unroll;     /* VEC: 16-B loads in flight per lane (4, 8 or 16); 0 = default */
    int32_t schedule;   /* work distribution: 0 = default (static), DYNA_SCHED_STATIC, DYNA_SCHED_DYNAMIC */
} dyna_kv_opts;
#define DYNA_SCHED_STATIC  1   /* round-robin items over a balanced persistent grid */
#define DYNA_SCHED_DYNAMIC 2   /* workers grab items from a per-launch atomic counter: the decoder warp of the
                                  BULK ring and of the tile kernel grabs up to 32 consecutive items per atomic,
                                  fewer towards the end (guided) — the default (0) for those launches from 24
                                  pieces per SM of payload with at most a fifth of the item slots empty,
                                  outside graph capture (measured +1-3%).  Asked for explicitly on the VEC
                                  engine, each warp grabs up to 32 items per atomic the same way: faster
                                  than static on long single calls (one 4-GiB call 0.93 -> 1.01 of the copy
                                  peak), slower on short or overlapped ones — an option, not a default */

/* Calibration table used by DYNA_VARIANT_AUTO / DYNA_ENGINE_AUTO (SURVEY §8 a6:
 * "chosen over the staged variant per chunk size by measured bandwidth").
 * An entry applies to migrations whose row bytes (H*d*e) equal row_bytes
 * (0 = any), whose destination locality matches peer (0 = same GPU, 1 = other
 * GPU), and whose call size (tokens in token_range) <= max_chunk_tokens (in
 * the paper's per-chunk push, a call moves one chunk, so this is the
 * chunk size).  Entries for the exact row size are preferred over generic
 * ones; within each class the smallest covering max_chunk_tokens wins.  The
 * library starts with the table measured on B200 (profiles/), replaceable at
 * run time (or measured on the caller's own pools: dyna_kv_calibrate).  An
 * entry may name DYNA_ENGINE_TILES (the built-in one does for long calls of
 * small rows).  Measured rules apply on top of the table when the engine is
 * AUTO: for a row size without an exact entry, a contiguous run
 * (min(gcd(bs_src, bs_dst), chunk_tokens) * row bytes) shorter than 32 KiB in
 * a call of at least 1024 tokens with the destination on the source device
 * moves as TMA tensor tiles (DYNA_ENGINE_TILES, with the ring slot as
 * piece_bytes); tiles never run under CUDA-graph capture before the library's
 * tile-map cache holds the geometry; otherwise no BULK engine for runs shorter
 * than 16 KiB. */
typedef struct {
    int32_t row_bytes;
    int32_t peer;
    int32_t max_chunk_tokens;
    int32_t variant;      /* DYNA_VARIANT_FUSED / STAGED */
    int32_t engine;       /* DYNA_ENGINE_VEC / BULK / BULK_WS / TILES */
    int32_t piece_bytes;  /* 0 = engine default */
    int32_t stages;
    int32_t unroll;
} dyna_kv_calib_entry;

/* Bytes a pool of this geometry needs: L*2*NB*bs*H*d*e.  0 if desc invalid. */
DYNA_API size_t dyna_kv_pool_bytes(const dyna_kv_pool_desc* desc);

/* Wrap caller memory as a pool.  device_base: device pointer on desc->device,
 * 256-B aligned, at least dyna_kv_pool_bytes(desc) bytes, BORROWED (the
 * library never frees it; keep it alive until dyna_kv_pool_destroy).  The
 * library allocates a small per-pool inbox of chunk flags on desc->device. */
DYNA_API dyna_status dyna_kv_pool_create(const dyna_kv_pool_desc* desc, void* device_base, dyna_kv_pool_t* out);
/* Destroy calls (pool, ready board, channel) never synchronise the device:
 * the library's allocations are retired and released by the next call that
 * allocates anyway (pool / board / channel create or import), so a destroy —
 * e.g. from a binding object's garbage collection — cannot deadlock against a
 * waiting producer-coupled migration.  Every migration using the object must
 * have completed (dyna_kv_wait) before it is destroyed. */
DYNA_API dyna_status dyna_kv_pool_destroy(dyna_kv_pool_t pool);

/* Migrate src -> dst for token_range x layer_range in chunks of chunk_tokens
 * (chunk k = [begin + k*c, min(begin + (k+1)*c, end)), reading R5).
 * Work is enqueued on `stream`, which must belong to the SOURCE pool's
 * device; it runs after prior work on that stream (so a caller orders each
 * chunk's migrate after the prefill that produced it — P:556).  The source
 * rows must not be written until completion (KV is append-only); the
 * destination rows must not be read before completion (or their chunk flag).
 * An empty token or layer range returns DYNA_OK with nothing enqueued.
 * *out receives a handle that must be passed to dyna_kv_wait exactly once. */
DYNA_API dyna_status dyna_kv_migrate(dyna_block_table src, dyna_block_table dst,
                            dyna_range token_range, dyna_range layer_range,
                            int32_t chunk_tokens, struct CUstream_st* stream,
                            dyna_kv_xfer_t* out);

/* Same, with explicit options (opts may be NULL = all defaults). */
DYNA_API dyna_status dyna_kv_migrate_ex(dyna_block_table src, dyna_block_table dst,
                               dyna_range token_range, dyna_range layer_range,
                               int32_t chunk_tokens, struct CUstream_st* stream,
                               const dyna_kv_opts* opts, dyna_kv_xfer_t* out);

/* Head resharding between tensor-parallel instances of different degree
 * (§5 P:595-596 deploys r^alpha and r^beta as TP
 * groups).  A TP-sharded instance keeps, per rank, a pool of its own heads;
 * when the sender's and receiver's TP degrees differ, a rank pair exchanges
 * only some heads of every row.  This call moves, for every layer in
 * layer_range, K and V, token in token_range, the KV heads
 * [src_heads.begin, src_heads.end) of the source row (reached through the
 * source table) into heads [dst_head_begin, dst_head_begin + n) of the
 * destination row (reached through the destination table); every other head
 * of the destination row, and every other row, is untouched.  Pools must agree
 * on L, d and e; H may differ.  The head slice (n*d*e bytes) and d*e must be
 * multiples of 16.  When both slices are whole rows (n == H_src == H_dst) this
 * is dyna_kv_migrate_ex.  Otherwise: FUSED variant (DYNA_ENOTSUP for STAGED).
 * Engines: DYNA_ENGINE_TILES (and BULK / BULK_WS, its aliases here) = TMA tensor tiles (a block's slices of
 * several (layer, K|V) slabs per tensor load / store; DYNA_ENOTSUP when no tensor
 * map can describe the slice: slices over 2 KiB that are not a multiple of
 * 2 KiB, or a miss of the library's tile-map cache under CUDA-graph capture);
 * DYNA_ENGINE_VEC = 16-B vector copies; AUTO = tiles when they apply and the
 * destination is on the source device, else VEC.  Per-chunk signalling
 * (DYNA_MIGRATE_SIGNAL) as for
 * dyna_kv_migrate_ex, with a chunk's bytes counted as its slices.  An empty
 * head range is an empty migration.  Errors as dyna_kv_migrate_ex, plus
 * DYNA_ERANGE for head ranges outside either pool. */
DYNA_API dyna_status dyna_kv_migrate_heads(dyna_block_table src, dyna_block_table dst,
                                           dyna_range token_range, dyna_range layer_range,
                                           dyna_range src_heads, int32_t dst_head_begin,
                                           int32_t chunk_tokens, struct CUstream_st* stream,
                                           const dyna_kv_opts* opts, dyna_kv_xfer_t* out);

/* A whole TP reshard of one request in ONE launch (reading R14): n
 * head-sliced migrations (e.g. the rank pairs of dist.tp_reshard_plan) over the same
 * token_range, layer_range and chunk_tokens, each moving heads [src_heads) of its source rows
 * into heads [dst_head_begin, ...) of its destination rows, exactly as dyna_kv_migrate_heads
 * would.  All entries move slices of one size (n_heads*d*e) over one block grid
 * (gcd(bs_src, bs_dst)) and have their sources on the launching device.  One launch
 * instead of n (entries one after the other in the launch's work order).  Destination aliasing
 * (R7) is checked per head: entries may write different heads of the same rows.  Per-chunk
 * signalling gives every entry its own epoch and slots (dyna_kv_batch_info with the entry's
 * index).  FUSED variant (DYNA_ENOTSUP otherwise); engines as dyna_kv_migrate_heads
 * (one engine for the whole launch); other rules as dyna_kv_migrate_batch. */
typedef struct {
    dyna_block_table src, dst;
    dyna_range src_heads;
    int32_t dst_head_begin;
    int32_t reserved;        /* 0 */
} dyna_kv_head_migration;
DYNA_API dyna_status dyna_kv_reshard(const dyna_kv_head_migration* migs, int32_t n, dyna_range token_range,
                                     dyna_range layer_range, int32_t chunk_tokens, struct CUstream_st* stream,
                                     const dyna_kv_opts* opts, dyna_kv_xfer_t* out);

/* Chunk streams (§4.3 P:556 "once chunk k completes, its
 * KV block is immediately DMA-pushed"; decoded tokens join the open chunk,
 * which closes when full or when r^alpha ends).  A stream is one logical migration of
 * tokens [begin, ...) whose end is not known yet: the caller reports tokens as their KV
 * is written (prefill chunks, then decoded tokens) and every chunk that became full is
 * pushed at once (one fused launch on `stream`, ordered after the producer's work on it);
 * closing pushes the open partial chunk.  With DYNA_MIGRATE_SIGNAL, chunk k of the stream
 * (tokens [begin + k*c, ...)) raises inbox slot [sender][first_slot + k] to the stream's
 * epoch, exactly as one dyna_kv_migrate_ex over the whole range would; the stream reserves
 * its slots at open, as many as the destination table can hold chunks (at most
 * DYNA_MAX_CHUNKS; a push beyond them fails with DYNA_ERANGE).  Tables must cover every token
 * reported and stay valid until dyna_kv_chunkstream_finish; FUSED variant, SM engines.
 * One chunk stream is driven by one thread at a time (the object is not locked). */
typedef struct dyna_kv_chunkstream* dyna_kv_chunkstream_t;
DYNA_API dyna_status dyna_kv_chunkstream_open(dyna_block_table src, dyna_block_table dst, int64_t begin,
                                         dyna_range layer_range, int32_t chunk_tokens, struct CUstream_st* stream,
                                         const dyna_kv_opts* opts, dyna_kv_chunkstream_t* out);
/* n_tokens more tokens have KV; *pushed (may be NULL) = chunks pushed by this call. */
DYNA_API dyna_status dyna_kv_chunkstream_produced(dyna_kv_chunkstream_t s, int64_t n_tokens, int32_t* pushed);
/* r^alpha ended: push the open partial chunk (if any); later produced() calls fail. */
DYNA_API dyna_status dyna_kv_chunkstream_close(dyna_kv_chunkstream_t s, int32_t* pushed);
DYNA_API dyna_status dyna_kv_chunkstream_info(dyna_kv_chunkstream_t s, uint64_t* epoch, int32_t* sender,
                                              int32_t* first_slot, int64_t* produced_end, int64_t* pushed_end,
                                              int32_t* num_pushed);
/* Wait for every pushed chunk, free the stream; returns the first deferred error. */
DYNA_API dyna_status dyna_kv_chunkstream_finish(dyna_kv_chunkstream_t s);

/* The push's two halves as calls of their own (§4.3 P:556:
 * the sender packs the chunk, the receiver places it through its own table), for callers
 * that carry the bytes between the two themselves — e.g. the NCCL send/recv baseline
 * or a host/RDMA hop.  The buffer is contiguous device memory readable and
 * writable from the pool's device, 16-B aligned, laid out [l - l0][kv][t - t0][row]
 * (row = H*d*e bytes; reading R3), at least (l1-l0)*2*(t1-t0)*row bytes.
 *   dyna_kv_pack    rows of `src` for token_range x layer_range (through its table) -> buf
 *   dyna_kv_unpack  buf -> rows of `dst` (through its table); nothing else changes
 * Enqueued on `stream` (the pool's device); opts select the engine / SM budget like
 * dyna_kv_migrate_ex (no per-chunk flags: DYNA_EINVAL; no staged variant: DYNA_ENOTSUP).
 * unpack's table follows the destination rules of dyna_block_table (host ids, or
 * DYNA_MIGRATE_UNCHECKED).  Errors and completion as dyna_kv_migrate_ex; an empty range
 * enqueues nothing. */
DYNA_API dyna_status dyna_kv_pack(dyna_block_table src, dyna_range token_range, dyna_range layer_range,
                                  void* buf, uint64_t buf_bytes, struct CUstream_st* stream,
                                  const dyna_kv_opts* opts, dyna_kv_xfer_t* out);
DYNA_API dyna_status dyna_kv_unpack(const void* buf, uint64_t buf_bytes, dyna_block_table dst,
                                    dyna_range token_range, dyna_range layer_range, struct CUstream_st* stream,
                                    const dyna_kv_opts* opts, dyna_kv_xfer_t* out);

/* Many migrations in ONE kernel launch (a batch of short
 * requests, e.g. configs[2]'s 64-request skewed batch).  Every non-empty entry
 * is validated like dyna_kv_migrate; all sources must live on one device (the
 * launching device, `stream`'s) and share one row size; destinations may be
 * any reachable pools.  FUSED variant only (DYNA_ENOTSUP otherwise).
 * n <= DYNA_MAX_BATCH.  The descriptors are copied before the call
 * returns; block tables follow dyna_block_table's rules, and aliasing (R7) is
 * checked across entries: no destination row written by two entries, none
 * read as a source row by any entry.
 * Per-chunk signalling (opts->flags & DYNA_MIGRATE_SIGNAL; VEC engine): every
 * entry gets its own epoch and a disjoint range of inbox slots of its
 * (sender, destination pool) — see dyna_kv_batch_info — so each request's
 * r^beta can start as soon as its own chunks landed.  The signalled chunks of
 * one batch from one sender into one destination pool must fit in
 * DYNA_MAX_CHUNKS (DYNA_ERANGE otherwise): the entries of one launch never
 * share a slot. */
#define DYNA_MAX_BATCH 16384
typedef struct {
    dyna_block_table src, dst;
    dyna_range token_range;
} dyna_kv_migration;
DYNA_API dyna_status dyna_kv_migrate_batch(const dyna_kv_migration* migs, int32_t n, dyna_range layer_range,
                                           int32_t chunk_tokens, struct CUstream_st* stream,
                                           const dyna_kv_opts* opts, dyna_kv_xfer_t* out);
/* Signalled batch: chunk j (0-based, of that entry's token range) of entry
 * `index` is resident when the destination inbox slot [sender][first_slot + j]
 * holds a value >= epoch (dyna_kv_stream_wait_chunk / dyna_kv_copy_flags with
 * chunk = first_slot + j).  Empty entries report num_chunks = 0.  DYNA_EINVAL
 * for a handle that is not a signalled batch. */
DYNA_API dyna_status dyna_kv_batch_info(dyna_kv_xfer_t xfer, int32_t index, uint64_t* epoch, int32_t* first_slot,
                                        int32_t* num_chunks, int32_t* sender);

/* Prepared batches: plan once, launch many (CUDA-graph friendly).  dyna_kv_prepare_batch
 * validates the batch exactly as dyna_kv_migrate_batch (same rules and errors; R7 checked once,
 * here), resolves the engine, and uploads the plans, item bases, tile maps and any host-resident
 * block tables into device memory owned by the handle (a synchronous, startup-time call: it
 * allocates).  dyna_kv_prepared_launch enqueues the whole batch on `stream` with ONE kernel and no
 * host-side validation, upload or allocation, so it can be captured into a CUDA graph and
 * replayed; each launch re-reads the rows and the device block tables as they are then (the tables
 * must keep their entries).  No per-chunk flags (DYNA_EINVAL with DYNA_MIGRATE_SIGNAL).  The
 * launches of one handle share its deferred-error word: dyna_kv_wait of any of them reports, and
 * clears, the errors of every earlier launch.  The handle must outlive every launch made from it
 * (until dyna_kv_wait); dyna_kv_prepared_destroy never synchronises the device. */
typedef struct dyna_kv_prepared* dyna_kv_prepared_t;
DYNA_API dyna_status dyna_kv_prepare_batch(const dyna_kv_migration* migs, int32_t n, dyna_range layer_range,
                                           int32_t chunk_tokens, const dyna_kv_opts* opts, dyna_kv_prepared_t* out);
/* The same for a whole TP reshard (dyna_kv_reshard's arguments and rules; one launch). */
DYNA_API dyna_status dyna_kv_prepare_reshard(const dyna_kv_head_migration* migs, int32_t n, dyna_range token_range,
                                             dyna_range layer_range, int32_t chunk_tokens, const dyna_kv_opts* opts,
                                             dyna_kv_prepared_t* out);
DYNA_API dyna_status dyna_kv_prepared_launch(dyna_kv_prepared_t prepared, struct CUstream_st* stream,
                                             dyna_kv_xfer_t* out);
DYNA_API dyna_status dyna_kv_prepared_destroy(dyna_kv_prepared_t prepared);

/* Producer-coupled push (§4.3: "once chunk
 * k completes, its KV block is immediately DMA-pushed ... while Server1
 * continues with chunk k+1").  A ready board is an array of u64 slots on the
 * source device.  The producer (the prefill) marks chunk k on ITS stream after
 * the kernels that wrote chunk k's KV; one dyna_kv_migrate_on_ready launch on
 * another stream covers the whole range and copies chunk k as soon as its
 * mark (>= epoch) is visible — no host round trip per chunk.
 * Chunk k = tokens [begin + k*c, min(begin + (k+1)*c, end)) of that call.
 * The migration kernel stays resident while it waits, so its grid is capped
 * (opts->max_ctas, default and maximum: half the SMs) to leave the producer
 * room to run; FUSED variant with the VEC engine only.  A board is reused
 * across requests with increasing epochs (dyna_kv_ready_begin).
 * HAZARD: while such a migration waits, anything that synchronises the whole
 * device (cudaDeviceSynchronize, cudaMalloc/cudaFree that sync — including
 * this library's create / import calls, which allocate — synchronous copies
 * on the legacy stream, e.g. a framework's host-to-device copy on the default
 * stream when the coupled migration runs there) before the last chunk is marked
 * deadlocks (this library's migration calls themselves initialise what they
 * create on first use — a pool pair's chunk counters, tile-map cache entries —
 * on a non-blocking library stream, never on the legacy stream): the
 * device waits for the migration, the migration for a mark that is never
 * issued.  The same holds for the FIRST launch of any kernel in the process
 * while the migration waits: CUDA loads kernels lazily and a module load
 * synchronises the context.  This library preloads all of its own kernels;
 * run the producer's kernels once before the first coupled migration (or set
 * CUDA_MODULE_LOADING=EAGER).  Each chunk wait therefore gives up after the board's timeout
 * (default 10 s; dyna_kv_ready_set_timeout) and dyna_kv_wait then returns
 * DYNA_ETIMEDOUT (a chunk whose wait timed out is skipped: no flag, rows unspecified). */
typedef struct dyna_kv_ready* dyna_kv_ready_t;
DYNA_API dyna_status dyna_kv_ready_create(int32_t device, int32_t max_chunks, dyna_kv_ready_t* out);
DYNA_API dyna_status dyna_kv_ready_destroy(dyna_kv_ready_t board);
DYNA_API dyna_status dyna_kv_ready_set_timeout(dyna_kv_ready_t board, uint64_t timeout_ns);
/* A fresh epoch for the next request on this board (host counter; no device work). */
DYNA_API dyna_status dyna_kv_ready_begin(dyna_kv_ready_t board, uint64_t* epoch);
/* Enqueue on the producer's stream: slot[chunk] = epoch (release, GPU scope). */
DYNA_API dyna_status dyna_kv_ready_mark(dyna_kv_ready_t board, int32_t chunk, uint64_t epoch,
                                        struct CUstream_st* producer_stream);
/* Layer-granular marks (opts->flags & DYNA_READY_PER_LAYER; §4.3
 * chunk-level transfer "can be composed with" layer-level transfer):
 * the producer marks slot k*(l1-l0) + (l-l0) once layer l of chunk k has
 * written its KV, and those rows move as soon as that mark is visible, while
 * the prefill still computes the chunk's later layers.  The board then needs
 * num_chunks*(l1-l0) slots.
 * Tail: with one mark per chunk, the chunk marked last is moved by the capped
 * grid after the producer ends (at 512-MiB chunks that exposes more than one
 * whole-range push).  Cover every chunk but the last with the
 * coupled launch and push the last chunk with dyna_kv_migrate (full width) on
 * a stream that waits for the producer — or mark per (chunk, layer).
 * Cancellation (when r^alpha ends before s, "its
 * transfer is aborted"): see dyna_kv_ready_cancel.  The board must outlive
 * every migration launched on it (until dyna_kv_wait returns). */
DYNA_API dyna_status dyna_kv_migrate_on_ready(dyna_block_table src, dyna_block_table dst,
                                              dyna_range token_range, dyna_range layer_range,
                                              int32_t chunk_tokens, dyna_kv_ready_t board, uint64_t epoch,
                                              struct CUstream_st* stream, const dyna_kv_opts* opts,
                                              dyna_kv_xfer_t* out);
/* Cancel, from the host and with immediate effect, every migration on this
 * board whose epoch is <= `epoch` (the cancel epoch reaches the device word
 * the waiting warps poll by an 8-byte DMA on the board's own non-blocking
 * stream; the call returns once it has landed and needs no free SM).  A running migration stops waiting: a slot
 * whose mark is visible when a warp reaches it is still copied (so every
 * MARKED chunk is delivered whole, and its per-chunk flag is raised when
 * signalling); the items of a slot whose mark is not visible are skipped, and
 * a chunk with any skipped item never gets its flag.  dyna_kv_wait of a
 * cancelled migration returns DYNA_ECANCELED; destination rows of chunks
 * without a flag are unspecified (partially written), rows outside the
 * token range are untouched as always.  Cancelling is monotone (an epoch
 * below the board's current cancel epoch is a no-op). */
DYNA_API dyna_status dyna_kv_ready_cancel(dyna_kv_ready_t board, uint64_t epoch);

/* Receiver-steered placement across processes (the STAGED shape, SURVEY §8a
 * a2-a4; §4.3: "messages steering placement on the receiver
 * side").  The RECEIVER owns a channel: a ring of staging slots plus one
 * "full" and one "credit" sequence word per slot, in its own device memory.
 * It exports the channel; the SENDER imports it and pushes: for every
 * sub-chunk (chunks cut to fit one slot) a kernel gathers the source rows
 * straight into the receiver's slot over NVLink and releases the slot's full
 * word (system scope), after waiting for the slot's credit.  The receiver
 * places: it waits for the full word, scatters the slot through ITS OWN block
 * table, optionally raises its per-chunk inbox flags, and returns the credit.
 * The sender never sees the destination table.  Both sides must describe the
 * same migration (token range, layer range, chunk_tokens) in the same order;
 * each channel carries one sender's pushes to one destination pool. */
typedef struct dyna_kv_channel* dyna_kv_channel_t;
typedef struct {
    uint8_t mem[64];         /* cudaIpcMemHandle_t of the channel allocation */
    uint64_t slot_bytes;
    int32_t slots;
    int32_t sender;          /* sender instance id (inbox row for the chunk flags) */
    dyna_kv_pool_desc desc;  /* the receiver pool's geometry */
} dyna_kv_channel_handle;

/* Receiver: a channel into `dst` for sender `sender` (slots >= 2, slot_bytes a
 * multiple of 16 holding at least one token of the migrations to come). */
DYNA_API dyna_status dyna_kv_channel_create(dyna_kv_pool_t dst, int32_t sender, int32_t slots, uint64_t slot_bytes,
                                            dyna_kv_channel_t* out);
DYNA_API dyna_status dyna_kv_channel_export(dyna_kv_channel_t ch, dyna_kv_channel_handle* out);
/* Sender: map a receiver's channel into `local_device`. */
DYNA_API dyna_status dyna_kv_channel_import(const dyna_kv_channel_handle* h, int32_t local_device,
                                            dyna_kv_channel_t* out);
DYNA_API dyna_status dyna_kv_channel_destroy(dyna_kv_channel_t ch);
/* Device-side waits of push (credits) and place (full words) give up after this
 * long (default 10 s) and report DYNA_ETIMEDOUT at dyna_kv_wait. */
DYNA_API dyna_status dyna_kv_channel_set_timeout(dyna_kv_channel_t ch, uint64_t timeout_ns);
/* Sender: push tokens x layers of `src` into the channel, chunk by chunk, on `stream` (source device). */
DYNA_API dyna_status dyna_kv_push(dyna_block_table src, dyna_range token_range, dyna_range layer_range,
                                  int32_t chunk_tokens, dyna_kv_channel_t ch, struct CUstream_st* stream,
                                  dyna_kv_xfer_t* out);
/* Receiver: place the pushed rows through `dst` (a table of the channel's pool) on `stream`
 * (receiver device).  opts->flags may request per-chunk inbox flags (sender = the channel's). */
DYNA_API dyna_status dyna_kv_place(dyna_kv_channel_t ch, dyna_block_table dst, dyna_range token_range,
                                   dyna_range layer_range, int32_t chunk_tokens, struct CUstream_st* stream,
                                   const dyna_kv_opts* opts, dyna_kv_xfer_t* out);

/* Head-sliced channel traffic (TP resharding in the receiver-steered form;
 * reading R14): the sender pushes its heads [src_heads) of every row, packed
 * as [layer][K|V][token][n_heads*d*e] into the receiver's slots; the receiver
 * places them into its heads [dst_head_begin, dst_head_begin + num_heads).
 * Both sides must describe the same token range, layer range, chunk_tokens
 * and head count, in the same order; the pools may differ in H (L, d, e
 * agree with the channel's pool).  Everything else as dyna_kv_push / _place. */
DYNA_API dyna_status dyna_kv_push_heads(dyna_block_table src, dyna_range token_range, dyna_range layer_range,
                                        dyna_range src_heads, int32_t chunk_tokens, dyna_kv_channel_t ch,
                                        struct CUstream_st* stream, dyna_kv_xfer_t* out);
DYNA_API dyna_status dyna_kv_place_heads(dyna_kv_channel_t ch, dyna_block_table dst, dyna_range token_range,
                                         dyna_range layer_range, int32_t dst_head_begin, int32_t num_heads,
                                         int32_t chunk_tokens, struct CUstream_st* stream,
                                         const dyna_kv_opts* opts, dyna_kv_xfer_t* out);

/* CUDA graphs: dyna_kv_migrate / _ex with DEVICE block tables may be captured
 * into a CUDA graph (stream capture) and replayed; release each handle with
 * dyna_kv_wait after the capture ends (it returns at once — the captured work
 * runs at replay).  Host-resident tables and dyna_kv_migrate_batch (whose
 * descriptors travel through the upload ring) are refused during capture
 * (DYNA_ENOTSUP).  Per-chunk signalling inside a replayed graph reuses the
 * epoch assigned at capture time. */

/* Block the host until every chunk is resident in the destination, report
 * deferred errors (DYNA_ECUDA; DYNA_ERANGE from device-side id checks,
 * DYNA_ETIMEDOUT from device-side waits) of THIS migration — each handle has
 * its own deferred-error word, so concurrent migrations never see each
 * other's errors — and free the handle.  (Migrations captured into a CUDA
 * graph report through dyna_kv_poll_error instead.) */
DYNA_API dyna_status dyna_kv_wait(dyna_kv_xfer_t xfer);

/* Non-blocking: DYNA_OK if complete, DYNA_EAGAIN if in flight.  Does not free. */
DYNA_API dyna_status dyna_kv_query(dyna_kv_xfer_t xfer);

/* Enqueue on `stream` (work is ordered after it) a wait until the whole
 * migration is complete — the device-side form of dyna_kv_wait, for a
 * consumer (r^beta's compute) on another stream of the source device. */
DYNA_API dyna_status dyna_kv_stream_wait(dyna_kv_xfer_t xfer, struct CUstream_st* stream);

/* Per-chunk readiness (DYNA_MIGRATE_SIGNAL).  Each signalled migration gets
 * an epoch, monotone per (sender instance, destination pool), and its own
 * range of consecutive inbox slots [first_slot, first_slot + num_chunks) of
 * that (sender, destination pool).  Chunk k of the migration is resident when
 * inbox slot [sender][first_slot + k] holds a value >= epoch.  Concurrent
 * signalled migrations (any streams, any threads, chunk streams included) use
 * disjoint slots; a slot is reused only after DYNA_MAX_CHUNKS further chunks
 * were reserved by the same sender for the same pool (a migration must have
 * completed by then: its per-slot byte counters are reused too), and flags
 * are raised with an atomic max (never lowered).  Epochs and slots are keyed on the
 * destination pool's identity, which an IPC export carries, and start above
 * every flag already in the row, so a restarted sender or a re-imported pool
 * never reuses an epoch.  Any pointer may be NULL. */
DYNA_API dyna_status dyna_kv_xfer_info(dyna_kv_xfer_t xfer, uint64_t* epoch, int32_t* num_chunks, int32_t* sender,
                                       int32_t* first_slot);

/* What a migration resolved to (AUTO choices included) and how many kernels
 * it launched — for logs and benchmarks.  Any pointer may be NULL. */
DYNA_API dyna_status dyna_kv_xfer_plan(dyna_kv_xfer_t xfer, int32_t* variant, int32_t* engine, int32_t* piece_bytes,
                                       int32_t* stages, int32_t* unroll, int32_t* launches);

/* Enqueue on `stream` (a stream of the DESTINATION pool's device) a device
 * wait (acquire, system scope) until inbox slot `chunk` (= first_slot + k for
 * chunk k of a migration, dyna_kv_xfer_info) from `sender` reaches `epoch`;
 * work after it on `stream` sees the chunk's rows.  timeout_ns 0 = no
 * timeout; on timeout the kernel records DYNA_ETIMEDOUT for the next
 * dyna_kv_poll_error on that process. */
DYNA_API dyna_status dyna_kv_stream_wait_chunk(dyna_kv_pool_t dst, int32_t sender, int32_t chunk,
                                      uint64_t epoch, uint64_t timeout_ns,
                                      struct CUstream_st* stream);

/* Enqueue on `stream` a copy of inbox slots [sender][first, first+n) of
 * `dst` into host memory `host_out` (n uint64 values; pinned memory makes it
 * asynchronous).  Lets a host-side scheduler see which chunks have landed
 * (r^beta may start once all chunks covering [0, s) are resident). */
DYNA_API dyna_status dyna_kv_copy_flags(dyna_kv_pool_t dst, int32_t sender, int32_t first, int32_t n,
                                        uint64_t* host_out, struct CUstream_st* stream);

/* Replace the calibration table (copied; n <= 256).  n = 0 restores the built-in table. */
DYNA_API dyna_status dyna_kv_calib_set(const dyna_kv_calib_entry* entries, int32_t n);
/* Copy up to cap entries of the current table into out; returns the entry count (>= 0). */
DYNA_API int32_t dyna_kv_calib_get(dyna_kv_calib_entry* out, int32_t cap);

/* Measure AUTO's choice on this hardware for one (source pool, destination pool) pair and
 * install it (north_star item 4: the fused variant "chosen over the staged variant
 * per chunk size by measured bandwidth").  For each of the n chunk sizes chunk_tokens[i], every
 * candidate below migrates `reps` calls of that many tokens (all layers; token offsets cycling
 * through the tables so a call does not find the previous one's rows in L2) back to back while
 * the stream is held by a device-side gate, so the CUDA events around them time device work
 * only; the fastest candidate becomes the entry (row bytes of the pair, its locality: same
 * GPU = 0, other GPU or imported pool = 1, max_chunk_tokens = chunk_tokens[i]; the largest size
 * also covers every longer call), replacing the table's entries for that (row bytes, locality).
 * Candidates, in order (DYNA_CALIB_CANDIDATES): FUSED VEC 4 KiB x U8, FUSED VEC 8 KiB x U4,
 * FUSED VEC 16 KiB x U16, FUSED BULK ring 32 KiB x 4, STAGED VEC 8 KiB x U8, STAGED BULK
 * 32 KiB x 4, FUSED TILES (STAGED is skipped — 0 GB/s — into an imported pool or a destination
 * table without device ids on another GPU; TILES when no tensor map fits the rows, and for
 * destinations on another GPU or imported).  out[i] receives the entry for chunk_tokens[i]; gbps (NULL or
 * n x DYNA_CALIB_CANDIDATES floats) the payload GB/s of every candidate.  Tables: as
 * dyna_kv_migrate_ex (host ids or DYNA_MIGRATE_UNCHECKED semantics: the destination rows must
 * be distinct); both must cover at least the largest chunk size.  The call OVERWRITES the
 * destination rows its tables map, and synchronises `stream` (a startup-time call).  Errors:
 * DYNA_EINVAL (n <= 0, chunk sizes <= 0 or not ascending, reps < 1), DYNA_ERANGE (a chunk size
 * longer than the tables), or any error of the migrations it runs. */
#define DYNA_CALIB_CANDIDATES 7
DYNA_API dyna_status dyna_kv_calibrate(dyna_block_table src, dyna_block_table dst, const int32_t* chunk_tokens,
                                       int32_t n, int32_t reps, struct CUstream_st* stream,
                                       dyna_kv_calib_entry* out, float* gbps);

/* Thread-local description of the last error on this thread. */
DYNA_API const char* dyna_kv_last_error(void);

/* Deferred device-side error recorded since the last call (and clear it). */
DYNA_API dyna_status dyna_kv_poll_error(void);

/* Number of kernels this library has launched in this process. */
DYNA_API uint64_t dyna_kv_launch_count(void);

/* ---------------- peers ---------------- */

/* Enable P2P from `device` to `peer` (both in this process).  DYNA_EPEER if
 * the pair cannot access each other.  dyna_kv_migrate also does this lazily. */
DYNA_API dyna_status dyna_kv_enable_peer(int32_t device, int32_t peer);

/* Cross-process pools (one process per GPU): the owner exports its pool, a
 * peer imports it and can then use it as a migration destination (or
 * source).  The handle is plain bytes; send it with any channel (e.g.
 * torch.distributed all_gather_object). */
typedef struct {
    uint8_t pool_mem[64];    /* cudaIpcMemHandle_t of the allocation holding the pool */
    uint8_t inbox_mem[64];   /* cudaIpcMemHandle_t of the pool's flag inbox */
    uint64_t pool_offset;    /* byte offset of device_base inside its allocation */
    dyna_kv_pool_desc desc;  /* the owner's geometry */
    uint64_t uid;            /* the pool's identity (flag epochs / slots and alias checks key on it) */
} dyna_kv_ipc_handle;

DYNA_API dyna_status dyna_kv_pool_export(dyna_kv_pool_t pool, dyna_kv_ipc_handle* out);
/* Map a peer's pool into `local_device`'s address space. */
DYNA_API dyna_status dyna_kv_pool_import(const dyna_kv_ipc_handle* handle, int32_t local_device, dyna_kv_pool_t* out);

/* ---------------- test-input generator (NOT part of the migration) -------------
 * Fill `bytes` (multiple of 16) at device pointer `dst` with the kvgen stream
 * for `seed`, starting at stream byte `byte_offset` (multiple of 8):
 *   word(w) = splitmix64(splitmix64(seed) ^ (w * 0xD1B54A32D192ED03)).
 * Same counter generator as kvgen/__init__.py (each side implements it). */
DYNA_API dyna_status dyna_kv_debug_fill(void* dst, uint64_t bytes, uint64_t seed, uint64_t byte_offset,
                               struct CUstream_st* stream);

#ifdef __cplusplus
}
#endif
#endif /* DYNA_KV_H */
