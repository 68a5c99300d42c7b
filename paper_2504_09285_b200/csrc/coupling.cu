// coupling.cu — the two ways a migration is coupled to the instances around it:
// producer-coupled ready boards (one launch waits per chunk for the prefill's
// mark) and receiver-steered placement channels (the sender
// fills the receiver's staging slots, the receiver scatters with its own block
// table; §4.3, SURVEY §8 a2-a4 across processes).
#include "runtime.cuh"

using namespace dynakv;
using namespace dynakv::rt;

extern "C" {

dyna_status dyna_kv_ready_create(int32_t device, int32_t max_chunks, dyna_kv_ready_t* out) {
  if (!out || device < 0 || max_chunks <= 0 || max_chunks > (1 << 24)) return fail(DYNA_EINVAL, "bad argument");
  *out = nullptr;
  flush_retired();
  auto* b = new dyna_kv_ready();
  b->dev = device;
  b->max_chunks = max_chunks;
  DeviceGuard g(device);
  // cudaMalloc of a board (like any allocation) may synchronise the device: create boards
  // before starting coupled migrations (dyna_kv.h).  The initialisation itself runs on the
  // board's own non-blocking control stream.
  const size_t sb = sizeof(unsigned long long) * max_chunks;
  bool ok = cudaStreamCreateWithFlags(&b->ctrl, cudaStreamNonBlocking) == cudaSuccess &&
            cudaMalloc(&b->slots, sb) == cudaSuccess &&
            cudaMalloc(&b->cancel_dev, sizeof(unsigned long long)) == cudaSuccess &&
            cudaHostAlloc(&b->cancel_stage, sizeof(unsigned long long), cudaHostAllocPortable) == cudaSuccess;
  ok = ok && cudaMemsetAsync(b->slots, 0, sb, b->ctrl) == cudaSuccess &&
       cudaMemsetAsync(b->cancel_dev, 0, sizeof(unsigned long long), b->ctrl) == cudaSuccess &&
       cudaStreamSynchronize(b->ctrl) == cudaSuccess;
  if (!ok) {
    cudaFree(b->slots);
    cudaFree(b->cancel_dev);
    if (b->cancel_stage) cudaFreeHost(b->cancel_stage);
    if (b->ctrl) cudaStreamDestroy(b->ctrl);
    delete b;
    return fail(DYNA_ENOMEM, "ready board of %d slots", max_chunks);
  }
  dev_info(device);
  *out = b;
  return DYNA_OK;
}

dyna_status dyna_kv_ready_destroy(dyna_kv_ready_t b) {
  if (!b) return fail(DYNA_EINVAL, "NULL board");
  retire(b->dev, b->slots, Mem::Device);  // released by the next allocating call (no device sync here)
  retire(b->dev, b->cancel_dev, Mem::Device);
  retire(b->dev, b->cancel_stage, Mem::Host);
  {
    DeviceGuard g(b->dev);
    cudaStreamDestroy(b->ctrl);
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

dyna_status dyna_kv_ready_cancel(dyna_kv_ready_t b, uint64_t epoch) {
  if (!b) return fail(DYNA_EINVAL, "NULL board");
  std::lock_guard<std::mutex> lk(b->cancel_mu);
  if (epoch <= b->cancel_epoch.load()) return DYNA_OK;  // monotone
  b->cancel_epoch.store(epoch);
  // one 8-byte DMA on the board's own non-blocking stream: it does not wait for the
  // (possibly still waiting) migration kernels, and no SM is needed to deliver it
  DeviceGuard g(b->dev);
  *b->cancel_stage = epoch;
  CUDA_TRY(cudaMemcpyAsync(b->cancel_dev, b->cancel_stage, sizeof(unsigned long long), cudaMemcpyHostToDevice,
                           b->ctrl));
  CUDA_TRY(cudaStreamSynchronize(b->ctrl));
  return DYNA_OK;
}

dyna_status dyna_kv_ready_mark(dyna_kv_ready_t b, int32_t chunk, uint64_t epoch, struct CUstream_st* stream) {
  if (!b) return fail(DYNA_EINVAL, "NULL board");
  if (chunk < 0 || chunk >= b->max_chunks) return fail(DYNA_ERANGE, "chunk %d outside the board", chunk);
  DeviceGuard g(b->dev);
  launch_mark_ready(b->slots + chunk, epoch, reinterpret_cast<cudaStream_t>(stream));
  CUDA_TRY(cudaGetLastError());
  return DYNA_OK;
}

// ---------------------------------------------------------------- receiver-steered placement channel

static int64_t chan_subchunk(const dyna_kv_channel* ch, int64_t row, int lm, int64_t c) {
  const int64_t tok = row * lm * 2;
  return std::min<int64_t>(c, (int64_t)ch->slot_bytes / tok);
}

dyna_status dyna_kv_channel_create(dyna_kv_pool_t dst, int32_t sender, int32_t slots, uint64_t slot_bytes,
                                   dyna_kv_channel_t* out) {
  if (!out || !dst) return fail(DYNA_EINVAL, "NULL argument");
  *out = nullptr;
  if (dst->imported) return fail(DYNA_EINVAL, "create the channel on the destination pool's owner");
  flush_retired();
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

dyna_status dyna_kv_channel_set_timeout(dyna_kv_channel_t ch, uint64_t timeout_ns) {
  if (!ch || timeout_ns == 0) return fail(DYNA_EINVAL, "bad argument");
  ch->timeout_ns = timeout_ns;
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
  flush_retired();
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
  retire(ch->push_counters_dev, ch->push_counters, Mem::Device);  // no device sync in a destroy
  retire(ch->dev, ch->place_counters, Mem::Device);
  retire(ch->dev, ch->base, ch->imported ? Mem::Ipc : Mem::Device);
  delete ch;
  return DYNA_OK;
}

// Shared checks of push / place: geometry against the channel, ranges, a device table.
// slice > 0: head-sliced push / place of `slice` bytes per token (H may differ from the channel's).
static dyna_status chan_check(const dyna_kv_channel* ch, const dyna_block_table& t, dyna_range tr, dyna_range lr,
                              int32_t c, bool* empty, int64_t slice = 0) {
  if (!ch || !t.pool) return fail(DYNA_EINVAL, "NULL channel or pool");
  const dyna_kv_pool_desc &g = t.pool->desc, &cg = ch->desc;
  if (g.num_layers != cg.num_layers || (!slice && g.num_kv_heads != cg.num_kv_heads) || g.head_dim != cg.head_dim ||
      g.elem_bytes != cg.elem_bytes)
    return fail(DYNA_EGEOM, "pool geometry differs from the channel's");
  if (lr.begin < 0 || lr.begin > lr.end || lr.end > g.num_layers) return fail(DYNA_ERANGE, "bad layer range");
  if (tr.begin < 0 || tr.begin > tr.end || tr.end >= (int64_t(1) << 31)) return fail(DYNA_ERANGE, "bad token range");
  *empty = tr.begin == tr.end || lr.begin == lr.end;
  if (*empty) return DYNA_OK;
  if (c <= 0) return fail(DYNA_ERANGE, "chunk_tokens must be > 0");
  if (tr.end > t.len * g.block_size) return fail(DYNA_ERANGE, "token range exceeds the block table");
  if (!t.block_ids) return fail(DYNA_EINVAL, "push/place need device block_ids");
  if (chan_subchunk(ch, slice ? slice : t.pool->row, (int)(lr.end - lr.begin), c) < 1)
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
  return zeroed_alloc(reinterpret_cast<void**>(c), sizeof(unsigned long long) * DYNA_MAX_CHUNKS, dev);
}

dyna_status dyna_kv_push(dyna_block_table src, dyna_range tr, dyna_range lr, int32_t c, dyna_kv_channel_t ch,
                         struct CUstream_st* stream_, dyna_kv_xfer_t* out) {
  if (!out) return fail(DYNA_EINVAL, "NULL out");
  *out = nullptr;
  bool empty = false;
  dyna_status r = chan_check(ch, src, tr, lr, c, &empty);
  if (r) return r;
  dyna_kv_pool* S = src.pool;
  if (empty) {
    auto* x = new dyna_kv_xfer();
    x->dev = S->dev;
    x->sender = ch->sender;
    x->empty = true;
    *out = x;
    return DYNA_OK;
  }
  if (ch->imported ? ch->dev != S->dev : (ch->dev != S->dev && (r = ensure_peer(S->dev, ch->dev)) != DYNA_OK))
    return r ? r : fail(DYNA_EPEER, "channel mapped on device %d, source on %d", ch->dev, S->dev);
  dyna_kv_xfer* x = nullptr;
  if ((r = new_xfer(S->dev, ch->sender, reinterpret_cast<cudaStream_t>(stream_), &x))) return r;
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
        launch_wait_flag(ch->credit + slot, q - ch->slots + 1, ch->timeout_ns, stream, x->err);
      }
      // gather straight into the receiver's slot; the last writer releases full[slot] = q + 1
      Plan p = make_plan(paged(S, src.block_ids), linear(ch->base + (size_t)slot * ch->slot_bytes), S->row, sa,
                         sb, l0, lm, sb - sa, S->desc.block_size, kVecPiece);
      p.err = x->err;
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
  if (empty) {
    auto* x = new dyna_kv_xfer();
    x->dev = D->dev;
    x->sender = ch->sender;
    x->empty = true;
    *out = x;
    return DYNA_OK;
  }
  dyna_kv_xfer* x = nullptr;
  if ((r = new_xfer(D->dev, ch->sender, reinterpret_cast<cudaStream_t>(stream_), &x))) return r;
  x->nchunks = (int32_t)nchunks;
  std::lock_guard<std::mutex> lk(ch->mu);
  unsigned long long *flags = nullptr, *counters = nullptr;
  if (signal) {
    if ((r = chan_counters(&ch->place_counters, D->dev)) ||
        (r = flag_reserve(ch->sender, D, nchunks, &x->epoch, &x->first_slot))) {
      delete x;
      return r;
    }
    flags = D->inbox + (size_t)ch->sender * DYNA_MAX_CHUNKS + x->first_slot;
    counters = ch->place_counters + x->first_slot;
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
      launch_wait_flag(ch->full + slot, q + 1, ch->timeout_ns, stream, x->err);
      Plan p = make_plan(linear(ch->base + (size_t)slot * ch->slot_bytes), paged(D, dst.block_ids), D->row, sa, sb,
                         l0, lm, sb - sa, D->desc.block_size, kVecPiece);
      set_chunking(p, tr.begin, tr.end, c);
      p.err = x->err;
      if (signal) {
        p.counters = counters;
        p.flags = flags;
        p.epoch = x->epoch;
      }
      r = launch_copy(p, DYNA_ENGINE_VEC, o.max_ctas, kBulkStages, kVecU, D->dev, stream, 0);
      launch_release_sys(ch->credit + slot, q + 1, stream);  // the slot may be refilled
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

// ---------------------------------------------------------------- head-sliced channel (TP resharding)
// The slot holds packed slices [l][kv][t][n_heads*d*e]: the sender gathers its heads
// [h0, h0 + n) of every row, the receiver scatters them into its heads [hd0, hd0 + n).
static dyna_status head_slice(const dyna_kv_pool_desc& g, int64_t h0, int64_t n, int64_t* slice) {
  const int64_t he = (int64_t)g.head_dim * g.elem_bytes;
  if (h0 < 0 || n <= 0 || h0 + n > g.num_kv_heads)
    return fail(DYNA_ERANGE, "heads [%lld, %lld) outside [0, %d)", (long long)h0, (long long)(h0 + n), g.num_kv_heads);
  if (he % 16) return fail(DYNA_EGEOM, "head slices must be multiples of 16 bytes (d*e = %lld)", (long long)he);
  *slice = n * he;
  return DYNA_OK;
}

dyna_status dyna_kv_push_heads(dyna_block_table src, dyna_range tr, dyna_range lr, dyna_range src_heads, int32_t c,
                               dyna_kv_channel_t ch, struct CUstream_st* stream_, dyna_kv_xfer_t* out) {
  if (!out) return fail(DYNA_EINVAL, "NULL out");
  *out = nullptr;
  if (!src.pool) return fail(DYNA_EINVAL, "NULL pool");
  int64_t slice = 0;
  dyna_status r = head_slice(src.pool->desc, src_heads.begin, src_heads.end - src_heads.begin, &slice);
  if (r) return r;
  bool empty = false;
  if ((r = chan_check(ch, src, tr, lr, c, &empty, slice))) return r;
  dyna_kv_pool* S = src.pool;
  if (empty) {
    auto* x = new dyna_kv_xfer();
    x->dev = S->dev;
    x->sender = ch->sender;
    x->empty = true;
    *out = x;
    return DYNA_OK;
  }
  if (ch->imported ? ch->dev != S->dev : (ch->dev != S->dev && (r = ensure_peer(S->dev, ch->dev)) != DYNA_OK))
    return r ? r : fail(DYNA_EPEER, "channel mapped on device %d, source on %d", ch->dev, S->dev);
  dyna_kv_xfer* x = nullptr;
  if ((r = new_xfer(S->dev, ch->sender, reinterpret_cast<cudaStream_t>(stream_), &x))) return r;
  std::lock_guard<std::mutex> lk(ch->mu);
  if ((r = chan_counters(&ch->push_counters, S->dev))) {
    delete x;
    return r;
  }
  ch->push_counters_dev = S->dev;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  DeviceGuard guard(S->dev);
  const int l0 = (int)lr.begin, lm = (int)(lr.end - lr.begin);
  const int64_t sc = chan_subchunk(ch, slice, lm, c);
  const int64_t he = (int64_t)S->desc.head_dim * S->desc.elem_bytes;
  const uint64_t seq0 = ch->push_seq;
  const uint64_t launches0 = g_launches.load();
  for (int64_t a = tr.begin; a < tr.end && !r; a += c) {
    const int64_t b = std::min<int64_t>(a + c, tr.end);
    for (int64_t sa = a; sa < b && !r; sa += sc) {
      const int64_t sb = std::min(sa + sc, b);
      const uint64_t q = ch->push_seq++;
      const int slot = (int)(q % ch->slots);
      if (q >= (uint64_t)ch->slots) launch_wait_flag(ch->credit + slot, q - ch->slots + 1, ch->timeout_ns, stream, x->err);
      Plan p = make_plan_sliced(paged(S, src.block_ids), linear(ch->base + (size_t)slot * ch->slot_bytes), slice,
                                S->row, src_heads.begin * he, slice, 0, sa, sb, l0, lm, sb - sa, S->desc.block_size,
                                kVecPiece);
      p.err = x->err;
      p.counters = ch->push_counters;
      p.flags = ch->full + slot;
      p.epoch = q + 1;
      p.sys_fence = 1;
      r = launch_rows(p, 0, S->dev, stream);
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

dyna_status dyna_kv_place_heads(dyna_kv_channel_t ch, dyna_block_table dst, dyna_range tr, dyna_range lr,
                                int32_t dst_head_begin, int32_t num_heads, int32_t c, struct CUstream_st* stream_,
                                const dyna_kv_opts* opts, dyna_kv_xfer_t* out) {
  if (!out) return fail(DYNA_EINVAL, "NULL out");
  *out = nullptr;
  if (!dst.pool) return fail(DYNA_EINVAL, "NULL pool");
  int64_t slice = 0;
  dyna_status r = head_slice(dst.pool->desc, dst_head_begin, num_heads, &slice);
  if (r) return r;
  bool empty = false;
  if ((r = chan_check(ch, dst, tr, lr, c, &empty, slice))) return r;
  if (ch->imported || dst.pool != ch->dst) return fail(DYNA_EINVAL, "place on the channel's owner, into its pool");
  dyna_kv_opts o{};
  if ((r = check_opts(opts, &o))) return r;
  const bool signal = (o.flags & DYNA_MIGRATE_SIGNAL) != 0;
  dyna_kv_pool* D = dst.pool;
  const int64_t nchunks = empty ? 0 : (tr.end - tr.begin + c - 1) / c;
  if (signal && nchunks > DYNA_MAX_CHUNKS) return fail(DYNA_ERANGE, "too many chunks for signalling");
  if (empty) {
    auto* x = new dyna_kv_xfer();
    x->dev = D->dev;
    x->sender = ch->sender;
    x->empty = true;
    *out = x;
    return DYNA_OK;
  }
  dyna_kv_xfer* x = nullptr;
  if ((r = new_xfer(D->dev, ch->sender, reinterpret_cast<cudaStream_t>(stream_), &x))) return r;
  x->nchunks = (int32_t)nchunks;
  std::lock_guard<std::mutex> lk(ch->mu);
  unsigned long long *flags = nullptr, *counters = nullptr;
  if (signal) {
    if ((r = chan_counters(&ch->place_counters, D->dev)) ||
        (r = flag_reserve(ch->sender, D, nchunks, &x->epoch, &x->first_slot))) {
      delete x;
      return r;
    }
    flags = D->inbox + (size_t)ch->sender * DYNA_MAX_CHUNKS + x->first_slot;
    counters = ch->place_counters + x->first_slot;
  }
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  DeviceGuard guard(D->dev);
  const int l0 = (int)lr.begin, lm = (int)(lr.end - lr.begin);
  const int64_t sc = chan_subchunk(ch, slice, lm, c);
  const int64_t he = (int64_t)D->desc.head_dim * D->desc.elem_bytes;
  const uint64_t launches0 = g_launches.load();
  for (int64_t a = tr.begin; a < tr.end && !r; a += c) {
    const int64_t b = std::min<int64_t>(a + c, tr.end);
    for (int64_t sa = a; sa < b && !r; sa += sc) {
      const int64_t sb = std::min(sa + sc, b);
      const uint64_t q = ch->place_seq++;
      const int slot = (int)(q % ch->slots);
      launch_wait_flag(ch->full + slot, q + 1, ch->timeout_ns, stream, x->err);
      Plan p = make_plan_sliced(linear(ch->base + (size_t)slot * ch->slot_bytes), paged(D, dst.block_ids), slice,
                                slice, 0, D->row, (int64_t)dst_head_begin * he, sa, sb, l0, lm, sb - sa,
                                D->desc.block_size, kVecPiece);
      set_chunking(p, tr.begin, tr.end, c);
      p.err = x->err;
      if (signal) {
        p.counters = counters;
        p.flags = flags;
        p.epoch = x->epoch;
      }
      r = launch_rows(p, o.max_ctas, D->dev, stream);
      launch_release_sys(ch->credit + slot, q + 1, stream);  // the slot may be refilled
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

}  // extern "C"
