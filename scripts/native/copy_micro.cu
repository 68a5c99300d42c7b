// copy_micro.cu — engine micro-benchmark behind DESIGN.md §6d (not the product path).
//
// Question: why does the BULK engine's throughput scale with the bytes per TMA
// bulk op (8 KiB 831, 16 KiB 1595, 32 KiB 2746 GB/s payload on 2-KiB-row blocks,
// profiles/r01_l3_probe.json), and which engine shape moves random 32-KiB blocks
// (Llama-3-8B: 16 tokens x 2 KiB rows) at the HBM copy peak?
//
// Workload: n_items copies of `piece` bytes between two 2-GiB buffers; blocks of
// `blk` bytes are placed at random (permuted) block slots on both sides, each cut
// into blk/piece consecutive items — the item list the production decode yields,
// precomputed here so that decode cost is out of the picture.  512 MiB payload.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o copy_micro copy_micro.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e = (x);                                                                   \
    if (e != cudaSuccess) {                                                                \
      fprintf(stderr, "%s: %s (%s:%d)\n", #x, cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

struct It {
  int64_t s, d;
};

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n .reg .pred P;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W_%=;\n}\n" ::"r"(
          sa(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void bl(void* s, const void* g, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(s)),
               "l"(g), "r"(n), "r"(sa(b))
               : "memory");
}
__device__ __forceinline__ void bs(void* g, const void* s, uint32_t n) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(sa(s)), "r"(n) : "memory");
}
__device__ __forceinline__ void bcommit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bwait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bwait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// ---- A: W independent single-thread TMA rings per CTA (lane 0 of each warp)
__global__ void k_bulk(const It* __restrict__ items, int64_t n, const char* S, char* D, int piece, int stages, int W,
                       int lag) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[64];
  __shared__ int64_t pd[64];
  __shared__ uint32_t pn[64];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) != 0) return;
  uint64_t* f = full + w * stages;
  int64_t* PD = pd + w * stages;
  uint32_t* PN = pn + w * stages;
  unsigned char* ring = sm + (size_t)w * stages * piece;
  for (int s = 0; s < stages; ++s) mb_init(&f[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  int64_t next = (int64_t)blockIdx.x * W + w;
  const int64_t stride = (int64_t)gridDim.x * W;
  auto refill = [&](int s) {
    if (next < n) {
      const It it = items[next];
      next += stride;
      mb_tx(&f[s], piece);
      bl(ring + (size_t)s * piece, S + it.s, piece, &f[s]);
      PD[s] = it.d;
      PN[s] = piece;
    } else {
      PN[s] = 0;
    }
  };
  for (int s = 0; s < stages; ++s) refill(s);
  for (int64_t i = 0;; ++i) {
    const int s = (int)(i % stages);
    if (PN[s] == 0) break;
    mb_wait(&f[s], (uint32_t)((i / stages) & 1));
    bs(D + PD[s], ring + (size_t)s * piece, PN[s]);
    bcommit();
    if (i >= lag) {
      if (lag == 3) bwait_read<3>(); else if (lag == 2) bwait_read<2>(); else bwait_read<1>();
      refill((int)((i - lag) % stages));
    }
  }
  bwait0();
}

// ---- B: warp per item, U 16-B loads per lane in flight
template <int U, int HINT>
__global__ void __launch_bounds__(256) k_vec(const It* __restrict__ items, int64_t n, const char* S, char* D,
                                             int piece) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nw) {
    const It it = items[i];
    const int4* s = reinterpret_cast<const int4*>(S + it.s);
    int4* d = reinterpret_cast<int4*>(D + it.d);
    const int nv = piece >> 4;
    for (int b = 0; b < nv; b += 32 * U) {
      int4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int4* p = s + b + u * 32 + lane;
        if (HINT == 1)
          asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                       : "l"(p));
        else
          asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                       : "l"(p));
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(d + b + u * 32 + lane),
                     "r"(v[u].x), "r"(v[u].y), "r"(v[u].z), "r"(v[u].w)
                     : "memory");
    }
  }
}

// ---- C: TMA bulk load by one thread, stores by the CTA's warps from shared memory
// (st.global.v4); slots handed back with an mbarrier of all storing warps.
__global__ void k_tma_stg(const It* __restrict__ items, int64_t n, const char* S, char* D, int piece, int stages) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[32], empty[32];
  __shared__ int64_t pd[32];
  __shared__ uint32_t pn[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nst = (blockDim.x >> 5) - 1;  // storing warps
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], nst);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane) return;
    int64_t next = blockIdx.x;
    for (int64_t i = 0;; ++i) {
      const int s = (int)(i % stages);
      if (i >= stages) mb_wait(&empty[s], (uint32_t)(((i / stages) - 1) & 1));
      if (next >= n) {
        pn[s] = 0;
        mb_arrive(&full[s]);
        break;
      }
      const It it = items[next];
      next += gridDim.x;
      pd[s] = it.d;
      pn[s] = piece;
      mb_tx(&full[s], piece);
      bl(ring + (size_t)s * piece, S + it.s, piece, &full[s]);
    }
    return;
  }
  const int sw = warp - 1;
  for (int64_t i = 0;; ++i) {
    const int s = (int)(i % stages);
    mb_wait(&full[s], (uint32_t)((i / stages) & 1));
    const uint32_t nb = pn[s];
    if (nb == 0) break;
    const int4* src = reinterpret_cast<const int4*>(ring + (size_t)s * piece);
    int4* dst = reinterpret_cast<int4*>(D + pd[s]);
    const int nv = nb >> 4;
    for (int v = sw * 32 + lane; v < nv; v += nst * 32) {
      int4 x = src[v];
      asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(dst + v), "r"(x.x), "r"(x.y),
                   "r"(x.z), "r"(x.w)
                   : "memory");
    }
    __syncwarp();
    if (lane == 0) mb_arrive(&empty[s]);
  }
}

// ---- D: like A but each refill also issues an L2 prefetch `ahead` items further
__global__ void k_bulk_pf(const It* __restrict__ items, int64_t n, const char* S, char* D, int piece, int stages,
                          int ahead) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t f[32];
  __shared__ int64_t PD[32];
  __shared__ uint32_t PN[32];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s) mb_init(&f[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  int64_t next = blockIdx.x;
  const int64_t stride = gridDim.x;
  for (int a = 0; a < ahead; ++a) {
    const int64_t j = next + (int64_t)(stages + a) * stride;
    if (j < n)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(S + items[j].s), "r"(piece) : "memory");
  }
  auto refill = [&](int s) {
    if (next < n) {
      const It it = items[next];
      const int64_t j = next + (int64_t)(stages + ahead) * stride;
      if (j < n)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(S + items[j].s), "r"(piece) : "memory");
      next += stride;
      mb_tx(&f[s], piece);
      bl(ring + (size_t)s * piece, S + it.s, piece, &f[s]);
      PD[s] = it.d;
      PN[s] = piece;
    } else {
      PN[s] = 0;
    }
  };
  for (int s = 0; s < stages; ++s) refill(s);
  const int lag = 2;
  for (int64_t i = 0;; ++i) {
    const int s = (int)(i % stages);
    if (PN[s] == 0) break;
    mb_wait(&f[s], (uint32_t)((i / stages) & 1));
    bs(D + PD[s], ring + (size_t)s * piece, PN[s]);
    bcommit();
    if (i >= lag) {
      bwait_read<2>();
      refill((int)((i - lag) % stages));
    }
  }
  bwait0();
}

// ---- E: cooperative loads into registers by all warps, then staged through smem and
// written back by ONE bulk store per item (loads on the LSU path, stores on TMA).
template <int U>
__global__ void __launch_bounds__(256) k_ldg_bulkst(const It* __restrict__ items, int64_t n, const char* S, char* D,
                                                    int piece) {
  extern __shared__ __align__(128) unsigned char buf[];  // 2 x piece per warp
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned char* mine = buf + (size_t)w * 2 * piece;
  int par = 0;
  for (int64_t i = warp; i < n; i += nw, par ^= 1) {
    const It it = items[i];
    const int4* s = reinterpret_cast<const int4*>(S + it.s);
    int4* sb = reinterpret_cast<int4*>(mine + (size_t)par * piece);
    if (lane == 0) bwait_read<1>();  // the store from this half (two items ago) has read it
    __syncwarp();
    const int nv = piece >> 4;
    for (int b = 0; b < nv; b += 32 * U) {
      int4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                     : "l"(s + b + u * 32 + lane));
#pragma unroll
      for (int u = 0; u < U; ++u) sb[b + u * 32 + lane] = v[u];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      bs(D + it.d, sb, piece);
      bcommit();
    }
  }
  if (lane == 0) bwait0();
}

// ---- F: head-sliced rows: an item = `rows` rows of `slice` bytes at `spitch` (source) / `dpitch`
// (destination) strides, copied lane-major over 16-B vectors, U in flight per lane (k_copy_rows).
template <int U>
__global__ void __launch_bounds__(256, 3) k_rows(const It* __restrict__ items, int64_t n, const char* S, char* D,
                                                 int rows, int slice, int spitch, int dpitch) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int vps = slice >> 4;
  const int nv = rows * vps;
  for (int64_t i = warp; i < n; i += nw) {
    const It it = items[i];
    for (int b = 0; b < nv; b += 32 * U) {
      int4 v[U];
      int r[U], c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = b + u * 32 + lane;
        r[u] = idx / vps;
        c[u] = idx - r[u] * vps;
        if (idx < nv)
          asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                       : "l"(S + it.s + (int64_t)r[u] * spitch + c[u] * 16));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = b + u * 32 + lane;
        if (idx < nv)
          asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(D + it.d + (int64_t)r[u] * dpitch +
                                                                                     c[u] * 16),
                       "r"(v[u].x), "r"(v[u].y), "r"(v[u].z), "r"(v[u].w)
                       : "memory");
      }
    }
  }
}

struct Bench {
  char *S, *D;
  It* items;
  int64_t n;
  int piece;
};

static float time_it(void (*fn)(const Bench&, void*), const Bench& b, void* arg, int reps = 12) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  std::vector<float> ms;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    fn(b, arg);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float t;
    CK(cudaEventElapsedTime(&t, e0, e1));
    if (r >= 2) ms.push_back(t);
  }
  std::sort(ms.begin(), ms.end());
  return ms[ms.size() / 2];
}

struct ACfg {
  int stages, W, ctas_per_sm, lag, sms;
};
static void run_a(const Bench& b, void* a) {
  const ACfg& c = *(const ACfg*)a;
  const size_t smem = (size_t)c.W * c.stages * b.piece;
  k_bulk<<<c.sms * c.ctas_per_sm, 32 * c.W, smem>>>(b.items, b.n, b.S, b.D, b.piece, c.stages, c.W, c.lag);
}
struct VCfg {
  int U, hint, ctas;
};
static void run_v(const Bench& b, void* a) {
  const VCfg& c = *(const VCfg*)a;
  if (c.U == 8 && c.hint == 0) k_vec<8, 0><<<c.ctas, 256>>>(b.items, b.n, b.S, b.D, b.piece);
  if (c.U == 8 && c.hint == 1) k_vec<8, 1><<<c.ctas, 256>>>(b.items, b.n, b.S, b.D, b.piece);
  if (c.U == 16 && c.hint == 0) k_vec<16, 0><<<c.ctas, 256>>>(b.items, b.n, b.S, b.D, b.piece);
  if (c.U == 16 && c.hint == 1) k_vec<16, 1><<<c.ctas, 256>>>(b.items, b.n, b.S, b.D, b.piece);
}
struct CCfg {
  int stages, warps, sms;
};
static void run_c(const Bench& b, void* a) {
  const CCfg& c = *(const CCfg*)a;
  k_tma_stg<<<c.sms, 32 * c.warps, (size_t)c.stages * b.piece>>>(b.items, b.n, b.S, b.D, b.piece, c.stages);
}
struct DCfg {
  int stages, ahead, sms;
};
static void run_d(const Bench& b, void* a) {
  const DCfg& c = *(const DCfg*)a;
  k_bulk_pf<<<c.sms, 32, (size_t)c.stages * b.piece>>>(b.items, b.n, b.S, b.D, b.piece, c.stages, c.ahead);
}
struct ECfg {
  int ctas, warps;
};
static void run_e(const Bench& b, void* a) {
  const ECfg& c = *(const ECfg*)a;
  k_ldg_bulkst<8><<<c.ctas, 256, (size_t)8 * 2 * b.piece>>>(b.items, b.n, b.S, b.D, b.piece);
}
static void run_memcpy(const Bench& b, void*) {
  CK(cudaMemcpyAsync(b.D, b.S, (size_t)b.n * b.piece, cudaMemcpyDeviceToDevice));
}

int main(int argc, char** argv) {
  int dev = 0;
  CK(cudaSetDevice(dev));
  int sms = 0, optin = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  for (auto k : {(const void*)k_bulk, (const void*)k_tma_stg, (const void*)k_bulk_pf, (const void*)k_ldg_bulkst<8>})
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 2048));
  const size_t pool = 2ull << 30;
  const size_t payload = 512ull << 20;
  char *S, *D;
  CK(cudaMalloc(&S, pool));
  CK(cudaMalloc(&D, pool));
  CK(cudaMemset(S, 1, pool));
  CK(cudaMemset(D, 2, pool));
  It* dItems;
  CK(cudaMalloc(&dItems, sizeof(It) * (payload / 4096)));
  std::mt19937_64 rng(250409285);

  auto make = [&](size_t blk, int piece, bool contiguous) {
    const int64_t nblk_pool = pool / blk, nblk = payload / blk;
    std::vector<int64_t> ps(nblk_pool), pd(nblk_pool);
    std::iota(ps.begin(), ps.end(), 0);
    std::iota(pd.begin(), pd.end(), 0);
    if (!contiguous) {
      std::shuffle(ps.begin(), ps.end(), rng);
      std::shuffle(pd.begin(), pd.end(), rng);
    }
    std::vector<It> v;
    for (int64_t j = 0; j < nblk; ++j)
      for (size_t o = 0; o < blk; o += piece) v.push_back({(int64_t)(ps[j] * blk + o), (int64_t)(pd[j] * blk + o)});
    CK(cudaMemcpy(dItems, v.data(), sizeof(It) * v.size(), cudaMemcpyHostToDevice));
    return Bench{S, D, dItems, (int64_t)v.size(), piece};
  };
  auto report = [&](const char* eng, const char* cfg, size_t blk, int piece, bool contig, float ms) {
    printf("{\"engine\": \"%s\", \"cfg\": \"%s\", \"blk\": %zu, \"piece\": %d, \"tables\": \"%s\", \"ms\": %.4f, "
           "\"payload_GBps\": %.1f}\n",
           eng, cfg, blk, piece, contig ? "contiguous" : "random", ms, payload / (ms * 1e-3) / 1e9);
    fflush(stdout);
  };
  const char* only = argc > 1 ? argv[1] : "";
  if (*only == 'F') {  // head slices: 16-row items of `slice` bytes out of 2-KiB rows (Llama-3-8B), 512 MiB payload
    CK(cudaFuncSetAttribute((const void*)k_rows<8>, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    for (int slice : {2048, 1024, 512, 256})
      for (int dcontig : {0, 1})
        for (int contig : {0, 1}) {
          // source: blocks of 16 rows x 2 KiB at random block slots; an item reads `slice` bytes of
          // each row at a random column; destination: rows of `slice` (dcontig) or 2 KiB pitch
          const int64_t blk = 16 * 2048, nblk_pool = pool / blk;
          const int64_t nitems = (int64_t)payload / (16 * slice);
          std::vector<int64_t> ps(nblk_pool), pd(nblk_pool);
          std::iota(ps.begin(), ps.end(), 0);
          std::iota(pd.begin(), pd.end(), 0);
          if (!contig) {
            std::shuffle(ps.begin(), ps.end(), rng);
            std::shuffle(pd.begin(), pd.end(), rng);
          }
          const int per = 2048 / slice;  // slices per row
          std::vector<It> v;
          for (int64_t i = 0; i < nitems; ++i) {
            const int64_t b = i / per, col = (i % per) * slice;   // all slices of a block, one after the other
            v.push_back({ps[b % nblk_pool] * blk + col,
                         dcontig ? (pd[b % nblk_pool] * blk + col * 16) : (pd[b % nblk_pool] * blk + col)});
          }
          CK(cudaMemcpy(dItems, v.data(), sizeof(It) * v.size(), cudaMemcpyHostToDevice));
          Bench bb{S, D, dItems, (int64_t)v.size(), slice};
          struct FCfg { int slice, dpitch; } fc{slice, dcontig ? slice : 2048};
          auto run_f = [](const Bench& b, void* a) {
            const FCfg& c = *(const FCfg*)a;
            int sms = 0;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
            k_rows<8><<<sms * 3, 256>>>(b.items, b.n, b.S, b.D, 16, c.slice, 2048, c.dpitch);
          };
          char cfg[128];
          snprintf(cfg, sizeof cfg, "slice%d dst_%s", slice, dcontig ? "contig" : "pitch2048");
          report("rows", cfg, blk, slice, contig, time_it(run_f, bb, &fc));
        }
    return 0;
  }
  char cfg[256];
  {
    Bench b = make(32768, 32768, true);
    report("memcpy", "cudaMemcpyAsync D2D", 0, 0, true, time_it(run_memcpy, b, nullptr));
  }
  for (int contig = 0; contig < 2; ++contig)
    for (size_t blk : {(size_t)32768, (size_t)131072}) {
      for (int piece : {8192, 16384, 32768, 65536}) {
        if ((size_t)piece > blk) continue;
        Bench b = make(blk, piece, contig);
        if (!*only || only[0] == 'A')
          for (int W : {1, 2, 4})
            for (int cps : {1, 2})
              for (int stages : {3, 4, 6, 8}) {
                const size_t smem = (size_t)W * stages * piece * cps;
                if (smem > (size_t)optin - 4096 || W * stages > 64) continue;
                for (int lag : {1, 2}) {
                  if (lag >= stages - 1) continue;
                  ACfg c{stages, W, cps, lag, sms};
                  snprintf(cfg, sizeof cfg, "W%d cps%d st%d lag%d", W, cps, stages, lag);
                  report("bulk", cfg, blk, piece, contig, time_it(run_a, b, &c));
                }
              }
        if (contig) continue;
        if (!*only || only[0] == 'V')
          for (int U : {8, 16})
            for (int hint : {0, 1})
              for (int cps : {2, 3, 4}) {
                VCfg c{U, hint, sms * cps};
                snprintf(cfg, sizeof cfg, "U%d hint%d ctas%dx", U, hint, cps);
                report("vec", cfg, blk, piece, contig, time_it(run_v, b, &c));
              }
        if (!*only || only[0] == 'C')
          for (int warps : {5, 9, 17})
            for (int stages : {3, 4, 6}) {
              if ((size_t)stages * piece > (size_t)optin - 4096) continue;
              CCfg c{stages, warps, sms};
              snprintf(cfg, sizeof cfg, "warps%d st%d", warps, stages);
              report("tma_ld+stg", cfg, blk, piece, contig, time_it(run_c, b, &c));
            }
        if (!*only || only[0] == 'D')
          for (int stages : {4, 6})
            for (int ahead : {2, 4, 8}) {
              if ((size_t)stages * piece > (size_t)optin - 4096) continue;
              DCfg c{stages, ahead, sms};
              snprintf(cfg, sizeof cfg, "st%d ahead%d", stages, ahead);
              report("bulk+L2pf", cfg, blk, piece, contig, time_it(run_d, b, &c));
            }
        if ((!*only || only[0] == 'E') && piece <= 8192)
          for (int cps : {1}) {
            ECfg c{sms * cps, 8};
            snprintf(cfg, sizeof cfg, "ctas%dx", cps);
            report("ldg+bulkst", cfg, blk, piece, contig, time_it(run_e, b, &c));
          }
      }
    }
  return 0;
}
