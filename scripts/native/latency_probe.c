/* Launch-bound regime of the C ABI (no Python): per-call host cost and end-to-end latency of
 * small migrations.  Toy geometry (configs[0]) and one Llama-3-8B chunk.
 *
 *   nvcc -O2 -o latency_probe scripts/native/latency_probe.c -I include \
 *        -L paper_2504_09285_b200 -ldyna_kv -Xlinker -rpath=$PWD/paper_2504_09285_b200
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "dyna_kv.h"

static double now_us(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e6 + ts.tv_nsec * 1e-3;
}

#define CK(x)                                                                         \
  do {                                                                                \
    dyna_status s_ = (x);                                                             \
    if (s_) {                                                                         \
      fprintf(stderr, "%s failed: %d %s\n", #x, (int)s_, dyna_kv_last_error());       \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

static void run(const char* name, dyna_kv_pool_desc d, int ntok, int chunk, int reps) {
  const size_t bytes = dyna_kv_pool_bytes(&d);
  void *a = NULL, *b = NULL;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  CK(dyna_kv_debug_fill(a, bytes, 1, 0, st));
  CK(dyna_kv_debug_fill(b, bytes, 2, 0, st));
  dyna_kv_pool_t ps, pd;
  CK(dyna_kv_pool_create(&d, a, &ps));
  CK(dyna_kv_pool_create(&d, b, &pd));
  const int nb = (ntok + d.block_size - 1) / d.block_size;
  int32_t* hs = (int32_t*)malloc(nb * 4);
  int32_t* hd = (int32_t*)malloc(nb * 4);
  for (int i = 0; i < nb; ++i) {
    hs[i] = (i * 7) % d.num_blocks;  /* distinct while nb <= NB and gcd(7, NB) = 1 */
    hd[i] = (i * 11 + 3) % d.num_blocks;
  }
  int32_t *ds, *dd;
  cudaMalloc((void**)&ds, nb * 4);
  cudaMalloc((void**)&dd, nb * 4);
  cudaMemcpy(ds, hs, nb * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dd, hd, nb * 4, cudaMemcpyHostToDevice);
  cudaDeviceSynchronize();
  dyna_block_table ts_dev = {ps, ds, NULL, nb}, td_dev = {pd, dd, NULL, nb};
  dyna_block_table ts_both = {ps, ds, hs, nb}, td_both = {pd, dd, hd, nb};
  dyna_block_table ts_host = {ps, NULL, hs, nb}, td_host = {pd, NULL, hd, nb};
  dyna_range tr = {0, ntok}, lr = {0, d.num_layers};
  dyna_kv_xfer_t* xs = (dyna_kv_xfer_t*)malloc(sizeof(dyna_kv_xfer_t) * reps);
  dyna_kv_opts unchecked;
  memset(&unchecked, 0, sizeof unchecked);
  unchecked.flags = DYNA_MIGRATE_UNCHECKED;   /* device-only tables: the caller vouches for distinct rows */
  struct { const char* n; dyna_block_table s, t; const dyna_kv_opts* o; } modes[] = {
      {"device ids (DYNA_MIGRATE_UNCHECKED)", ts_dev, td_dev, &unchecked},
      {"device+host ids (host checks)", ts_both, td_both, NULL},
      {"host ids only (upload)", ts_host, td_host, NULL}};
  for (int m = 0; m < 3; ++m) {
    for (int i = 0; i < 50; ++i) {  /* warm */
      CK(dyna_kv_migrate_ex(modes[m].s, modes[m].t, tr, lr, chunk, st, modes[m].o, &xs[0]));
      CK(dyna_kv_wait(xs[0]));
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaStreamSynchronize(st);
    /* (1) host cost per enqueued call, (2) device time for the back-to-back calls */
    cudaEventRecord(e0, st);
    double t0 = now_us();
    for (int i = 0; i < reps; ++i) CK(dyna_kv_migrate_ex(modes[m].s, modes[m].t, tr, lr, chunk, st, modes[m].o, &xs[i]));
    double t1 = now_us();
    cudaEventRecord(e1, st);
    for (int i = 0; i < reps; ++i) CK(dyna_kv_wait(xs[i]));
    cudaEventSynchronize(e1);
    float dev_ms = 0;
    cudaEventElapsedTime(&dev_ms, e0, e1);
    double t2 = now_us();
    /* (3) latency of one call + wait, serial */
    double lat0 = now_us();
    for (int i = 0; i < reps; ++i) {
      CK(dyna_kv_migrate_ex(modes[m].s, modes[m].t, tr, lr, chunk, st, modes[m].o, &xs[0]));
      CK(dyna_kv_wait(xs[0]));
    }
    double lat1 = now_us();
    const double payload = (double)ntok * 2 * d.num_layers * d.num_kv_heads * d.head_dim * d.elem_bytes;
    printf("{\"case\": \"%s\", \"tables\": \"%s\", \"tokens\": %d, \"payload_bytes\": %.0f, "
           "\"host_us_per_call\": %.2f, \"device_us_per_call\": %.2f, \"wall_us_per_call_pipelined\": %.2f, "
           "\"latency_us_call_plus_wait\": %.2f, \"pipelined_GBps\": %.1f}\n",
           name, modes[m].n, ntok, payload, (t1 - t0) / reps, dev_ms * 1e3 / reps, (t2 - t0) / reps,
           (lat1 - lat0) / reps, payload * reps / ((t2 - t0) * 1e3));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  dyna_kv_pool_destroy(ps);
  dyna_kv_pool_destroy(pd);
  cudaFree(a);
  cudaFree(b);
  cudaFree(ds);
  cudaFree(dd);
  free(hs);
  free(hd);
  free(xs);
  cudaStreamDestroy(st);
}

int main(void) {
  dyna_kv_pool_desc toy = {2, 2, 64, 2, 16, 64, 0, 0};            /* configs[0] */
  dyna_kv_pool_desc l3 = {32, 8, 128, 2, 16, 1024, 0, 0};         /* Llama-3-8B rows */
  run("configs[0] toy s=100 c=32", toy, 100, 32, 2000);
  run("Llama-3-8B 16-token request", l3, 16, 16, 2000);
  run("Llama-3-8B 256-token chunk", l3, 256, 256, 1000);
  run("Llama-3-8B 4096-token chunk", l3, 4096, 4096, 200);
  return 0;
}
