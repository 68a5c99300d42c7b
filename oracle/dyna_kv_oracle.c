/*
 * dyna_kv_oracle.c — CPU oracle for DynaServe's chunked KV-cache migration.
 *
 * TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2504_09285_b200/csrc); the two meet only through kvgen's seeded
 * inputs.
 *
 * What it computes.  PAPER.md §3.1: a request of L tokens is split
 * at s into r^alpha (tokens 1..s) and r^beta (tokens s+1..L); when the two
 * micro-requests run on different instances "the instances exchange the
 * required KV cache blocks".  §4.3: r^alpha is processed in
 * equal-sized chunks, and "once chunk k completes, its KV block is ... pushed
 * to Server2", placement on the receiver steered by a message.  The result of
 * all of that is a plain definition:
 *
 *   Pd' = Pd, except for every layer l in [l0,l1), kv in {K,V}, token t in
 *   [t0,t1), head h < H, element i < d:
 *     the e bytes at off_d(l,kv,Td[t/bs_d], t mod bs_d, h, i)
 *     := the e bytes at off_s(l,kv,Ts[t/bs_s], t mod bs_s, h, i);   Ps' = Ps.
 *
 * with the paged pool layout [L][2][NB][bs][H][d] of e-byte elements
 * (reading R3 in DESIGN.md) and 0-based half-open token ranges (reading R1:
 * paper token i <-> index i-1, so r^alpha = [0, s)).
 *
 * oracle_migrate() is that definition written out element by element.
 * oracle_migrate_chunked() follows P:556 step by step (pack chunk k of the
 * source into a contiguous buffer, then place it through the destination
 * table) for any chunk size and any chunk order; it exists so the tests can
 * pin that chunking does not change the result.
 * oracle_migrate_heads() is the same definition restricted to a run of KV
 * heads, for instances of different tensor-parallel degree (§5
 * P:595-596 deploys r^alpha / r^beta as TP groups): the
 * source heads [h0,h1) land in destination heads [hd0, hd0 + h1 - h0), every
 * other head untouched (reading R14).
 *
 * No blocking, fusion or reordering: loops run in the order of the
 * definition.  Copies are bitwise (reading R8), so NaN payloads, -0 and
 * subnormals pass through untouched.
 */
#include <stddef.h>
#include <stdint.h>
#include <string.h>

typedef struct {
    int64_t L;   /* layers */
    int64_t H;   /* KV heads */
    int64_t d;   /* head_dim */
    int64_t e;   /* element bytes */
    int64_t bs;  /* block size (tokens per block) */
    int64_t NB;  /* number of blocks in the pool */
} oracle_geom;

/* off(l,kv,b,slot,h,i) = (((((l*2+kv)*NB + b)*bs + slot)*H + h)*d + i)*e */
int64_t oracle_off(const oracle_geom* g, int64_t l, int64_t kv, int64_t b,
                   int64_t slot, int64_t h, int64_t i)
{
    return (((((l * 2 + kv) * g->NB + b) * g->bs + slot) * g->H + h) * g->d + i) * g->e;
}

/* Logical view through a block table: KV_T(l,kv,t,h,i) lives at
 * off(l, kv, T[t div bs], t mod bs, h, i). */
int64_t oracle_logical_off(const oracle_geom* g, const int32_t* T, int64_t l,
                           int64_t kv, int64_t t, int64_t h, int64_t i)
{
    return oracle_off(g, l, kv, (int64_t)T[t / g->bs], t % g->bs, h, i);
}

int64_t oracle_pool_bytes(const oracle_geom* g)
{
    return g->L * 2 * g->NB * g->bs * g->H * g->d * g->e;
}

/* The plain definition.  Ps/Ts: source pool and table; Pd/Td: destination.
 * Token range [t0,t1), layer range [l0,l1).  An empty range changes nothing
 * (s = 0 means r^alpha is empty). */
void oracle_migrate(const uint8_t* Ps, const oracle_geom* gs, const int32_t* Ts,
                    uint8_t* Pd, const oracle_geom* gd, const int32_t* Td,
                    int64_t t0, int64_t t1, int64_t l0, int64_t l1)
{
    for (int64_t l = l0; l < l1; ++l)
        for (int64_t kv = 0; kv < 2; ++kv)
            for (int64_t t = t0; t < t1; ++t)
                for (int64_t h = 0; h < gs->H; ++h)
                    for (int64_t i = 0; i < gs->d; ++i)
                        memcpy(Pd + oracle_logical_off(gd, Td, l, kv, t, h, i),
                               Ps + oracle_logical_off(gs, Ts, l, kv, t, h, i),
                               (size_t)gs->e);
}

/* P:556 step by step.  The range [t0,t1) is cut into chunks of c tokens
 * relative to t0 (reading R5): chunk k = [t0 + k*c, min(t0 + (k+1)*c, t1)).
 * Chunks are taken in the order given by order[0..n_order) (reading R9: no
 * order is promised).  Each chunk is packed into `staging` as
 * [l - l0][kv][t - a][h][i] (reading R3), then placed through Td.
 * `staging` must hold (l1-l0)*2*c*H*d*e bytes. */
void oracle_migrate_chunked(const uint8_t* Ps, const oracle_geom* gs, const int32_t* Ts,
                            uint8_t* Pd, const oracle_geom* gd, const int32_t* Td,
                            int64_t t0, int64_t t1, int64_t l0, int64_t l1,
                            int64_t c, const int64_t* order, int64_t n_order,
                            uint8_t* staging)
{
    const int64_t H = gs->H, d = gs->d, e = gs->e;
    for (int64_t o = 0; o < n_order; ++o) {
        const int64_t k = order[o];
        const int64_t a = t0 + k * c;
        const int64_t b = (a + c < t1) ? a + c : t1;
        const int64_t n = b - a;
        if (n <= 0) continue;
        /* chunk k of the source is complete: pack it */
        for (int64_t l = l0; l < l1; ++l)
            for (int64_t kv = 0; kv < 2; ++kv)
                for (int64_t t = a; t < b; ++t)
                    for (int64_t h = 0; h < H; ++h)
                        for (int64_t i = 0; i < d; ++i)
                            memcpy(staging + (((((l - l0) * 2 + kv) * n + (t - a)) * H + h) * d + i) * e,
                                   Ps + oracle_logical_off(gs, Ts, l, kv, t, h, i), (size_t)e);
        /* the receiver places it through its block table */
        for (int64_t l = l0; l < l1; ++l)
            for (int64_t kv = 0; kv < 2; ++kv)
                for (int64_t t = a; t < b; ++t)
                    for (int64_t h = 0; h < H; ++h)
                        for (int64_t i = 0; i < d; ++i)
                            memcpy(Pd + oracle_logical_off(gd, Td, l, kv, t, h, i),
                                   staging + (((((l - l0) * 2 + kv) * n + (t - a)) * H + h) * d + i) * e,
                                   (size_t)e);
    }
}

/* Head-restricted definition (reading R14).  Pools may differ in H (the
 * head count of each TP shard); L, d, e agree.  For every l in [l0,l1), kv,
 * t in [t0,t1), head h in [h0,h1), i < d:
 *   the e bytes at off_d(l,kv,Td[t/bs_d], t mod bs_d, hd0 + (h - h0), i)
 *   := the e bytes at off_s(l,kv,Ts[t/bs_s], t mod bs_s, h, i). */
void oracle_migrate_heads(const uint8_t* Ps, const oracle_geom* gs, const int32_t* Ts,
                          uint8_t* Pd, const oracle_geom* gd, const int32_t* Td,
                          int64_t t0, int64_t t1, int64_t l0, int64_t l1,
                          int64_t h0, int64_t h1, int64_t hd0)
{
    for (int64_t l = l0; l < l1; ++l)
        for (int64_t kv = 0; kv < 2; ++kv)
            for (int64_t t = t0; t < t1; ++t)
                for (int64_t h = h0; h < h1; ++h)
                    for (int64_t i = 0; i < gs->d; ++i)
                        memcpy(Pd + oracle_logical_off(gd, Td, l, kv, t, hd0 + (h - h0), i),
                               Ps + oracle_logical_off(gs, Ts, l, kv, t, h, i),
                               (size_t)gs->e);
}

/* The two halves of P:556's push on their own — "once chunk k completes, its KV
 * block is ... pushed", placement "steered on the receiver side" — as the staged
 * transfer and the NCCL baseline carry them: the sender packs
 * tokens [t0,t1) x layers [l0,l1) of its pool through Ts into one contiguous
 * buffer laid out [l - l0][kv][t - t0][h][i] (reading R3, the same canonical
 * layout as oracle_migrate_chunked's staging), the receiver places that buffer
 * through Td.  oracle_unpack(oracle_pack(...)) is oracle_migrate. */
void oracle_pack(const uint8_t* Ps, const oracle_geom* gs, const int32_t* Ts,
                 int64_t t0, int64_t t1, int64_t l0, int64_t l1, uint8_t* out)
{
    const int64_t n = t1 - t0, H = gs->H, d = gs->d, e = gs->e;
    for (int64_t l = l0; l < l1; ++l)
        for (int64_t kv = 0; kv < 2; ++kv)
            for (int64_t t = t0; t < t1; ++t)
                for (int64_t h = 0; h < H; ++h)
                    for (int64_t i = 0; i < d; ++i)
                        memcpy(out + (((((l - l0) * 2 + kv) * n + (t - t0)) * H + h) * d + i) * e,
                               Ps + oracle_logical_off(gs, Ts, l, kv, t, h, i), (size_t)e);
}

void oracle_unpack(const uint8_t* in, uint8_t* Pd, const oracle_geom* gd, const int32_t* Td,
                   int64_t t0, int64_t t1, int64_t l0, int64_t l1)
{
    const int64_t n = t1 - t0, H = gd->H, d = gd->d, e = gd->e;
    for (int64_t l = l0; l < l1; ++l)
        for (int64_t kv = 0; kv < 2; ++kv)
            for (int64_t t = t0; t < t1; ++t)
                for (int64_t h = 0; h < H; ++h)
                    for (int64_t i = 0; i < d; ++i)
                        memcpy(Pd + oracle_logical_off(gd, Td, l, kv, t, h, i),
                               in + (((((l - l0) * 2 + kv) * n + (t - t0)) * H + h) * d + i) * e, (size_t)e);
}
