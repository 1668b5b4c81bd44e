/* A C caller of the OMPCCL collectives (include/diomp_b200.h), no Python:
 * two endpoints on two GPUs (argv), one host thread each, as two reference
 * ranks would drive collectives.py:232-405.  Device-synchronised teams:
 * allreduce (one entry handshake per call, diomp_team_barrier as the exit),
 * bcast, reduce, then the small-message path through diomp_ll_call (epochs
 * kept in each endpoint's RMA context).  Integer-valued f32 data, so every
 * expected value is exact.  Exit 0 = every check passed. */
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "diomp_b200.h"

#define K 2
static const uint64_t SEG = 64ull << 20;
static const uint64_t SEND = 0, RECV = 16ull << 20, FLAG = 32ull << 20;
static const uint64_t CNT = (32ull << 20) + 2048, LL = (32ull << 20) + 32768, LLSLOT = 64ull << 10;
static const uint64_t N = (1ull << 20) + 3;   /* f32 elements of the big calls */

static int gpu[K];
static uint64_t base[K];
static int failures = 0;
static pthread_barrier_t bar;

#define CHECK(cond, what)                                                        \
    do {                                                                         \
        if (!(cond)) {                                                           \
            fprintf(stderr, "FAIL pos %d: %s (line %d)\n", pos, what, __LINE__); \
            __sync_fetch_and_add(&failures, 1);                                  \
            return NULL;                                                         \
        }                                                                        \
    } while (0)

static void advance(diomp_team *t, int n) {
    for (int q = 0; q < K; ++q)
        if (q != t->pos) {
            t->epoch_to[q] += n;
            t->epoch_from[q] += n;
        }
}

static int fill(int pos, uint64_t off, uint64_t n, float scale) {
    float *h = malloc(n * sizeof(float));
    for (uint64_t i = 0; i < n; ++i) h[i] = (float)((i % 1000) * scale + pos);
    int rc = diomp_memcpy_sync(gpu[pos], base[pos] + off, (uint64_t)h, n * sizeof(float), DIOMP_H2D);
    free(h);
    return rc;
}

static uint64_t count_bad(int pos, uint64_t off, uint64_t n, float scale, int mode) {
    float *h = malloc(n * sizeof(float));
    uint64_t bad = 0;
    if (diomp_memcpy_sync(gpu[pos], (uint64_t)h, base[pos] + off, n * sizeof(float), DIOMP_D2H))
        bad = n;
    for (uint64_t i = 0; i < n && !bad; ++i) {
        float v = (float)((i % 1000) * scale);
        float want = mode == 0 ? 2 * v + 1 /* sum of v+0 and v+1 */ : v /* bcast from 0 */;
        if (h[i] != want) ++bad;
    }
    free(h);
    return bad;
}

static void *rank_main(void *arg) {
    const int pos = (int)(intptr_t)arg;
    void *stream = NULL, *ctx = NULL;
    CHECK(diomp_stream_create(gpu[pos], &stream) == DIOMP_OK, "stream_create");
    diomp_team t;
    memset(&t, 0, sizeof t);
    t.k = K; t.pos = pos; t.device = gpu[pos]; t.sync = 1;
    t.flag_off = FLAG; t.counter_off = CNT;
    for (int q = 0; q < K; ++q) { t.base[q] = base[q]; t.slot[q] = (uint32_t)q; }
    pthread_barrier_wait(&bar);

    /* allreduce, out of place, twice back to back, then the exit handshake */
    CHECK(fill(pos, SEND, N, 3.0f) == DIOMP_OK, "fill send");
    pthread_barrier_wait(&bar);
    for (int rep = 0; rep < 2; ++rep) {
        CHECK(diomp_allreduce(&t, SEND, RECV, N, DIOMP_F32, DIOMP_SUM, stream) == DIOMP_OK,
              "allreduce");
        advance(&t, 1);
    }
    CHECK(diomp_team_barrier(&t, stream) == DIOMP_OK, "exit barrier");
    advance(&t, 1);
    CHECK(diomp_stream_sync(stream) == DIOMP_OK && diomp_device_error(gpu[pos]) == DIOMP_OK,
          "allreduce drained");
    CHECK(count_bad(pos, RECV, N, 3.0f, 0) == 0, "allreduce exact");
    pthread_barrier_wait(&bar);

    /* bcast from position 0 (in place in SEND) */
    CHECK(fill(pos, SEND, N, pos == 0 ? 5.0f : 7.0f) == DIOMP_OK, "fill bcast");
    if (pos == 0) CHECK(fill(pos, SEND, N, 5.0f) == DIOMP_OK, "root payload");
    pthread_barrier_wait(&bar);
    CHECK(diomp_bcast(&t, SEND, N * sizeof(float) - 1, 0, stream) == DIOMP_OK, "bcast");
    advance(&t, 1);
    CHECK(diomp_team_barrier(&t, stream) == DIOMP_OK, "exit barrier");
    advance(&t, 1);
    CHECK(diomp_stream_sync(stream) == DIOMP_OK, "bcast drained");
    if (pos == 1) {
        /* every byte but the last equals the root's (v + 0 for pos 0) */
        float *h = malloc(N * sizeof(float));
        CHECK(diomp_memcpy_sync(gpu[pos], (uint64_t)h, base[pos] + SEND, N * sizeof(float),
                                DIOMP_D2H) == DIOMP_OK, "read bcast");
        uint64_t bad = 0;
        for (uint64_t i = 0; i + 1 < N; ++i)
            if (h[i] != (float)((i % 1000) * 5.0f)) ++bad;
        free(h);
        CHECK(bad == 0, "bcast byte-exact");
    }
    pthread_barrier_wait(&bar);

    /* small messages: LL allreduce through the RMA context (epochs in C) */
    CHECK(diomp_rma_ctx_create(K, 1, &ctx) == DIOMP_OK, "ctx_create");
    CHECK(diomp_rma_set_local(ctx, 0, gpu[pos], gpu[pos]) == DIOMP_OK, "set_local");
    for (int q = 0; q < K; ++q)
        CHECK(diomp_peer_table_set(ctx, q, 0, base[q], SEG, gpu[q]) == DIOMP_OK, "peer table");
    diomp_ll_args x;
    memset(&x, 0, sizeof x);
    x.k = K; x.pos = pos; x.device = gpu[pos]; x.dtype = DIOMP_F32; x.op = DIOMP_SUM;
    x.root = 0; x.mode = 0;
    for (int q = 0; q < K; ++q) { x.base[q] = base[q]; x.slot[q] = (uint32_t)q; }
    x.ll_off = LL; x.slot_bytes = LLSLOT;
    x.send_off = SEND; x.recv_off = RECV; x.count = 999;
    CHECK(fill(pos, SEND, 999, 1.0f) == DIOMP_OK, "fill LL");
    pthread_barrier_wait(&bar);
    for (int rep = 0; rep < 50; ++rep) {
        CHECK(diomp_ll_call(ctx, &x, stream, NULL, 1) == DIOMP_OK, "ll_call blocking");
        CHECK(x.epoch_to[1 - pos] == (uint32_t)(rep + 1) && x.epoch_from[1 - pos] == (uint32_t)(rep + 1),
              "ll epochs advance once per call");
    }
    CHECK(count_bad(pos, RECV, 999, 1.0f, 0) == 0, "LL allreduce exact");
    CHECK(diomp_rma_ctx_destroy(ctx) == DIOMP_OK, "ctx_destroy");
    diomp_stream_destroy(stream);
    return NULL;
}

int main(int argc, char **argv) {
    gpu[0] = argc > 1 ? atoi(argv[1]) : 0;
    gpu[1] = argc > 2 ? atoi(argv[2]) : 1;
    if (gpu[0] == gpu[1]) {
        /* device-synchronised endpoints never share a GPU (their kernels wait
         * on each other) */
        fprintf(stderr, "needs two distinct GPUs\n");
        return 3;
    }
    for (int p = 0; p < K; ++p)
        if (diomp_seg_create(gpu[p], SEG, &base[p]) != DIOMP_OK) return 2;
    if (diomp_peer_enable(gpu[0], gpu[1]) || diomp_peer_enable(gpu[1], gpu[0])) return 2;
    pthread_barrier_init(&bar, NULL, K);
    pthread_t th[K];
    for (int p = 0; p < K; ++p) pthread_create(&th[p], NULL, rank_main, (void *)(intptr_t)p);
    for (int p = 0; p < K; ++p) pthread_join(th[p], NULL);
    for (int p = 0; p < K; ++p) diomp_seg_destroy(gpu[p], base[p]);
    if (failures) return 1;
    printf("all ok\n");
    return 0;
}
