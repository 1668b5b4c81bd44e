/* A C caller of the rank-addressed RMA context (include/diomp_b200.h):
 * everything the reference's put/get/fence path offers, reached without
 * Python.  Two endpoints ("ranks" 0 and 1, one device each) on GPUs A and B
 * (argv; the same GPU twice on a one-GPU box), segments from
 * diomp_seg_create, the peer table filled by hand.  Exit 0 = every check
 * passed; prints one line per check. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "diomp_b200.h"

#define CHECK(cond, what)                                   \
    do {                                                    \
        if (!(cond)) {                                      \
            fprintf(stderr, "FAIL %s (line %d)\n", what, __LINE__); \
            return 1;                                       \
        }                                                   \
        printf("ok %s\n", what);                            \
    } while (0)

int main(int argc, char **argv) {
    int ga = argc > 1 ? atoi(argv[1]) : 0, gb = argc > 2 ? atoi(argv[2]) : 0;
    const uint64_t SEG = 64ull << 20, N = (3ull << 20) + 17;
    uint64_t base_a = 0, base_b = 0;
    CHECK(diomp_seg_create(ga, SEG, &base_a) == DIOMP_OK, "seg_create A");
    CHECK(diomp_seg_create(gb, SEG, &base_b) == DIOMP_OK, "seg_create B");
    if (ga != gb) {
        CHECK(diomp_peer_enable(ga, gb) == DIOMP_OK, "peer_enable A->B");
        CHECK(diomp_peer_enable(gb, ga) == DIOMP_OK, "peer_enable B->A");
    }
    void *ctx = NULL;
    CHECK(diomp_rma_ctx_create(2, 1, &ctx) == DIOMP_OK, "ctx_create");
    CHECK(diomp_rma_set_local(ctx, 0, ga, 0) == DIOMP_OK, "set_local");
    CHECK(diomp_peer_table_set(ctx, 0, 0, base_a, SEG, 0) == DIOMP_OK, "peer_table_set rank 0");
    CHECK(diomp_peer_table_set(ctx, 1, 0, base_b, SEG, ga == gb ? 0 : 1) == DIOMP_OK,
          "peer_table_set rank 1");
    void *stream = NULL;
    CHECK(diomp_stream_create(ga, &stream) == DIOMP_OK, "stream_create");

    unsigned char *src = malloc(N), *back = malloc(N);
    for (uint64_t i = 0; i < N; ++i) src[i] = (unsigned char)(i * 131u + 7u);
    uint64_t op = 0;
    /* H2D put of host bytes into rank 0's segment at offset 4096+3 */
    CHECK(diomp_rma_put(ctx, 0, 0, 4099, (uint64_t)src, N, DIOMP_H2D, 0, stream, &op) == DIOMP_OK,
          "put H2D");
    CHECK(diomp_op_wait(ctx, op, 30.0) == DIOMP_OK, "op_wait H2D");
    /* D2D put rank 0 -> rank 1 (offset 8192+3), fence toward rank 1 */
    CHECK(diomp_rma_put(ctx, 1, 0, 8195, base_a + 4099, N, DIOMP_D2D, 0, stream, &op) == DIOMP_OK,
          "put D2D to rank 1");
    uint64_t pending = 99;
    CHECK(diomp_rma_outstanding(ctx, 1ull << 0, &pending) == DIOMP_OK && pending == 0,
          "no ops toward rank 0");
    CHECK(diomp_fence_group(ctx, 1ull << 1) == DIOMP_OK, "fence_group {rank 1}");
    CHECK(diomp_op_query(ctx, op) == DIOMP_OK, "fenced op reads complete");
    /* D2D get rank 1 -> rank 0 (offset 16M), then D2H get of it */
    CHECK(diomp_rma_get(ctx, 1, 0, 8195, base_a + (16u << 20), N, DIOMP_D2D, 0, stream, &op) ==
              DIOMP_OK, "get D2D from rank 1");
    CHECK(diomp_op_wait(ctx, op, 30.0) == DIOMP_OK, "op_wait get");
    memset(back, 0, N);
    CHECK(diomp_rma_get(ctx, 0, 0, 16u << 20, (uint64_t)back, N, DIOMP_D2H, 0, stream, &op) ==
              DIOMP_OK, "get D2H");
    CHECK(diomp_op_wait(ctx, op, 30.0) == DIOMP_OK, "op_wait D2H");
    CHECK(memcmp(back, src, N) == 0, "round trip byte-exact");
    /* small puts: many in flight, one fence */
    for (int i = 0; i < 1000; ++i)
        if (diomp_rma_put(ctx, 1, 0, 64 * (uint64_t)i, base_a + 4099, 8, DIOMP_D2D, 0, stream,
                          &op) != DIOMP_OK)
            return 2;
    CHECK(diomp_fence_group(ctx, 3ull) == DIOMP_OK, "fence after 1000 puts");
    /* errors: out of the segment, unknown rank, bad kind */
    CHECK(diomp_rma_put(ctx, 1, 0, SEG - 4, base_a, 8, DIOMP_D2D, 0, stream, &op) ==
              DIOMP_INVALID_ADDRESS, "range past the segment -> INVALID_ADDRESS");
    CHECK(diomp_rma_get(ctx, 2, 0, 0, base_a, 8, DIOMP_D2D, 0, stream, &op) ==
              DIOMP_INVALID_ADDRESS, "unknown rank -> INVALID_ADDRESS");
    CHECK(diomp_rma_put(ctx, 1, 0, 0, base_a, 8, DIOMP_D2H, 0, stream, &op) == DIOMP_BAD_REQUEST,
          "put with a get kind -> BAD_REQUEST");
    CHECK(diomp_rma_ctx_destroy(ctx) == DIOMP_OK, "ctx_destroy");
    diomp_stream_destroy(stream);
    diomp_seg_destroy(ga, base_a);
    diomp_seg_destroy(gb, base_b);
    free(src);
    free(back);
    printf("all ok\n");
    return 0;
}
