// FP64 DGEMM C += A @ B, warp-specialised TMA pipeline (sm_100a).
//
// The Cannon block product (apps/cannon.py:138, BLAS in the reference).
// tcgen05 has no f64 kind, so the FP64 tensor instruction on Blackwell is
// DMMA (mma.sync.m8n8k4.f64); this kernel is built so the DMMA pipe never
// waits on anything but its own operands:
//
//   * persistent: one 256-thread CTA per SM walks the 128x128 output tiles
//     (grouped 8 m-tiles at a time for L2 reuse of B);
//   * TMA loads of every k-tile (A: one 128x16 box, B: eight 16x16 boxes)
//     into a STAGES-deep ring with transaction-count full barriers, issued by
//     whichever warp releases a slot last: it refills the slot with the
//     k-tile STAGES ahead at once (across tile boundaries, so the next tile
//     streams in during the epilogue) -- every slot is refilled the moment
//     it frees, no thread ever waits to produce.  No separate producer warp:
//     with 9 warps ptxas caps registers at 168 (3 warps share an SMSP's 16K
//     registers) and the 64x32 warp tile spills (measured: a lane-0
//     producer LEAD = STAGES-2 ahead left 7 % of warp samples waiting on
//     the full barrier, ncu);
//   * eight warps (64x32 each, 2 per SMSP, up to 255 registers): wait on the
//     stage's full barrier, run 2 x 32 DMMAs per 8 k, release the stage with
//     one arrive per warp -- no CTA-wide barrier anywhere in the main loop,
//     no cp.async issue slots;
//   * 128-byte swizzled tiles, conflict-free fragment loads without padding:
//     A fragments are 16-byte loads of two consecutive k ("paired k": lane tq
//     takes k = kk+2tq for the first DMMA and kk+2tq+1 for the second) from a
//     row permutation gq -> (gq>>1) + 4(gq&1), so the two rows a quarter-warp
//     touches sit in opposite halves of the 128-byte swizzle pattern; B
//     fragments (8 consecutive n of 4 rows k = kk+2tq) land in distinct chunks
//     because k&7 spans both halves;
//   * TMA zero-fills out-of-range rows/columns, so ragged M / N / K need no
//     predication in the main loop.
//
// Requirements (else diomp_dgemm uses the cp.async kernel of gemm.cuh): A and
// B 16-byte aligned with even leading dimensions; no fused forward.
#pragma once

#include "common.cuh"

namespace diomp {
namespace gemm_tma {

constexpr int BM = 128, BK = 16;
constexpr int A_BYTES = BM * BK * 8;            // 16 KiB
constexpr int B_BOX_BYTES = BK * 16 * 8;        // 2 KiB: one 16-column box

// Tile shapes: BN columns per CTA, MINB CTAs per SM, STAGES-deep ring.
template <int BN_, int MINB_, int STAGES_, int WM_ = 8, int WN_ = 4>
struct Shape {
    static constexpr int BN = BN_, MINB = MINB_, STAGES = STAGES_;
    static constexpr int WM = WM_, WN = WN_;    // 8x8 fragments per warp (8x4: 64 x 32)
    static constexpr int WARPS_N = BN / (WN * 8);
    static constexpr int NCW = (BM / (WM * 8)) * WARPS_N;     // warps (all compute)
    static constexpr int THREADS = NCW * 32;
    static constexpr int B_BYTES = BK * BN * 8;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 1024 + 2 * STAGES * 8 + STAGES * 4;
};
// 128x128, 8 warps of 64x32, 1 CTA/SM, 7 x 32 KiB.  Measured on B200
// (tools/probe.py dgemm, 8192^3 / 16384^3 TFLOP/s, cuBLAS 35.4 / 36.1):
//   Shape<128,1,7>        34.3 / 34.9   (this one; DMMA pipe 93.4 % active)
//   Shape<64,2,4>         33.6 / 34.2   (128x64, 2 CTAs/SM)
//   Shape<128,1,7,4,4>    31.9 / 32.5   (16 warps of 32x32)
//   Shape<128,1,7,8,2>    31.7 / 32.8   (16 warps of 64x16)
using Big = Shape<128, 1, 7>;

struct Params {
    int64_t M, N, K;
    double *C;
    int64_t ldc;
    int64_t mtiles, ntiles;
    int32_t cvec;   // C 16 B aligned with an even ldc: double2 epilogue stores
};

__device__ __forceinline__ uint32_t su32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bar_init(uint64_t *b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W;\n}\n" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma2d(void *dst, const CUtensorMap *map, int x, int y,
                                      uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// tile -> (m-tile, n-tile), 8 m-tiles per group so consecutive CTAs share B
__device__ __forceinline__ void tile_coords(const Params &p, int64_t t, int64_t &mi, int64_t &ni) {
    const int64_t group = 8, per_group = group * p.ntiles;
    const int64_t g = t / per_group, first_m = g * group;
    const int64_t gsize = (p.mtiles - first_m) < group ? (p.mtiles - first_m) : group;
    mi = first_m + (t % per_group) % gsize;
    ni = (t % per_group) / gsize;
}

template <class SH>
__global__ void __launch_bounds__(SH::THREADS, SH::MINB)
    dgemm_tma_kernel(const __grid_constant__ CUtensorMap amap,
                     const __grid_constant__ CUtensorMap bmap, const __grid_constant__ Params p) {
    constexpr int BN = SH::BN, STAGES = SH::STAGES, NCW = SH::NCW, WARPS_N = SH::WARPS_N;
    constexpr int WM = SH::WM, WN = SH::WN;
    constexpr int STAGE_BYTES = SH::STAGE_BYTES;
    extern __shared__ uint8_t raw[];
    // 1024-byte aligned for the 128-byte swizzle.  The cast through uintptr_t
    // makes the fragment reads generic LD.E; keeping the pointer in the shared
    // window (LDS, 223 instead of 254 registers) measured slower -- the
    // compiler then issues each k-step's fragment loads just before their
    // DMMAs: 8192^3 34.3 -> 32.4 TFLOP/s, DMMA pipe 93.4 -> 88.4 %
    // (profiles/r02_dgemm_lds_variant.txt)
    uint8_t *sm = (uint8_t *)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    uint64_t *full = (uint64_t *)(sm + (size_t)STAGES * STAGE_BYTES);
    uint64_t *empty = full + STAGES;
    unsigned int *released = (unsigned int *)(empty + STAGES);   // warps done with a slot
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t ktiles = (uint32_t)ceil_div(p.K, BK);
    const int64_t ntotal = p.mtiles * p.ntiles;
    const uint32_t my_tiles =
        blockIdx.x < ntotal ? (uint32_t)((ntotal - 1 - blockIdx.x) / gridDim.x + 1) : 0u;
    const uint32_t total_it = my_tiles * ktiles;

    // load k-iteration j (this CTA's tile j / ktiles, k-tile j % ktiles) into slot s
    auto refill = [&](uint32_t j, int s) {
        if (j >= total_it) return;
        const uint32_t tl = j / ktiles, kt = j - tl * ktiles;
        int64_t mi, ni;
        tile_coords(p, blockIdx.x + (int64_t)tl * gridDim.x, mi, ni);
        uint8_t *st = sm + (size_t)s * STAGE_BYTES;
        bar_expect(&full[s], STAGE_BYTES);
        tma2d(st, &amap, (int)(kt * BK), (int)(mi * BM), &full[s]);
#pragma unroll
        for (int b = 0; b < BN / 16; ++b)
            tma2d(st + A_BYTES + b * B_BOX_BYTES, &bmap, (int)(ni * BN + b * 16), (int)(kt * BK),
                  &full[s]);
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], NCW);
            released[s] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int s = 0; s < STAGES; ++s) refill((uint32_t)s, s);
    }
    __syncthreads();

    const int gq = lane >> 2, tq = lane & 3;
    const int wm = (warp / WARPS_N) * (WM * 8), wn = (warp % WARPS_N) * (WN * 8);
    const int prow = (gq >> 1) + 4 * (gq & 1);      // fragment row gq -> tile row (mod 8)
    // per-lane byte offsets inside a stage: A row base (the swizzle XOR of
    // the row is `prow`), B box base + 8-byte half + 16-byte chunk index
    const uint32_t a_base = (uint32_t)(wm + prow) * 128u;
    const uint32_t b_base = (uint32_t)(A_BYTES + (wn >> 4) * B_BOX_BYTES + (gq & 1) * 8);
    const int bc0 = ((wn & 15) + gq) >> 1;   // chunk of fragment j = 0 (j odd: chunk ^ 4)

    uint32_t it = 0;
    int s = 0;
    uint32_t ph = 0;
    for (uint32_t tl = 0; tl < my_tiles; ++tl) {
        int64_t mi, ni;
        tile_coords(p, blockIdx.x + (int64_t)tl * gridDim.x, mi, ni);
        double acc[WM][WN][2];
#pragma unroll
        for (int i = 0; i < WM; ++i)
#pragma unroll
            for (int j = 0; j < WN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

        for (uint32_t kt = 0; kt < ktiles; ++kt, ++it) {
            bar_wait(&full[s], ph);
            const uint8_t *st = sm + (size_t)s * STAGE_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK; kk += 8) {
                double2 a2[WM];
                double b0[WN], b1[WN];
                const int ac = (kk >> 1) + tq;            // 16 B chunk of k = kk+2tq, +1
                const uint8_t *ap = st + a_base + ((ac ^ prow) << 4);
#pragma unroll
                for (int i = 0; i < WM; ++i)
                    a2[i] = *reinterpret_cast<const double2 *>(ap + i * 8 * 128);
                const int k0 = kk + 2 * tq, k1 = k0 + 1;
                // fragment j: box (wn + 8j) / 16, chunk bc0 ^ (4 if j odd)
                const uint8_t *bp0 = st + b_base + k0 * 128;
                const uint8_t *bp1 = st + b_base + k1 * 128;
#pragma unroll
                for (int j = 0; j < WN; ++j) {
                    const int ch = bc0 ^ ((j & 1) << 2);
                    const int box = (j >> 1) * B_BOX_BYTES;
                    b0[j] = *reinterpret_cast<const double *>(bp0 + box + ((ch ^ (k0 & 7)) << 4));
                    b1[j] = *reinterpret_cast<const double *>(bp1 + box + ((ch ^ (k1 & 7)) << 4));
                }
#pragma unroll
                for (int i = 0; i < WM; ++i)
#pragma unroll
                    for (int j = 0; j < WN; ++j) dmma(acc[i][j], a2[i].x, b0[j]);
#pragma unroll
                for (int i = 0; i < WM; ++i)
#pragma unroll
                    for (int j = 0; j < WN; ++j) dmma(acc[i][j], a2[i].y, b1[j]);
            }
            // release the slot; the last warp to do so refills it with
            // iteration it + STAGES right away (its mbarrier wait completes at
            // once and orders every warp's reads before the TMA writes)
            __syncwarp();
            if (lane == 0) {
                bar_arrive(&empty[s]);
                if (atomicAdd(&released[s], 1u) == NCW - 1) {
                    released[s] = 0;
                    bar_wait(&empty[s], ph);
                    refill(it + STAGES, s);
                }
            }
            if (++s == STAGES) {
                s = 0;
                ph ^= 1u;
            }
        }

        // epilogue: C = C + acc (numpy's `C += A_blk @ B`: product, then add)
        const int64_t m0 = mi * BM + wm, n0 = ni * BN + wn;
#pragma unroll
        for (int i = 0; i < WM; ++i)
#pragma unroll
            for (int j = 0; j < WN; ++j) {
                const int64_t r = m0 + i * 8 + prow;
                const int64_t c = n0 + j * 8 + 2 * tq;
                if (r >= p.M) continue;
                double *cp = p.C + r * p.ldc + c;
                if (p.cvec && c + 1 < p.N) {
                    double2 v = *reinterpret_cast<double2 *>(cp);
                    v.x = __dadd_rn(v.x, acc[i][j][0]);
                    v.y = __dadd_rn(v.y, acc[i][j][1]);
                    *reinterpret_cast<double2 *>(cp) = v;
                } else {
                    if (c < p.N) cp[0] = __dadd_rn(cp[0], acc[i][j][0]);
                    if (c + 1 < p.N) cp[1] = __dadd_rn(cp[1], acc[i][j][1]);
                }
            }
    }
}

static int encode_2d(CUtensorMap *map, const double *base, int64_t inner, int64_t outer, int64_t ld,
                     uint32_t box_inner, uint32_t box_outer) {
    auto encode = diomp::stencil::get_encode_fn();
    if (!encode) return DIOMP_INTERNAL;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void *)base, dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? DIOMP_OK : DIOMP_BAD_REQUEST;
}

// Eligible: A/B 16 B aligned, even leading dimensions, 32-bit TMA coordinates.
static bool eligible(const diomp_dgemm_args *x) {
    if (x->fwd || x->sync || ((x->A | x->B) & 15) || (x->lda & 1) || (x->ldb & 1) || x->K <= 0 ||
        x->M >= (1ll << 31) || x->N >= (1ll << 31) || x->K >= (1ll << 31))
        return false;
    // k-iterations per CTA are counted in 32 bits
    const int64_t tiles = ceil_div(x->M, BM) * ceil_div(x->N, 64);
    return ceil_div(tiles, kNumSMs) * ceil_div(x->K, BK) < (1ll << 31);
}

template <class SH>
static int launch_shape(const diomp_dgemm_args *x, cudaStream_t s) {
    static bool attr_set[64] = {false};
    if (x->device < 64 && !attr_set[x->device]) {
        DIOMP_CUDA_TRY(cudaFuncSetAttribute(dgemm_tma_kernel<SH>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)SH::SMEM));
        attr_set[x->device] = true;
    }
    constexpr int BN = SH::BN;
    CUtensorMap amap, bmap;
    int rc = encode_2d(&amap, (const double *)x->A, x->K, x->M, x->lda, BK, BM);
    if (!rc) rc = encode_2d(&bmap, (const double *)x->B, x->N, x->K, x->ldb, 16, BK);
    if (rc) return rc;
    Params p{};
    p.M = x->M; p.N = x->N; p.K = x->K;
    p.C = (double *)x->C;
    p.ldc = x->ldc;
    p.mtiles = ceil_div(x->M, BM);
    p.ntiles = ceil_div(x->N, BN);
    p.cvec = !((x->C & 15) || (x->ldc & 1));
    const int64_t tiles = p.mtiles * p.ntiles;
    const int64_t slots = (int64_t)kNumSMs * SH::MINB;
    const int grid = (int)(tiles < slots ? tiles : slots);
    dgemm_tma_kernel<SH><<<grid, SH::THREADS, SH::SMEM, s>>>(amap, bmap, p);
    DIOMP_LAUNCH_CHECK();
    return DIOMP_OK;
}

static int launch(const diomp_dgemm_args *x, cudaStream_t s) { return launch_shape<Big>(x, s); }

}  // namespace gemm_tma
}  // namespace diomp
