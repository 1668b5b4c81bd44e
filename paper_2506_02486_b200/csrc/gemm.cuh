// FP64 matrix multiply (sm_100a).
//
// 1. diomp_matmul_f64 -- the kernel seam of kernels/__init__.py:31
//    (_core.pyx:35-46): c = a @ b with each element a left fold over k in
//    ascending order, multiplies and adds separately rounded (no FMA), so the
//    result is bit-identical to the reference oracle.  Register-blocked 4x4
//    per thread, 64x64 tiles, operands staged through shared memory.
//
// 2. diomp_dgemm -- the Cannon block product of apps/cannon.py:138
//    (C += A_blk @ B_s, BLAS in the reference, tolerance-checked).  tcgen05
//    has no f64 kind, so the FP64 tensor path on Blackwell is DMMA
//    (mma.sync.m8n8k4.f64; the larger f64 shapes expand to the same DMMA.8x8x4
//    on sm_100a).  Default tiles 128x64x16, 8 warps of 32x32, 2 CTAs/SM,
//    3-stage cp.async pipeline into bank-conflict-free padded tiles, A
//    fragments of two k-steps fetched with one 16 B shared load.  When `fwd` is
//    set, every B tile is additionally stored once to the predecessor's spare
//    stripe over NVLink straight from shared memory (CTA row mi forwards the
//    k-tiles kt with kt % n_mtiles == mi), fusing the ring shift of
//    cannon.py:124-131 into the product.
#pragma once

#include "common.cuh"
#include "dgemm_tma.cuh"

namespace diomp {
namespace gemm {

// ---------------------------------------------------------------------------
// exact k-ordered matmul
// ---------------------------------------------------------------------------
constexpr int XT = 64;  // output tile
constexpr int XK = 16;  // k tile

__global__ void __launch_bounds__(256) matmul_exact_kernel(int64_t n, int64_t kk, int64_t m,
                                                           const double *__restrict__ a,
                                                           const double *__restrict__ b,
                                                           double *__restrict__ c) {
    __shared__ double As[XK][XT + 1];
    __shared__ double Bs[XK][XT + 1];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int64_t i0 = (int64_t)blockIdx.y * XT, j0 = (int64_t)blockIdx.x * XT;
    double acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int s = 0; s < 4; ++s) acc[r][s] = 0.0;
    for (int64_t k0 = 0; k0 < kk; k0 += XK) {
        for (int e = threadIdx.x; e < XT * XK; e += 256) {
            const int mi = e / XK, ki = e % XK;  // A: row mi, col ki
            const int64_t gi = i0 + mi, gk = k0 + ki;
            As[ki][mi] = (gi < n && gk < kk) ? a[gi * kk + gk] : 0.0;
            const int kb = e / XT, nj = e % XT;  // B: row kb, col nj
            const int64_t gkb = k0 + kb, gj = j0 + nj;
            Bs[kb][nj] = (gkb < kk && gj < m) ? b[gkb * m + gj] : 0.0;
        }
        __syncthreads();
        const int kmax = (int)((kk - k0) < XK ? (kk - k0) : XK);
        for (int q = 0; q < kmax; ++q) {
            double av[4], bv[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) av[r] = As[q][ty + 16 * r];
#pragma unroll
            for (int s = 0; s < 4; ++s) bv[s] = Bs[q][tx + 16 * s];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int s = 0; s < 4; ++s) acc[r][s] = __dadd_rn(acc[r][s], __dmul_rn(av[r], bv[s]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int64_t gi = i0 + ty + 16 * r, gj = j0 + tx + 16 * s;
            if (gi < n && gj < m) c[gi * m + gj] = acc[r][s];
        }
}

// ---------------------------------------------------------------------------
// DMMA DGEMM: C += A @ B
// ---------------------------------------------------------------------------
// Tile configurations.  WM x WN = 8x8 DMMA fragments per warp; WARPS_M x
// WARPS_N warps per CTA; MINB CTAs per SM (register budget).
template <int WM_, int WN_, int WARPS_M_, int WARPS_N_, int BK_, int STAGES_, int MINB_,
          bool PAIRK_ = false, int APADX_ = 4, int BPADX_ = 4>
struct Cfg {
    static constexpr int WM = WM_, WN = WN_, WARPS_M = WARPS_M_, WARPS_N = WARPS_N_;
    static constexpr bool PAIRK = PAIRK_;
    static constexpr int BM = WM * 8 * WARPS_M, BN = WN * 8 * WARPS_N, BK = BK_;
    static constexpr int STAGES = STAGES_, MINB = MINB_;
    static constexpr int THREADS = WARPS_M * WARPS_N * 32;
    static constexpr int APAD = BK + APADX_;  // A tile row pitch (doubles): conflict-free fragments
    // B tile row pitch (doubles).  A warp's 8 B fragment load is served per
    // half-warp (lanes gq 0..3 x tq 0..3): its rows step by `kstep` = 1
    // (single-k) or 2 (paired-k) x BPAD, so conflict-free needs
    // kstep * BPAD = 4 (mod 16): BN + 4 single-k, BN + 2 paired-k.
    static constexpr int BPAD = BN + BPADX_;
    static constexpr int A_STAGE = BM * APAD, B_STAGE = BK * BPAD;
    static constexpr size_t SMEM = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double);
};
using CfgBig = Cfg<8, 4, 2, 4, 16, 4, 1>;    // 128x128 CTA, 64x32 warps, 1 CTA/SM
using CfgDual = Cfg<4, 4, 4, 2, 16, 3, 2>;   // 128x64 CTA, 32x32 warps, 2 CTAs/SM
using CfgDeepK = Cfg<8, 4, 2, 4, 32, 3, 1>;  // 128x128 CTA, BK=32 (half the barriers)
#ifndef DIOMP_DGEMM_P2_BPADX
#define DIOMP_DGEMM_P2_BPADX 2
#endif
using CfgP2 = Cfg<4, 4, 4, 2, 16, 3, 2, true, 8, DIOMP_DGEMM_P2_BPADX>;  // CfgDual, paired-k A loads, A pitch 24, B pitch 66
using CfgQ4 = Cfg<4, 8, 2, 2, 16, 3, 2, false, 4>; // 64x128 CTA, 4 warps of 32x64 (cuBLAS's shape)

struct GemmParams {
    int64_t M, N, K;
    const double *A;
    const double *B;
    double *C;
    double *fwd;
    int64_t lda, ldb, ldc, ldf;
    int32_t sync;
    const uint64_t *wait_addr[2];
    uint64_t wait_value[2];
    uint64_t *sig_addr[2];
    uint64_t sig_value[2];
    unsigned int *counter;
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool pred) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    const int n = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem, bool pred) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    const int n = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(n)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

template <class C, bool VEC>
__device__ __forceinline__ void load_tiles(const GemmParams &p, double *As, double *Bs, int64_t m0,
                                           int64_t n0, int64_t k0) {
    // A: BM x BK, B: BK x BN, in 16 B chunks (VEC: even K/N/ld, 16 B aligned
    // bases) or single doubles (any shape); trip counts are compile-time so
    // the loops unroll
    constexpr int W = VEC ? 2 : 1;
    constexpr int NA = C::BM * C::BK / W, NB = C::BK * C::BN / W;
#pragma unroll
    for (int it = 0; it < (NA + C::THREADS - 1) / C::THREADS; ++it) {
        const int e = threadIdx.x + it * C::THREADS;
        if (NA % C::THREADS && e >= NA) break;
        const int r = e / (C::BK / W), ch = e % (C::BK / W);
        const int64_t gr = m0 + r, gk = k0 + ch * W;
        const bool ok = gr < p.M && gk < p.K;
        const void *g = ok ? (const void *)(p.A + gr * p.lda + gk) : (const void *)p.A;
        if (VEC) cp_async16(As + r * C::APAD + ch * W, g, ok);
        else cp_async8(As + r * C::APAD + ch * W, g, ok);
    }
#pragma unroll
    for (int it = 0; it < (NB + C::THREADS - 1) / C::THREADS; ++it) {
        const int e = threadIdx.x + it * C::THREADS;
        if (NB % C::THREADS && e >= NB) break;
        const int r = e / (C::BN / W), ch = e % (C::BN / W);
        const int64_t gk = k0 + r, gn = n0 + ch * W;
        const bool ok = gk < p.K && gn < p.N;
        const void *g = ok ? (const void *)(p.B + gk * p.ldb + gn) : (const void *)p.B;
        if (VEC) cp_async16(Bs + r * C::BPAD + ch * W, g, ok);
        else cp_async8(Bs + r * C::BPAD + ch * W, g, ok);
    }
}

template <class C, bool VEC>
__global__ void __launch_bounds__(C::THREADS, C::MINB) dgemm_dmma_kernel(const __grid_constant__ GemmParams p) {
    extern __shared__ __align__(16) double gsm[];
    double *As = gsm;
    double *Bs = gsm + C::STAGES * C::A_STAGE;

    // swizzle CTAs in groups of 8 m-tiles for L2 reuse of B
    const int64_t mtiles = ceil_div(p.M, C::BM), ntiles = ceil_div(p.N, C::BN);
    const int64_t bid = blockIdx.x;
    const int64_t group = 8;
    const int64_t per_group = group * ntiles;
    const int64_t g = bid / per_group;
    const int64_t first_m = g * group;
    const int64_t gsize = (mtiles - first_m) < group ? (mtiles - first_m) : group;
    const int64_t mi = first_m + (bid % per_group) % gsize;
    const int64_t ni = (bid % per_group) / gsize;
    const int64_t m0 = mi * C::BM, n0 = ni * C::BN;

    if (p.sync) {
        if (threadIdx.x < 2 && p.wait_addr[threadIdx.x])
            wait_ge(p.wait_addr[threadIdx.x], p.wait_value[threadIdx.x]);
        __syncthreads();
    }

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = (warp / C::WARPS_N) * C::WM * 8, wn = (warp % C::WARPS_N) * C::WN * 8;
    const int gq = lane >> 2, tq = lane & 3;

    double acc[C::WM][C::WN][2];
#pragma unroll
    for (int i = 0; i < C::WM; ++i)
#pragma unroll
        for (int j = 0; j < C::WN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int64_t ktiles = ceil_div(p.K, C::BK);
#pragma unroll
    for (int s = 0; s < C::STAGES - 1; ++s) {
        if (s < ktiles) load_tiles<C, VEC>(p, As + s * C::A_STAGE, Bs + s * C::B_STAGE, m0, n0, (int64_t)s * C::BK);
        cp_async_commit();
    }
    for (int64_t kt = 0; kt < ktiles; ++kt) {
        cp_async_wait<C::STAGES - 2>();
        __syncthreads();
        const int st = (int)(kt % C::STAGES);
        const double *a_s = As + st * C::A_STAGE;
        const double *b_s = Bs + st * C::B_STAGE;
        // prefetch tile kt + STAGES - 1 into the slot consumed at kt-1
        const int64_t nk = kt + C::STAGES - 1;
        if (nk < ktiles) {
            const int ns = (int)(nk % C::STAGES);
            load_tiles<C, VEC>(p, As + ns * C::A_STAGE, Bs + ns * C::B_STAGE, m0, n0, nk * C::BK);
        }
        cp_async_commit();
        // fused ring shift: forward this B tile once to the predecessor
        if (p.fwd && (kt % mtiles) == mi) {
            for (int e = threadIdx.x; e < C::BK * C::BN / 2; e += C::THREADS) {
                const int r = e / (C::BN / 2), ch = e % (C::BN / 2);
                const int64_t gk = kt * C::BK + r, gn = n0 + ch * 2;
                if (gk < p.K && gn < p.N) {
                    if (VEC) {
                        *reinterpret_cast<double2 *>(p.fwd + gk * p.ldf + gn) =
                            *reinterpret_cast<const double2 *>(b_s + r * C::BPAD + ch * 2);
                    } else {
                        p.fwd[gk * p.ldf + gn] = b_s[r * C::BPAD + ch * 2];
                        if (gn + 1 < p.N) p.fwd[gk * p.ldf + gn + 1] = b_s[r * C::BPAD + ch * 2 + 1];
                    }
                }
            }
        }
        if (C::PAIRK) {
            // k pairs: lane tq takes k = kk+2tq (first DMMA) and kk+2tq+1
            // (second) -- one 16 B shared load gives both A fragments; the
            // 8-wide k slice is summed in a different (still exact-product,
            // rounded-add) order, inside the GEMM's stated tolerance.
#pragma unroll
            for (int kk = 0; kk < C::BK; kk += 8) {
                double2 a2[C::WM];
                double b0[C::WN], b1[C::WN];
#pragma unroll
                for (int i = 0; i < C::WM; ++i)
                    a2[i] = *reinterpret_cast<const double2 *>(a_s + (wm + i * 8 + gq) * C::APAD + kk + 2 * tq);
#pragma unroll
                for (int j = 0; j < C::WN; ++j) {
                    b0[j] = b_s[(kk + 2 * tq) * C::BPAD + wn + j * 8 + gq];
                    b1[j] = b_s[(kk + 2 * tq + 1) * C::BPAD + wn + j * 8 + gq];
                }
#pragma unroll
                for (int i = 0; i < C::WM; ++i)
#pragma unroll
                    for (int j = 0; j < C::WN; ++j) dmma(acc[i][j], a2[i].x, b0[j]);
#pragma unroll
                for (int i = 0; i < C::WM; ++i)
#pragma unroll
                    for (int j = 0; j < C::WN; ++j) dmma(acc[i][j], a2[i].y, b1[j]);
            }
        } else {
#pragma unroll
            for (int kk = 0; kk < C::BK; kk += 4) {
                double af[C::WM], bf[C::WN];
#pragma unroll
                for (int i = 0; i < C::WM; ++i) af[i] = a_s[(wm + i * 8 + gq) * C::APAD + kk + tq];
#pragma unroll
                for (int j = 0; j < C::WN; ++j) bf[j] = b_s[(kk + tq) * C::BPAD + wn + j * 8 + gq];
#pragma unroll
                for (int i = 0; i < C::WM; ++i)
#pragma unroll
                    for (int j = 0; j < C::WN; ++j) dmma(acc[i][j], af[i], bf[j]);
            }
        }
    }
    cp_async_wait<0>();

    // epilogue: C = C + acc (numpy's `C += A_blk @ B` order: product, then add)
#pragma unroll
    for (int i = 0; i < C::WM; ++i)
#pragma unroll
        for (int j = 0; j < C::WN; ++j) {
            const int64_t r = m0 + wm + i * 8 + gq;
            const int64_t cidx = n0 + wn + j * 8 + tq * 2;
            if (VEC && r < p.M && cidx + 1 < p.N) {
                double2 *cp = reinterpret_cast<double2 *>(p.C + r * p.ldc + cidx);
                double2 cv = *cp;
                cv.x = __dadd_rn(cv.x, acc[i][j][0]);
                cv.y = __dadd_rn(cv.y, acc[i][j][1]);
                *cp = cv;
            } else if (r < p.M && cidx < p.N) {
                p.C[r * p.ldc + cidx] = __dadd_rn(p.C[r * p.ldc + cidx], acc[i][j][0]);
                if (!VEC && cidx + 1 < p.N)
                    p.C[r * p.ldc + cidx + 1] = __dadd_rn(p.C[r * p.ldc + cidx + 1], acc[i][j][1]);
            }
        }

    if (p.sync && last_cta_done(p.counter, gridDim.x) && threadIdx.x < 2 && p.sig_addr[threadIdx.x])
        st_release_sys(p.sig_addr[threadIdx.x], p.sig_value[threadIdx.x]);
}

template <class C, bool VEC = true>
static int launch_dgemm(const GemmParams &p, int device, cudaStream_t s) {
    static bool attr_set[64] = {false};
    if (device < 64 && !attr_set[device]) {
        DIOMP_CUDA_TRY(cudaFuncSetAttribute(dgemm_dmma_kernel<C, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)C::SMEM));
        attr_set[device] = true;
    }
    const int64_t tiles = ceil_div(p.M, C::BM) * ceil_div(p.N, C::BN);
    dgemm_dmma_kernel<C, VEC><<<(unsigned)tiles, C::THREADS, C::SMEM, s>>>(p);
    DIOMP_LAUNCH_CHECK();
    return DIOMP_OK;
}

}  // namespace gemm
}  // namespace diomp

extern "C" {

int diomp_matmul_f64(int device, int64_t n, int64_t k, int64_t m, uint64_t a, uint64_t b,
                     uint64_t c, void *stream) {
    using namespace diomp;
    using namespace diomp::gemm;
    if (n <= 0 || m <= 0) return DIOMP_OK;
    DIOMP_CUDA_TRY(cudaSetDevice(device));
    dim3 grid((unsigned)ceil_div(m, XT), (unsigned)ceil_div(n, XT));
    matmul_exact_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(n, k, m, (const double *)a,
                                                                 (const double *)b, (double *)c);
    DIOMP_LAUNCH_CHECK();
    return DIOMP_OK;
}

int diomp_dgemm(const diomp_dgemm_args *x, void *stream) {
    using namespace diomp;
    using namespace diomp::gemm;
    if (x->M <= 0 || x->N <= 0) return DIOMP_OK;
    if (x->K < 0 || x->lda < x->K || x->ldb < x->N || x->ldc < x->N || (x->fwd && x->ldf < x->N) ||
        ((x->A | x->B | x->C | x->fwd) & 7))
        return DIOMP_BAD_REQUEST;
    // 16 B cp.async needs even leading dimensions / K / N and 16 B aligned
    // bases; any other shape (e.g. an odd ring stripe width n/P) takes the
    // same kernel with 8 B operand copies and scalar epilogue stores
    const bool vec = !((x->K & 1) || (x->N & 1) || (x->lda & 1) || (x->ldb & 1) || (x->ldc & 1) ||
                       ((x->A | x->B | x->C | x->fwd) & 15) || (x->fwd && (x->ldf & 1)));
    DIOMP_CUDA_TRY(cudaSetDevice(x->device));
    GemmParams p{};
    p.M = x->M; p.N = x->N; p.K = x->K;
    p.A = (const double *)x->A; p.B = (const double *)x->B; p.C = (double *)x->C;
    p.fwd = (double *)x->fwd;
    p.lda = x->lda; p.ldb = x->ldb; p.ldc = x->ldc; p.ldf = x->ldf;
    p.sync = x->sync;
    for (int i = 0; i < 2; ++i) {
        p.wait_addr[i] = (const uint64_t *)x->wait_addr[i];
        p.wait_value[i] = x->wait_value[i];
        p.sig_addr[i] = (uint64_t *)x->sig_addr[i];
        p.sig_value[i] = x->sig_value[i];
    }
    p.counter = (unsigned int *)x->counter;
    // default: 2 CTAs/SM with 32x32 warp tiles and paired-k A fragments
    // (16 B shared loads, pitch 24): 0.92 of cuBLAS DGEMM at 8192^3, DMMA pipe
    // 88 % active vs cuBLAS 96.5 % (profiles/r01_dgemm_dmma_pipe.json).  The
    // single-k layout measured 0.91, cuBLAS's own 64x128 / 32x64-warp shape
    // 0.91-0.93, the 1-CTA 64x32 variants 0.86-0.87, BK=32 0.89, 4 stages at
    // 1 CTA/SM 0.74.  A CUTLASS-style mainloop (next k-step's fragments
    // loaded while the current DMMAs issue, tile boundary crossed before the
    // last step's DMMAs) measured 0.76 (spills at 128 regs) / 0.78 (BK=32,
    // 1 CTA/SM) / 0.90 (64x128 CTA) -- the compiler's own schedule is better.
    // 16 warps of 32x32 in a 128x128 CTA (4 stages, 1 CTA/SM): 0.81-0.83.
    // B pitch BN+2 removed the paired-k B loads' 2-way bank conflicts (1.07e9 ->
    // 1.1e6 at 8192^3) for only +0.3 %: the gap to cuBLAS is not shared memory.
    // default: the warp-specialised TMA kernel (dgemm_tma.cuh); the cp.async
    // kernels below serve the fused-forward / device-flag ring step, operands
    // TMA cannot describe, and DIOMP_DGEMM_TMA=0
    static const bool tma_on = [] {
        const char *e = getenv("DIOMP_DGEMM_TMA");
        return !(e && atoi(e) == 0);
    }();
    if (tma_on && gemm_tma::eligible(x)) return gemm_tma::launch(x, (cudaStream_t)stream);
    if (!vec) return launch_dgemm<CfgP2, false>(p, x->device, (cudaStream_t)stream);
    const char *v = getenv("DIOMP_DGEMM_CFG");
    if (v && atoi(v) == 0) return launch_dgemm<CfgBig>(p, x->device, (cudaStream_t)stream);
    if (v && atoi(v) == 1) return launch_dgemm<CfgDual>(p, x->device, (cudaStream_t)stream);
    if (v && atoi(v) == 2) return launch_dgemm<CfgDeepK>(p, x->device, (cudaStream_t)stream);
    if (v && atoi(v) == 3) return launch_dgemm<CfgQ4>(p, x->device, (cudaStream_t)stream);
    return launch_dgemm<CfgP2>(p, x->device, (cudaStream_t)stream);
}

}  // extern "C"
