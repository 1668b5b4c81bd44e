// Minimod 8th-order acoustic-isotropic stencil (sm_100a).
//
// Reference: kernels/reference.py:14-31, kernels/_core.pyx:9-32 (per-point
// order), apps/stencil.py:113-126 (driver step), apps/halo_onesided.py:12-25
// (Listing-1 halo).  Arithmetic is bit-identical to the reference: every
// operation is an explicitly rounded __dmul_rn/__dadd_rn/__dsub_rn in the
// reference's order (acc = c*u; x taps t=1..4; y taps; z taps;
// (2u - u_prev) + acc), so no FMA contraction can occur.
//
// Fast path (R=4, NZ even, 16 B aligned): one CTA per SM owns a 14(y) x 128(z)
// column of the domain and streams along x through a chunk of planes.  The CTA
// is warp-specialised:
//   * a producer warp issues TMA (cp.async.bulk.tensor.3d) loads: u_cur plane
//     tiles with their 4-wide y/z halo (22 x 136 f64, 1088-byte rows) into a
//     7-slot ring and u_prev tiles (14 x 128) into a 4-slot ring, each slot
//     with a "full" (transaction-count) and an "empty" (consumer-arrival)
//     mbarrier -- no CTA-wide barrier per plane;
//   * 14 compute warps (7 row pairs x 2 halves of the 128 columns), 2(y) x 2(z)
//     points per thread, keep the 9-plane x-window of each point in registers
//     (the plane loop is unrolled 9x so the window rotates by register
//     renaming; 128 registers, no spills); y/z taps come from the centre
//     plane's slot with 16 B shared loads (conflict-free rows), interleaved
//     tap by tap so only a sliding pair of rows is live;
//   * u_next is stored with 16 B coalesced stores.
// Measured (1024^3, one B200): 262.5 Gpts/s = 0.962 of the measured HBM copy
// peak at 24 B/point, DRAM traffic 1.024x the minimum.  Round 1's 24 x 64
// tiles (576-byte TMA rows, 12 compute warps) ran 243-246: the longer rows
// and the two extra compute warps are each worth about half of the gain to
// 258.6 (profiles/r02_stencil_shapes.txt); the instantiation without the halo
// epilogue for launches without neighbours the rest
// (profiles/r02_stencil_halo_codegen.txt).
// Fused driver epilogue: output planes [R,2R) / [nxl, nxl+R) are also stored
// into the left / right neighbour's u_next ghost planes over NVLink (peer
// pointers), the point source is added in-register (one extra rounded add,
// exactly like stencil.py:124-125), and with sync on, edge CTAs wait for the
// neighbours' "previous step done" flag, which block 0 of each step's kernel
// raises for the step before it (kernel order makes that step's stores
// complete) -- the device-side replacement of fence+barrier.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include <map>
#include <mutex>
#include <queue>
#include <vector>

#include "common.cuh"

namespace diomp {
namespace stencil {

constexpr int R = 4;
#ifndef DIOMP_STENCIL_NCW
#define DIOMP_STENCIL_NCW 14
#endif
constexpr int NCW = DIOMP_STENCIL_NCW;  // compute warps (2 rows x 64 columns each)
#ifndef DIOMP_STENCIL_WZ
#define DIOMP_STENCIL_WZ 2
#endif
constexpr int WZ = DIOMP_STENCIL_WZ;    // compute warps side by side along z
constexpr int TY = 2 * NCW / WZ;
constexpr int TZ = 64 * WZ;
constexpr int BY = TY + 2 * R;  // rows per slot
constexpr int BZ = TZ + 2 * R;  // columns per slot
constexpr int SLOT = BY * BZ;   // doubles per slot
// smem budget (227 KB): u_cur ring of BY x BZ tiles + u_prev ring of TY x TZ tiles
#ifndef DIOMP_STENCIL_NSLOT
#define DIOMP_STENCIL_NSLOT (NCW >= 16 ? 7 : (NCW >= 14 ? 7 : (NCW >= 12 ? 8 : 11)))
#endif
#ifndef DIOMP_STENCIL_NPREV
#define DIOMP_STENCIL_NPREV (NCW >= 16 ? 3 : (NCW >= 14 ? 4 : (NCW >= 12 ? 5 : 8)))
#endif
constexpr int NSLOT = DIOMP_STENCIL_NSLOT;  // 5 in use + the rest in flight
constexpr int NPREV = DIOMP_STENCIL_NPREV;  // u_prev tile ring
constexpr int PREV_AHEAD = NPREV - 2;     // u_prev tiles issued this many outputs ahead
constexpr int PSLOT = TY * TZ;            // doubles per u_prev tile
constexpr int THREADS = (NCW + 1) * 32;   // + one TMA producer warp
constexpr uint32_t SLOT_BYTES = SLOT * 8;
constexpr uint32_t PSLOT_BYTES = PSLOT * 8;
constexpr size_t SMEM_BYTES =
    (size_t)NSLOT * SLOT_BYTES + (size_t)NPREV * PSLOT_BYTES + 2 * (NSLOT + NPREV) * 8;
static_assert(SMEM_BYTES <= 232448, "stencil rings exceed 227 KB of shared memory");
static_assert(BZ <= 256 && BY <= 256, "TMA box dimensions are at most 256");
static_assert(NCW % WZ == 0, "compute warps must tile the rows evenly");

struct Params {
    double *u_next;
    const double *u_prev;
    int64_t NX, NY, NZ;
    int32_t ntz, ncols;
    int32_t chunk, nch;
    double c0;
    double wx[R + 1], wy[R + 1], wz[R + 1];
    // fused driver
    double *left_next;
    double *right_next;
    int64_t nxl;
    int64_t src_x, src_y, src_z;  // src_x < 0: no source
    double amp;
    // device sync
    int32_t sync;
    const uint64_t *wait_l;
    const uint64_t *wait_r;
    uint64_t wl, wr;
    uint64_t *sig_l;
    uint64_t *sig_r;
    uint64_t sl, sr;
    unsigned int *counter;
    int32_t edge_first;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}

__device__ __forceinline__ void tma_load_plane(double *dst, const CUtensorMap *map, int z, int y,
                                               int x, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(z), "r"(y), "r"(x), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ double2 lds2(const double *p) {
    return *reinterpret_cast<const double2 *>(p);
}

__device__ __forceinline__ double tap(double acc, double w, double a, double b) {
    return __dadd_rn(acc, __dmul_rn(w, __dadd_rn(a, b)));
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Per-thread streaming state (pointers advance by one plane per output plane).
struct Lane {
    double *pn;         // u_next at (x, y, z) of the thread's first point
    int64_t x;          // current output plane (full-array index)
    int so;             // slot offset (doubles) of the thread's first point
    int src_pt;         // which of the 4 points is the source (y/z match), -1: none
    bool yv0, yv1, zv0, zv1, full;
};

template <bool FULL>
__device__ __forceinline__ void store4(double *b, int64_t NZ, const double (&o)[4], const Lane &ln) {
    if (FULL) {
        *reinterpret_cast<double2 *>(b) = make_double2(o[0], o[1]);
        *reinterpret_cast<double2 *>(b + NZ) = make_double2(o[2], o[3]);
        return;
    }
    if (ln.yv0 && ln.zv1) *reinterpret_cast<double2 *>(b) = make_double2(o[0], o[1]);
    else if (ln.yv0 && ln.zv0) b[0] = o[0];
    if (ln.yv1 && ln.zv1) *reinterpret_cast<double2 *>(b + NZ) = make_double2(o[2], o[3]);
    else if (ln.yv1 && ln.zv0) b[NZ] = o[2];
}

// One loaded plane q for a compute thread's 2x2 points.  J is the
// register-window rotation: window index t (0..8 = planes q-8..q) lives in
// bank (J+1+t)%9.  Per point the operation order is exactly the reference's;
// the 4 points are interleaved tap by tap, keeping only a sliding pair of
// neighbour rows live (rows -t / 1+t of tap t are rows 1-(t+1) / (t+1) of
// tap t+1).  The slot of plane q-R is released (empty barrier) after its
// last use here.
template <int J, bool FULL, bool HALO>
__device__ __forceinline__ void step_plane(const Params &p, const double *sm, uint64_t *full,
                                           uint64_t *empty, const double *psm, uint64_t *pfull,
                                           uint64_t *pempty, double (&Q)[9][4], Lane &ln, int q,
                                           int L, int &s, uint32_t &ph) {
    // s / ph: ring slot and mbarrier phase of plane q (advanced incrementally,
    // no division by NSLOT); the centre plane q-R sits R slots behind.
    const bool out_plane = q >= 2 * R;
    const int sc = s >= R ? s - R : s - R + NSLOT;
    mbar_wait(&full[s], ph);
    {
        const double *c = sm + s * SLOT + ln.so;
        const double2 a = lds2(c), b = lds2(c + BZ);
        Q[J][0] = a.x; Q[J][1] = a.y; Q[J][2] = b.x; Q[J][3] = b.y;
    }
    if (out_plane) {
        constexpr int C = (J + 5) % 9;  // centre bank
        const double *cr = sm + sc * SLOT + ln.so;
        double acc[4];
#ifdef DIOMP_STENCIL_MEMONLY
        // experiment build: same loads / barriers / stores, no taps
#pragma unroll
        for (int pt = 0; pt < 4; ++pt) acc[pt] = Q[C][pt] + cr[pt & 1];
        if (false)
#endif
        {
#pragma unroll
        for (int pt = 0; pt < 4; ++pt) acc[pt] = __dmul_rn(p.c0, Q[C][pt]);
#pragma unroll
        for (int t = 1; t <= R; ++t)
#pragma unroll
            for (int pt = 0; pt < 4; ++pt)
                acc[pt] = tap(acc[pt], p.wx[t], Q[(J + 5 + t) % 9][pt], Q[(J + 5 - t + 9) % 9][pt]);
        {
            double2 rp0 = make_double2(Q[C][2], Q[C][3]);  // row +1 (own row 1)
            double2 rm1 = make_double2(Q[C][0], Q[C][1]);  // row 0  (own row 0)
#pragma unroll
            for (int t = 1; t <= R; ++t) {
                const double2 rm0 = lds2(cr - t * BZ);
                const double2 rp1 = lds2(cr + (1 + t) * BZ);
                acc[0] = tap(acc[0], p.wy[t], rp0.x, rm0.x);
                acc[1] = tap(acc[1], p.wy[t], rp0.y, rm0.y);
                acc[2] = tap(acc[2], p.wy[t], rp1.x, rm1.x);
                acc[3] = tap(acc[3], p.wy[t], rp1.y, rm1.y);
                rp0 = rp1;
                rm1 = rm0;
            }
        }
#pragma unroll
        for (int a = 0; a < 2; ++a) {
            const double *rr = cr + a * BZ;
            const double2 m43 = lds2(rr - 4), m21 = lds2(rr - 2), p23 = lds2(rr + 2), p45 = lds2(rr + 4);
            const double o0 = Q[C][a * 2], o1 = Q[C][a * 2 + 1];
            double &c0 = acc[a * 2], &c1 = acc[a * 2 + 1];
            c0 = tap(c0, p.wz[1], o1, m21.y);    c1 = tap(c1, p.wz[1], p23.x, o0);
            c0 = tap(c0, p.wz[2], p23.x, m21.x); c1 = tap(c1, p.wz[2], p23.y, m21.y);
            c0 = tap(c0, p.wz[3], p23.y, m43.y); c1 = tap(c1, p.wz[3], p45.x, m21.x);
            c0 = tap(c0, p.wz[4], p45.x, m43.x); c1 = tap(c1, p.wz[4], p45.y, m43.y);
        }
        }
        // u_prev of this output plane from its TMA-filled tile, then free the tile
        const int o = q - 2 * R;
        const int ps = o % NPREV;
        mbar_wait(&pfull[ps], (uint32_t)((o / NPREV) & 1));
        const double *pt0 = psm + ps * PSLOT + (ln.so / BZ - R) * TZ + (ln.so % BZ - R);
        const double2 pa = lds2(pt0), pb = lds2(pt0 + TZ);
        const double pv[4] = {pa.x, pa.y, pb.x, pb.y};
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&pempty[ps]);
        double out[4];
#pragma unroll
        for (int pt = 0; pt < 4; ++pt)
            out[pt] = __dadd_rn(__dsub_rn(__dmul_rn(2.0, Q[C][pt]), pv[pt]), acc[pt]);
        if (ln.src_pt >= 0 && ln.x == p.src_x) {
#pragma unroll
            for (int pt = 0; pt < 4; ++pt)
                if (pt == ln.src_pt) out[pt] = __dadd_rn(out[pt], p.amp);
        }
        store4<FULL>(ln.pn, p.NZ, out, ln);
        const int64_t pstride = p.NY * p.NZ;
        if (HALO) {
            // pn's copies in the neighbours' ghost planes, from the parameters
            // (no per-plane pointer bookkeeping in the loop: N=2 512 -> 517,
            // N=4 988 -> 994 Gpts/s, profiles/r02_stencil_halo_codegen.txt)
            if (ln.x < 2 * R && p.left_next)
                store4<FULL>(p.left_next + p.nxl * pstride + (ln.pn - p.u_next), p.NZ, out, ln);
            if (ln.x >= p.nxl && p.right_next)
                store4<FULL>(p.right_next - p.nxl * pstride + (ln.pn - p.u_next), p.NZ, out, ln);
        }
        ln.pn += pstride;
        ln.x += 1;
    }
    if (q >= R) {  // plane q-R had its last read (centre of this output plane)
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[sc]);
    }
    if (++s == NSLOT) {
        s = 0;
        ph ^= 1u;
    }
}

template <bool FULL, bool HALO>
__device__ __forceinline__ void consume(const Params &p, const double *sm, uint64_t *full,
                                       uint64_t *empty, const double *psm, uint64_t *pfull,
                                       uint64_t *pempty, Lane &ln, int L) {
    double Q[9][4];
#pragma unroll
    for (int i = 0; i < 9; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) Q[i][j] = 0.0;
    int s = 0;
    uint32_t ph = 0;
#define DIOMP_STEP(JJ) \
    if (q + JJ < L) \
        step_plane<JJ, FULL, HALO>(p, sm, full, empty, psm, pfull, pempty, Q, ln, q + JJ, L, s, ph);
    for (int q = 0; q < L; q += 9) {
        DIOMP_STEP(0) DIOMP_STEP(1) DIOMP_STEP(2) DIOMP_STEP(3) DIOMP_STEP(4)
        DIOMP_STEP(5) DIOMP_STEP(6) DIOMP_STEP(7) DIOMP_STEP(8)
    }
#undef DIOMP_STEP
}

// HALO: the kernel carries the epilogue stores into the neighbours' ghost
// planes.  Launches without neighbours use the instantiation without them:
// merely having those (never executed) stores in the loop body costs 2 %
// (profiles/r02_stencil_halo_codegen.txt).
template <bool HALO>
__global__ void __launch_bounds__(THREADS, 1)
    stencil_tma_kernel(const __grid_constant__ CUtensorMap map, const __grid_constant__ CUtensorMap pmap,
                       const __grid_constant__ Params p) {
    extern __shared__ __align__(1024) double sm[];
    double *psm = sm + NSLOT * SLOT;                      // u_prev tiles
    uint64_t *full = reinterpret_cast<uint64_t *>(psm + NPREV * PSLOT);
    uint64_t *empty = full + NSLOT;
    uint64_t *pfull = empty + NSLOT;
    uint64_t *pempty = pfull + NPREV;

    // Unit decode: interior chunks first, the two edge chunks (which wait on
    // and write to the neighbours) last -- or, with edge_first, the edge
    // chunks first so their NVLink halo stores drain under the interior.
    int c = blockIdx.x / p.ncols;
    const int col = blockIdx.x % p.ncols;
    if (p.nch > 2 && !p.edge_first) c = (c < p.nch - 2) ? c + 1 : (c == p.nch - 2 ? 0 : p.nch - 1);
    if (p.nch > 2 && p.edge_first) c = (c == 0) ? 0 : (c == 1 ? p.nch - 1 : c - 1);
    const int ty = col / p.ntz, tz = col % p.ntz;
    const int y0 = R + ty * TY, z0 = R + tz * TZ;
    const int64_t xa = R + (int64_t)c * p.chunk;
    int64_t xb = xa + p.chunk;
    if (xb > p.NX - R) xb = p.NX - R;
    const int L = (int)(xb - xa) + 2 * R;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < NSLOT; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
#pragma unroll
        for (int s = 0; s < NPREV; ++s) {
            mbar_init(&pfull[s], 1);
            mbar_init(&pempty[s], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // Programmatic dependent launch: this grid may have been scheduled while
    // the previous step's grid was still running; everything above touched
    // only shared memory.  Let the next step's grid be scheduled as early,
    // then wait until the previous grid has completed and its memory
    // operations are visible (returns at once without PDL).
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) {
        // this step's kernel started, so the previous step's kernel -- its
        // u_next stores and its halo stores into the neighbours -- has
        // completed: block 0 tells both neighbours (the previous step's
        // completion signal, sent here instead of by a last-CTA count at the
        // end of every step, which cost each CTA a fence and an atomic)
        if (p.sync && blockIdx.x == 0 && (p.sig_l || p.sig_r)) {
            __threadfence_system();
            if (p.sig_l) st_release_sys(p.sig_l, p.sl);
            if (p.sig_r) st_release_sys(p.sig_r, p.sr);
        }
        if (p.sync) {
            if (xa < 2 * R && p.wait_l) wait_ge(p.wait_l, p.wl);
            if (xb > p.NX - 2 * R && p.wait_r) wait_ge(p.wait_r, p.wr);
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
    }
    __syncthreads();

    if (warp == NCW) {
        // ---- producer warp: TMA loads of u_cur planes and u_prev tiles into their rings
        if (lane == 0) {
            const int nout = L - 2 * R;
            auto issue_prev = [&](int o) {  // u_prev tile of output plane o
                const int ps = o % NPREV;
                if (o >= NPREV) mbar_wait(&pempty[ps], (uint32_t)(((o / NPREV) - 1) & 1));
                mbar_expect_tx(&pfull[ps], PSLOT_BYTES);
                tma_load_plane(psm + ps * PSLOT, &pmap, z0, y0, (int)(xa + o), &pfull[ps]);
            };
            int next_prev = 0;
            for (int q = 0; q < L; ++q) {
                const int s = q % NSLOT;
                if (q >= NSLOT) mbar_wait(&empty[s], (uint32_t)(((q / NSLOT) - 1) & 1));
                mbar_expect_tx(&full[s], SLOT_BYTES);
                tma_load_plane(sm + s * SLOT, &map, z0 - R, y0 - R, (int)(xa - R + q), &full[s]);
                // keep u_prev PREV_AHEAD output planes ahead of the plane that completes
                for (; next_prev < nout && next_prev <= q - 2 * R + PREV_AHEAD; ++next_prev)
                    issue_prev(next_prev);
            }
        }
    } else {
        // ---- compute warps: 2 rows x 64 columns each, 2x2 points per thread
        const int ry = 2 * (warp / WZ), zz = 64 * (warp % WZ) + 2 * lane;
        const int64_t y = y0 + ry, z = z0 + zz;
        Lane ln;
        ln.yv0 = y < p.NY - R;
        ln.yv1 = y + 1 < p.NY - R;
        ln.zv0 = z < p.NZ - R;
        ln.zv1 = z + 1 < p.NZ - R;
        ln.full = (y0 + TY <= p.NY - R) && (z0 + TZ <= p.NZ - R);  // uniform per CTA
        ln.so = (R + ry) * BZ + R + zz;
        const int64_t g0 = (xa * p.NY + y) * p.NZ + z;
        ln.pn = p.u_next + g0;
        ln.x = xa;
        ln.src_pt = -1;
        if (p.src_x >= xa && p.src_x < xb) {
            const int64_t dy = p.src_y - y, dz = p.src_z - z;
            if (dy >= 0 && dy < 2 && dz >= 0 && dz < 2) ln.src_pt = (int)(dy * 2 + dz);
        }
        if (ln.full) consume<true, HALO>(p, sm, full, empty, psm, pfull, pempty, ln, L);
        else consume<false, HALO>(p, sm, full, empty, psm, pfull, pempty, ln, L);
    }

}

// Generic path: any radius <= 8, any even/odd extents, no alignment needs.
// One thread per interior point, operands straight from global (L1/L2).
struct GenericParams {
    double *u_next;
    const double *u_cur;
    const double *u_prev;
    int64_t NX, NY, NZ;
    int32_t r;
    double c0;
    double wx[9], wy[9], wz[9];
    int64_t src_x, src_y, src_z;
    double amp;
};

__global__ void __launch_bounds__(256) stencil_generic_kernel(const __grid_constant__ GenericParams p) {
    const int64_t ni = p.NX - 2 * p.r, nj = p.NY - 2 * p.r, nk = p.NZ - 2 * p.r;
    const int64_t total = ni * nj * nk;
    const int64_t sy = p.NZ, sx = p.NY * p.NZ;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = idx % nk + p.r;
        const int64_t j = (idx / nk) % nj + p.r;
        const int64_t i = idx / (nk * nj) + p.r;
        const int64_t g = i * sx + j * sy + k;
        const double u = p.u_cur[g];
        double acc = __dmul_rn(p.c0, u);
        for (int t = 1; t <= p.r; ++t)
            acc = __dadd_rn(acc, __dmul_rn(p.wx[t], __dadd_rn(p.u_cur[g + t * sx], p.u_cur[g - t * sx])));
        for (int t = 1; t <= p.r; ++t)
            acc = __dadd_rn(acc, __dmul_rn(p.wy[t], __dadd_rn(p.u_cur[g + t * sy], p.u_cur[g - t * sy])));
        for (int t = 1; t <= p.r; ++t)
            acc = __dadd_rn(acc, __dmul_rn(p.wz[t], __dadd_rn(p.u_cur[g + t], p.u_cur[g - t])));
        double out = __dadd_rn(__dsub_rn(__dmul_rn(2.0, u), p.u_prev[g]), acc);
        if (i == p.src_x && j == p.src_y && k == p.src_z) out = __dadd_rn(out, p.amp);
        p.u_next[g] = out;
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)ptr;
    });
    return fn;
}

static int make_plane_map(CUtensorMap *map, const double *u, int64_t NX, int64_t NY, int64_t NZ,
                          bool halo = true) {
    auto encode = get_encode_fn();
    if (!encode) return DIOMP_INTERNAL;
    cuuint64_t dims[3] = {(cuuint64_t)NZ, (cuuint64_t)NY, (cuuint64_t)NX};
    cuuint64_t strides[2] = {(cuuint64_t)NZ * 8, (cuuint64_t)NY * NZ * 8};
    cuuint32_t box[3] = {halo ? (cuuint32_t)BZ : (cuuint32_t)TZ, halo ? (cuuint32_t)BY : (cuuint32_t)TY, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    // L2 promotion of the TMA fills (DIOMP_STENCIL_L2PROMO=0/64/128/256, default 256)
    static const CUtensorMapL2promotion promo = [] {
        const char *e = getenv("DIOMP_STENCIL_L2PROMO");
        const int v = e ? atoi(e) : 256;
        return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
               : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
               : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                          : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    }();
    CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)u, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? DIOMP_OK : DIOMP_BAD_REQUEST;
}

static bool fast_path_ok(uint64_t u_next, uint64_t u_cur, uint64_t u_prev, int64_t NX, int64_t NY,
                         int64_t NZ, int radius) {
    if (radius != R) return false;
    if ((NZ & 1) || NX < 3 * R || NY <= 2 * R || NZ <= 2 * R) return false;
    if ((u_next | u_cur | u_prev) & 15) return false;
    if (NX > (1ll << 31) || NY > (1ll << 31) || NZ > (1ll << 31)) return false;
    return true;
}

// Chunking along x.  Units (column, chunk) are handed to SMs in blockIdx
// order as CTAs retire, so the step time is the makespan of that list
// schedule on kNumSMs slots with unit cost (planes + W); W = 4 planes of
// warm-up (the 2R extra u_cur planes and the pipeline fill) was fitted to
// chunk sweeps at 128 and 256 planes on B200 (tools/probe.py stencil 1024 NX
// with DIOMP_STENCIL_CHUNK).  Simulate each chunk count, keep the best;
// results are cached per shape.
static double list_makespan(int64_t nx_int, int ncols, int64_t chunk) {
    constexpr double W = 4.0;
    const int64_t nch = ceil_div(nx_int, chunk);
    std::priority_queue<double, std::vector<double>, std::greater<double>> slot;
    for (int i = 0; i < kNumSMs; ++i) slot.push(0.0);
    for (int64_t b = 0; b < nch; ++b) {
        int64_t c = b;  // interior chunks first, then the two edge chunks
        if (nch > 2) c = (b < nch - 2) ? b + 1 : (b == nch - 2 ? 0 : nch - 1);
        const double len = (double)(c == nch - 1 ? nx_int - c * chunk : chunk) + W;
        for (int u = 0; u < ncols; ++u) {
            const double t = slot.top();
            slot.pop();
            slot.push(t + len);
        }
    }
    double t = 0;
    while (!slot.empty()) {
        t = slot.top();
        slot.pop();
    }
    return t;
}

static void pick_chunks(int64_t nx_int, int ncols, int *chunk_out, int *nch_out) {
    const char *env = getenv("DIOMP_STENCIL_CHUNK");
    if (env && atoi(env) > 0) {
        int ch = atoi(env);
        if (ch < 2 * R) ch = 2 * R;
        *chunk_out = ch;
        *nch_out = (int)ceil_div(nx_int, ch);
        return;
    }
    static std::mutex mu;
    static std::map<std::pair<int64_t, int>, int64_t> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(nx_int, ncols);
    auto it = cache.find(key);
    int64_t chunk;
    if (it != cache.end()) {
        chunk = it->second;
    } else {
        double best = 1e300;
        chunk = nx_int;
        // chunk counts 1..16, and uneven splits (a long chunk plus a short
        // tail) between consecutive counts
        for (int nch = 1; nch <= 16; ++nch) {
            const int64_t hi = ceil_div(nx_int, nch), lo = ceil_div(nx_int, nch + 1);
            if (nch > 1 && hi < 2 * R) break;
            for (int j = 0; j < 8; ++j) {
                const int64_t ch = hi - (hi - lo) * j / 8;
                if (ch < 2 * R || (j && ch == hi)) continue;
                const double t = list_makespan(nx_int, ncols, ch);
                if (t < best * 0.999) {
                    best = t;
                    chunk = ch;
                }
            }
        }
        cache[key] = chunk;
    }
    *chunk_out = (int)chunk;
    *nch_out = (int)ceil_div(nx_int, chunk);
}

static int launch_fast(const CUtensorMap &map, const CUtensorMap &pmap, Params &p, cudaStream_t s) {
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_set[dev]) {
        DIOMP_CUDA_TRY(cudaFuncSetAttribute(stencil_tma_kernel<true>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)SMEM_BYTES));
        DIOMP_CUDA_TRY(cudaFuncSetAttribute(stencil_tma_kernel<false>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)SMEM_BYTES));
        attr_set[dev] = true;
    }
    const int64_t ny_int = p.NY - 2 * R, nz_int = p.NZ - 2 * R, nx_int = p.NX - 2 * R;
    const int nty = (int)ceil_div(ny_int, TY);
    p.ntz = (int)ceil_div(nz_int, TZ);
    p.ncols = nty * p.ntz;
    pick_chunks(nx_int, p.ncols, &p.chunk, &p.nch);
    const int64_t units = (int64_t)p.ncols * p.nch;
    if (units > 0x7fffffff) return DIOMP_BAD_REQUEST;
    // Small grids without device flags (one GPU; a step of a few tens of
    // microseconds is launch- and prologue-bound) let consecutive steps
    // overlap launch and prologue (programmatic dependent launch):
    // configs[0] on one GPU, 128^3 x 100 steps, 144 -> 163 Gpts/s.  Measured
    // slower elsewhere (profiles/r02_stencil_pdl.txt): large grids by 0.5 %
    // (1024^3: 257.4 -> 256.1), the device-flag multi-GPU steps by 8 %
    // (128^3 on two GPUs: 116 -> 107), so those launch plainly.
    // DIOMP_STENCIL_PDL=0/1 forces it.
    static const int pdl_env = getenv("DIOMP_STENCIL_PDL") ? atoi(getenv("DIOMP_STENCIL_PDL")) : -1;
    const bool pdl = pdl_env >= 0 ? pdl_env != 0
                                  : (!p.sync && nx_int * ny_int * nz_int <= (int64_t(1) << 25));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)units);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    if (p.left_next || p.right_next)
        DIOMP_CUDA_TRY(cudaLaunchKernelEx(&cfg, stencil_tma_kernel<true>, map, pmap, p));
    else
        DIOMP_CUDA_TRY(cudaLaunchKernelEx(&cfg, stencil_tma_kernel<false>, map, pmap, p));
    return DIOMP_OK;
}

static int launch_generic(const GenericParams &g, cudaStream_t s) {
    const int64_t total = (g.NX - 2 * g.r) * (g.NY - 2 * g.r) * (g.NZ - 2 * g.r);
    if (total <= 0) return DIOMP_OK;
    int64_t blocks = ceil_div(total, 256);
    if (blocks > kNumSMs * 16) blocks = kNumSMs * 16;
    stencil_generic_kernel<<<(unsigned)blocks, 256, 0, s>>>(g);
    DIOMP_LAUNCH_CHECK();
    return DIOMP_OK;
}

}  // namespace stencil
}  // namespace diomp

extern "C" {

int diomp_stencil_update(int device, const diomp_stencil_args *a, void *stream) {
    using namespace diomp::stencil;
    if (a->radius < 0 || a->radius > 8) return DIOMP_BAD_REQUEST;
    if (a->NX <= 2 * a->radius || a->NY <= 2 * a->radius || a->NZ <= 2 * a->radius) return DIOMP_OK;
    DIOMP_CUDA_TRY(cudaSetDevice(device));
    cudaStream_t s = (cudaStream_t)stream;
    if (fast_path_ok(a->u_next, a->u_cur, a->u_prev, a->NX, a->NY, a->NZ, a->radius) &&
        !getenv("DIOMP_STENCIL_GENERIC")) {
        CUtensorMap map, pmap;
        int rc = make_plane_map(&map, (const double *)a->u_cur, a->NX, a->NY, a->NZ);
        if (rc == DIOMP_OK)
            rc = make_plane_map(&pmap, (const double *)a->u_prev, a->NX, a->NY, a->NZ, false);
        if (rc == DIOMP_OK) {
            Params p{};
            p.u_next = (double *)a->u_next;
            p.u_prev = (const double *)a->u_prev;
            p.NX = a->NX; p.NY = a->NY; p.NZ = a->NZ;
            p.c0 = a->center;
            for (int t = 0; t <= R; ++t) { p.wx[t] = a->wx[t]; p.wy[t] = a->wy[t]; p.wz[t] = a->wz[t]; }
            p.src_x = -1;
            return launch_fast(map, pmap, p, s);
        }
    }
    GenericParams g{};
    g.u_next = (double *)a->u_next;
    g.u_cur = (const double *)a->u_cur;
    g.u_prev = (const double *)a->u_prev;
    g.NX = a->NX; g.NY = a->NY; g.NZ = a->NZ;
    g.r = a->radius;
    g.c0 = a->center;
    for (int t = 0; t <= a->radius; ++t) { g.wx[t] = a->wx[t]; g.wy[t] = a->wy[t]; g.wz[t] = a->wz[t]; }
    g.src_x = -1;
    return launch_generic(g, s);
}

int diomp_stencil_run(const diomp_stencil_plan *pl, int64_t step0, int64_t nsteps, void *stream) {
    using namespace diomp;
    using namespace diomp::stencil;
    if (pl->radius != R) return DIOMP_BAD_REQUEST;
    DIOMP_CUDA_TRY(cudaSetDevice(pl->device));
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nxl = pl->NX - 2 * R;
    bool fast = fast_path_ok(pl->field[0], pl->field[1], pl->field[0], pl->NX, pl->NY, pl->NZ, R) &&
                (pl->left_field[0] | pl->left_field[1] | pl->right_field[0] | pl->right_field[1]) % 16 == 0 &&
                nxl >= 2 * R && !getenv("DIOMP_STENCIL_GENERIC");
    CUtensorMap maps[2], pmaps[2];
    if (fast) {
        for (int b = 0; b < 2 && fast; ++b)
            fast = make_plane_map(&maps[b], (const double *)pl->field[b], pl->NX, pl->NY, pl->NZ) == DIOMP_OK &&
                   make_plane_map(&pmaps[b], (const double *)pl->field[b], pl->NX, pl->NY, pl->NZ, false) == DIOMP_OK;
    }
    const int64_t plane = pl->NY * pl->NZ;
    const bool nbrs = (pl->left_field[0] | pl->left_field[1] | pl->right_field[0] | pl->right_field[1]) != 0;
    // the generic path stores halos before its update: without device flags
    // nothing would order those stores after the neighbour's reads
    if (!fast && nbrs && !pl->sync) return DIOMP_BAD_REQUEST;
    static const int edge_first = getenv("DIOMP_STENCIL_EDGE_FIRST") ? atoi(getenv("DIOMP_STENCIL_EDGE_FIRST")) : 0;
    // Device flags per neighbour pair, nsteps + 1 signals per call:
    //   +1        entry: this call's first kernel started, so everything the
    //             caller enqueued before it on this stream (field init, H2D
    //             copies, the previous call) is complete
    //   +1+k+1    step step0+k finished (k = 0 .. nsteps-1)
    // Step k stores into a neighbour's ghost planes only once the neighbour
    // reported +1+k (entered, and finished its step step0+k-1, the last
    // reader of those planes).
    if (!fast && pl->sync && nbrs) {
        if (pl->left_field[0]) {
            signal_kernel<<<1, 1, 0, s>>>((uint64_t *)pl->sig_left, pl->to_left + 1);
            wait_kernel<<<1, 1, 0, s>>>((const uint64_t *)pl->wait_left, pl->from_left + 1);
        }
        if (pl->right_field[0]) {
            signal_kernel<<<1, 1, 0, s>>>((uint64_t *)pl->sig_right, pl->to_right + 1);
            wait_kernel<<<1, 1, 0, s>>>((const uint64_t *)pl->wait_right, pl->from_right + 1);
        }
        DIOMP_LAUNCH_CHECK();
    }
    for (int64_t st = step0; st < step0 + nsteps; ++st) {
        const int pb = (int)(st & 1), cb = 1 - pb;  // prev = field[s%2], cur = field[(s+1)%2]
        const int64_t k = st - step0;
        if (fast) {
            Params p{};
            p.u_next = (double *)pl->field[pb];
            p.u_prev = (const double *)pl->field[pb];
            p.NX = pl->NX; p.NY = pl->NY; p.NZ = pl->NZ;
            p.c0 = pl->center;
            for (int t = 0; t <= R; ++t) p.wx[t] = p.wy[t] = p.wz[t] = pl->w[t];
            p.left_next = (double *)pl->left_field[pb];
            p.right_next = (double *)pl->right_field[pb];
            p.nxl = nxl;
            p.src_x = pl->src_i; p.src_y = pl->src_j; p.src_z = pl->src_k;
            p.amp = pl->amp;
            p.sync = pl->sync;
            p.edge_first = edge_first;
            if (p.sync) {
                p.wait_l = pl->left_field[pb] ? (const uint64_t *)pl->wait_left : nullptr;
                p.wait_r = pl->right_field[pb] ? (const uint64_t *)pl->wait_right : nullptr;
                p.wl = pl->from_left + 1 + k;   // left entered / finished step st-1
                p.wr = pl->from_right + 1 + k;
                // block 0 announces entry (k = 0) or step st-1's completion
                p.sig_l = pl->left_field[pb] ? (uint64_t *)pl->sig_left : nullptr;
                p.sig_r = pl->right_field[pb] ? (uint64_t *)pl->sig_right : nullptr;
                p.sl = pl->to_left + 1 + k;
                p.sr = pl->to_right + 1 + k;
                p.counter = (unsigned int *)pl->counter;
            }
            int rc = launch_fast(maps[cb], pmaps[pb], p, s);
            if (rc) return rc;
            if (p.sync && st == step0 + nsteps - 1) {
                // the last step's completion: a one-thread kernel behind it
                if (pl->left_field[pb])
                    signal_kernel<<<1, 1, 0, s>>>((uint64_t *)pl->sig_left, pl->to_left + k + 2);
                if (pl->right_field[pb])
                    signal_kernel<<<1, 1, 0, s>>>((uint64_t *)pl->sig_right, pl->to_right + k + 2);
                DIOMP_LAUNCH_CHECK();
            }
        } else {
            // Listing-1 order: halo puts, flag exchange, update (+ source).
            const uint64_t cur = pl->field[cb];
            const uint64_t slab = (uint64_t)R * plane * 8;
            if (pl->left_field[cb]) {
                int rc = launch_copy(pl->left_field[cb] + (uint64_t)(R + nxl) * plane * 8,
                                     cur + (uint64_t)R * plane * 8, slab, s);
                if (rc) return rc;
            }
            if (pl->right_field[cb]) {
                int rc = launch_copy(pl->right_field[cb], cur + (uint64_t)nxl * plane * 8, slab, s);
                if (rc) return rc;
            }
            if (pl->sync) {
                if (pl->left_field[cb]) {
                    signal_kernel<<<1, 1, 0, s>>>((uint64_t *)pl->sig_left, pl->to_left + k + 2);
                    wait_kernel<<<1, 1, 0, s>>>((const uint64_t *)pl->wait_left, pl->from_left + k + 2);
                }
                if (pl->right_field[cb]) {
                    signal_kernel<<<1, 1, 0, s>>>((uint64_t *)pl->sig_right, pl->to_right + k + 2);
                    wait_kernel<<<1, 1, 0, s>>>((const uint64_t *)pl->wait_right, pl->from_right + k + 2);
                }
                DIOMP_LAUNCH_CHECK();
            }
            GenericParams g{};
            g.u_next = (double *)pl->field[pb];
            g.u_cur = (const double *)cur;
            g.u_prev = (const double *)pl->field[pb];
            g.NX = pl->NX; g.NY = pl->NY; g.NZ = pl->NZ;
            g.r = R;
            g.c0 = pl->center;
            for (int t = 0; t <= R; ++t) g.wx[t] = g.wy[t] = g.wz[t] = pl->w[t];
            g.src_x = pl->src_i; g.src_y = pl->src_j; g.src_z = pl->src_k;
            g.amp = pl->amp;
            int rc = launch_generic(g, s);
            if (rc) return rc;
        }
    }
    return DIOMP_OK;
}

}  // extern "C"
