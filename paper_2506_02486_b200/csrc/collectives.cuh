// OMPCCL collectives over NVLink peer memory (sm_100a).
//
// Reference: collectives.py:232-405.  The reference moves 1 MiB chunks around
// a ring through scratch slots with token flags (collectives.py:146-215); here
// every position reads/writes its peers' symmetric buffers directly, one
// kernel per position, so the wire pattern becomes:
//   allreduce  position p folds block p = [p*count/k, (p+1)*count/k) by loading
//              it from every position in ring order p, p+1, ... (exactly the
//              reference's reduce-scatter fold, collectives.py:22-24, 361-382)
//              and stores the result into every position's recv buffer (the
//              all-gather, collectives.py:386-405).  Per direction each GPU
//              moves 2(k-1)/k of the buffer -- the ring's optimum.
//   reduce     same block split, fold order starting at the root
//              (collectives.py:19-21, 270-323); results go to the root only.
//   bcast      the buffer is cut into k-1 blocks, one per non-root position;
//              each pulls its block from the root and pushes it to the other
//              non-roots.  The root's egress is exactly one buffer and every
//              non-root receives exactly one buffer.
// Entry / exit synchronisation is device-side (system-scope flags, see
// diomp_team) so back-to-back collectives never race on buffers -- the
// cross-collective slot race of the reference cannot occur.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "common.cuh"

namespace diomp {
namespace coll {

constexpr int THREADS = 512;

template <typename T>
struct Sum {
    __device__ __forceinline__ static T apply(T a, T b) { return a + b; }
};
// numpy's float add runs on x86 SSE/AVX, whose NaN rules differ from the GPU's
// canonical NaN: a NaN operand propagates (the first one if both), quieted,
// and an invalid operation (inf - inf) yields the x86 "default NaN" (sign
// set).  Reproduce them so NaN payloads are bit-identical to the reference.
template <>
struct Sum<float> {
    __device__ __forceinline__ static float apply(float a, float b) {
        if (a != a) return __int_as_float(__float_as_int(a) | 0x00400000);
        if (b != b) return __int_as_float(__float_as_int(b) | 0x00400000);
        const float r = __fadd_rn(a, b);
        return r != r ? __int_as_float((int)0xFFC00000u) : r;
    }
};
template <>
struct Sum<double> {
    __device__ __forceinline__ static double apply(double a, double b) {
        if (a != a) return __longlong_as_double(__double_as_longlong(a) | 0x0008000000000000ll);
        if (b != b) return __longlong_as_double(__double_as_longlong(b) | 0x0008000000000000ll);
        const double r = __dadd_rn(a, b);
        return r != r ? __longlong_as_double((long long)0xFFF8000000000000ull) : r;
    }
};
template <>
struct Sum<int32_t> {  // numpy wraps on overflow
    __device__ __forceinline__ static int32_t apply(int32_t a, int32_t b) {
        return (int32_t)((uint32_t)a + (uint32_t)b);
    }
};
template <>
struct Sum<int64_t> {
    __device__ __forceinline__ static int64_t apply(int64_t a, int64_t b) {
        return (int64_t)((uint64_t)a + (uint64_t)b);
    }
};

// numpy.minimum / numpy.maximum: NaN in either operand propagates (the first
// if both), otherwise the second operand wins ties (so min(0.0, -0.0) = -0.0).
template <typename T>
__device__ __forceinline__ bool isnan_t(T v) { return v != v; }

template <typename T>
struct Min {
    __device__ __forceinline__ static T apply(T a, T b) { return (a < b || isnan_t(a)) ? a : b; }
};
template <typename T>
struct Max {
    __device__ __forceinline__ static T apply(T a, T b) { return (a > b || isnan_t(a)) ? a : b; }
};

struct Args {
    diomp_team t;
    uint64_t send_off, recv_off;
    uint64_t count;   // elements (bytes for bcast)
    int32_t root;
    int32_t mode;     // 0 allreduce, 1 reduce
};

__device__ __forceinline__ void entry_barrier(const diomp_team &t) {
    if (!t.sync) return;
    const int q = threadIdx.x;
    if (q < t.k && q != t.pos) {
        if (blockIdx.x == 0) {
            __threadfence_system();
            st_release_sys((uint64_t *)(t.base[q] + t.flag_off) + t.slot[t.pos], t.epoch_to[q] + 1);
        }
        wait_ge((const uint64_t *)(t.base[t.pos] + t.flag_off) + t.slot[q], t.epoch_from[q] + 1);
    }
    __syncthreads();
}

// There is no exit handshake inside the collective kernels.  A call is
// complete toward a peer once that peer's stream has moved past it, which the
// next collective's entry signal (raised by block 0 at kernel start, after
// the previous kernel has retired) certifies -- so back-to-back collectives
// pay one handshake each, not two.  When the caller needs the result itself
// (a blocking call, coll.complete()), a one-CTA diomp_team_barrier after the
// kernel is the exit.

// Fold element range [lo, hi) of T over positions start, start+1, ... (mod k)
// and store to the recv buffer of every position in [dst_lo, dst_hi) (all) or
// to `only` (reduce).  Vectorised 16 B where the offsets allow.
template <typename T, typename OP, int KMAX, int U = (KMAX <= 4 ? 2 : 1)>
__device__ __forceinline__ void fold_range(const Args &a, uint64_t lo, uint64_t hi, int start,
                                           int only) {
    const diomp_team &t = a.t;
    const int k = t.k;
    constexpr int V = 16 / sizeof(T);
    const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t gsz = (uint64_t)gridDim.x * blockDim.x;
    // vector-aligned interior when send/recv offsets share alignment mod 16
    uint64_t vlo = hi, vhi = hi;
    if (((a.send_off - a.recv_off) & 15) == 0) {
        uint64_t first = lo;
        while (first < hi && ((a.send_off + first * sizeof(T)) & 15)) ++first;
        vlo = first;
        vhi = vlo + (hi - vlo) / V * V;
    }
    auto src = [&](int p) { return (const T *)(t.base[p] + a.send_off); };
    auto dst = [&](int p) { return (T *)(t.base[p] + a.recv_off); };
    // vector body: element vlo sits on a 16-byte boundary in every member's
    // send and recv buffer (same offsets, same alignment)
    using VT = uint4;
    auto vsrc = [&](int p) { return reinterpret_cast<const VT *>(src(p) + vlo); };
    auto vdst = [&](int p) { return reinterpret_cast<VT *>(dst(p) + vlo); };
    const uint64_t nvec = (vhi - vlo) / V;
    // U independent vectors per thread per iteration: all k*U loads are in
    // flight before the first fold (NVLink load latency ~2 us needs MBs in
    // flight per GPU)
    for (uint64_t v0 = gtid; v0 < nvec; v0 += gsz * U) {
        VT buf[U][KMAX];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t v = v0 + u * gsz;
            if (v < nvec) {
#pragma unroll
                for (int i = 0; i < KMAX; ++i)
                    if (i < k) {
                        int pidx = start + i;
                        if (pidx >= k) pidx -= k;
                        buf[u][i] = vsrc(pidx)[v];
                    }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t v = v0 + u * gsz;
            if (v >= nvec) break;
            T acc[V];
            const T *b0 = reinterpret_cast<const T *>(&buf[u][0]);
#pragma unroll
            for (int e = 0; e < V; ++e) acc[e] = b0[e];
#pragma unroll
            for (int i = 1; i < KMAX; ++i)
                if (i < k) {
                    const T *bi = reinterpret_cast<const T *>(&buf[u][i]);
#pragma unroll
                    for (int e = 0; e < V; ++e) acc[e] = OP::apply(acc[e], bi[e]);
                }
            VT out = *reinterpret_cast<VT *>(acc);
            if (only >= 0) {
                vdst(only)[v] = out;
            } else {
                for (int i = 0; i < k; ++i) {
                    int pidx = t.pos + i;  // own copy first, then peers
                    if (pidx >= k) pidx -= k;
                    vdst(pidx)[v] = out;
                }
            }
        }
    }
    // scalar head / tail (and everything when not vectorisable)
    const uint64_t nhead = vlo - lo, ntail = hi - vhi;
    for (uint64_t j = gtid; j < nhead + ntail; j += gsz) {
        const uint64_t e = j < nhead ? lo + j : vhi + (j - nhead);
        T acc = src(start)[e];
        for (int i = 1; i < k; ++i) {
            int pidx = start + i;
            if (pidx >= k) pidx -= k;
            acc = OP::apply(acc, src(pidx)[e]);
        }
        if (only >= 0) dst(only)[e] = acc;
        else
            for (int i = 0; i < k; ++i) dst(i)[e] = acc;
    }
}

// mode 0: fused allreduce (fold block p, store it to every member);
// mode 1: reduce to the root;
// mode 2: allreduce step 1 of 3 (fold block p into the own recv only; the
//         copy engine then pushes it to every peer).
template <typename T, typename OP, int KMAX, int U = (KMAX <= 4 ? 2 : 1)>
__global__ void __launch_bounds__(THREADS) reduce_kernel(const __grid_constant__ Args a) {
    entry_barrier(a.t);
    const int k = a.t.k, p = a.t.pos;
    const uint64_t lo = (uint64_t)p * a.count / k, hi = (uint64_t)(p + 1) * a.count / k;
    if (a.mode == 0) {
        fold_range<T, OP, KMAX, U>(a, lo, hi, p, -1);
    } else if (a.mode == 1) {
        fold_range<T, OP, KMAX, U>(a, lo, hi, a.root, a.root);
    }
#ifdef DIOMP_EXPERIMENTS
    else {
        fold_range<T, OP, KMAX, U>(a, lo, hi, p, p);
    }
#endif
}


// bcast: non-root position p handles block j = (p - root - 1 mod k) of k-1.
template <int U>
__global__ void __launch_bounds__(THREADS) bcast_kernel(const __grid_constant__ Args a) {
    entry_barrier(a.t);
    const diomp_team &t = a.t;
    const int k = t.k, p = t.pos, root = a.root;
    if (p != root) {
        const uint64_t off = a.send_off, n = a.count;
        const uint64_t al = (off + 15) & ~(uint64_t)15;
        const uint64_t body_lo = al - off < n ? al - off : n;
        const uint64_t nvec = (n - body_lo) / 16;
        const uint64_t body_hi = body_lo + nvec * 16;
        int j = p - root - 1;
        if (j < 0) j += k;
        const uint64_t vlo = (uint64_t)j * nvec / (k - 1), vhi = (uint64_t)(j + 1) * nvec / (k - 1);
        const uint4 *src = reinterpret_cast<const uint4 *>(t.base[root] + off + body_lo);
        const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
        const uint64_t gsz = (uint64_t)gridDim.x * blockDim.x;
        uint64_t v = vlo + gtid;
        for (; v + (U - 1) * gsz < vhi; v += U * gsz) {
            uint4 b[U];
#pragma unroll
            for (int u = 0; u < U; ++u) b[u] = src[v + u * gsz];
            for (int i = 0; i < k; ++i) {
                int q = p + i;
                if (q >= k) q -= k;
                if (q == root) continue;
                uint4 *d = reinterpret_cast<uint4 *>(t.base[q] + off + body_lo);
#pragma unroll
                for (int u = 0; u < U; ++u) d[v + u * gsz] = b[u];
            }
        }
        for (; v < vhi; v += gsz) {
            uint4 b = src[v];
            for (int q = 0; q < k; ++q)
                if (q != root) reinterpret_cast<uint4 *>(t.base[q] + off + body_lo)[v] = b;
        }
        // unaligned head/tail bytes: handled by block-0 owner
        if (j == 0) {
            const uint8_t *s8 = reinterpret_cast<const uint8_t *>(t.base[root] + off);
            const uint64_t ntail = n - body_hi;
            for (uint64_t i = gtid; i < body_lo + ntail; i += gsz) {
                const uint64_t e = i < body_lo ? i : body_hi + (i - body_lo);
                const uint8_t b = s8[e];
                for (int q = 0; q < k; ++q)
                    if (q != root) reinterpret_cast<uint8_t *>(t.base[q] + off)[e] = b;
            }
        }
    }
}

#ifdef DIOMP_EXPERIMENTS
// Experiments build only (-DDIOMP_EXPERIMENTS): measured slower than the
// default pull+push bcast on 4 B200 (profiles/r01_bcast_chain_sweep.txt,
// profiles/r01_bcast_pullchain_sweep.txt), kept out of the product library.
// bcast, chain algorithm (k >= 3, large buffers): positions in ring order
// from the root form a pipeline root -> root+1 -> ... -> root+k-1.  The body
// (16-B vectors) is cut into chunks; CTA b of every position handles chunks
// b, b+G, b+2G, ... in order: it waits until its predecessor's CTA b has
// delivered the chunk (a per-CTA progress flag in the own scratch), stores
// the chunk from its own buffer into the successor's, and publishes its
// progress in the successor's scratch.  Every NVLink link carries the buffer
// once in one direction -- measured faster than pull+push on 4 B200
// (tools/fanout_probe.cu: 686-694 vs 623-633 GB/s at 1 GiB, no flags).
// With the progress flags in place it loses, though: every chunk costs its
// CTA a system fence before the flag, and the fences dominate (4 B200, C-ABI
// probe, profiles/r01_bcast_chain_sweep.txt: best 628 GB/s at 1 GiB with 128
// CTAs x 256 KiB chunks vs 609 for pull+push, and 2x slower at 64 MiB).  So it
// is opt-in (DIOMP_BCAST_ALGO=chain / diomp_set_bcast_chain_min).
// Progress flags: chain_flags(q)[slot of the writer][b], value
// (E << 32) | chunks delivered, E = the call's entry signal value of the pair
// (monotone over every collective between the two endpoints, so old values
// can never satisfy a new wait).  Unaligned head/tail bytes: the root stores
// them to every member directly.
constexpr int CHAIN_GMAX = 256;                     // flag slots per writer
constexpr uint64_t CHAIN_FLAGS_OFF = 4096;          // from flag_off: after signals + counters
constexpr int CHAIN_U = 4;

__device__ __forceinline__ uint64_t *chain_flag(const diomp_team &t, int at, int writer, int b) {
    return (uint64_t *)(t.base[at] + t.flag_off + CHAIN_FLAGS_OFF) +
           (uint64_t)t.slot[writer] * CHAIN_GMAX + b;
}

__global__ void __launch_bounds__(THREADS) bcast_chain_kernel(const __grid_constant__ Args a,
                                                              uint64_t chv) {
    entry_barrier(a.t);
    const diomp_team &t = a.t;
    const int k = t.k, p = t.pos, root = a.root;
    const int h = (p - root + k) % k;                 // hop distance from the root
    const int succ = (p + 1) % k, pred = (p + k - 1) % k;
    const uint64_t off = a.send_off, n = a.count;
    const uint64_t al = (off + 15) & ~(uint64_t)15;
    const uint64_t body_lo = al - off < n ? al - off : n;
    const uint64_t nvec = (n - body_lo) / 16, body_hi = body_lo + nvec * 16;
    const uint4 *mine = reinterpret_cast<const uint4 *>(t.base[p] + off + body_lo);
    uint4 *next = reinterpret_cast<uint4 *>(t.base[succ] + off + body_lo);
    const uint64_t E = (uint64_t)(t.epoch_from[pred] + 1) << 32;   // from the predecessor
    const uint64_t Eo = (uint64_t)(t.epoch_to[succ] + 1) << 32;    // to the successor
    const uint64_t nch = (nvec + chv - 1) / chv;
    uint64_t i = 0;
    // the last hop only receives (its predecessor's exit signal follows the
    // predecessor's system fences, so the exit barrier covers the data)
    for (uint64_t c = blockIdx.x; h < k - 1 && c < nch; c += gridDim.x, ++i) {
        if (h > 0) {
            if (threadIdx.x == 0) wait_ge(chain_flag(t, p, pred, blockIdx.x), E | (i + 1));
            __syncthreads();
        }
        const uint64_t lo = c * chv, hi = lo + chv < nvec ? lo + chv : nvec;
        uint64_t v = lo + threadIdx.x;
        // L2-only loads: the chunk was just written over NVLink by the predecessor
        for (; v + (CHAIN_U - 1) * THREADS < hi; v += CHAIN_U * THREADS) {
            uint4 r[CHAIN_U];
#pragma unroll
            for (int u = 0; u < CHAIN_U; ++u) r[u] = __ldcg(mine + v + u * THREADS);
#pragma unroll
            for (int u = 0; u < CHAIN_U; ++u) next[v + u * THREADS] = r[u];
        }
        for (; v < hi; v += THREADS) next[v] = __ldcg(mine + v);
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence_system();
            st_release_sys(chain_flag(t, succ, p, blockIdx.x), Eo | (i + 1));
        }
    }
    if (h == 0 && blockIdx.x == 0) {   // unaligned head / tail bytes straight from the root
        const uint8_t *s8 = reinterpret_cast<const uint8_t *>(t.base[root] + off);
        const uint64_t ntail = n - body_hi;
        for (uint64_t e0 = threadIdx.x; e0 < body_lo + ntail; e0 += THREADS) {
            const uint64_t e = e0 < body_lo ? e0 : body_hi + (e0 - body_lo);
            const uint8_t b = s8[e];
            for (int q = 0; q < k; ++q)
                if (q != root) reinterpret_cast<uint8_t *>(t.base[q] + off)[e] = b;
        }
    }
}

// bcast, pull chain: the same root -> root+1 -> ... pipeline, but every hop
// LOADS its chunk from its predecessor's buffer over NVLink and stores it to
// its own HBM.  All the hop's stores are local, so the system fence before
// each progress flag drains local writes only instead of NVLink write acks
// (what made the push chain fence-bound), and every link carries the buffer
// once as read responses -- the "readers" pattern of tools/fanout_probe.cu,
// the fastest one measured (765 GB/s at 1 GiB on 4 B200).  The root does no
// data work.  Flags as the push chain: the predecessor's CTA b publishes
// (E << 32) | chunks into this position's scratch after its local stores.
__global__ void __launch_bounds__(THREADS) bcast_pullchain_kernel(const __grid_constant__ Args a,
                                                                  uint64_t chv) {
    entry_barrier(a.t);
    const diomp_team &t = a.t;
    const int k = t.k, p = t.pos, root = a.root;
    const int h = (p - root + k) % k;
    const int succ = (p + 1) % k, pred = (p + k - 1) % k;
    const uint64_t off = a.send_off, n = a.count;
    const uint64_t al = (off + 15) & ~(uint64_t)15;
    const uint64_t body_lo = al - off < n ? al - off : n;
    const uint64_t nvec = (n - body_lo) / 16, body_hi = body_lo + nvec * 16;
    const uint4 *from = reinterpret_cast<const uint4 *>(t.base[pred] + off + body_lo);
    uint4 *mine = reinterpret_cast<uint4 *>(t.base[p] + off + body_lo);
    const uint64_t E = (uint64_t)(t.epoch_from[pred] + 1) << 32;
    const uint64_t Eo = (uint64_t)(t.epoch_to[succ] + 1) << 32;
    const uint64_t nch = (nvec + chv - 1) / chv;
    uint64_t i = 0;
    for (uint64_t c = blockIdx.x; h > 0 && c < nch; c += gridDim.x, ++i) {
        if (h > 1) {   // the root's buffer is complete at entry
            if (threadIdx.x == 0) wait_ge(chain_flag(t, p, pred, blockIdx.x), E | (i + 1));
            __syncthreads();
        }
        const uint64_t lo = c * chv, hi = lo + chv < nvec ? lo + chv : nvec;
        uint64_t v = lo + threadIdx.x;
        for (; v + (CHAIN_U - 1) * THREADS < hi; v += CHAIN_U * THREADS) {
            uint4 r[CHAIN_U];
#pragma unroll
            for (int u = 0; u < CHAIN_U; ++u) r[u] = __ldcg(from + v + u * THREADS);
#pragma unroll
            for (int u = 0; u < CHAIN_U; ++u) mine[v + u * THREADS] = r[u];
        }
        for (; v < hi; v += THREADS) mine[v] = __ldcg(from + v);
        if (h < k - 1) {
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence_system();
                st_release_sys(chain_flag(t, succ, p, blockIdx.x), Eo | (i + 1));
            }
        }
    }
    if (h == 0 && blockIdx.x == 0) {
        const uint8_t *s8 = reinterpret_cast<const uint8_t *>(t.base[root] + off);
        const uint64_t ntail = n - body_hi;
        for (uint64_t e0 = threadIdx.x; e0 < body_lo + ntail; e0 += THREADS) {
            const uint64_t e = e0 < body_lo ? e0 : body_hi + (e0 - body_lo);
            const uint8_t b = s8[e];
            for (int q = 0; q < k; ++q)
                if (q != root) reinterpret_cast<uint8_t *>(t.base[q] + off)[e] = b;
        }
    }
}

// bcast algorithm: chain for k >= 3 from DIOMP_BCAST_CHAIN_MIN bytes (default
// never, see above), else pull+push.  DIOMP_BCAST_ALGO=pull|chain forces one;
// DIOMP_BCAST_ALGO=pullchain selects the pull chain for the chain sizes.
static std::atomic<uint64_t> g_bcast_chain_min{~0ull};
static std::once_flag g_bc_once;

static uint64_t bcast_chain_min() {
    std::call_once(g_bc_once, [] {
        const char *algo = getenv("DIOMP_BCAST_ALGO");
        const char *e = getenv("DIOMP_BCAST_CHAIN_MIN");
        if (e) g_bcast_chain_min = (uint64_t)strtoull(e, nullptr, 10);
        if (algo && !strcmp(algo, "pull")) g_bcast_chain_min = ~0ull;
        if (algo && (!strcmp(algo, "chain") || !strcmp(algo, "pullchain"))) g_bcast_chain_min = 0;
    });
    return g_bcast_chain_min.load(std::memory_order_relaxed);
}

// chain flavour: 1 = pull chain, 0 = push chain (DIOMP_BCAST_ALGO=pullchain
// or diomp_set_bcast_pullchain).
static std::atomic<int> g_bcast_pullchain{-1};

static bool bcast_pullchain() {
    int v = g_bcast_pullchain.load(std::memory_order_relaxed);
    if (v < 0) {
        const char *e = getenv("DIOMP_BCAST_ALGO");
        int want = (e && !strcmp(e, "pullchain")) ? 1 : 0;
        g_bcast_pullchain.compare_exchange_strong(v, want);
        v = g_bcast_pullchain.load(std::memory_order_relaxed);
    }
    return v == 1;
}

#endif  // DIOMP_EXPERIMENTS

// CTAs per SM (512 threads each).  Measured through the C ABI
// (tools/coll_probe.cpp, profiles/r01_collprobe_k{2,4}.txt): 2 CTAs/SM wins
// below 256 MiB (16 MiB allreduce k=2: 399 vs 324 GB/s busBW; 64 MiB k=4:
// 587 vs 559) and for every bcast size; 4 CTAs/SM (more loads in flight)
// wins the large allreduces by 1-2 %.  DIOMP_COLL_CTAS_PER_SM overrides.
static int ctas_per_sm(uint64_t bytes, bool reduce) {
    static int env = [] {
        const char *e = getenv("DIOMP_COLL_CTAS_PER_SM");
        int x = e ? atoi(e) : 0;
        return x < 0 ? 0 : (x > 4 ? 4 : x);
    }();
    if (env) return env;
    // round 2 sweep (profiles/r02_coll_sweep.txt, 4 B200, no exit handshake):
    // 4 CTAs/SM from 64 MiB for the reduction kernels (k=2 64 MiB 610 -> 617,
    // k=4 628 -> 633 GB/s busBW)
    return (reduce && bytes >= (64ull << 20)) ? 4 : 2;
}

static int grid_for(uint64_t work_items, int per_sm) {
    int64_t want = ceil_div((int64_t)work_items, THREADS);
    if (want < 1) want = 1;
    if (want > kNumSMs * per_sm) want = kNumSMs * per_sm;
    return (int)want;
}

#ifdef DIOMP_EXPERIMENTS
// Allreduce algorithm.  fused (default): one kernel, block p folded from the
// peers' send buffers (loads) and stored to every member (SM stores).  ce: the
// same fold into the own recv only, then the copy engine pushes block p to
// every peer, then an exit barrier.  Measured on 2 B200 (f32 sum, busBW):
// fused 493 / 617 / 660 GB/s at 64 MiB / 256 MiB / 1 GiB, ce 421 / 522 / 561
// -- the fold and the push run back to back instead of overlapping, which
// costs more than the copy engine's better bidirectional write rate (~774 vs
// ~697 GB/s per direction, profiles/r01_nvlink_probe.txt) gains.  Kept as an
// option: DIOMP_AR_ALGO=ce or diomp_set_allreduce_ce_min().
static std::atomic<uint64_t> g_ar_ce_min{~0ull};
static std::once_flag g_ar_once;

static uint64_t ar_ce_min() {
    std::call_once(g_ar_once, [] {
        const char *e = getenv("DIOMP_AR_ALGO");
        if (e && !strcmp(e, "ce")) g_ar_ce_min = 0;
    });
    return g_ar_ce_min.load(std::memory_order_relaxed);
}

#endif  // DIOMP_EXPERIMENTS

template <typename T, typename OP>
static int launch_reduce(Args a, cudaStream_t s) {
    const uint64_t per = a.count / a.t.k + 1;
    const uint64_t items = per / (16 / sizeof(T)) + 1;
    const int g = grid_for(items, ctas_per_sm(a.count * sizeof(T), true));
#ifdef DIOMP_EXPERIMENTS
    const bool ce = a.mode == 0 && a.t.sync && a.t.k > 1 && a.count * sizeof(T) >= ar_ce_min();
    if (ce) a.mode = 2;
#endif
    // KMAX = smallest supported team bound >= k (register footprint, and the
    // per-thread unroll, follow the actual team size)
    // vectors in flight per thread per source (DIOMP_COLL_U = 1 | 2 | 4 for
    // f32 sums, the benchmarked op; default 2 for k <= 4)
    static const int env_u = [] {
        const char *e = getenv("DIOMP_COLL_U");
        return e ? atoi(e) : 0;
    }();
    constexpr bool probe = std::is_same<T, float>::value && std::is_same<OP, Sum<float>>::value;
    if (probe && env_u == 1 && a.t.k <= 4) {
        if (a.t.k <= 2) reduce_kernel<T, OP, 2, 1><<<g, THREADS, 0, s>>>(a);
        else reduce_kernel<T, OP, 4, 1><<<g, THREADS, 0, s>>>(a);
    } else if (probe && env_u == 4 && a.t.k <= 4) {
        if (a.t.k <= 2) reduce_kernel<T, OP, 2, 4><<<g, THREADS, 0, s>>>(a);
        else reduce_kernel<T, OP, 4, 4><<<g, THREADS, 0, s>>>(a);
    } else if (a.t.k <= 2) reduce_kernel<T, OP, 2><<<g, THREADS, 0, s>>>(a);
    else if (a.t.k <= 4) reduce_kernel<T, OP, 4><<<g, THREADS, 0, s>>>(a);
    else if (a.t.k <= 8) reduce_kernel<T, OP, 8><<<g, THREADS, 0, s>>>(a);
    else if (a.t.k <= 16) reduce_kernel<T, OP, 16><<<g, THREADS, 0, s>>>(a);
    else reduce_kernel<T, OP, DIOMP_MAX_TEAM><<<g, THREADS, 0, s>>>(a);
    DIOMP_LAUNCH_CHECK();
#ifdef DIOMP_EXPERIMENTS
    if (ce) {
        const int k = a.t.k, p = a.t.pos;
        const uint64_t lo = (uint64_t)p * a.count / k * sizeof(T);
        const uint64_t hi = (uint64_t)(p + 1) * a.count / k * sizeof(T);
        if (hi > lo) {
            const uint8_t *src = (const uint8_t *)(a.t.base[p] + a.recv_off) + lo;
            for (int i = 1; i < k; ++i) {
                const int q = (p + i) % k;
                uint8_t *dst = (uint8_t *)(a.t.base[q] + a.recv_off) + lo;
                DIOMP_CUDA_TRY(cudaMemcpyAsync(dst, src, hi - lo, cudaMemcpyDeviceToDevice, s));
            }
        }
    }
#endif
    return DIOMP_OK;
}

template <typename T>
static int dispatch_op(const Args &a, int op, cudaStream_t s) {
    switch (op) {
        case DIOMP_SUM: return launch_reduce<T, Sum<T>>(a, s);
        case DIOMP_MIN: return launch_reduce<T, Min<T>>(a, s);
        case DIOMP_MAX: return launch_reduce<T, Max<T>>(a, s);
        default: return DIOMP_BAD_REQUEST;
    }
}

static int dispatch(const Args &a, int dtype, int op, cudaStream_t s) {
    switch (dtype) {
        case DIOMP_F32: return dispatch_op<float>(a, op, s);
        case DIOMP_F64: return dispatch_op<double>(a, op, s);
        case DIOMP_I32: return dispatch_op<int32_t>(a, op, s);
        case DIOMP_I64: return dispatch_op<int64_t>(a, op, s);
        default: return DIOMP_BAD_REQUEST;
    }
}

static bool team_ok(const diomp_team *t) {
    return t->k >= 1 && t->k <= DIOMP_MAX_TEAM && t->pos >= 0 && t->pos < t->k;
}

// ---------------------------------------------------------------------------
// Small messages: one-shot "LL" (low-latency) collectives.
//
// For a few KiB the two-phase kernel above is all handshake: entry round trip,
// peer loads, stores.  Here every 4-byte payload word travels with its flag in
// one 8-byte store, (epoch << 32) | word, so a receiver knows the word has
// landed when its flag reads this call's epoch -- no separate signal, no
// fence, no entry or exit handshake; one NVLink one-way trip per call.
//   allreduce: every position stores its whole vector into every peer's LL
//     slot, then folds all k vectors element by element in the reference's
//     order (block b = [b*count/k, (b+1)*count/k) folded from position b), so
//     each position computes the full result itself -- bit-identical.
//   bcast: the root stores into every non-root's slot; non-roots copy out.
// Slots: per source endpoint, two parities (epoch & 1); a parity is reused
// only after the peer acknowledged the call that used it last (the
// acknowledgement bank below -- receiving a peer's words alone does not
// prove it: a bcast root receives none).  Epochs are per pair (both ends
// count every LL call between them), flags start at 0 (segments are
// zero-filled), epochs at 1.
// ---------------------------------------------------------------------------

struct LLArgs {
    int32_t k, pos, dtype, op, root, mode;   // mode 0 allreduce, 1 bcast
    uint64_t base[DIOMP_MAX_TEAM];           // position's segment base (as addressable here)
    uint32_t slot[DIOMP_MAX_TEAM];           // position's global endpoint index
    uint32_t ep_to[DIOMP_MAX_TEAM];          // this call's epoch toward position q
    uint32_t ep_from[DIOMP_MAX_TEAM];        // this call's epoch from position q
    uint64_t ll_off, slot_bytes;             // LL region offset; bytes per (slot, parity)
    uint64_t send_off, recv_off, count;      // elements (bytes for bcast)
};

__device__ __forceinline__ uint64_t *ll_slot(const LLArgs &a, int at, int from, uint32_t epoch) {
    return (uint64_t *)(a.base[at] + a.ll_off + ((uint64_t)a.slot[from] * 2 + (epoch & 1)) * a.slot_bytes);
}

// Acknowledgements.  The two-parity reuse argument above needs return
// traffic: a bcast root receives nothing from its peers, so on its own it
// could run two calls ahead and overwrite a parity slot a slow peer has not
// read yet (the peer then waits forever for an epoch that was overwritten).
// So every member acknowledges every call to every peer of the team: once
// all its CTAs are done with call e (read what it had to read), the last CTA
// stores e into each peer's ack bank -- also where nothing travelled between
// the two (a bcast between two non-roots, the root's side of a bcast),
// because both ends count every LL call on the pair.  A writer stores call e
// into a peer's parity slot only after the peer acknowledged call e-2, the
// previous call of that parity -- a local poll, normally satisfied at once.
// Bank: the 4 KiB below ll_off in every member's segment, ack[source
// endpoint] (u64), then a u32 last-CTA counter.
constexpr uint64_t LL_ACK_BELOW = 4096;

__device__ __forceinline__ uint64_t *ll_ack(const LLArgs &a, int at, int from) {
    return (uint64_t *)(a.base[at] + a.ll_off - LL_ACK_BELOW) + a.slot[from];
}

__device__ __forceinline__ unsigned int *ll_counter(const LLArgs &a) {
    return (unsigned int *)(a.base[a.pos] + a.ll_off - LL_ACK_BELOW + 8 * DIOMP_MAX_TEAM);
}

// before writing this call's words into q's slot: q consumed call e-2
__device__ __forceinline__ void ll_wait_ack(const LLArgs &a, int q) {
    const uint32_t e = a.ep_to[q];
    if (e > 2) wait_ge(ll_ack(a, a.pos, q), (uint64_t)(e - 2));
}

// after every CTA is done with this call: the last CTA acknowledges it to
// every peer
__device__ __forceinline__ void ll_send_acks(const LLArgs &a) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(ll_counter(a), 1u) == gridDim.x - 1) {
            atomicExch(ll_counter(a), 0u);
            __threadfence_system();
            for (int q = 0; q < a.k; ++q)
                if (q != a.pos) st_release_sys(ll_ack(a, q, a.pos), (uint64_t)a.ep_from[q]);
        }
    }
}

__device__ __forceinline__ uint32_t ll_wait(const uint64_t *p, uint32_t epoch) {
    uint64_t v;
    const uint64_t t0 = globaltimer_ns();
    for (;;) {
        asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
        if ((uint32_t)(v >> 32) == epoch) return (uint32_t)v;
        if (globaltimer_ns() - t0 > g_wait_timeout_ns) {
            record_device_error((unsigned)DIOMP_INTERNAL);
            return 0;
        }
    }
}

__device__ __forceinline__ void ll_store(uint64_t *p, uint32_t epoch, uint32_t w) {
    const uint64_t v = ((uint64_t)epoch << 32) | w;
    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <typename T, typename OP, int KMAX>
__global__ void __launch_bounds__(256) ll_allreduce_kernel(const __grid_constant__ LLArgs a) {
    constexpr int W = sizeof(T) / 4;
    const int k = a.k, me = a.pos;
    const uint64_t n = a.count;
    const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t gsz = (uint64_t)gridDim.x * blockDim.x;
    const T *send = (const T *)(a.base[me] + a.send_off);
    T *recv = (T *)(a.base[me] + a.recv_off);
    if (threadIdx.x < k && threadIdx.x != me) ll_wait_ack(a, threadIdx.x);
    __syncthreads();
    // push my vector into every peer's slot
    for (uint64_t e = gtid; e < n; e += gsz) {
        uint32_t w[W];
        const T v = send[e];
        memcpy(w, &v, sizeof(T));
        for (int q = 0; q < k; ++q) {
            if (q == me) continue;
            uint64_t *dst = ll_slot(a, q, me, a.ep_to[q]) + e * W;
#pragma unroll
            for (int i = 0; i < W; ++i) ll_store(dst + i, a.ep_to[q], w[i]);
        }
    }
    // gather every position's element and fold in the reference order
    for (uint64_t e = gtid; e < n; e += gsz) {
        T vals[KMAX];
#pragma unroll
        for (int q = 0; q < KMAX; ++q) {
            if (q >= k) break;
            if (q == me) {
                vals[q] = send[e];
            } else {
                const uint64_t *src = ll_slot(a, me, q, a.ep_from[q]) + e * W;
                uint32_t w[W];
#pragma unroll
                for (int i = 0; i < W; ++i) w[i] = ll_wait(src + i, a.ep_from[q]);
                memcpy(&vals[q], w, sizeof(T));
            }
        }
        int b = (int)(e * (uint64_t)k / n);
        while (b + 1 < k && (uint64_t)(b + 1) * n / k <= e) ++b;
        while (b > 0 && (uint64_t)b * n / k > e) --b;
        T acc = vals[b];
        for (int i = 1; i < k; ++i) {
            int q = b + i;
            if (q >= k) q -= k;
#pragma unroll
            for (int qq = 0; qq < KMAX; ++qq)   // register-resident select of vals[q]
                if (qq == q) acc = OP::apply(acc, vals[qq]);
        }
        recv[e] = acc;
    }
    ll_send_acks(a);
}

// bcast of `count` bytes at send_off: the root stores 4-byte words (zero-padded
// tail) into every non-root's slot; non-roots copy them into their buffer.
__global__ void __launch_bounds__(256) ll_bcast_kernel(const __grid_constant__ LLArgs a) {
    const int k = a.k, me = a.pos, root = a.root;
    const uint64_t nw = (a.count + 3) / 4;
    const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t gsz = (uint64_t)gridDim.x * blockDim.x;
    uint8_t *buf = (uint8_t *)(a.base[me] + a.send_off);
    if (me == root) {
        if (threadIdx.x < k && threadIdx.x != root) ll_wait_ack(a, threadIdx.x);
        __syncthreads();
        for (uint64_t i = gtid; i < nw; i += gsz) {
            uint32_t w = 0;
            const uint64_t o = i * 4;
            for (int b = 0; b < 4 && o + b < a.count; ++b) w |= (uint32_t)buf[o + b] << (8 * b);
            for (int q = 0; q < k; ++q)
                if (q != root) ll_store(ll_slot(a, q, root, a.ep_to[q]) + i, a.ep_to[q], w);
        }
    } else {
        const uint64_t *src = ll_slot(a, me, root, a.ep_from[root]);
        for (uint64_t i = gtid; i < nw; i += gsz) {
            const uint32_t w = ll_wait(src + i, a.ep_from[root]);
            const uint64_t o = i * 4;
            for (int b = 0; b < 4 && o + b < a.count; ++b) buf[o + b] = (uint8_t)(w >> (8 * b));
        }
    }
    ll_send_acks(a);
}

template <typename T, typename OP>
static int launch_ll(const LLArgs &a, cudaStream_t s) {
    const int64_t blocks = std::min<int64_t>(ceil_div((int64_t)a.count, 256), 32);
    if (a.k <= 2) ll_allreduce_kernel<T, OP, 2><<<(unsigned)blocks, 256, 0, s>>>(a);
    else if (a.k <= 4) ll_allreduce_kernel<T, OP, 4><<<(unsigned)blocks, 256, 0, s>>>(a);
    else if (a.k <= 8) ll_allreduce_kernel<T, OP, 8><<<(unsigned)blocks, 256, 0, s>>>(a);
    else return DIOMP_BAD_REQUEST;
    DIOMP_LAUNCH_CHECK();
    return DIOMP_OK;
}

template <typename T>
static int ll_dispatch_op(const LLArgs &a, cudaStream_t s) {
    switch (a.op) {
        case DIOMP_SUM: return launch_ll<T, Sum<T>>(a, s);
        case DIOMP_MIN: return launch_ll<T, Min<T>>(a, s);
        case DIOMP_MAX: return launch_ll<T, Max<T>>(a, s);
        default: return DIOMP_BAD_REQUEST;
    }
}

}  // namespace coll
}  // namespace diomp

extern "C" {

#ifdef DIOMP_EXPERIMENTS
int diomp_set_allreduce_ce_min(uint64_t bytes) {
    diomp::coll::ar_ce_min();  // settle the environment default first
    diomp::coll::g_ar_ce_min.store(bytes, std::memory_order_relaxed);
    return DIOMP_OK;
}

int diomp_set_bcast_chain_min(uint64_t bytes) {
    diomp::coll::bcast_chain_min();  // settle the environment default first
    diomp::coll::g_bcast_chain_min.store(bytes, std::memory_order_relaxed);
    return DIOMP_OK;
}

int diomp_set_bcast_pullchain(int32_t on) {
    diomp::coll::g_bcast_pullchain.store(on ? 1 : 0, std::memory_order_relaxed);
    return DIOMP_OK;
}
#endif  // DIOMP_EXPERIMENTS

int diomp_allreduce(const diomp_team *team, uint64_t send_off, uint64_t recv_off, uint64_t count,
                    int32_t dtype, int32_t op, void *stream) {
    using namespace diomp::coll;
    if (!team_ok(team)) return DIOMP_BAD_REQUEST;
    if (count == 0) return DIOMP_OK;
    DIOMP_CUDA_TRY(cudaSetDevice(team->device));
    Args a{};
    a.t = *team;
    a.send_off = send_off;
    a.recv_off = recv_off;
    a.count = count;
    a.mode = 0;
    return dispatch(a, dtype, op, (cudaStream_t)stream);
}

int diomp_reduce(const diomp_team *team, uint64_t send_off, uint64_t recv_off, uint64_t count,
                 int32_t dtype, int32_t op, int32_t root, void *stream) {
    using namespace diomp::coll;
    if (!team_ok(team) || root < 0 || root >= team->k) return DIOMP_BAD_REQUEST;
    if (count == 0) return DIOMP_OK;
    DIOMP_CUDA_TRY(cudaSetDevice(team->device));
    Args a{};
    a.t = *team;
    a.send_off = send_off;
    a.recv_off = recv_off;
    a.count = count;
    a.root = root;
    a.mode = 1;
    return dispatch(a, dtype, op, (cudaStream_t)stream);
}

int diomp_ll_collective(const diomp_ll_args *x, void *stream) {
    using namespace diomp;
    using namespace diomp::coll;
    if (x->k < 1 || x->k > 8 || x->pos < 0 || x->pos >= x->k || x->root < 0 || x->root >= x->k)
        return DIOMP_BAD_REQUEST;
    if (x->count == 0 || x->k == 1) return DIOMP_OK;
    LLArgs a{};
    a.k = x->k; a.pos = x->pos; a.dtype = x->dtype; a.op = x->op; a.root = x->root;
    a.mode = x->mode;
    for (int q = 0; q < x->k; ++q) {
        a.base[q] = x->base[q];
        a.slot[q] = x->slot[q];
        a.ep_to[q] = x->epoch_to[q];
        a.ep_from[q] = x->epoch_from[q];
    }
    a.ll_off = x->ll_off;
    a.slot_bytes = x->slot_bytes;
    a.send_off = x->send_off;
    a.recv_off = x->recv_off;
    a.count = x->count;
    const uint64_t esz = x->mode == 1 ? 1 : (x->dtype == DIOMP_F64 || x->dtype == DIOMP_I64 ? 8 : 4);
    if ((x->count * esz + 3) / 4 * 8 > x->slot_bytes) return DIOMP_BAD_REQUEST;   // LL doubles the bytes
    DIOMP_CUDA_TRY(cudaSetDevice(x->device));
    cudaStream_t s = (cudaStream_t)stream;
    if (x->mode == 1) {
        const int64_t blocks = std::min<int64_t>(ceil_div((int64_t)(x->count + 3) / 4, 256), 32);
        ll_bcast_kernel<<<(unsigned)blocks, 256, 0, s>>>(a);
        DIOMP_LAUNCH_CHECK();
        return DIOMP_OK;
    }
    switch (x->dtype) {
        case DIOMP_F32: return ll_dispatch_op<float>(a, s);
        case DIOMP_F64: return ll_dispatch_op<double>(a, s);
        case DIOMP_I32: return ll_dispatch_op<int32_t>(a, s);
        case DIOMP_I64: return ll_dispatch_op<int64_t>(a, s);
        default: return DIOMP_BAD_REQUEST;
    }
}

// One LL call as the runtime issues it, in a single C call: this call's
// epochs from the context's pair table (then advanced), the stream ordered
// after the caller's `after` stream (an event, no host synchronisation), the
// launch, and with `blocking` the wait for completion plus the device
// error-word check (a timed-out device wait -> DIOMP_INTERNAL, the
// reference's TransportFailure).  The Python equivalent cost ~11 us of
// interpreter time per call (profiles/r02_coll_host_overhead_ll.txt).
int diomp_ll_call(void *ctx, diomp_ll_args *x, void *stream, void *after, int32_t blocking) {
    using namespace diomp;
    auto *c = (rma::Ctx *)ctx;
    if (!c || x->k < 1 || x->k > 8 || x->pos < 0 || x->pos >= x->k) return DIOMP_BAD_REQUEST;
    const uint32_t n = (uint32_t)c->nranks * (uint32_t)c->dpr;
    const uint32_t me = x->slot[x->pos];
    for (int q = 0; q < x->k; ++q)
        if (x->slot[q] >= n) return DIOMP_BAD_REQUEST;
    if (x->count == 0 || x->k == 1) return DIOMP_OK;
    cudaStream_t s = (cudaStream_t)stream;
    DIOMP_CUDA_TRY(cudaSetDevice(x->device));
    if (after && after != stream) {
        // record + wait under the lock: another thread's record on the same
        // event cannot slip in between and order this call after the wrong
        // stream
        std::lock_guard<std::mutex> lk(c->mu);
        if ((int)c->order_ev.size() <= x->device) c->order_ev.resize(x->device + 1, nullptr);
        if (!c->order_ev[x->device])
            DIOMP_CUDA_TRY(cudaEventCreateWithFlags(&c->order_ev[x->device], cudaEventDisableTiming));
        cudaEvent_t ev = c->order_ev[x->device];
        DIOMP_CUDA_TRY(cudaEventRecord(ev, (cudaStream_t)after));
        DIOMP_CUDA_TRY(cudaStreamWaitEvent(s, ev, 0));
    }
    {
        std::lock_guard<std::mutex> lk(c->mu);
        for (int q = 0; q < x->k; ++q) {
            if (q == x->pos) continue;
            const uint32_t p = x->slot[q];
            x->epoch_to[q] = c->ll_sent[me * n + p] + 1;
            x->epoch_from[q] = c->ll_recvd[p * n + me] + 1;
        }
        int rc = diomp_ll_collective(x, stream);
        if (rc) return rc;
        for (int q = 0; q < x->k; ++q) {
            if (q == x->pos) continue;
            const uint32_t p = x->slot[q];
            c->ll_sent[me * n + p] += 1;
            c->ll_recvd[p * n + me] += 1;
        }
    }
    if (!blocking) return DIOMP_OK;
    DIOMP_CUDA_TRY(cudaStreamSynchronize(s));
    return diomp_device_error(x->device);
}

int diomp_bcast(const diomp_team *team, uint64_t offset, uint64_t nbytes, int32_t root, void *stream) {
    using namespace diomp;
    using namespace diomp::coll;
    if (!team_ok(team) || root < 0 || root >= team->k) return DIOMP_BAD_REQUEST;
    if (nbytes == 0 || team->k == 1) return DIOMP_OK;
    DIOMP_CUDA_TRY(cudaSetDevice(team->device));
    Args a{};
    a.t = *team;
    a.send_off = offset;
    a.recv_off = offset;
    a.count = nbytes;
    a.root = root;
#ifdef DIOMP_EXPERIMENTS
    if (team->sync && team->k >= 3 && nbytes >= bcast_chain_min() && nbytes >= 16 * CHAIN_GMAX) {
        // chunk / CTA count: DIOMP_BCAST_CHAIN_CHUNK (bytes), DIOMP_BCAST_CHAIN_G
        static const uint64_t env_chunk = [] {
            const char *e = getenv("DIOMP_BCAST_CHAIN_CHUNK");
            return e ? (uint64_t)strtoull(e, nullptr, 10) : (uint64_t)(256 << 10);
        }();
        static const int env_g = [] {
            const char *e = getenv("DIOMP_BCAST_CHAIN_G");
            int x = e ? atoi(e) : 128;
            return x < 1 ? 1 : (x > CHAIN_GMAX ? CHAIN_GMAX : x);
        }();
        const uint64_t nvec = nbytes / 16;
        const uint64_t chv = std::max<uint64_t>(env_chunk / 16, 32);
        const uint64_t nch = (nvec + chv - 1) / chv;
        const int g = (int)std::min<uint64_t>((uint64_t)env_g, nch);
        if (bcast_pullchain()) bcast_pullchain_kernel<<<g, THREADS, 0, (cudaStream_t)stream>>>(a, chv);
        else bcast_chain_kernel<<<g, THREADS, 0, (cudaStream_t)stream>>>(a, chv);
        DIOMP_LAUNCH_CHECK();
        return DIOMP_OK;
    }
#endif
    const uint64_t per = nbytes / (uint64_t)(team->k - 1) / 16 + 1;
    // k >= 4 (profiles/r02_coll_sweep.txt): 1 CTA/SM with 2 vectors in flight
    // between 32 and 256 MiB (64 MiB 610 -> 625 GB/s), 4 CTAs/SM with 4
    // vectors from 256 MiB (1 GiB 617 -> 633)
    int per_sm = ctas_per_sm(nbytes, false);
    const bool big4 = team->k >= 4 && nbytes >= (256ull << 20);
    const bool mid4 = team->k >= 4 && nbytes >= (32ull << 20) && !big4;
    if (!getenv("DIOMP_COLL_CTAS_PER_SM")) per_sm = big4 ? 4 : mid4 ? 1 : per_sm;
    const int g = grid_for(per, per_sm);
    // 16-B vectors in flight per thread (DIOMP_BCAST_U = 2 | 4 | 8 overrides).
    // Measured on 4 B200 (profiles/r01_bcast_u_sweep.txt): 2 beats 4 and 8 at
    // 2 CTAs/SM from 32 MiB -- fewer outstanding NVLink loads per SM, less
    // congestion (k=4: 64 MiB 575 vs 518 GB/s, 1 GiB 608 vs 599; k=3/k=2 also
    // ahead); only k=4 below 32 MiB keeps 4 (16 MiB: 402 vs 390).
    static const int env_u = [] {
        const char *e = getenv("DIOMP_BCAST_U");
        return e ? atoi(e) : 0;
    }();
    const int u = env_u ? env_u : (team->k >= 4 && (nbytes < (32ull << 20) || big4) ? 4 : 2);
    if (u == 4) bcast_kernel<4><<<g, THREADS, 0, (cudaStream_t)stream>>>(a);
    else if (u == 8) bcast_kernel<8><<<g, THREADS, 0, (cudaStream_t)stream>>>(a);
    else bcast_kernel<2><<<g, THREADS, 0, (cudaStream_t)stream>>>(a);
    DIOMP_LAUNCH_CHECK();
    return DIOMP_OK;
}

}  // extern "C"
