// Segments, IPC, streams/events and the one-sided data plane.
//
// Replaces the reference's simulated arenas (global_memory.py:190-206) and
// frame transport (transport.py:508-566, 830-861): a segment is one
// cudaMalloc per device, peers reach it through CUDA IPC or peer access, and
// put/get move bytes over NVLink directly on the initiator's stream -- no
// frames, no progress thread: SM copy kernels (small transfers, local copies),
// the copy engine for large remote puts, a bulk-async TMA kernel for large
// remote gets (see diomp_put / diomp_get for the measured crossovers).
#pragma once

#include <cstring>
#include <mutex>

#include "common.cuh"

namespace diomp {

// ---------------------------------------------------------------------------
// copy kernel (put / get)
// ---------------------------------------------------------------------------

// 16-byte vector body: each thread keeps UNROLL independent 16 B loads in
// flight before storing, which is what hides the ~2 us NVLink round trip of
// peer loads (get) and keeps enough posted stores outstanding (put).
template <int UNROLL>
__global__ void __launch_bounds__(512) copy16_kernel(uint4 *__restrict__ dst,
                                                     const uint4 *__restrict__ src,
                                                     uint64_t n16) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (UNROLL - 1) * stride < n16; i += UNROLL * stride) {
        uint4 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) v[u] = src[i + u * stride];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) dst[i + u * stride] = v[u];
    }
    for (; i < n16; i += stride) dst[i] = src[i];
}

// Unaligned head/tail bytes (and wholly misaligned pairs): plain byte copy.
__global__ void copy1_kernel(uint8_t *__restrict__ dst, const uint8_t *__restrict__ src,
                             uint64_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        dst[i] = src[i];
}

__global__ void copy8_kernel(uint64_t *__restrict__ dst, const uint64_t *__restrict__ src,
                             uint64_t n8) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += stride)
        dst[i] = src[i];
}

// Bulk-async (TMA engine) copy for large peer reads: one thread per CTA keeps
// STAGES chunk loads (peer HBM -> smem, cp.async.bulk + mbarrier) in flight and
// drains each landed chunk with a bulk store to local HBM.  No per-byte SM
// instructions, so ~148 CTAs keep enough NVLink reads outstanding to reach the
// link peak (probe: 785 GB/s at 1 GiB vs 774 for the SM loop;
// profiles/r01_nvlink_probe.txt).  dst, src, n and chunk are multiples of 16.
namespace bulk {
constexpr int STAGES = 4;
constexpr uint32_t CHUNK = 32768;
constexpr int CTAS = kNumSMs;

__device__ __forceinline__ uint32_t saddr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void load_chunk(char *smem, const char *src, uint32_t bytes,
                                           uint64_t *bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(saddr(smem)),
        "l"(src), "r"(bytes), "r"(saddr(bar))
        : "memory");
}

__global__ void __launch_bounds__(32) bulk_copy_kernel(char *__restrict__ dst,
                                                       const char *__restrict__ src, uint64_t n) {
    extern __shared__ __align__(128) char ring[];
    __shared__ __align__(8) uint64_t full[STAGES];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < STAGES; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&full[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint64_t nchunks = (n + CHUNK - 1) / CHUNK;
    auto chunk_bytes = [&](uint64_t c) {
        return (uint32_t)((c + 1) * CHUNK <= n ? CHUNK : n - c * CHUNK);
    };
    uint64_t next = blockIdx.x;
    for (int s = 0; s < STAGES && next < nchunks; ++s, next += gridDim.x)
        load_chunk(ring + (size_t)s * CHUNK, src + next * CHUNK, chunk_bytes(next), &full[s]);
    uint32_t phase = 0;
    int s = 0;
    for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        asm volatile(
            "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::
                "r"(saddr(&full[s])),
            "r"(phase)
            : "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                         dst + c * CHUNK),
                     "r"(saddr(ring + (size_t)s * CHUNK)), "r"(chunk_bytes(c))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (next < nchunks) {  // refill slot s once its store has read it
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            load_chunk(ring + (size_t)s * CHUNK, src + next * CHUNK, chunk_bytes(next), &full[s]);
            next += gridDim.x;
        }
        if (++s == STAGES) {
            s = 0;
            phase ^= 1;
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
}  // namespace bulk

static int launch_bulk_copy(int device, uint64_t dst, uint64_t src, uint64_t n, cudaStream_t s) {
    static bool configured[64] = {};
    const int smem = bulk::STAGES * (int)bulk::CHUNK;
    if (device < 0 || device >= 64) return DIOMP_BAD_REQUEST;
    if (!configured[device]) {
        DIOMP_CUDA_TRY(cudaFuncSetAttribute(bulk::bulk_copy_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        configured[device] = true;
    }
    const int64_t chunks = ceil_div((int64_t)n, (int64_t)bulk::CHUNK);
    const int ctas = (int)(chunks < bulk::CTAS ? chunks : bulk::CTAS);
    bulk::bulk_copy_kernel<<<ctas, 32, smem, s>>>((char *)dst, (const char *)src, n);
    DIOMP_LAUNCH_CHECK();
    return DIOMP_OK;
}

static int launch_copy(uint64_t dst, uint64_t src, uint64_t n, cudaStream_t s) {
    if (n == 0) return DIOMP_OK;
    if (((dst ^ src) & 15) == 0) {
        uint64_t head = (16 - (dst & 15)) & 15;
        if (head > n) head = n;
        if (head) {
            copy1_kernel<<<1, 32, 0, s>>>((uint8_t *)dst, (const uint8_t *)src, head);
            DIOMP_LAUNCH_CHECK();
        }
        uint64_t body = (n - head) / 16;
        if (body) {
            const int threads = 512;
            const int unroll = 4;
            int64_t want = ceil_div((int64_t)body, (int64_t)threads * unroll);
            int blocks = (int)(want < kNumSMs * 4 ? want : kNumSMs * 4);
            copy16_kernel<unroll><<<blocks, threads, 0, s>>>((uint4 *)(dst + head),
                                                             (const uint4 *)(src + head), body);
            DIOMP_LAUNCH_CHECK();
        }
        uint64_t tail = n - head - body * 16;
        if (tail) {
            uint64_t off = head + body * 16;
            copy1_kernel<<<1, 32, 0, s>>>((uint8_t *)(dst + off), (const uint8_t *)(src + off),
                                          tail);
            DIOMP_LAUNCH_CHECK();
        }
        return DIOMP_OK;
    }
    if (((dst | src) & 7) == 0) {
        uint64_t n8 = n / 8;
        int64_t want = ceil_div((int64_t)n8, 512);
        int blocks = (int)(want < kNumSMs * 4 ? want : kNumSMs * 4);
        if (n8) {
            copy8_kernel<<<blocks, 512, 0, s>>>((uint64_t *)dst, (const uint64_t *)src, n8);
            DIOMP_LAUNCH_CHECK();
        }
        if (n % 8) {
            copy1_kernel<<<1, 32, 0, s>>>((uint8_t *)(dst + n8 * 8),
                                          (const uint8_t *)(src + n8 * 8), n % 8);
            DIOMP_LAUNCH_CHECK();
        }
        return DIOMP_OK;
    }
    int64_t want = ceil_div((int64_t)n, 512);
    int blocks = (int)(want < kNumSMs * 4 ? want : kNumSMs * 4);
    copy1_kernel<<<blocks, 512, 0, s>>>((uint8_t *)dst, (const uint8_t *)src, n);
    DIOMP_LAUNCH_CHECK();
    return DIOMP_OK;
}

// ---------------------------------------------------------------------------
// flags
// ---------------------------------------------------------------------------

__global__ void signal_kernel(uint64_t *flag, uint64_t value) {
    __threadfence_system();
    st_release_sys(flag, value);
}

__global__ void wait_kernel(const uint64_t *flag, uint64_t value) { wait_ge(flag, value); }

// Team barrier: thread q signals position q and waits for q's signal.
__global__ void team_barrier_kernel(diomp_team t) {
    int q = threadIdx.x;
    if (q < t.k && q != t.pos) {
        __threadfence_system();
        uint64_t *remote = (uint64_t *)(t.base[q] + t.flag_off) + t.slot[t.pos];
        st_release_sys(remote, t.epoch_to[q] + 1);
        const uint64_t *mine = (const uint64_t *)(t.base[t.pos] + t.flag_off) + t.slot[q];
        wait_ge(mine, t.epoch_from[q] + 1);
    }
}

}  // namespace diomp

// ===========================================================================
// C ABI
// ===========================================================================
using namespace diomp;

extern "C" {

const char *diomp_status_string(int status) {
    switch (status) {
        case DIOMP_OK: return "ok";
        case DIOMP_INVALID_ADDRESS: return "invalid address";
        case DIOMP_BAD_REQUEST: return "bad request";
        case DIOMP_INTERNAL: return "internal error (device wait timed out)";
        case DIOMP_PENDING: return "pending";
        case DIOMP_OUT_OF_SEGMENT: return "out of segment";
        case DIOMP_DOUBLE_FREE: return "double free";
        default: break;
    }
    if (status >= DIOMP_CUDA_ERROR_BASE) return cudaGetErrorString((cudaError_t)(status - DIOMP_CUDA_ERROR_BASE));
    return "unknown status";
}

int diomp_version(void) { return 10000; }

int diomp_device_count(int *count) {
    DIOMP_CUDA_TRY(cudaGetDeviceCount(count));
    return DIOMP_OK;
}

int diomp_device_sync(int device) {
    DIOMP_CUDA_TRY(cudaSetDevice(device));
    DIOMP_CUDA_TRY(cudaDeviceSynchronize());
    return DIOMP_OK;
}

static unsigned int *g_host_error_word[64] = {};
static std::mutex g_error_word_mu;

static int ensure_error_word(int device) {
    if (device < 0 || device >= 64) return DIOMP_OK;
    std::lock_guard<std::mutex> lk(g_error_word_mu);
    if (g_host_error_word[device]) return DIOMP_OK;
    void *p = nullptr, *dp = nullptr;
    DIOMP_CUDA_TRY(cudaHostAlloc(&p, 64, cudaHostAllocMapped | cudaHostAllocPortable));
    memset(p, 0, 64);
    DIOMP_CUDA_TRY(cudaHostGetDevicePointer(&dp, p, 0));
    DIOMP_CUDA_TRY(cudaMemcpyToSymbol(g_error_word, &dp, sizeof(dp)));
    g_host_error_word[device] = (unsigned int *)p;
    return DIOMP_OK;
}

int diomp_device_error(int device) {
    unsigned int *w = (device >= 0 && device < 64) ? g_host_error_word[device] : nullptr;
    if (w) {  // mapped mirror: no CUDA call unless an error was recorded
        unsigned int err = __atomic_exchange_n(w, 0u, __ATOMIC_ACQ_REL);
        if (!err) return DIOMP_OK;
        unsigned int zero = 0;
        DIOMP_CUDA_TRY(cudaSetDevice(device));
        DIOMP_CUDA_TRY(cudaMemcpyToSymbol(g_device_error, &zero, sizeof(zero)));
        return (int)err;
    }
    DIOMP_CUDA_TRY(cudaSetDevice(device));
    unsigned int err = 0, zero = 0;
    DIOMP_CUDA_TRY(cudaMemcpyFromSymbol(&err, g_device_error, sizeof(err)));
    if (err) DIOMP_CUDA_TRY(cudaMemcpyToSymbol(g_device_error, &zero, sizeof(zero)));
    return err ? (int)err : DIOMP_OK;
}

int diomp_set_wait_timeout(int device, double seconds) {
    DIOMP_CUDA_TRY(cudaSetDevice(device));
    int rc = ensure_error_word(device);
    if (rc) return rc;
    unsigned long long ns = (unsigned long long)(seconds * 1e9);
    DIOMP_CUDA_TRY(cudaMemcpyToSymbol(g_wait_timeout_ns, &ns, sizeof(ns)));
    return DIOMP_OK;
}

// ---- segments ------------------------------------------------------------

int diomp_seg_create(int device, uint64_t bytes, uint64_t *base_out) {
    DIOMP_CUDA_TRY(cudaSetDevice(device));
    void *p = nullptr;
    DIOMP_CUDA_TRY(cudaMalloc(&p, bytes));
    cudaError_t e = cudaMemset(p, 0, bytes);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        cudaFree(p);
        return DIOMP_CUDA_ERROR_BASE + (int)e;
    }
    *base_out = (uint64_t)p;
    return DIOMP_OK;
}

int diomp_seg_destroy(int device, uint64_t base) {
    DIOMP_CUDA_TRY(cudaSetDevice(device));
    DIOMP_CUDA_TRY(cudaDeviceSynchronize());
    DIOMP_CUDA_TRY(cudaFree((void *)base));
    return DIOMP_OK;
}

int diomp_seg_ipc_export(int device, uint64_t base, uint8_t handle_out[64]) {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
    DIOMP_CUDA_TRY(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    DIOMP_CUDA_TRY(cudaIpcGetMemHandle(&h, (void *)base));
    memcpy(handle_out, &h, 64);
    return DIOMP_OK;
}

int diomp_seg_ipc_import(int device, const uint8_t handle[64], uint64_t *base_out) {
    DIOMP_CUDA_TRY(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    void *p = nullptr;
    DIOMP_CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    *base_out = (uint64_t)p;
    return DIOMP_OK;
}

int diomp_seg_ipc_close(int device, uint64_t base) {
    DIOMP_CUDA_TRY(cudaSetDevice(device));
    DIOMP_CUDA_TRY(cudaIpcCloseMemHandle((void *)base));
    return DIOMP_OK;
}

int diomp_peer_enable(int device, int peer_device) {
    if (device == peer_device) return DIOMP_OK;
    DIOMP_CUDA_TRY(cudaSetDevice(device));
    int can = 0;
    DIOMP_CUDA_TRY(cudaDeviceCanAccessPeer(&can, device, peer_device));
    if (!can) return DIOMP_BAD_REQUEST;
    cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return DIOMP_OK;
    }
    DIOMP_CUDA_TRY(e);
    return DIOMP_OK;
}

// ---- streams / events -------------------------------------------------------

int diomp_stream_create(int device, void **stream_out) {
    DIOMP_CUDA_TRY(cudaSetDevice(device));
    cudaStream_t s;
    DIOMP_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    *stream_out = (void *)s;
    return DIOMP_OK;
}

int diomp_stream_destroy(void *stream) {
    DIOMP_CUDA_TRY(cudaStreamDestroy((cudaStream_t)stream));
    return DIOMP_OK;
}

int diomp_stream_sync(void *stream) {
    DIOMP_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    return DIOMP_OK;
}

int diomp_event_create(int device, void **event_out) {
    DIOMP_CUDA_TRY(cudaSetDevice(device));
    cudaEvent_t e;
    DIOMP_CUDA_TRY(cudaEventCreate(&e));
    *event_out = (void *)e;
    return DIOMP_OK;
}

int diomp_event_create_sync(int device, void **event_out) {
    DIOMP_CUDA_TRY(cudaSetDevice(device));
    cudaEvent_t e;
    DIOMP_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    *event_out = (void *)e;
    return DIOMP_OK;
}

int diomp_event_record(void *event, void *stream) {
    DIOMP_CUDA_TRY(cudaEventRecord((cudaEvent_t)event, (cudaStream_t)stream));
    return DIOMP_OK;
}

int diomp_event_query(void *event) {
    cudaError_t e = cudaEventQuery((cudaEvent_t)event);
    if (e == cudaSuccess) return DIOMP_OK;
    if (e == cudaErrorNotReady) {
        cudaGetLastError();
        return DIOMP_PENDING;
    }
    return DIOMP_CUDA_ERROR_BASE + (int)e;
}

int diomp_event_sync(void *event) {
    DIOMP_CUDA_TRY(cudaEventSynchronize((cudaEvent_t)event));
    return DIOMP_OK;
}

int diomp_event_destroy(void *event) {
    DIOMP_CUDA_TRY(cudaEventDestroy((cudaEvent_t)event));
    return DIOMP_OK;
}

int diomp_event_elapsed_ms(void *start, void *stop, float *ms_out) {
    DIOMP_CUDA_TRY(cudaEventElapsedTime(ms_out, (cudaEvent_t)start, (cudaEvent_t)stop));
    return DIOMP_OK;
}

int diomp_stream_wait_event(void *stream, void *event) {
    DIOMP_CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)event, 0));
    return DIOMP_OK;
}

int diomp_stream_query(void *stream) {
    cudaError_t e = cudaStreamQuery((cudaStream_t)stream);
    if (e == cudaSuccess) return DIOMP_OK;
    if (e == cudaErrorNotReady) {
        cudaGetLastError();
        return DIOMP_PENDING;
    }
    return DIOMP_CUDA_ERROR_BASE + (int)e;
}

// ---- data plane ---------------------------------------------------------------

int diomp_copy(int device, uint64_t dst, uint64_t src, uint64_t nbytes, void *stream) {
    DIOMP_CUDA_TRY(cudaSetDevice(device));
    return launch_copy(dst, src, nbytes, (cudaStream_t)stream);
}

// Engine choice for one-sided transfers, from the NVLink probe on B200
// (profiles/r01_nvlink_probe.txt): SM-issued stores to a peer saturate at
// ~715 GB/s whatever the kernel shape (16/32 B vectors, TMA bulk stores), while
// the copy engine reaches 717 / 765 / 779 GB/s at 64 MiB / 256 MiB / 1 GiB and
// is also ahead from 1 MiB; peer reads are fastest through the bulk-async (TMA)
// kernel from 16 MiB (785 GB/s at 1 GiB) and through the SM loop below that.
// Small transfers stay on the SM kernel (lowest issue latency).
// DIOMP_PUT_ENGINE = auto|sm|ce, DIOMP_GET_ENGINE = auto|sm|tma.
// Small transfers (tools/lat_probe.cu on 2 B200, 8 B peer copy, host issue +
// event wait): copy engine 8.55 us (1.3 us to issue) vs 10.7 us (2.6 us) for
// a one-thread SM kernel -- an empty kernel alone is 8.7 us -- so remote
// puts of any size go to the copy engine.  Small remote gets measured the
// other way through the Python API (8 B get+wait 15.3 us on the copy engine
// vs 14.2 on the SM kernel), so they stay on the kernel
// (DIOMP_GET_ENGINE=ce: copy engine up to 64 KiB).
static uint64_t g_put_ce_min = ~0ull, g_get_bulk_min = ~0ull, g_get_ce_max = 0;
static std::once_flag g_engine_once;

static void init_engines() {
    std::call_once(g_engine_once, [] {
        const char *pe = getenv("DIOMP_PUT_ENGINE");
        const char *ge = getenv("DIOMP_GET_ENGINE");
        g_put_ce_min = (pe && !strcmp(pe, "sm")) ? ~0ull : 1;
        g_get_bulk_min = (ge && !strcmp(ge, "sm")) ? ~0ull : (ge && !strcmp(ge, "tma")) ? 16 : (16ull << 20);
        g_get_ce_max = (ge && !strcmp(ge, "ce")) ? (64ull << 10) : 0;
    });
}

static inline int current_device_is(int device) {
    int cur = -1;
    return cudaGetDevice(&cur) == cudaSuccess && cur == device;
}

int diomp_put(int device, uint64_t dst, uint64_t src, uint64_t nbytes, int remote, void *stream) {
    if (nbytes == 0) return DIOMP_OK;
    init_engines();
    if (!current_device_is(device)) DIOMP_CUDA_TRY(cudaSetDevice(device));
    if (remote && nbytes >= g_put_ce_min) {
        DIOMP_CUDA_TRY(cudaMemcpyAsync((void *)dst, (const void *)src, nbytes,
                                       cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
        return DIOMP_OK;
    }
    return launch_copy(dst, src, nbytes, (cudaStream_t)stream);
}

int diomp_get(int device, uint64_t dst, uint64_t src, uint64_t nbytes, int remote, void *stream) {
    if (nbytes == 0) return DIOMP_OK;
    init_engines();
    if (!current_device_is(device)) DIOMP_CUDA_TRY(cudaSetDevice(device));
    cudaStream_t s = (cudaStream_t)stream;
    if (remote && nbytes <= g_get_ce_max) {
        DIOMP_CUDA_TRY(cudaMemcpyAsync((void *)dst, (const void *)src, nbytes,
                                       cudaMemcpyDeviceToDevice, s));
        return DIOMP_OK;
    }
    if (remote && nbytes >= g_get_bulk_min && ((dst ^ src) & 15) == 0) {
        uint64_t head = (16 - (dst & 15)) & 15;
        uint64_t body = (nbytes - head) / 16 * 16;
        uint64_t tail = nbytes - head - body;
        int rc;
        if (head && (rc = launch_copy(dst, src, head, s))) return rc;
        if (body && (rc = launch_bulk_copy(device, dst + head, src + head, body, s))) return rc;
        if (tail && (rc = launch_copy(dst + head + body, src + head + body, tail, s))) return rc;
        return DIOMP_OK;
    }
    return launch_copy(dst, src, nbytes, s);
}

int diomp_memcpy_async(uint64_t dst, uint64_t src, uint64_t nbytes, int kind, void *stream) {
    if (nbytes == 0) return DIOMP_OK;
    cudaMemcpyKind k = kind == DIOMP_H2D   ? cudaMemcpyHostToDevice
                       : kind == DIOMP_D2H ? cudaMemcpyDeviceToHost
                                           : cudaMemcpyDeviceToDevice;
    if (kind != DIOMP_H2D && kind != DIOMP_D2H && kind != DIOMP_D2D) return DIOMP_BAD_REQUEST;
    DIOMP_CUDA_TRY(cudaMemcpyAsync((void *)dst, (const void *)src, nbytes, k, (cudaStream_t)stream));
    return DIOMP_OK;
}

int diomp_memset_async(uint64_t dst, int value, uint64_t nbytes, void *stream) {
    DIOMP_CUDA_TRY(cudaMemsetAsync((void *)dst, value, nbytes, (cudaStream_t)stream));
    return DIOMP_OK;
}

int diomp_memcpy_sync(int device, uint64_t dst, uint64_t src, uint64_t nbytes, int kind) {
    if (nbytes == 0) return DIOMP_OK;
    if (kind != DIOMP_H2D && kind != DIOMP_D2H && kind != DIOMP_D2D) return DIOMP_BAD_REQUEST;
    DIOMP_CUDA_TRY(cudaSetDevice(device));
    DIOMP_CUDA_TRY(cudaDeviceSynchronize());
    DIOMP_CUDA_TRY(cudaMemcpy((void *)dst, (const void *)src, nbytes, cudaMemcpyDefault));
    // A pageable H2D cudaMemcpy may return once the bytes are staged, before
    // the DMA lands; work on other (non-blocking) streams is not ordered
    // after it, so drain the device before reporting the write done.
    DIOMP_CUDA_TRY(cudaDeviceSynchronize());
    return DIOMP_OK;
}

int diomp_signal(int device, uint64_t flag_addr, uint64_t value, void *stream) {
    DIOMP_CUDA_TRY(cudaSetDevice(device));
    signal_kernel<<<1, 1, 0, (cudaStream_t)stream>>>((uint64_t *)flag_addr, value);
    DIOMP_LAUNCH_CHECK();
    return DIOMP_OK;
}

int diomp_wait(int device, uint64_t flag_addr, uint64_t value, void *stream) {
    DIOMP_CUDA_TRY(cudaSetDevice(device));
    wait_kernel<<<1, 1, 0, (cudaStream_t)stream>>>((const uint64_t *)flag_addr, value);
    DIOMP_LAUNCH_CHECK();
    return DIOMP_OK;
}

int diomp_team_barrier(const diomp_team *team, void *stream) {
    if (team->k < 1 || team->k > DIOMP_MAX_TEAM || team->pos < 0 || team->pos >= team->k)
        return DIOMP_BAD_REQUEST;
    if (team->k == 1 || !team->sync) return DIOMP_OK;
    DIOMP_CUDA_TRY(cudaSetDevice(team->device));
    team_barrier_kernel<<<1, 64, 0, (cudaStream_t)stream>>>(*team);
    DIOMP_LAUNCH_CHECK();
    return DIOMP_OK;
}

}  // extern "C"
