// NVLink one-sided copy probe (2 GPUs, one process, peer access).
// Compares the put/get kernel shapes the runtime could use:
//   sm-store  : kernel on the source GPU, 16 B loads local, 16 B stores remote (put)
//   sm-load   : kernel on the destination GPU, 16 B loads remote (get)
//   tma-store : cp.async.bulk HBM->smem, cp.async.bulk smem->remote (put)
//   ce        : cudaMemcpyPeerAsync (copy engine)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gpurun_out/nvlink_probe tools/nvlink_probe.cu
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <int U>
__global__ void __launch_bounds__(1024) copy16(uint4 *__restrict__ dst, const uint4 *__restrict__ src,
                                               uint64_t n16) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n16; i += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = src[i + u * stride];
#pragma unroll
        for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
    }
    for (; i < n16; i += stride) dst[i] = src[i];
}

// Contiguous-chunk variant: each CTA owns a contiguous range; warps move 16 B x U per lane.
template <int U>
__global__ void __launch_bounds__(1024) copy16_chunk(uint4 *__restrict__ dst,
                                                     const uint4 *__restrict__ src, uint64_t n16) {
    uint64_t per = (n16 + gridDim.x - 1) / gridDim.x;
    uint64_t b = blockIdx.x * per, e = b + per < n16 ? b + per : n16;
    const uint64_t step = (uint64_t)blockDim.x * U;
    uint64_t i = b + threadIdx.x;
    for (; i + (U - 1) * blockDim.x < e; i += step) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = src[i + u * blockDim.x];
#pragma unroll
        for (int u = 0; u < U; ++u) dst[i + u * blockDim.x] = v[u];
    }
    for (; i < e; i += blockDim.x) dst[i] = src[i];
}

template <int U, int MODE>
__global__ void __launch_bounds__(1024) copy32(uint4 *__restrict__ dst, const uint4 *__restrict__ src,
                                               uint64_t n32) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i < n32; i += stride) {
        const char *s = (const char *)src + i * 32;
        char *d = (char *)dst + i * 32;
        uint32_t r[8];
        asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "l"(s));
        if (MODE == 0)
            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(d), "r"(r[0]), "r"(r[1]), "r"(r[2]),
                         "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
        else
            asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(d), "r"(r[0]), "r"(r[1]), "r"(r[2]),
                         "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// TMA bulk copy: one elected thread per CTA drives a ring of S stages of C bytes.
template <int S>
__global__ void __launch_bounds__(32) tma_copy(char *__restrict__ dst, const char *__restrict__ src,
                                               uint64_t n, uint32_t chunk) {
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t full[S];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < S; ++s)
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    uint64_t nchunks = (n + chunk - 1) / chunk;
    uint32_t phase[S];
    for (int s = 0; s < S; ++s) phase[s] = 0;
    uint64_t c0 = blockIdx.x;
    // prologue: issue up to S loads
    int issued = 0;
    for (uint64_t c = c0; c < nchunks && issued < S; c += gridDim.x, ++issued) {
        uint32_t bytes = (uint32_t)((c + 1) * chunk <= n ? chunk : n - c * chunk);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&full[issued])),
                     "r"(bytes));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(sm + (size_t)issued * chunk)),
            "l"(src + c * chunk), "r"(bytes), "r"(smem_u32(&full[issued]))
            : "memory");
    }
    int s = 0;
    uint64_t cl = c0 + (uint64_t)issued * gridDim.x;  // next chunk to load
    for (uint64_t c = c0; c < nchunks; c += gridDim.x) {
        uint32_t bytes = (uint32_t)((c + 1) * chunk <= n ? chunk : n - c * chunk);
        // wait full[s]
        asm volatile(
            "{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" ::"r"(
                smem_u32(&full[s])),
            "r"(phase[s]));
        phase[s] ^= 1;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * chunk),
                     "r"(smem_u32(sm + (size_t)s * chunk)), "r"(bytes)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        if (cl < nchunks) {
            // slot s is reused: wait until its store has read smem (allow S-1 outstanding)
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            uint32_t b2 = (uint32_t)((cl + 1) * chunk <= n ? chunk : n - cl * chunk);
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                         "r"(b2));
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(sm + (size_t)s * chunk)),
                "l"(src + cl * chunk), "r"(b2), "r"(smem_u32(&full[s]))
                : "memory");
            cl += gridDim.x;
        }
        s = (s + 1) % S;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static float time_it(int dev, cudaStream_t st, int iters, void (*fn)(void *), void *arg) {
    CK(cudaSetDevice(dev));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int i = 0; i < 3; ++i) fn(arg);
    CK(cudaStreamSynchronize(st));
    CK(cudaEventRecord(a, st));
    for (int i = 0; i < iters; ++i) fn(arg);
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms / iters;
}

struct Args {
    char *dst, *src;
    uint64_t n;
    int blocks, threads, kind, u;
    uint32_t chunk;
    int stages;
    cudaStream_t st, st2;
    cudaEvent_t ev;
    int srcdev, dstdev;
};

static void run(void *p) {
    Args *a = (Args *)p;
    uint64_t n16 = a->n / 16;
    switch (a->kind) {
    case 0:
        if (a->u == 4) copy16<4><<<a->blocks, a->threads, 0, a->st>>>((uint4 *)a->dst, (uint4 *)a->src, n16);
        else if (a->u == 8) copy16<8><<<a->blocks, a->threads, 0, a->st>>>((uint4 *)a->dst, (uint4 *)a->src, n16);
        else copy16<2><<<a->blocks, a->threads, 0, a->st>>>((uint4 *)a->dst, (uint4 *)a->src, n16);
        break;
    case 1:
        if (a->u == 4) copy16_chunk<4><<<a->blocks, a->threads, 0, a->st>>>((uint4 *)a->dst, (uint4 *)a->src, n16);
        else copy16_chunk<8><<<a->blocks, a->threads, 0, a->st>>>((uint4 *)a->dst, (uint4 *)a->src, n16);
        break;
    case 2: {
        size_t smem = (size_t)a->stages * a->chunk;
        if (a->stages == 4) tma_copy<4><<<a->blocks, 32, smem, a->st>>>(a->dst, a->src, a->n, a->chunk);
        else tma_copy<8><<<a->blocks, 32, smem, a->st>>>(a->dst, a->src, a->n, a->chunk);
        break;
    }
    case 4:
        copy32<1, 0><<<a->blocks, a->threads, 0, a->st>>>((uint4 *)a->dst, (uint4 *)a->src, a->n / 32);
        break;
    case 5:
        copy32<1, 1><<<a->blocks, a->threads, 0, a->st>>>((uint4 *)a->dst, (uint4 *)a->src, a->n / 32);
        break;
    case 6: {  // CE for 3/4, SM for 1/4 on a second stream
        uint64_t h = a->n / 4 * 3 / 16 * 16;
        CK(cudaMemcpyPeerAsync(a->dst, a->dstdev, a->src, a->srcdev, h, a->st));
        copy16<4><<<a->blocks, a->threads, 0, a->st2>>>((uint4 *)(a->dst + h), (uint4 *)(a->src + h), (a->n - h) / 16);
        cudaEventRecord(a->ev, a->st2);
        cudaStreamWaitEvent(a->st, a->ev, 0);
        break;
    }
    case 3:
        CK(cudaMemcpyPeerAsync(a->dst, a->dstdev, a->src, a->srcdev, a->n, a->st));
        break;
    }
}

int main(int argc, char **argv) {
    int ndev;
    CK(cudaGetDeviceCount(&ndev));
    if (ndev < 2) { printf("need 2 GPUs\n"); return 1; }
    const uint64_t maxn = 1ull << 30;
    char *buf[2][2];
    cudaStream_t st[2], st2[2];
    cudaEvent_t ev[2];
    for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceEnablePeerAccess(1 - d, 0));
        CK(cudaMalloc(&buf[d][0], maxn));
        CK(cudaMalloc(&buf[d][1], maxn));
        CK(cudaMemset(buf[d][0], d + 1, maxn));
        CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&st2[d], cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ev[d], cudaEventDisableTiming));
        CK(cudaFuncSetAttribute(tma_copy<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CK(cudaFuncSetAttribute(tma_copy<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    }
    CK(cudaDeviceSynchronize());
    uint64_t sizes[] = {1ull << 20, 8ull << 20, 64ull << 20, 256ull << 20, 1ull << 30};
    struct V { const char *name; int kind, side, blocks, threads, u; uint32_t chunk; int stages; } vs[] = {
        {"put sm 592x512 u4", 0, 0, 592, 512, 4, 0, 0},
        {"put ce", 3, 0, 0, 0, 0, 0, 0},
        {"get sm 592x512 u4", 0, 1, 592, 512, 4, 0, 0},
        {"get tma 148 x 4x32K", 2, 1, 148, 32, 0, 32768, 4},
    };
    printf("{\"probe\": \"nvlink\", \"rows\": [\n");
    bool first = true;
    for (auto &v : vs) {
        for (uint64_t n : sizes) {
            Args a;
            a.n = n; a.blocks = v.blocks; a.threads = v.threads; a.kind = v.kind; a.u = v.u;
            a.chunk = v.chunk; a.stages = v.stages;
            int launch;
            if (v.side == 0) {        // put: launched on GPU0, src GPU0, dst GPU1
                launch = 0; a.src = buf[0][0]; a.dst = buf[1][1]; a.srcdev = 0; a.dstdev = 1;
            } else if (v.side == 1) { // get: launched on GPU1, src GPU0, dst GPU1
                launch = 1; a.src = buf[0][0]; a.dst = buf[1][1]; a.srcdev = 0; a.dstdev = 1;
            } else {
                launch = 0; a.src = buf[0][0]; a.dst = buf[0][1]; a.srcdev = 0; a.dstdev = 0;
            }
            a.st = st[launch]; a.st2 = st2[launch]; a.ev = ev[launch];
            int iters = n >= (256ull << 20) ? 10 : 50;
            float ms = time_it(launch, a.st, iters, run, &a);
            CK(cudaGetLastError());
            double gbs = n / (ms * 1e-3) / 1e9;
            printf("%s{\"v\": \"%s\", \"bytes\": %llu, \"us\": %.2f, \"GBps\": %.1f}", first ? "" : ",\n",
                   v.name, (unsigned long long)n, ms * 1e3, gbs);
            first = false;
        }
    }
    printf("\n]}\n");
    // bidirectional: both GPUs move n bytes toward each other at once (host-timed)
    struct B { const char *name; int kind, mode, blocks, threads, u; uint32_t chunk; int stages; } bs[] = {
        {"bidir put sm", 0, 0, 592, 512, 4, 0, 0},
        {"bidir put ce", 3, 0, 0, 0, 0, 0, 0},
        {"bidir get sm", 0, 1, 592, 512, 4, 0, 0},
        {"bidir get tma", 2, 1, 148, 32, 0, 32768, 4},
        {"bidir get ce", 3, 1, 0, 0, 0, 0, 0},
        {"bidir put ce + get tma", 9, 2, 148, 32, 0, 32768, 4},
    };
    uint64_t bsz[] = {64ull << 20, 256ull << 20, 1ull << 30};
    for (auto &b : bs) {
        for (uint64_t n : bsz) {
            Args a[2];
            for (int g = 0; g < 2; ++g) {
                Args &x = a[g];
                x.n = n; x.blocks = b.blocks; x.threads = b.threads; x.u = b.u; x.chunk = b.chunk; x.stages = b.stages;
                x.kind = b.kind;
                int o = 1 - g;
                if (b.mode == 0 || (b.mode == 2 && g == 0)) {  // put from g to o
                    if (b.mode == 2) x.kind = 3;
                    x.src = buf[g][0]; x.dst = buf[o][1]; x.srcdev = g; x.dstdev = o;
                } else {  // get on g from o
                    if (b.mode == 2) x.kind = 2;
                    x.src = buf[o][0]; x.dst = buf[g][1]; x.srcdev = o; x.dstdev = g;
                }
                x.st = st[g]; x.st2 = st2[g]; x.ev = ev[g];
            }
            int iters = n >= (256ull << 20) ? 10 : 40;
            for (int w = 0; w < 2; ++w) for (int g = 0; g < 2; ++g) { CK(cudaSetDevice(g)); run(&a[g]); }
            for (int g = 0; g < 2; ++g) { CK(cudaSetDevice(g)); CK(cudaStreamSynchronize(st[g])); }
            auto t0 = std::chrono::steady_clock::now();
            for (int i = 0; i < iters; ++i) for (int g = 0; g < 2; ++g) { CK(cudaSetDevice(g)); run(&a[g]); }
            for (int g = 0; g < 2; ++g) { CK(cudaSetDevice(g)); CK(cudaStreamSynchronize(st[g])); }
            double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / iters;
            printf("BIDIR %-26s %6llu MiB  %.1f GB/s per direction\n", b.name, (unsigned long long)(n >> 20), n / sec / 1e9);
        }
    }
    // verify last put byte pattern once
    CK(cudaSetDevice(0));
    Args a{buf[1][1], buf[0][0], 1ull << 20, 592, 512, 0, 4, 0, 0, st[0], st2[0], ev[0], 0, 1};
    CK(cudaMemset(buf[1][1], 0, 1 << 20));
    CK(cudaDeviceSynchronize());
    a.kind = 2; a.blocks = 148; a.chunk = 16384; a.stages = 8;
    run(&a);
    CK(cudaStreamSynchronize(st[0]));
    unsigned char h[16];
    CK(cudaMemcpy(h, buf[1][1] + (1 << 20) - 16, 16, cudaMemcpyDeviceToHost));
    printf("verify tma tail byte = %d (want 1)\n", h[15]);
    return 0;
}
