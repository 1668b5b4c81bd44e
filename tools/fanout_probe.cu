// Root fan-out probe (K GPUs, one process): how fast can GPU 0's data leave
// it when the other K-1 GPUs each need a third of it?
//   readers : K-1 GPUs each load S/(K-1) from GPU 0 (SM loads, concurrent)
//   writer  : GPU 0 stores S/(K-1) into each of the K-1 GPUs (SM stores)
//   ce-push : GPU 0 copy-engine pushes S/(K-1) to each (one stream per peer)
//   ce-pull : each of the K-1 GPUs copy-engine pulls S/(K-1) from GPU 0
// Rate = S / t (the root's egress).  Host-timed over back-to-back reps.
// nvcc -O3 -std=c++20 -gencode arch=compute_100a,code=sm_100a -o tools/fanout_probe.bin tools/fanout_probe.cu
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void __launch_bounds__(512) copy16(uint4 *__restrict__ dst, const uint4 *__restrict__ src, uint64_t n) {
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * gs < n; i += 4 * gs) {
        uint4 a = src[i], b = src[i + gs], c = src[i + 2 * gs], d = src[i + 3 * gs];
        dst[i] = a; dst[i + gs] = b; dst[i + 2 * gs] = c; dst[i + 3 * gs] = d;
    }
    for (; i < n; i += gs) dst[i] = src[i];
}

// root writer: one launch, block j of the grid range goes to destination j
struct Dst { uint4 *d[8]; };
__global__ void __launch_bounds__(512) fan_store(Dst D, const uint4 *__restrict__ src, uint64_t per, int nd) {
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < per * nd; i += gs) {
        const int j = (int)(i / per);
        D.d[j][i - j * per] = src[i];
    }
}

// bcast data patterns on non-root p (no flags, timing only), block j = p-1:
//   mode 0 (library today): pull block j from the root, push it to the other non-roots
//   mode 1 (pull-only):     pull block j from the root, pull every other block b from non-root b
//   mode 2 (push-only):     the root stores block j into non-root j; non-root j stores its
//                           (local) block into the other non-roots
struct Team { char *b[8]; };
__global__ void __launch_bounds__(512) bc_pattern(Team T, int k, int p, uint64_t per16, int mode) {
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int j = p - 1;
    if (mode == 0) {
        const uint4 *src = (const uint4 *)T.b[0] + j * per16;
        for (uint64_t i = g; i < per16; i += gs) {
            uint4 v = src[i];
            for (int q = 1; q < k; ++q) ((uint4 *)T.b[q])[j * per16 + i] = v;
        }
    } else if (mode == 3) {  // chain: position p stores the whole buffer into p+1
        const uint64_t n = per16 * (k - 1);
        if (p + 1 < k)
            for (uint64_t i = g; i < n; i += gs) ((uint4 *)T.b[p + 1])[i] = ((const uint4 *)T.b[p])[i];
    } else if (mode == 2) {
        const uint4 *src = (const uint4 *)T.b[p] + j * per16;
        for (uint64_t i = g; i < per16; i += gs) {
            uint4 v = src[i];
            for (int q = 1; q < k; ++q) if (q != p) ((uint4 *)T.b[q])[j * per16 + i] = v;
        }
    } else {
        // CTA slices: 1/(k-1) of the grid for the own block, the rest for peer blocks
        const uint64_t items = per16 * (k - 1);
        for (uint64_t i = g; i < items; i += gs) {
            const int bi = (int)(i / per16);          // block index 0..k-2
            const uint64_t e = i - bi * per16;
            const int srcpos = bi == j ? 0 : bi + 1;  // own block from the root, others from their owner
            ((uint4 *)T.b[p])[bi * per16 + e] = ((const uint4 *)T.b[srcpos])[bi * per16 + e];
        }
    }
}

int main(int argc, char **argv) {
    int K; CK(cudaGetDeviceCount(&K));
    const uint64_t S = 1ull << 30;
    std::vector<char *> buf(K);
    std::vector<std::vector<cudaStream_t>> st(K);
    for (int g = 0; g < K; ++g) {
        CK(cudaSetDevice(g));
        for (int h = 0; h < K; ++h) if (h != g) CK(cudaDeviceEnablePeerAccess(h, 0));
        CK(cudaMalloc(&buf[g], S));
        CK(cudaMemset(buf[g], g, S));
        st[g].resize(K);
        for (auto &s : st[g]) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    }
    for (uint64_t sz : {64ull << 20, 256ull << 20, 1ull << 30}) {
        if (getenv("SKIP_FANOUT")) break;
        const uint64_t per = sz / (K - 1) / 16 * 16;
        for (int v = 0; v < 4; ++v) {
            for (int ctas : {296, 592}) {
                if (v >= 2 && ctas == 592) continue;
                auto run = [&] {
                    if (v == 0) for (int g = 1; g < K; ++g) { CK(cudaSetDevice(g));
                        copy16<<<ctas, 512, 0, st[g][0]>>>((uint4 *)buf[g], (const uint4 *)(buf[0] + (g - 1) * per), per / 16); }
                    if (v == 1) { CK(cudaSetDevice(0)); Dst D{}; for (int g = 1; g < K; ++g) D.d[g - 1] = (uint4 *)(buf[g] + (g - 1) * per);
                        fan_store<<<ctas, 512, 0, st[0][0]>>>(D, (const uint4 *)buf[0], per / 16, K - 1); }
                    if (v == 2) { CK(cudaSetDevice(0)); for (int g = 1; g < K; ++g)
                        CK(cudaMemcpyAsync(buf[g] + (g - 1) * per, buf[0] + (g - 1) * per, per, cudaMemcpyDeviceToDevice, st[0][g])); }
                    if (v == 3) for (int g = 1; g < K; ++g) { CK(cudaSetDevice(g));
                        CK(cudaMemcpyAsync(buf[g] + (g - 1) * per, buf[0] + (g - 1) * per, per, cudaMemcpyDeviceToDevice, st[g][0])); }
                };
                auto sync = [&] { for (int g = 0; g < K; ++g) { CK(cudaSetDevice(g)); for (auto &s : st[g]) CK(cudaStreamSynchronize(s)); } };
                run(); sync();
                const int reps = sz >= (256ull << 20) ? 10 : 30;
                auto t0 = std::chrono::steady_clock::now();
                for (int r = 0; r < reps; ++r) run();
                sync();
                double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / reps;
                const char *nm[] = {"readers", "writer", "ce-push", "ce-pull"};
                printf("K=%d %-8s ctas=%3d %5llu MiB  root egress %6.1f GB/s\n", K, nm[v], v < 2 ? ctas : 0,
                       (unsigned long long)(sz >> 20), (double)per * (K - 1) / t / 1e9);
                fflush(stdout);
            }
        }
    }
    for (uint64_t sz : {64ull << 20, 256ull << 20, 1ull << 30}) {
        const uint64_t per = sz / (K - 1) / 16 * 16;
        Team T{}; for (int g = 0; g < K; ++g) T.b[g] = buf[g];
        for (int mode = 0; mode < 4; ++mode) for (int ctas : {296, 592}) {
            if (mode == 2 || (ctas == 296 && !getenv("ALL_CTAS"))) continue;
            auto run = [&] {
                if (mode == 2) { CK(cudaSetDevice(0)); Dst D{}; for (int g = 1; g < K; ++g) D.d[g - 1] = (uint4 *)(buf[g] + (g - 1) * per);
                    fan_store<<<ctas, 512, 0, st[0][0]>>>(D, (const uint4 *)buf[0], per / 16, K - 1); }
                for (int g = mode == 3 ? 0 : 1; g < K; ++g) { CK(cudaSetDevice(g));
                bc_pattern<<<ctas, 512, 0, st[g][0]>>>(T, K, g, per / 16, mode); } };
            auto sync = [&] { for (int g = 0; g < K; ++g) { CK(cudaSetDevice(g)); CK(cudaDeviceSynchronize()); } };
            run(); sync();
            const int reps = sz >= (256ull << 20) ? 10 : 30;
            auto t0 = std::chrono::steady_clock::now();
            for (int r = 0; r < reps; ++r) run();
            sync();
            double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / reps;
            printf("K=%d bcast-pattern %-9s ctas=%3d %5llu MiB  S/t %6.1f GB/s\n", K, mode == 3 ? "chain" : mode == 2 ? "push-only" : mode ? "pull-only" : "pull+push",
                   ctas, (unsigned long long)(sz >> 20), (double)per * (K - 1) / t / 1e9);
            fflush(stdout);
        }
    }
    // copy-engine bcast pattern, all dependencies local: non-root j gets its
    // block from the root chunk by chunk (stream 0) and, per chunk, pushes it to
    // the other non-roots (one stream per destination) after an event
    if (K >= 3) {
        std::vector<std::vector<cudaEvent_t>> ev(K);
        for (int g = 1; g < K; ++g) { CK(cudaSetDevice(g)); ev[g].resize(64);
            for (auto &evx : ev[g]) CK(cudaEventCreateWithFlags(&evx, cudaEventDisableTiming)); }
        for (uint64_t sz : {64ull << 20, 256ull << 20, 1ull << 30}) {
            const uint64_t per = sz / (K - 1) / 16 * 16;
            for (uint64_t ch : {8ull << 20, 16ull << 20, 32ull << 20, 64ull << 20}) {
                auto run = [&] {
                    for (int g = 1; g < K; ++g) {
                        CK(cudaSetDevice(g));
                        const uint64_t base = (g - 1) * per;
                        int c = 0;
                        for (uint64_t o = 0; o < per; o += ch, ++c) {
                            const uint64_t len = std::min(ch, per - o);
                            CK(cudaMemcpyAsync(buf[g] + base + o, buf[0] + base + o, len, cudaMemcpyDeviceToDevice, st[g][0]));
                            CK(cudaEventRecord(ev[g][c % 64], st[g][0]));
                            for (int q = 1; q < K; ++q) if (q != g) {
                                CK(cudaStreamWaitEvent(st[g][q], ev[g][c % 64], 0));
                                CK(cudaMemcpyAsync(buf[q] + base + o, buf[g] + base + o, len, cudaMemcpyDeviceToDevice, st[g][q]));
                            }
                        }
                    }
                };
                auto sync = [&] { for (int g = 0; g < K; ++g) { CK(cudaSetDevice(g)); CK(cudaDeviceSynchronize()); } };
                run(); sync();
                const int reps = sz >= (256ull << 20) ? 10 : 30;
                auto t0 = std::chrono::steady_clock::now();
                for (int r = 0; r < reps; ++r) run();
                sync();
                double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / reps;
                printf("K=%d bcast-pattern ce-get+ce-push chunk=%2llu MiB %5llu MiB  S/t %6.1f GB/s\n", K,
                       (unsigned long long)(ch >> 20), (unsigned long long)(sz >> 20), (double)per * (K - 1) / t / 1e9);
                fflush(stdout);
            }
        }
    }
    return 0;
}
