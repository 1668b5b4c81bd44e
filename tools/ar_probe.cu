// Allreduce engine probe (K GPUs, one process, one host thread per GPU).
// f32 sum, block p = [p*n/K, (p+1)*n/K) folded by position p (the reference's
// reduce-scatter order) and delivered to every member.  Variants:
//   sm        : the library's fused kernel shape -- SM loads of the block from
//               every peer, fold, SM stores to every member
//   ce CH     : copy engines only on NVLink: per chunk, K-1 CE gets of the
//               peers' block chunk into local scratch (one stream per peer),
//               a local fold kernel (HBM), K-1 CE pushes of the result
//   smce CH   : SM-load fold straight from the peers into the own recv chunk,
//               CE pushes of the result (one stream per peer), pipelined
// Times: all threads released by a barrier, each enqueues + syncs its GPU;
// op time = max over threads; busBW = 2(K-1)/K * bytes / t.
// nvcc -O3 -std=c++20 -gencode arch=compute_100a,code=sm_100a -o tools/ar_probe.bin tools/ar_probe.cu
#include <algorithm>
#include <barrier>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int KM = 8;
struct Ptrs { const float *src[KM]; float *dst[KM]; };

// fused SM allreduce block: fold positions p, p+1, ... ; store to all dst
template <int KMAX>
__global__ void __launch_bounds__(512) sm_fused(Ptrs P, int k, int p, uint64_t lo4, uint64_t n4, int ndst) {
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, gs = (uint64_t)gridDim.x * blockDim.x;
    constexpr int U = KMAX <= 4 ? 2 : 1;
    for (uint64_t v0 = g; v0 < n4; v0 += gs * U) {
        float4 b[U][KMAX];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint64_t v = v0 + u * gs;
            if (v < n4)
#pragma unroll
                for (int i = 0; i < KMAX; ++i)
                    if (i < k) { int q = p + i; if (q >= k) q -= k; b[u][i] = reinterpret_cast<const float4 *>(P.src[q])[lo4 + v]; }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint64_t v = v0 + u * gs;
            if (v >= n4) break;
            float4 a = b[u][0];
#pragma unroll
            for (int i = 1; i < KMAX; ++i)
                if (i < k) { a.x = __fadd_rn(a.x, b[u][i].x); a.y = __fadd_rn(a.y, b[u][i].y); a.z = __fadd_rn(a.z, b[u][i].z); a.w = __fadd_rn(a.w, b[u][i].w); }
            for (int i = 0; i < ndst; ++i) { int q = p + i; if (q >= k) q -= k; reinterpret_cast<float4 *>(P.dst[q])[lo4 + v] = a; }
        }
    }
}

int K = 2;
std::vector<float *> sendb, recvb, scratch;
std::vector<cudaStream_t> smain;
std::vector<std::vector<cudaStream_t>> sget, spush;
std::vector<std::vector<cudaEvent_t>> evpool;

struct Var { const char *name; int kind; uint64_t ch; int nslot; };

static void enqueue(int p, const Var &v, uint64_t n /*floats*/) {
    CK(cudaSetDevice(p));
    const uint64_t lo = (uint64_t)p * n / K, hi = (uint64_t)(p + 1) * n / K;
    cudaStream_t s = smain[p];
    Ptrs P{};
    for (int q = 0; q < K; ++q) { P.src[q] = sendb[q]; P.dst[q] = recvb[q]; }
    if (v.kind == 0) {
        uint64_t n4 = (hi - lo) / 4;
        int grid = 148 * 4;
        if (K <= 2) sm_fused<2><<<grid, 512, 0, s>>>(P, K, p, lo / 4, n4, K);
        else if (K <= 4) sm_fused<4><<<grid, 512, 0, s>>>(P, K, p, lo / 4, n4, K);
        else sm_fused<8><<<grid, 512, 0, s>>>(P, K, p, lo / 4, n4, K);
        return;
    }
    auto &ev = evpool[p];
    size_t e = 0;
    auto nev = [&]() { return ev[e++]; };
    cudaEvent_t start = nev();
    CK(cudaEventRecord(start, s));
    const uint64_t chf = v.ch / 4;
    std::vector<cudaEvent_t> fold_done(v.nslot, nullptr);
    uint64_t c = 0;
    std::vector<cudaEvent_t> push_done;
    for (uint64_t off = lo; off < hi; off += chf, ++c) {
        const uint64_t len = std::min(chf, hi - off);
        const int slot = c % v.nslot;
        Ptrs F{};
        if (v.kind == 1) {
            // CE gets into scratch[slot][i]
            std::vector<cudaEvent_t> got;
            for (int i = 1; i < K; ++i) {
                int q = (p + i) % K;
                cudaStream_t g = sget[p][i];
                CK(cudaStreamWaitEvent(g, fold_done[slot] ? fold_done[slot] : start, 0));
                float *dst = scratch[p] + ((uint64_t)slot * (K - 1) + (i - 1)) * chf;
                CK(cudaMemcpyAsync(dst, sendb[q] + off, len * 4, cudaMemcpyDeviceToDevice, g));
                cudaEvent_t x = nev(); CK(cudaEventRecord(x, g)); got.push_back(x);
            }
            for (auto x : got) CK(cudaStreamWaitEvent(s, x, 0));
            F.src[0] = sendb[p] + off;
            for (int i = 1; i < K; ++i) F.src[i] = scratch[p] + ((uint64_t)slot * (K - 1) + (i - 1)) * chf;
            F.dst[0] = recvb[p] + off;
            // fold positions in ring order starting at p: src[i] = position p+i
            if (K <= 2) sm_fused<2><<<148 * 2, 512, 0, s>>>(F, K, 0, 0, len / 4, 1);
            else if (K <= 4) sm_fused<4><<<148 * 2, 512, 0, s>>>(F, K, 0, 0, len / 4, 1);
            else sm_fused<8><<<148 * 2, 512, 0, s>>>(F, K, 0, 0, len / 4, 1);
        } else {
            for (int i = 0; i < K; ++i) { int q = (p + i) % K; F.src[i] = sendb[q] + off; }
            F.dst[0] = recvb[p] + off;
            if (K <= 2) sm_fused<2><<<148 * 4, 512, 0, s>>>(F, K, 0, 0, len / 4, 1);
            else if (K <= 4) sm_fused<4><<<148 * 4, 512, 0, s>>>(F, K, 0, 0, len / 4, 1);
            else sm_fused<8><<<148 * 4, 512, 0, s>>>(F, K, 0, 0, len / 4, 1);
        }
        cudaEvent_t fd = nev(); CK(cudaEventRecord(fd, s));
        fold_done[slot] = fd;
        for (int i = 1; i < K; ++i) {
            int q = (p + i) % K;
            cudaStream_t ps = spush[p][i];
            CK(cudaStreamWaitEvent(ps, fd, 0));
            CK(cudaMemcpyAsync(recvb[q] + off, recvb[p] + off, len * 4, cudaMemcpyDeviceToDevice, ps));
        }
    }
    for (int i = 1; i < K; ++i) { cudaEvent_t x = nev(); CK(cudaEventRecord(x, spush[p][i])); CK(cudaStreamWaitEvent(s, x, 0)); }
    if (v.kind == 1) for (int i = 1; i < K; ++i) { cudaEvent_t x = nev(); CK(cudaEventRecord(x, sget[p][i])); CK(cudaStreamWaitEvent(s, x, 0)); }
    if (e > ev.size()) { printf("event pool overflow\n"); exit(1); }
}

__global__ void fill(float *d, uint64_t n, int g) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        d[i] = (float)((i % 13) + 3 * g);
}
__global__ void check(const float *d, uint64_t n, int K, unsigned long long *bad) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        float want = 0; for (int g = 0; g < K; ++g) want += (float)((i % 13) + 3 * g);
        if (d[i] != want) atomicAdd(bad, 1ull);
    }
}

int main(int argc, char **argv) {
    CK(cudaGetDeviceCount(&K));
    if (argc > 1) K = atoi(argv[1]);
    const uint64_t NMAX = 1ull << 30;
    sendb.resize(K); recvb.resize(K); scratch.resize(K); smain.resize(K); sget.resize(K); spush.resize(K); evpool.resize(K);
    for (int g = 0; g < K; ++g) {
        CK(cudaSetDevice(g));
        for (int h = 0; h < K; ++h) if (h != g) CK(cudaDeviceEnablePeerAccess(h, 0));
        CK(cudaMalloc(&sendb[g], NMAX)); CK(cudaMalloc(&recvb[g], NMAX));
        CK(cudaMalloc(&scratch[g], 4ull * (K - 1) * (64ull << 20)));
        CK(cudaStreamCreateWithFlags(&smain[g], cudaStreamNonBlocking));
        sget[g].resize(K); spush[g].resize(K);
        for (int i = 0; i < K; ++i) { CK(cudaStreamCreateWithFlags(&sget[g][i], cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&spush[g][i], cudaStreamNonBlocking)); }
        evpool[g].resize(20000);
        for (auto &x : evpool[g]) CK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
        fill<<<1184, 512>>>(sendb[g], NMAX / 4, g);
        CK(cudaDeviceSynchronize());
    }
    std::vector<Var> vars = {{"sm", 0, 0, 0}};
    for (uint64_t ch : {2ull << 20, 4ull << 20, 8ull << 20, 16ull << 20, 32ull << 20})
        { vars.push_back({"ce", 1, ch, 3}); vars.push_back({"smce", 2, ch, 3}); }
    std::vector<uint64_t> sizes = {16ull << 20, 64ull << 20, 256ull << 20, 1ull << 30};
    std::barrier bar(K + 1);
    std::vector<double> tsec(K);
    const Var *cur = nullptr; uint64_t curn = 0; int reps = 0; bool quit = false;
    std::vector<std::thread> th;
    for (int p = 0; p < K; ++p) th.emplace_back([&, p] {
        CK(cudaSetDevice(p));
        for (;;) {
            bar.arrive_and_wait();
            if (quit) return;
            double best = 1e30;
            for (int r = 0; r < reps; ++r) {
                bar.arrive_and_wait();  // common release per rep
                auto t0 = std::chrono::steady_clock::now();
                enqueue(p, *cur, curn);
                CK(cudaStreamSynchronize(smain[p]));
                tsec[p] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                bar.arrive_and_wait();  // done; main reads tsec
            }
            (void)best;
            bar.arrive_and_wait();
        }
    });
    printf("# K=%d  busBW GB/s (median over reps), host-timed per op incl. enqueue\n", K);
    for (auto &v : vars) {
        for (uint64_t bytes : sizes) {
            if (v.kind && v.ch * K > bytes * 2 && bytes > (64ull << 20)) {}
            cur = &v; curn = bytes / 4; reps = bytes >= (256ull << 20) ? 8 : 20;
            for (int g = 0; g < K; ++g) { CK(cudaSetDevice(g)); CK(cudaMemset(recvb[g], 0, bytes)); CK(cudaDeviceSynchronize()); }
            bar.arrive_and_wait();
            std::vector<double> ts;
            for (int r = 0; r < reps; ++r) {
                bar.arrive_and_wait();
                bar.arrive_and_wait();
                double m = 0; for (int p = 0; p < K; ++p) m = std::max(m, tsec[p]);
                ts.push_back(m);
            }
            bar.arrive_and_wait();
            std::sort(ts.begin(), ts.end());
            double t = ts[ts.size() / 2];
            unsigned long long bad = 0, *dbad;
            for (int g = 0; g < K; ++g) {
                CK(cudaSetDevice(g)); CK(cudaMalloc(&dbad, 8)); CK(cudaMemset(dbad, 0, 8));
                check<<<1184, 512>>>(recvb[g], bytes / 4, K, dbad);
                unsigned long long h; CK(cudaMemcpy(&h, dbad, 8, cudaMemcpyDeviceToHost)); bad += h; CK(cudaFree(dbad));
            }
            printf("%-5s ch=%3llu MiB  %5llu MiB  %8.1f us  busBW %6.1f GB/s  min %6.1f  %s\n", v.name,
                   (unsigned long long)(v.ch >> 20), (unsigned long long)(bytes >> 20), t * 1e6,
                   2.0 * (K - 1) / K * bytes / t / 1e9, 2.0 * (K - 1) / K * bytes / ts[0] / 1e9, bad ? "BAD" : "ok");
            fflush(stdout);
        }
    }
    quit = true;
    bar.arrive_and_wait();
    for (auto &t : th) t.join();
    return 0;
}
