// bcast over the copy engines, k GPUs in one process (peer access), root 0:
// non-root i pulls block i-1 (of k-1) from the root chunk by chunk and pushes
// every pulled chunk on to the other non-roots -- the pull+push schedule of
// bcast_kernel with cudaMemcpyPeerAsync instead of SM loads/stores.  Prints
// busBW = S / t per (size, chunks, push streams).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/bcast_ce_probe.cu -o tools/bcast_ce_probe.bin
#include <atomic>
#include <chrono>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void gate_kernel(volatile int *flag) {
    while (*flag == 0) {
    }
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

int main(int argc, char **argv) {
    setvbuf(stdout, nullptr, _IOLBF, 0);
    int k = 0;
    CK(cudaGetDeviceCount(&k));
    if (argc > 1) k = atoi(argv[1]);
    if (k < 3) { printf("need >= 3 GPUs\n"); return 0; }
    const size_t maxS = 1ull << 30;
    std::vector<char *> buf(k);
    std::vector<cudaStream_t> pull(k), push(k), push2(k);
    const int MAXC = 64;
    std::vector<std::vector<cudaEvent_t>> ev(k, std::vector<cudaEvent_t>(MAXC));
    for (int d = 0; d < k; ++d) {
        CK(cudaSetDevice(d));
        for (int p = 0; p < k; ++p)
            if (p != d) CK(cudaDeviceEnablePeerAccess(p, 0));
        CK(cudaMalloc(&buf[d], maxS));
        CK(cudaMemset(buf[d], d, maxS));
        CK(cudaStreamCreateWithFlags(&pull[d], cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&push[d], cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&push2[d], cudaStreamNonBlocking));
        for (int c = 0; c < MAXC; ++c) CK(cudaEventCreateWithFlags(&ev[d][c], cudaEventDisableTiming));
    }
    auto sync_all = [&] {
        for (int d = 0; d < k; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
    };
    // mode 0: pull+push, pushes on one stream; 1: one push stream per destination
    // (two streams); 2: root pushes everything (baseline); 3: non-roots pull everything
    auto run = [&](size_t S, int C, int mode) {
        const size_t blk = S / (k - 1);
        if (mode == 2) {
            CK(cudaSetDevice(0));
            for (int q = 1; q < k; ++q)
                CK(cudaMemcpyPeerAsync(buf[q], q, buf[0], 0, S, q % 2 ? push[0] : push2[0]));
            return;
        }
        if (mode == 3) {
            for (int q = 1; q < k; ++q) {
                CK(cudaSetDevice(q));
                CK(cudaMemcpyPeerAsync(buf[q], q, buf[0], 0, S, pull[q]));
            }
            return;
        }
        for (int i = 1; i < k; ++i) {
            CK(cudaSetDevice(i));
            const size_t off0 = (size_t)(i - 1) * blk;
            const size_t len = (i == k - 1) ? S - off0 : blk;
            for (int c = 0; c < C; ++c) {
                const size_t a = off0 + len * c / C, b = off0 + len * (c + 1) / C;
                CK(cudaMemcpyPeerAsync(buf[i] + a, i, buf[0] + a, 0, b - a, pull[i]));
                CK(cudaEventRecord(ev[i][c], pull[i]));
                CK(cudaStreamWaitEvent(push[i], ev[i][c], 0));
                if (mode == 1) CK(cudaStreamWaitEvent(push2[i], ev[i][c], 0));
                int n = 0;
                for (int q = 1; q < k; ++q) {
                    if (q == i) continue;
                    cudaStream_t s = (mode == 1 && (n++ & 1)) ? push2[i] : push[i];
                    CK(cudaMemcpyPeerAsync(buf[q] + a, q, buf[i] + a, i, b - a, s));
                }
            }
        }
    };
    // all reps are enqueued behind a gate (a kernel spinning on a pinned host
    // flag, every stream waits for it), then released: the wall clock sees
    // the copies, not the host's enqueue rate
    int *hflag, *dflag;
    CK(cudaHostAlloc(&hflag, 64, cudaHostAllocMapped | cudaHostAllocPortable));
    CK(cudaHostGetDevicePointer(&dflag, hflag, 0));
    cudaStream_t gs;
    cudaEvent_t gev;
    CK(cudaSetDevice(0));
    CK(cudaStreamCreateWithFlags(&gs, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&gev, cudaEventDisableTiming));
    auto gate = [&] {
        *(volatile int *)hflag = 0;
        CK(cudaSetDevice(0));
        gate_kernel<<<1, 1, 0, gs>>>(dflag);
        CK(cudaEventRecord(gev, gs));
        for (int d = 0; d < k; ++d) {
            CK(cudaSetDevice(d));
            for (cudaStream_t s : {pull[d], push[d], push2[d]}) CK(cudaStreamWaitEvent(s, gev, 0));
        }
    };
    using clk = std::chrono::steady_clock;
    printf("# k=%d  busBW = S/t GB/s (wall clock over reps, all devices synchronised)\n", k);
    for (size_t S : {64ull << 20, 256ull << 20, 1ull << 30}) {
        for (int mode : {0, 1, 2, 3}) {
            for (int C : {1, 2, 4, 8, 16, 32}) {
                if (mode >= 2 && C > 1) continue;
                // bounded so the gated queues stay short (a full stream queue would block
                // the host before it releases the gate)
                // (measured: ~100+ queued entries per stream block the host)
                int reps = S >= (1ull << 30) ? 4 : 24;
                if (reps * C > 24) reps = C >= 24 ? 1 : 24 / C;
                run(S, C, mode);
                sync_all();
                gate();
                // watchdog: if an enqueue blocks (full stream queue behind the
                // gate), release the gate anyway after 2 s and flag the row
                std::atomic<int> enq{0};
                std::atomic<bool> fired{false};
                std::thread wd([&] {
                    for (int i = 0; i < 2000 && !enq.load(); ++i)
                        std::this_thread::sleep_for(std::chrono::milliseconds(1));
                    if (!enq.load()) { fired = true; *(volatile int *)hflag = 1; }
                });
                for (int r = 0; r < reps; ++r) run(S, C, mode);
                auto t0 = clk::now();
                enq = 1;
                *(volatile int *)hflag = 1;
                wd.join();
                sync_all();
                if (fired) printf("(watchdog released the gate: host enqueue blocked)\n");
                const double t = std::chrono::duration<double>(clk::now() - t0).count() / reps;
                printf("S=%5zu MiB mode=%d (%s) chunks=%2d  %.1f us  busBW %.1f GB/s\n", S >> 20, mode,
                       (const char *[]){"pull+push 1 stream", "pull+push 2 streams", "root push all",
                                        "pull all from root"}[mode],
                       C, t * 1e6, S / t / 1e9);
            }
        }
    }
    // correctness of mode 0 at 1 GiB, 16 chunks
    {
        CK(cudaSetDevice(0));
        std::vector<unsigned char> h(maxS);
        for (size_t i = 0; i < maxS; ++i) h[i] = (unsigned char)(i * 2654435761u >> 24);
        CK(cudaMemcpy(buf[0], h.data(), maxS, cudaMemcpyHostToDevice));
        for (int d = 1; d < k; ++d) { CK(cudaSetDevice(d)); CK(cudaMemset(buf[d], 0, maxS)); }
        sync_all();
        run(maxS, 16, 0);
        sync_all();
        std::vector<unsigned char> g(maxS);
        int bad = 0;
        for (int d = 1; d < k; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaMemcpy(g.data(), buf[d], maxS, cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < maxS; ++i) if (g[i] != h[i]) { ++bad; break; }
        }
        printf("check 1 GiB pull+push: %s\n", bad ? "MISMATCH" : "byte-exact on every non-root");
    }
    return 0;
}
