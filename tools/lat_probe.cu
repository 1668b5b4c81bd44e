// Small-transfer latency probe (2 GPUs, or 1): host-visible cost of issuing an
// 8-byte peer put and waiting for its completion, per mechanism.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/lat_probe.cu -o tools/lat_probe.bin
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void copy8(unsigned long long *d, const unsigned long long *s) { *d = *s; }
__global__ void empty_k() {}
// completion published to pinned host memory: the host spins on it instead of
// an event / stream synchronisation
__global__ void copy8_flag(unsigned long long *d, const unsigned long long *s,
                           volatile unsigned long long *hflag, unsigned long long v) {
    *d = *s;
    __threadfence_system();
    *hflag = v;
}
__global__ void flag_only(volatile unsigned long long *hflag, unsigned long long v) { *hflag = v; }

using clk = std::chrono::steady_clock;
static double us_since(clk::time_point t0) {
    return std::chrono::duration<double, std::micro>(clk::now() - t0).count();
}

int main() {
    int n = 0;
    cudaGetDeviceCount(&n);
    int ga = 0, gb = n > 1 ? 1 : 0;
    unsigned long long *a, *b;
    cudaSetDevice(gb);
    cudaMalloc(&b, 1 << 20);
    cudaSetDevice(ga);
    if (ga != gb) cudaDeviceEnablePeerAccess(gb, 0);
    cudaMalloc(&a, 1 << 20);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    unsigned long long *hflag;
    cudaHostAlloc(&hflag, 64, cudaHostAllocMapped | cudaHostAllocPortable);
    *hflag = 0;
    unsigned long long *dflag;
    cudaHostGetDevicePointer(&dflag, hflag, 0);
    volatile unsigned long long *vf = hflag;
    unsigned long long seq = 0;
    // a one-node graph of copy8_flag (graph launch instead of a kernel launch)
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    copy8_flag<<<1, 1, 0, s>>>(b, a, dflag, 0);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    const int N = 2000;
    for (int mode = 0; mode < 10; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            double issue = 0, total = 0;
            for (int i = 0; i < N; ++i) {
                auto t0 = clk::now();
                switch (mode) {
                    case 0: copy8<<<1, 1, 0, s>>>(b, a); cudaEventRecord(ev, s); break;
                    case 1: cudaMemcpyAsync(b, a, 8, cudaMemcpyDeviceToDevice, s); cudaEventRecord(ev, s); break;
                    case 2: cudaMemcpyPeerAsync(b, gb, a, ga, 8, s); cudaEventRecord(ev, s); break;
                    case 3: empty_k<<<1, 1, 0, s>>>(); cudaEventRecord(ev, s); break;
                    case 4: copy8<<<1, 1, 0, s>>>(b, a); break;
                    case 5: copy8<<<1, 32, 0, s>>>(b, a); cudaEventRecord(ev, s); break;
                    case 6: cudaEventRecord(ev, s); break;
                    case 7: copy8_flag<<<1, 1, 0, s>>>(b, a, dflag, ++seq); break;
                    case 8: flag_only<<<1, 1, 0, s>>>(dflag, ++seq); break;
                    case 9: cudaGraphLaunch(ge, s); break;
                }
                issue += us_since(t0);
                if (mode == 4) cudaStreamSynchronize(s);
                else if (mode == 7 || mode == 8) { while (*vf != seq) {} }
                else if (mode == 9) cudaStreamSynchronize(s);
                else cudaEventSynchronize(ev);
                total += us_since(t0);
            }
            if (rep == 1)
                printf("mode %d %-34s issue %6.2f us  issue+wait %6.2f us\n", mode,
                       (const char *[]){"kernel+event, event sync", "memcpyAsync D2D + event",
                                        "memcpyPeerAsync + event", "empty kernel + event",
                                        "kernel, stream sync", "kernel 32 thr + event",
                                        "event only", "kernel + host-flag spin",
                                        "flag-only kernel + host spin", "graph launch, stream sync"}[mode],
                       issue / N, total / N);
        }
    }
    return 0;
}
