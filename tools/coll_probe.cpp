// Collective kernel probe through the C ABI (libdiomp_b200.so), one process,
// K GPUs (peer access), one host thread per GPU -- no Python in the loop.
// Each position enqueues ITERS back-to-back device-synchronised allreduces
// (f32 sum) or bcasts on its own stream; device time = CUDA events around the
// batch, max over positions.  busBW: allreduce 2(K-1)/K*S/t, bcast S/t.
// Results are checked against the exact integer-valued sums.
// g++ -O2 -std=c++20 tools/coll_probe.cpp -o tools/coll_probe.bin \
//     paper_2506_02486_b200/libdiomp_b200.so -Wl,-rpath,'$ORIGIN/../paper_2506_02486_b200'
#include <algorithm>
#include <barrier>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "../include/diomp_b200.h"

#define CK(x) do { int e = (int)(x); if (e) { printf("%s at %d: %d\n", #x, __LINE__, e); exit(1);} } while (0)

int main(int argc, char **argv) {
    int K = 0;
    CK(diomp_device_count(&K));
    const char *op = argc > 1 ? argv[1] : "allreduce";
    if (argc > 2) K = atoi(argv[2]);
    const bool ar = !strcmp(op, "allreduce");
    const uint64_t NMAX = 1ull << 30, SEG = 2 * NMAX + (64ull << 20);
    const uint64_t SEND = 0, RECV = NMAX, FLAG = 2 * NMAX, CNT = FLAG + 512;  // the runtime's scratch layout
    std::vector<uint64_t> base(K);
    std::vector<void *> st(K);
    for (int g = 0; g < K; ++g) {
        CK(diomp_seg_create(g, SEG, &base[g]));
        for (int h = 0; h < K; ++h) if (h != g) CK(diomp_peer_enable(g, h));
        CK(diomp_stream_create(g, &st[g]));
        std::vector<float> host(1 << 22);  // pattern repeats every 4 Mi elements
        for (size_t i = 0; i < host.size(); ++i) host[i] = (float)((i % 13) + 3 * g);
        for (uint64_t o = 0; o < NMAX; o += host.size() * 4)
            CK(diomp_memcpy_sync(g, base[g] + SEND + o, (uint64_t)host.data(), host.size() * 4, DIOMP_H2D));
    }
    std::vector<diomp_team> team(K);
    for (int p = 0; p < K; ++p) {
        diomp_team &t = team[p];
        memset(&t, 0, sizeof t);
        t.k = K; t.pos = p; t.device = p; t.sync = getenv("NOSYNC") ? 0 : 1;
        t.flag_off = FLAG; t.counter_off = CNT;
        for (int q = 0; q < K; ++q) { t.base[q] = base[q]; t.slot[q] = q; }
    }
    const int per = 1;   // one entry handshake per call; the exit is a team barrier
    std::vector<uint64_t> sizes;
    for (uint64_t s = 1 << 20; s <= NMAX; s <<= 2) sizes.push_back(s);
    std::barrier bar(K);
    std::vector<float> ms(K);
    std::vector<std::thread> th;
    printf("# %s K=%d sync=%d\n", op, K, team[0].sync);
    for (int p = 0; p < K; ++p) th.emplace_back([&, p] {
        void *a, *b;
        CK(diomp_event_create(p, &a)); CK(diomp_event_create(p, &b));
        diomp_team &t = team[p];
        auto once = [&](uint64_t bytes) {
            if (ar) CK(diomp_allreduce(&t, SEND, RECV, bytes / 4, DIOMP_F32, DIOMP_SUM, st[p]));
            else CK(diomp_bcast(&t, SEND, bytes, 0, st[p]));
            for (int q = 0; q < K; ++q) if (q != p) { t.epoch_to[q] += per; t.epoch_from[q] += per; }
        };
        auto exit_barrier = [&]() {
            if (!t.sync) return;
            CK(diomp_team_barrier(&t, st[p]));
            for (int q = 0; q < K; ++q) if (q != p) { t.epoch_to[q] += 1; t.epoch_from[q] += 1; }
        };
        for (uint64_t bytes : sizes) {
            const int iters = bytes >= (256ull << 20) ? 10 : 50;
            for (int w = 0; w < 3; ++w) once(bytes);
            exit_barrier();
            CK(diomp_stream_sync(st[p]));
            bar.arrive_and_wait();
            CK(diomp_event_record(a, st[p]));
            for (int i = 0; i < iters; ++i) once(bytes);
            exit_barrier();
            CK(diomp_event_record(b, st[p]));
            CK(diomp_event_sync(b));
            float m; CK(diomp_event_elapsed_ms(a, b, &m));
            ms[p] = m / iters;
            CK(diomp_device_error(p));
            bar.arrive_and_wait();
            if (p == 0) {
                float mx = *std::max_element(ms.begin(), ms.end());
                double bw = (ar ? 2.0 * (K - 1) / K : 1.0) * bytes / (mx * 1e-3) / 1e9;
                printf("%-9s %6llu KiB  %9.2f us  busBW %6.1f GB/s\n", op, (unsigned long long)(bytes >> 10), mx * 1e3, bw);
                fflush(stdout);
            }
            bar.arrive_and_wait();
        }
        // check the last (largest) result on this GPU
        std::vector<float> h(1 << 20);
        uint64_t off = ar ? RECV : SEND;
        uint64_t n = sizes.back() / 4;
        unsigned long long bad = 0;
        for (uint64_t i0 = 0; i0 < n; i0 += (n / 7)) {
            uint64_t cnt = std::min<uint64_t>(h.size(), n - i0);
            CK(diomp_memcpy_sync(p, (uint64_t)h.data(), base[p] + off + i0 * 4, cnt * 4, DIOMP_D2H));
            for (uint64_t j = 0; j < cnt; ++j) {
                uint64_t i = i0 + j;
                float want = 0;
                const uint64_t r = (i & ((1u << 22) - 1)) % 13;
                if (ar) for (int g = 0; g < K; ++g) want += (float)(r + 3 * g);
                else want = (float)r;
                if (h[j] != want) ++bad;
            }
        }
        if (bad) printf("position %d: %llu wrong values\n", p, bad);
    });
    for (auto &x : th) x.join();
    printf("done\n");
    return 0;
}
