// NVLS multicast probe (one process, all visible GPUs): bind one physical
// buffer per GPU to a multicast object, store from GPU 0 through the
// multicast address (multimem.st) and measure the fan-out rate; verify every
// GPU received the bytes.  Compared with SM peer stores to each GPU in turn.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/nvls_probe.bin tools/nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
#define CU(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char *s; cuGetErrorString(r, &s); \
    printf("CU %s at %d: %s\n", #x, __LINE__, s); exit(1);} } while (0)

__global__ void __launch_bounds__(512) mc_store(float4 *mc, const float4 *src, uint64_t n16) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
        float4 v = src[i];
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + i),
                     "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                     : "memory");
    }
}

__global__ void __launch_bounds__(512) uc_store(float4 *dst, const float4 *src, uint64_t n16) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) dst[i] = src[i];
}

__global__ void __launch_bounds__(512) mc_ldreduce(float4 *dst, const float4 *mc, uint64_t n16) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
        float4 v;
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                     : "l"(mc + i)
                     : "memory");
        dst[i] = v;
    }
}

int main() {
    CU(cuInit(0));
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (ndev < 2) { printf("need >= 2 GPUs\n"); return 1; }
    const size_t want = 1ull << 30;
    CUmulticastObjectProp mp = {};
    mp.numDevices = ndev;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = want;
    size_t gran = 0, rgran = 0;
    CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
    CU(cuMulticastGetGranularity(&rgran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    const size_t size = (want + rgran - 1) / rgran * rgran;
    mp.size = size;
    printf("multicast granularity min %zu recommended %zu, size %zu, devices %d\n", gran, rgran, size, ndev);
    CUmemGenericAllocationHandle mc;
    CU(cuMulticastCreate(&mc, &mp));
    for (int d = 0; d < ndev; ++d) {
        CUdevice dev;
        CU(cuDeviceGet(&dev, d));
        CU(cuMulticastAddDevice(mc, dev));
    }
    std::vector<CUmemGenericAllocationHandle> phys(ndev);
    std::vector<CUdeviceptr> uc(ndev);
    for (int d = 0; d < ndev; ++d) {
        CK(cudaSetDevice(d));
        CUmemAllocationProp p = {};
        p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        p.location.id = d;
        p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
        size_t pg = 0;
        CU(cuMemGetAllocationGranularity(&pg, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
        CU(cuMemCreate(&phys[d], size, &p, 0));
        CU(cuMulticastBindMem(mc, 0, phys[d], 0, size, 0));
        CU(cuMemAddressReserve(&uc[d], size, pg, 0, 0));
        CU(cuMemMap(uc[d], size, 0, phys[d], 0));
        std::vector<CUmemAccessDesc> ads(ndev);
        for (int e = 0; e < ndev; ++e) {
            ads[e] = {};
            ads[e].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
            ads[e].location.id = e;
            ads[e].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        }
        CU(cuMemSetAccess(uc[d], size, ads.data(), ndev));
        CK(cudaMemset((void *)uc[d], 0, size));
    }
    // multicast VA, mapped for device 0
    CK(cudaSetDevice(0));
    CUdeviceptr mva;
    CU(cuMemAddressReserve(&mva, size, rgran, 0, 0));
    CU(cuMemMap(mva, size, 0, mc, 0));
    CUmemAccessDesc ad = {};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = 0;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CU(cuMemSetAccess(mva, size, &ad, 1));
    // peer access for the unicast comparison
    for (int d = 1; d < ndev; ++d) cudaDeviceEnablePeerAccess(d, 0);
    cudaGetLastError();
    float *src;
    CK(cudaMalloc(&src, want));
    std::vector<float> h(want / 4);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)(i % 1000003);
    CK(cudaMemcpy(src, h.data(), want, cudaMemcpyHostToDevice));
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (size_t n : {64ull << 20, 256ull << 20, 1ull << 30}) {
        for (int blocks : {148, 296, 592}) {
            const uint64_t n16 = n / 16;
            mc_store<<<blocks, 512, 0, st>>>((float4 *)mva, (const float4 *)src, n16);
            CK(cudaStreamSynchronize(st));
            CK(cudaEventRecord(a, st));
            const int it = 10;
            for (int i = 0; i < it; ++i) mc_store<<<blocks, 512, 0, st>>>((float4 *)mva, (const float4 *)src, n16);
            CK(cudaEventRecord(b, st));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            printf("mc_store   %5zu MiB blocks %3d: %7.1f GB/s (root egress), each of %d GPUs receives it\n",
                   n >> 20, blocks, n * it / (ms * 1e-3) / 1e9, ndev);
        }
        // unicast: store to each peer in turn (what a P2P bcast root would need)
        const uint64_t n16 = n / 16;
        CK(cudaEventRecord(a, st));
        for (int d = 1; d < ndev; ++d)
            uc_store<<<592, 512, 0, st>>>((float4 *)uc[d], (const float4 *)src, n16);
        CK(cudaEventRecord(b, st));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        printf("uc_store   %5zu MiB to %d peers in turn: %7.1f GB/s per peer-copy\n", n >> 20, ndev - 1,
               n * (ndev - 1) / (ms * 1e-3) / 1e9);
        CK(cudaEventRecord(a, st));
        for (int i = 0; i < 10; ++i)
            mc_ldreduce<<<592, 512, 0, st>>>((float4 *)src, (const float4 *)mva, n16);
        CK(cudaEventRecord(b, st));
        CK(cudaEventSynchronize(b));
        CK(cudaEventElapsedTime(&ms, a, b));
        printf("ld_reduce  %5zu MiB: %7.1f GB/s of reduced output\n", n >> 20, n * 10 / (ms * 1e-3) / 1e9);
        CK(cudaMemcpy(src, h.data(), want, cudaMemcpyHostToDevice));
    }
    // verify: every GPU's physical buffer holds src (last mc_store wrote 1 GiB)
    mc_store<<<592, 512, 0, st>>>((float4 *)mva, (const float4 *)src, want / 16);
    CK(cudaStreamSynchronize(st));
    int bad = 0;
    std::vector<float> back(want / 4);
    for (int d = 0; d < ndev; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaMemcpy(back.data(), (void *)uc[d], want, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < back.size(); i += 4099)
            if (back[i] != h[i]) { ++bad; break; }
    }
    printf("verify: %s\n", bad ? "MISMATCH" : "all GPUs hold the root's bytes");
    return bad ? 1 : 0;
}
