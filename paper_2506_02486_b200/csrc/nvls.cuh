// NVSwitch multicast (NVLS) allreduce window (sm_100a).
//
// Reference: collectives.allreduce (collectives.py:326-405).  The exact
// allreduce (collectives.cuh) folds every block in the reference's ring order
// and is bit-identical to it.  This is the in-switch alternative: each member
// binds a window of its own HBM to one multicast object; position p reduces
// block p of the window with multimem.ld_reduce (the NVSwitch adds the k
// members' values) and writes the sum back to every member with one
// multimem.st -- per GPU the links carry about S + S/k each way instead of
// the ring's 2(k-1)/k S, and the SMs issue one load and one store per 16 B
// instead of k of each.  The switch's summation order is not the reference's,
// so float sums agree within rounding (tested at rel-L2 <= 1e-6 f32 /
// 1e-12 f64, the north-star tolerance); integer sum / min / max are exact.
//
// One call = rounds of up to `window` bytes:
//   K1 copy the round's send bytes into the own window (local HBM); the last
//      CTA adds 1 to flag F1 on every member (multimem.red.release);
//   K2 wait F1 == k*epoch; ld_reduce / st block p of the round through the
//      multicast address; the last CTA adds 1 to F2 on every member;
//   K3 wait F2 == k*epoch; copy the window into the round's recv bytes.
// A member's window is read (ld_reduce) and written (st) by its peers only
// between F1 and F2 of a round, so the next round's K1 (after this member's
// K3) never races them.  Flags are monotone u64 counters in the window header.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <mutex>
#include <type_traits>

#include "common.cuh"

namespace diomp {
namespace nvls {

constexpr int THREADS = 512;
constexpr uint64_t HEADER = 2ull << 20;  // flags page(s) ahead of the data window
constexpr uint64_t F1_OFF = 0, F2_OFF = 128;

struct Driver {
    PFN_cuMulticastCreate_v12010 create = nullptr;
    PFN_cuMulticastAddDevice_v12010 add_device = nullptr;
    PFN_cuMulticastBindMem_v12010 bind_mem = nullptr;
    PFN_cuMulticastUnbind_v12010 unbind = nullptr;
    PFN_cuMulticastGetGranularity_v12010 granularity = nullptr;
    PFN_cuMemCreate_v10020 mem_create = nullptr;
    PFN_cuMemRelease_v10020 mem_release = nullptr;
    PFN_cuMemAddressReserve_v10020 reserve = nullptr;
    PFN_cuMemAddressFree_v10020 addr_free = nullptr;
    PFN_cuMemMap_v10020 map = nullptr;
    PFN_cuMemUnmap_v10020 unmap = nullptr;
    PFN_cuMemSetAccess_v10020 set_access = nullptr;
    PFN_cuMemExportToShareableHandle_v10020 export_handle = nullptr;
    PFN_cuMemImportFromShareableHandle_v10020 import_handle = nullptr;
    PFN_cuDeviceGetAttribute_v2000 get_attr = nullptr;
    PFN_cuDeviceGet_v2000 device_get = nullptr;
    bool ok = false;
};

static const Driver &drv() {
    static Driver d;
    static std::once_flag once;
    std::call_once(once, [] {
        auto get = [](const char *name, void **out) {
            cudaDriverEntryPointQueryResult q;
            return cudaGetDriverEntryPoint(name, out, cudaEnableDefault, &q) == cudaSuccess &&
                   q == cudaDriverEntryPointSuccess;
        };
        bool ok = true;
        ok &= get("cuMulticastCreate", (void **)&d.create);
        ok &= get("cuMulticastAddDevice", (void **)&d.add_device);
        ok &= get("cuMulticastBindMem", (void **)&d.bind_mem);
        ok &= get("cuMulticastUnbind", (void **)&d.unbind);
        ok &= get("cuMulticastGetGranularity", (void **)&d.granularity);
        ok &= get("cuMemCreate", (void **)&d.mem_create);
        ok &= get("cuMemRelease", (void **)&d.mem_release);
        ok &= get("cuMemAddressReserve", (void **)&d.reserve);
        ok &= get("cuMemAddressFree", (void **)&d.addr_free);
        ok &= get("cuMemMap", (void **)&d.map);
        ok &= get("cuMemUnmap", (void **)&d.unmap);
        ok &= get("cuMemSetAccess", (void **)&d.set_access);
        ok &= get("cuMemExportToShareableHandle", (void **)&d.export_handle);
        ok &= get("cuMemImportFromShareableHandle", (void **)&d.import_handle);
        ok &= get("cuDeviceGetAttribute", (void **)&d.get_attr);
        ok &= get("cuDeviceGet", (void **)&d.device_get);
        d.ok = ok;
    });
    return d;
}

// driver-API failures: status DIOMP_CUDA_ERROR_BASE + 900 + CUresult, and the
// failing call on stderr (these run once per window, at setup / teardown)
#define DIOMP_CU_TRY(expr)                                                        \
    do {                                                                          \
        CUresult _r = (expr);                                                     \
        if (_r != CUDA_SUCCESS) {                                                 \
            fprintf(stderr, "diomp nvls: %s failed: CUresult %d\n", #expr, (int)_r); \
            return DIOMP_CUDA_ERROR_BASE + 900 + (int)_r;                         \
        }                                                                         \
    } while (0)

// ---- device helpers ----------------------------------------------------------

__device__ __forceinline__ void mc_signal(uint64_t *mc_flag) {
    asm volatile("multimem.red.release.sys.global.add.u64 [%0], %1;" ::"l"(mc_flag), "l"(1ull)
                 : "memory");
}

// thread 0 of every CTA waits until the local copy of the flag reaches target
__device__ __forceinline__ void cta_wait_flag(const uint64_t *uc_flag, uint64_t target) {
    if (threadIdx.x == 0) {
        wait_ge(uc_flag, target);
        asm volatile("fence.proxy.alias;" ::: "memory");
    }
    __syncthreads();
}

// all CTAs done (system fence per CTA), then the last one bumps the flag on
// every member through the multicast address
__device__ __forceinline__ void grid_signal(unsigned int *counter, uint64_t *mc_flag) {
    if (last_cta_done(counter, gridDim.x) && threadIdx.x == 0) {
        asm volatile("fence.proxy.alias;" ::: "memory");
        mc_signal(mc_flag);
    }
}

struct Args {
    uint64_t uc;        // own window (unicast VA), header first
    uint64_t mc;        // multicast VA of the window
    uint64_t src, dst;  // the round's send / recv bytes (own GPU)
    uint64_t bytes;     // round length (bytes, multiple of the element size)
    uint64_t count;     // round length (elements)
    int32_t k, pos;
    int32_t dtype, op;
    uint64_t target;    // k * epoch
    unsigned int *counter;
};

__global__ void __launch_bounds__(THREADS) copy_in_kernel(const __grid_constant__ Args a) {
    const uint4 *s = (const uint4 *)a.src;
    uint4 *d = (uint4 *)(a.uc + HEADER);
    const uint64_t n16 = a.bytes / 16;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) d[i] = s[i];
    const uint64_t rem = a.bytes - n16 * 16;
    if (blockIdx.x == 0 && threadIdx.x < rem)
        ((uint8_t *)d)[n16 * 16 + threadIdx.x] = ((const uint8_t *)s)[n16 * 16 + threadIdx.x];
    grid_signal(a.counter, (uint64_t *)(a.mc + F1_OFF));
}

__global__ void __launch_bounds__(THREADS) copy_out_kernel(const __grid_constant__ Args a) {
    cta_wait_flag((const uint64_t *)(a.uc + F2_OFF), a.target);
    const uint4 *s = (const uint4 *)(a.uc + HEADER);
    uint4 *d = (uint4 *)a.dst;
    const uint64_t n16 = a.bytes / 16;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) d[i] = s[i];
    const uint64_t rem = a.bytes - n16 * 16;
    if (blockIdx.x == 0 && threadIdx.x < rem)
        ((uint8_t *)d)[n16 * 16 + threadIdx.x] = ((const uint8_t *)s)[n16 * 16 + threadIdx.x];
}

template <typename T, int OP>
__device__ __forceinline__ T ld_reduce(const T *p);

#define DIOMP_LDRED(T, OPN, PTX, REG)                                                          \
    template <>                                                                                \
    __device__ __forceinline__ T ld_reduce<T, OPN>(const T *p) {                               \
        T v;                                                                                   \
        asm volatile("multimem.ld_reduce.relaxed.sys.global." PTX " %0, [%1];"                 \
                     : "=" REG(v)                                                              \
                     : "l"(p)                                                                  \
                     : "memory");                                                              \
        return v;                                                                              \
    }
DIOMP_LDRED(float, 0, "add.f32", "f")
DIOMP_LDRED(double, 0, "add.f64", "d")
DIOMP_LDRED(int32_t, 0, "add.s32", "r")
DIOMP_LDRED(int32_t, 1, "min.s32", "r")
DIOMP_LDRED(int32_t, 2, "max.s32", "r")
DIOMP_LDRED(long long, 0, "add.u64", "l")
DIOMP_LDRED(long long, 1, "min.s64", "l")
DIOMP_LDRED(long long, 2, "max.s64", "l")
#undef DIOMP_LDRED

__device__ __forceinline__ void mc_store(float *p, float v) {
    asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void mc_store(double *p, double v) {
    asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void mc_store(int32_t *p, int32_t v) {
    asm volatile("multimem.st.relaxed.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void mc_store(long long *p, long long v) {
    asm volatile("multimem.st.relaxed.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Block p of the round: element range [lo, hi).  f32 sums move 16 B per
// instruction (ld_reduce / st .v4.f32) on the 16-byte aligned interior; the
// other types are scalar (the only multimem vector forms are f32 / f16 / bf16).
template <typename T, int OP>
__global__ void __launch_bounds__(THREADS) reduce_kernel(const __grid_constant__ Args a) {
    cta_wait_flag((const uint64_t *)(a.uc + F1_OFF), a.target);
    const uint64_t lo = (uint64_t)a.pos * a.count / a.k, hi = (uint64_t)(a.pos + 1) * a.count / a.k;
    T *mc = (T *)(a.mc + HEADER);
    const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t gsz = (uint64_t)gridDim.x * blockDim.x;
    uint64_t vlo = hi, vhi = hi;
    if constexpr (std::is_same<T, float>::value && OP == 0) {
        vlo = (lo + 3) / 4 * 4;
        if (vlo > hi) vlo = hi;
        vhi = vlo + (hi - vlo) / 4 * 4;
        float4 *m4 = (float4 *)(a.mc + HEADER) + vlo / 4;
        const uint64_t n4 = (vhi - vlo) / 4;
        for (uint64_t i = gtid; i < n4; i += gsz) {
            float4 v;
            asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "l"(m4 + i)
                         : "memory");
            asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(m4 + i),
                         "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                         : "memory");
        }
    }
    const uint64_t nhead = vlo - lo, ntail = hi - vhi;
    for (uint64_t j = gtid; j < nhead + ntail; j += gsz) {
        const uint64_t e = j < nhead ? lo + j : vhi + (j - nhead);
        mc_store(mc + e, ld_reduce<T, OP>(mc + e));
    }
    grid_signal(a.counter, (uint64_t *)(a.mc + F2_OFF));
}

static int grid_for(uint64_t items) {
    int64_t want = ceil_div((int64_t)items, THREADS);
    if (want < 1) want = 1;
    if (want > kNumSMs * 4) want = kNumSMs * 4;
    return (int)want;
}

template <typename T, int OP>
static int launch_round(const Args &a, cudaStream_t s) {
    const int gc = grid_for(a.bytes / 16 + 1);
    copy_in_kernel<<<gc, THREADS, 0, s>>>(a);
    DIOMP_LAUNCH_CHECK();
    const uint64_t per = a.count / a.k + 1;
    const int gr = grid_for(std::is_same<T, float>::value && OP == 0 ? per / 4 + 1 : per);
    reduce_kernel<T, OP><<<gr, THREADS, 0, s>>>(a);
    DIOMP_LAUNCH_CHECK();
    copy_out_kernel<<<gc, THREADS, 0, s>>>(a);
    DIOMP_LAUNCH_CHECK();
    return DIOMP_OK;
}

}  // namespace nvls
}  // namespace diomp

extern "C" {

int diomp_mc_supported(int device, int *out) {
    using namespace diomp::nvls;
    *out = 0;
    const Driver &d = drv();
    if (!d.ok) return DIOMP_OK;
    CUdevice dev;
    DIOMP_CU_TRY(d.device_get(&dev, device));
    int v = 0;
    DIOMP_CU_TRY(d.get_attr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    *out = v;
    return DIOMP_OK;
}

// Window bytes (data, excluding the header) rounded so header + data is a
// multiple of the multicast granularity.
int diomp_mc_window_bytes(int nmembers, uint64_t want, uint64_t *total_out) {
    using namespace diomp::nvls;
    const Driver &d = drv();
    if (!d.ok) return DIOMP_BAD_REQUEST;
    CUmulticastObjectProp mp = {};
    mp.numDevices = (unsigned)nmembers;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = HEADER + want;
    size_t gran = 0;
    DIOMP_CU_TRY(d.granularity(&gran, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
    *total_out = (HEADER + want + gran - 1) / gran * gran;
    return DIOMP_OK;
}

int diomp_mc_create(int nmembers, uint64_t total, int *fd_out, uint64_t *mc_out) {
    using namespace diomp::nvls;
    const Driver &d = drv();
    if (!d.ok) return DIOMP_BAD_REQUEST;
    CUmulticastObjectProp mp = {};
    mp.numDevices = (unsigned)nmembers;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = total;
    CUmemGenericAllocationHandle h;
    DIOMP_CU_TRY(d.create(&h, &mp));
    int fd = -1;
    DIOMP_CU_TRY(d.export_handle(&fd, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
    *fd_out = fd;
    *mc_out = (uint64_t)h;
    return DIOMP_OK;
}

int diomp_mc_import(int fd, uint64_t *mc_out) {
    using namespace diomp::nvls;
    const Driver &d = drv();
    if (!d.ok) return DIOMP_BAD_REQUEST;
    CUmemGenericAllocationHandle h;
    DIOMP_CU_TRY(d.import_handle(&h, (void *)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
    *mc_out = (uint64_t)h;
    return DIOMP_OK;
}

int diomp_mc_add_device(uint64_t mc, int device) {
    using namespace diomp::nvls;
    const Driver &d = drv();
    CUdevice dev;
    DIOMP_CU_TRY(d.device_get(&dev, device));
    DIOMP_CU_TRY(d.add_device((CUmemGenericAllocationHandle)mc, dev));
    return DIOMP_OK;
}

// Back the window with this GPU's memory, bind it to the multicast object and
// map both views for `device`; the header (flags) starts zeroed.
int diomp_mc_bind(uint64_t mc, int device, uint64_t total, uint64_t *uc_out, uint64_t *mc_va_out,
                  uint64_t *phys_out) {
    using namespace diomp::nvls;
    const Driver &d = drv();
    DIOMP_CUDA_TRY(cudaSetDevice(device));
    CUmemAllocationProp p = {};
    p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    p.location.id = device;
    p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;  // as the multicast object
    CUmemGenericAllocationHandle ph;
    DIOMP_CU_TRY(d.mem_create(&ph, total, &p, 0));
    DIOMP_CU_TRY(d.bind_mem((CUmemGenericAllocationHandle)mc, 0, ph, 0, total, 0));
    CUmemAccessDesc ad = {};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = device;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CUdeviceptr uc = 0, mva = 0;
    DIOMP_CU_TRY(d.reserve(&uc, total, 2ull << 20, 0, 0));
    DIOMP_CU_TRY(d.map(uc, total, 0, ph, 0));
    DIOMP_CU_TRY(d.set_access(uc, total, &ad, 1));
    DIOMP_CU_TRY(d.reserve(&mva, total, 1ull << 29, 0, 0));  // multicast-granular VA
    DIOMP_CU_TRY(d.map(mva, total, 0, (CUmemGenericAllocationHandle)mc, 0));
    DIOMP_CU_TRY(d.set_access(mva, total, &ad, 1));
    DIOMP_CUDA_TRY(cudaMemset((void *)uc, 0, HEADER));
    DIOMP_CUDA_TRY(cudaDeviceSynchronize());
    *uc_out = (uint64_t)uc;
    *mc_va_out = (uint64_t)mva;
    *phys_out = (uint64_t)ph;
    return DIOMP_OK;
}

int diomp_mc_release(uint64_t mc, int device, uint64_t total, uint64_t uc, uint64_t mc_va,
                     uint64_t phys) {
    using namespace diomp::nvls;
    const Driver &d = drv();
    DIOMP_CUDA_TRY(cudaSetDevice(device));
    DIOMP_CUDA_TRY(cudaDeviceSynchronize());
    CUdevice dev;
    DIOMP_CU_TRY(d.device_get(&dev, device));
    if (mc_va) {
        DIOMP_CU_TRY(d.unmap(mc_va, total));
        DIOMP_CU_TRY(d.addr_free(mc_va, total));
    }
    if (uc) {
        DIOMP_CU_TRY(d.unmap(uc, total));
        DIOMP_CU_TRY(d.addr_free(uc, total));
    }
    if (phys) {
        DIOMP_CU_TRY(d.unbind((CUmemGenericAllocationHandle)mc, dev, 0, total));
        DIOMP_CU_TRY(d.mem_release((CUmemGenericAllocationHandle)phys));
    }
    DIOMP_CU_TRY(d.mem_release((CUmemGenericAllocationHandle)mc));
    return DIOMP_OK;
}

int diomp_allreduce_nvls(const diomp_nvls_args *x, void *stream) {
    using namespace diomp;
    using namespace diomp::nvls;
    if (x->k < 2 || x->pos < 0 || x->pos >= x->k || x->dtype < 0 || x->dtype > 3 || x->op < 0 ||
        x->op > 2)
        return DIOMP_BAD_REQUEST;
    if ((x->dtype == DIOMP_F32 || x->dtype == DIOMP_F64) && x->op != DIOMP_SUM)
        return DIOMP_BAD_REQUEST;  // the switch's float min/max NaN rules are not numpy's
    const int esz = (x->dtype == DIOMP_F32 || x->dtype == DIOMP_I32) ? 4 : 8;
    if (x->window < 16 || x->count == 0) return x->count == 0 ? DIOMP_OK : DIOMP_BAD_REQUEST;
    if ((x->send | x->recv) & 15) return DIOMP_BAD_REQUEST;
    DIOMP_CUDA_TRY(cudaSetDevice(x->device));
    cudaStream_t s = (cudaStream_t)stream;
    const uint64_t per_round = x->window / 16 * 16 / (uint64_t)esz;  // elements per round
    uint64_t epoch = x->epoch;
    for (uint64_t e0 = 0; e0 < x->count; e0 += per_round) {
        const uint64_t n = x->count - e0 < per_round ? x->count - e0 : per_round;
        ++epoch;
        Args a{};
        a.uc = x->uc;
        a.mc = x->mc;
        a.src = x->send + e0 * esz;
        a.dst = x->recv + e0 * esz;
        a.bytes = n * esz;
        a.count = n;
        a.k = x->k;
        a.pos = x->pos;
        a.dtype = x->dtype;
        a.op = x->op;
        a.target = (uint64_t)x->k * epoch;
        a.counter = (unsigned int *)x->counter;
        int rc;
        switch (x->dtype * 3 + x->op) {
            case DIOMP_F32 * 3 + DIOMP_SUM: rc = launch_round<float, 0>(a, s); break;
            case DIOMP_F64 * 3 + DIOMP_SUM: rc = launch_round<double, 0>(a, s); break;
            case DIOMP_I32 * 3 + DIOMP_SUM: rc = launch_round<int32_t, 0>(a, s); break;
            case DIOMP_I32 * 3 + DIOMP_MIN: rc = launch_round<int32_t, 1>(a, s); break;
            case DIOMP_I32 * 3 + DIOMP_MAX: rc = launch_round<int32_t, 2>(a, s); break;
            case DIOMP_I64 * 3 + DIOMP_SUM: rc = launch_round<long long, 0>(a, s); break;
            case DIOMP_I64 * 3 + DIOMP_MIN: rc = launch_round<long long, 1>(a, s); break;
            default: rc = launch_round<long long, 2>(a, s); break;
        }
        if (rc) return rc;
    }
    return DIOMP_OK;
}

int diomp_nvls_rounds(uint64_t count, int dtype, uint64_t window, uint64_t *rounds_out) {
    const int esz = (dtype == DIOMP_F32 || dtype == DIOMP_I32) ? 4 : 8;
    const uint64_t per_round = window / 16 * 16 / (uint64_t)esz;
    *rounds_out = per_round ? (count + per_round - 1) / per_round : 0;
    return DIOMP_OK;
}

}  // extern "C"
