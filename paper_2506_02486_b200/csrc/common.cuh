// Shared helpers for libdiomp_b200 (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/diomp_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libdiomp_b200 is built for sm_100a only"
#endif

#define DIOMP_CUDA_TRY(expr)                                                   \
    do {                                                                       \
        cudaError_t _e = (expr);                                               \
        if (_e != cudaSuccess) return DIOMP_CUDA_ERROR_BASE + (int)_e;         \
    } while (0)

#define DIOMP_LAUNCH_CHECK() DIOMP_CUDA_TRY(cudaGetLastError())

namespace diomp {

constexpr int kNumSMs = 148;

// Device-side error word: a spin-wait that exceeds the timeout records
// DIOMP_INTERNAL here and gives up instead of hanging the GPU.  The host
// reads and clears it after synchronising (diomp_device_error).  The library
// is one translation unit (diomp_b200.cu includes every component), so these
// are plain definitions.
__device__ unsigned int g_device_error = 0;
__device__ unsigned long long g_wait_timeout_ns = 30ull * 1000 * 1000 * 1000;
// Optional pinned, device-mapped mirror of the error word (set up by
// diomp_set_wait_timeout): the host then polls it with a plain load instead
// of a synchronous cudaMemcpyFromSymbol after every fence.
__device__ unsigned int *g_error_word = nullptr;

__device__ __forceinline__ void record_device_error(unsigned int code) {
    atomicExch(&g_device_error, code);
    unsigned int *w = g_error_word;
    if (w) {
        *(volatile unsigned int *)w = code;
        __threadfence_system();
    }
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void st_release_sys(uint64_t *p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Spin until *flag >= value (system scope acquire).  Returns false on timeout.
// Tight polling for the first DIOMP_SPIN_NS (cross-GPU flags land within a
// few microseconds of each other in back-to-back collectives and stencil
// steps; a sleeping poller adds up to its sleep to every handshake), then an
// exponential nanosleep backoff.
#ifndef DIOMP_SPIN_NS
#define DIOMP_SPIN_NS 20000
#endif
__device__ __forceinline__ bool wait_ge(const uint64_t *flag, uint64_t value) {
    if (ld_acquire_sys(flag) >= value) return true;
    const uint64_t t0 = globaltimer_ns();
    const uint64_t limit = g_wait_timeout_ns;
    unsigned ns = 64;
    while (ld_acquire_sys(flag) < value) {
        const uint64_t dt = globaltimer_ns() - t0;
        if (dt > DIOMP_SPIN_NS) {
            __nanosleep(ns);
            if (ns < 1024) ns <<= 1;
        }
        if (dt > limit) {
            record_device_error((unsigned)DIOMP_INTERNAL);
            return false;
        }
    }
    return true;
}

// "Last CTA out" detection: every CTA calls this once at the very end (after
// its own global / peer stores); exactly one CTA gets true, after all others
// have made their stores visible.  CTAs that stored to peer memory pass
// sys_fence (system-scope fence); CTAs that only touched their own GPU's
// memory need just a GPU-scope fence -- the winner's system fence and release
// store make the whole grid's work visible to the peers (cumulativity) -- and
// skip the costly system fence.  The counter self-resets.
__device__ __forceinline__ bool last_cta_done(unsigned int *counter, unsigned int nctas,
                                              bool sys_fence = true) {
    __shared__ unsigned int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        if (sys_fence) __threadfence_system();
        else __threadfence();
        unsigned int prev = atomicAdd(counter, 1u);
        s_last = (prev == nctas - 1);
        if (s_last) {
            atomicExch(counter, 0u);
            __threadfence_system();
        }
    }
    __syncthreads();
    return s_last != 0;
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace diomp
