// Rank-addressed one-sided RMA context: the C ABI a non-Python caller uses
// to reach the global address space: a peer table of mapped
// segment bases, put/get addressed by (rank, device, offset) returning an op
// handle, op query/wait, and a fence over a set of target endpoints.
//
// Replaces, per reference interface:
//   peer table      transport.py:313-454 (peer connections) +
//                   global_memory.py:73-84 (GlobalAddress -> arena)
//   rma_put/get     runtime.py:371-470 -> transport.py:508-566
//   op handles      transport.py:58-101 (CompletionHandle: Pending ->
//                   RemoteDone | Failed, done(), wait(timeout))
//   fence_group     runtime.py:535-556 (remote completion toward a group)
//
// An op is one pooled CUDA event recorded behind the transfer on the issuing
// stream; its handle is (generation << 32 | slot), so a handle outlives its
// slot safely: once the op is retired (waited or fenced) the slot's
// generation moves on and the stale handle reads as complete.  All host-side
// state sits behind one mutex: entry points are reentrant on distinct
// streams.
#pragma once

#include <chrono>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace diomp {
namespace rma {

struct Peer {
    uint64_t base = 0, bytes = 0;
    int32_t phys = -1;   // box-wide physical GPU id (remote = differs from the issuer's)
};

struct Local {
    int32_t cuda_device = -1, phys = -1;
};

struct Slot {
    cudaEvent_t ev = nullptr;
    uint32_t gen = 1;
    int32_t ep = -1;      // target endpoint while live, -1 when free
    int32_t dev = -1;     // CUDA device the event belongs to
    cudaStream_t stream = nullptr;
};

struct Ctx {
    int32_t nranks = 0, dpr = 0;
    int32_t force_remote = 0;
    std::vector<Peer> peers;               // index = rank * dpr + dev
    std::vector<Local> locals;             // index = local device index
    std::vector<Slot> slots;
    std::vector<uint32_t> free_slots;
    std::vector<uint32_t> live;            // slots with a pending op, issue order
    std::vector<std::vector<cudaEvent_t>> ev_pool;   // per CUDA device
    // LL collective epochs per ordered endpoint pair: ll_sent[me * n + peer] =
    // LL calls this endpoint made toward peer, ll_recvd[peer * n + me] = LL
    // calls it took from peer (both ends count every call between them)
    std::vector<uint32_t> ll_sent, ll_recvd;
    std::vector<cudaEvent_t> order_ev;     // per CUDA device: "after the caller's stream"
    std::mutex mu;
};

static int get_event(Ctx &c, int dev, cudaEvent_t *out) {
    if ((int)c.ev_pool.size() <= dev) c.ev_pool.resize(dev + 1);
    auto &pool = c.ev_pool[dev];
    if (!pool.empty()) {
        *out = pool.back();
        pool.pop_back();
        return DIOMP_OK;
    }
    DIOMP_CUDA_TRY(cudaEventCreateWithFlags(out, cudaEventDisableTiming));
    return DIOMP_OK;
}

static void retire(Ctx &c, uint32_t idx) {
    Slot &s = c.slots[idx];
    if (s.ep < 0) return;
    if ((int)c.ev_pool.size() <= s.dev) c.ev_pool.resize(s.dev + 1);
    c.ev_pool[s.dev].push_back(s.ev);
    s.ev = nullptr;
    s.ep = -1;
    s.gen += 1;
    c.free_slots.push_back(idx);
}

// Record the completion event of an op just issued on `stream` (mu held).
static int new_op(Ctx &c, int ep, int dev, cudaStream_t stream, uint64_t *op_out) {
    cudaEvent_t ev;
    int rc = get_event(c, dev, &ev);
    if (rc) return rc;
    cudaError_t e = cudaEventRecord(ev, stream);
    if (e != cudaSuccess) {
        c.ev_pool[dev].push_back(ev);
        return DIOMP_CUDA_ERROR_BASE + (int)e;
    }
    uint32_t idx;
    if (!c.free_slots.empty()) {
        idx = c.free_slots.back();
        c.free_slots.pop_back();
    } else {
        idx = (uint32_t)c.slots.size();
        c.slots.emplace_back();
    }
    Slot &s = c.slots[idx];
    s.ev = ev;
    s.ep = ep;
    s.dev = dev;
    s.stream = stream;
    c.live.push_back(idx);
    *op_out = ((uint64_t)s.gen << 32) | idx;
    return DIOMP_OK;
}

static void drop_live(Ctx &c, uint32_t idx) {
    for (size_t i = 0; i < c.live.size(); ++i)
        if (c.live[i] == idx) {
            c.live.erase(c.live.begin() + (long)i);
            return;
        }
}

// Resolve (rank, dev, off, n) to a pointer inside that endpoint's segment.
static int resolve(Ctx &c, int32_t rank, int32_t dev, uint64_t off, uint64_t n, int *ep_out,
                   uint64_t *ptr_out) {
    if (rank < 0 || rank >= c.nranks || dev < 0 || dev >= c.dpr) return DIOMP_INVALID_ADDRESS;
    const int ep = rank * c.dpr + dev;
    const Peer &p = c.peers[ep];
    if (!p.base || off > p.bytes || n > p.bytes - off) return DIOMP_INVALID_ADDRESS;
    *ep_out = ep;
    *ptr_out = p.base + off;
    return DIOMP_OK;
}

}  // namespace rma
}  // namespace diomp

extern "C" {

int diomp_rma_ctx_create(int32_t nranks, int32_t devices_per_rank, void **ctx_out) {
    using namespace diomp::rma;
    if (nranks < 1 || devices_per_rank < 1 || (int64_t)nranks * devices_per_rank > DIOMP_MAX_TEAM)
        return DIOMP_BAD_REQUEST;
    Ctx *c = new Ctx();
    c->nranks = nranks;
    c->dpr = devices_per_rank;
    c->peers.resize((size_t)nranks * devices_per_rank);
    c->locals.resize(devices_per_rank);
    const size_t n = (size_t)nranks * devices_per_rank;
    c->ll_sent.assign(n * n, 0);
    c->ll_recvd.assign(n * n, 0);
    *ctx_out = c;
    return DIOMP_OK;
}

int diomp_rma_ctx_destroy(void *ctx) {
    using namespace diomp::rma;
    Ctx *c = (Ctx *)ctx;
    if (!c) return DIOMP_OK;
    {
        std::lock_guard<std::mutex> lk(c->mu);
        for (uint32_t idx : c->live) {
            if (c->slots[idx].ev) cudaEventSynchronize(c->slots[idx].ev);
            retire(*c, idx);
        }
        c->live.clear();
        for (auto &pool : c->ev_pool)
            for (cudaEvent_t e : pool) cudaEventDestroy(e);
        for (cudaEvent_t e : c->order_ev)
            if (e) cudaEventDestroy(e);
    }
    delete c;
    return DIOMP_OK;
}

int diomp_rma_set_local(void *ctx, int32_t local_dev, int32_t cuda_device, int32_t phys_gpu) {
    using namespace diomp::rma;
    Ctx *c = (Ctx *)ctx;
    if (!c || local_dev < 0 || local_dev >= c->dpr) return DIOMP_BAD_REQUEST;
    std::lock_guard<std::mutex> lk(c->mu);
    c->locals[local_dev].cuda_device = cuda_device;
    c->locals[local_dev].phys = phys_gpu;
    return DIOMP_OK;
}

int diomp_rma_set_force_remote(void *ctx, int32_t on) {
    diomp::rma::Ctx *c = (diomp::rma::Ctx *)ctx;
    if (!c) return DIOMP_BAD_REQUEST;
    c->force_remote = on;
    return DIOMP_OK;
}

int diomp_peer_table_set(void *ctx, int32_t rank, int32_t dev, uint64_t base, uint64_t bytes,
                         int32_t phys_gpu) {
    using namespace diomp::rma;
    Ctx *c = (Ctx *)ctx;
    if (!c || rank < 0 || rank >= c->nranks || dev < 0 || dev >= c->dpr) return DIOMP_BAD_REQUEST;
    std::lock_guard<std::mutex> lk(c->mu);
    Peer &p = c->peers[(size_t)rank * c->dpr + dev];
    p.base = base;
    p.bytes = bytes;
    p.phys = phys_gpu;
    return DIOMP_OK;
}

// put: bytes at `src` (a host pointer for DIOMP_H2D, a device pointer on
// local device `local_dev` for DIOMP_D2D) into (dst_rank, dst_dev, dst_off).
int diomp_rma_put(void *ctx, int32_t dst_rank, int32_t dst_dev, uint64_t dst_off, uint64_t src,
                  uint64_t nbytes, int32_t kind, int32_t local_dev, void *stream,
                  uint64_t *op_out) {
    using namespace diomp;
    using namespace diomp::rma;
    Ctx *c = (Ctx *)ctx;
    if (!c || local_dev < 0 || local_dev >= c->dpr || (kind != DIOMP_H2D && kind != DIOMP_D2D))
        return DIOMP_BAD_REQUEST;
    std::lock_guard<std::mutex> lk(c->mu);
    int ep;
    uint64_t dst;
    int rc = resolve(*c, dst_rank, dst_dev, dst_off, nbytes, &ep, &dst);
    if (rc) return rc;
    const Local &L = c->locals[local_dev];
    if (L.cuda_device < 0) return DIOMP_BAD_REQUEST;
    cudaStream_t s = (cudaStream_t)stream;
    if (nbytes) {
        if (kind == DIOMP_H2D) {
            DIOMP_CUDA_TRY(cudaSetDevice(L.cuda_device));
            DIOMP_CUDA_TRY(cudaMemcpyAsync((void *)dst, (const void *)src, nbytes,
                                           cudaMemcpyHostToDevice, s));
        } else {
            const int remote = c->force_remote || c->peers[ep].phys != L.phys;
            rc = diomp_put(L.cuda_device, dst, src, nbytes, remote, stream);
            if (rc) return rc;
        }
    }
    return new_op(*c, ep, L.cuda_device, s, op_out);
}

// get: bytes of (src_rank, src_dev, src_off) into `dst` (a host pointer for
// DIOMP_D2H, a device pointer on local device `local_dev` for DIOMP_D2D).
int diomp_rma_get(void *ctx, int32_t src_rank, int32_t src_dev, uint64_t src_off, uint64_t dst,
                  uint64_t nbytes, int32_t kind, int32_t local_dev, void *stream,
                  uint64_t *op_out) {
    using namespace diomp;
    using namespace diomp::rma;
    Ctx *c = (Ctx *)ctx;
    if (!c || local_dev < 0 || local_dev >= c->dpr || (kind != DIOMP_D2H && kind != DIOMP_D2D))
        return DIOMP_BAD_REQUEST;
    std::lock_guard<std::mutex> lk(c->mu);
    int ep;
    uint64_t src;
    int rc = resolve(*c, src_rank, src_dev, src_off, nbytes, &ep, &src);
    if (rc) return rc;
    const Local &L = c->locals[local_dev];
    if (L.cuda_device < 0) return DIOMP_BAD_REQUEST;
    cudaStream_t s = (cudaStream_t)stream;
    if (nbytes) {
        if (kind == DIOMP_D2H) {
            DIOMP_CUDA_TRY(cudaSetDevice(L.cuda_device));
            DIOMP_CUDA_TRY(cudaMemcpyAsync((void *)dst, (const void *)src, nbytes,
                                           cudaMemcpyDeviceToHost, s));
        } else {
            const int remote = c->force_remote || c->peers[ep].phys != L.phys;
            rc = diomp_get(L.cuda_device, dst, src, nbytes, remote, stream);
            if (rc) return rc;
        }
    }
    return new_op(*c, ep, L.cuda_device, s, op_out);
}

// DIOMP_OK once the op's bytes have landed (or the op was retired),
// DIOMP_PENDING before; a CUDA error fails the op.
int diomp_op_query(void *ctx, uint64_t op) {
    using namespace diomp::rma;
    Ctx *c = (Ctx *)ctx;
    if (!c) return DIOMP_BAD_REQUEST;
    const uint32_t idx = (uint32_t)op, gen = (uint32_t)(op >> 32);
    std::lock_guard<std::mutex> lk(c->mu);
    if (idx >= c->slots.size()) return DIOMP_BAD_REQUEST;
    Slot &s = c->slots[idx];
    if (s.gen != gen || s.ep < 0) return DIOMP_OK;
    cudaError_t e = cudaEventQuery(s.ev);
    if (e == cudaErrorNotReady) {
        cudaGetLastError();
        return DIOMP_PENDING;
    }
    drop_live(*c, idx);
    retire(*c, idx);
    return e == cudaSuccess ? DIOMP_OK : DIOMP_CUDA_ERROR_BASE + (int)e;
}

// Block until the op completes (timeout_s < 0: no limit).  Spins on the event
// for the first 200 us, then yields; DIOMP_INTERNAL on timeout (the op stays
// pending and can be waited again).
int diomp_op_wait(void *ctx, uint64_t op, double timeout_s) {
    using clock = std::chrono::steady_clock;
    const auto t0 = clock::now();
    for (;;) {
        int rc = diomp_op_query(ctx, op);
        if (rc != DIOMP_PENDING) return rc;
        const double dt = std::chrono::duration<double>(clock::now() - t0).count();
        if (timeout_s >= 0 && dt > timeout_s) return DIOMP_INTERNAL;
        if (dt > 200e-6) std::this_thread::yield();
    }
}

// Remote completion of every op issued toward the endpoints in `mask` (bit
// e = endpoint rank * devices_per_rank + dev).  Ops toward other endpoints
// are untouched.
int diomp_fence_group(void *ctx, uint64_t mask) {
    using namespace diomp::rma;
    Ctx *c = (Ctx *)ctx;
    if (!c) return DIOMP_BAD_REQUEST;
    std::vector<std::pair<uint32_t, cudaEvent_t>> mine;
    {
        std::lock_guard<std::mutex> lk(c->mu);
        std::vector<uint32_t> keep;
        keep.reserve(c->live.size());
        for (uint32_t idx : c->live) {
            const Slot &s = c->slots[idx];
            if ((mask >> s.ep) & 1ull) mine.emplace_back(idx, s.ev);
            else keep.push_back(idx);
        }
        c->live.swap(keep);
    }
    // Ops on one stream complete in issue order: wait for the last one per
    // stream (`mine` is in issue order), the earlier ones are then done too.
    int first_err = DIOMP_OK;
    std::vector<cudaStream_t> seen;
    for (size_t i = mine.size(); i-- > 0;) {
        cudaStream_t st;
        {
            std::lock_guard<std::mutex> lk(c->mu);
            st = c->slots[mine[i].first].stream;
        }
        bool done = false;
        for (cudaStream_t x : seen) done = done || x == st;
        if (done) continue;
        seen.push_back(st);
        cudaError_t e = cudaEventSynchronize(mine[i].second);
        if (e != cudaSuccess && !first_err) first_err = DIOMP_CUDA_ERROR_BASE + (int)e;
    }
    std::lock_guard<std::mutex> lk(c->mu);
    for (auto &pe : mine) retire(*c, pe.first);
    return first_err;
}

// Ops issued and not yet retired toward the endpoints in `mask`.
int diomp_rma_outstanding(void *ctx, uint64_t mask, uint64_t *count_out) {
    using namespace diomp::rma;
    Ctx *c = (Ctx *)ctx;
    if (!c) return DIOMP_BAD_REQUEST;
    std::lock_guard<std::mutex> lk(c->mu);
    uint64_t n = 0;
    for (uint32_t idx : c->live) {
        const Slot &s = c->slots[idx];
        if (!((mask >> s.ep) & 1ull)) continue;
        cudaError_t e = cudaEventQuery(s.ev);
        if (e == cudaErrorNotReady) {
            cudaGetLastError();
            ++n;
        }
    }
    *count_out = n;
    return DIOMP_OK;
}

}  // extern "C"
