"""Host-side cost of small collectives and puts through the public API, one
process per GPU (torchrun --nproc-per-node 2 tools/probe_coll_overhead.py).
Rank 0 prints us/op (enqueue-only and blocking) and a cProfile of the
enqueue loop."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.getcwd())


def main():
    import numpy as np

    import paper_2506_02486_b200 as d
    from paper_2506_02486_b200 import collectives as coll
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("DIOMP_GPUS", str(local))
    os.environ.setdefault("DIOMP_SEGMENT_BYTES", str(64 << 20))
    rt = d.init()
    comm = coll.bootstrap(rt, rt.world)
    send = rt.alloc_symmetric(1 << 20, 0)
    recv = rt.alloc_symmetric(1 << 20, 0)
    op = coll.ReduceOp(coll.ReduceKind.Sum, coll.ElementType.f32)
    n = 2000
    out = {}
    for _ in range(200):
        coll.allreduce(comm, send.addr, recv.addr, 256, op)
    s = rt._rma_streams[0]
    rt.barrier(rt.world)
    t0 = time.perf_counter()
    for _ in range(n):
        coll.allreduce(comm, send.addr, recv.addr, 256, op, blocking=False)
    t1 = time.perf_counter()
    coll.complete(comm)
    t2 = time.perf_counter()
    out["allreduce_enqueue_us"] = (t1 - t0) / n * 1e6
    out["allreduce_drain_us"] = (t2 - t0) / n * 1e6
    rt.barrier(rt.world)
    t0 = time.perf_counter()
    for _ in range(500):
        coll.allreduce(comm, send.addr, recv.addr, 256, op)
    out["allreduce_blocking_us"] = (time.perf_counter() - t0) / 500 * 1e6
    rt.barrier(rt.world)
    if rt.rank == 0:
        dst = rt.translate(recv.addr, 1)
        src = d.GlobalAddress(0, 0, send.addr.offset)
        for _ in range(200):
            rt.put(dst, src, 8, d.TransferKind.D2D)
        rt.fence(rt.world)
        t0 = time.perf_counter()
        for _ in range(n):
            rt.put(dst, src, 8, d.TransferKind.D2D)
        t1 = time.perf_counter()
        rt.fence(rt.world)
        out["put_enqueue_us"] = (t1 - t0) / n * 1e6
        t0 = time.perf_counter()
        for _ in range(500):
            rt.put(dst, src, 8, d.TransferKind.D2D)
            rt.fence(rt.world)
        out["put_fence_us"] = (time.perf_counter() - t0) / 500 * 1e6
        t0 = time.perf_counter()
        for _ in range(500):
            rt.get(dst, src, 8, d.TransferKind.D2D).wait()
        out["get_wait_us"] = (time.perf_counter() - t0) / 500 * 1e6
    rt.barrier(rt.world)
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(n):
        coll.allreduce(comm, send.addr, recv.addr, 256, op, blocking=False)
    pr.disable()
    coll.complete(comm)
    if rt.rank == 0:
        print(out, flush=True)
        pstats.Stats(pr).sort_stats("tottime").print_stats(22)
        pr = cProfile.Profile()
        dst = rt.translate(recv.addr, 1)
        src = d.GlobalAddress(0, 0, send.addr.offset)
        pr.enable()
        for _ in range(n):
            rt.put(dst, src, 8, d.TransferKind.D2D)
        rt.fence(rt.world)
        pr.disable()
        pstats.Stats(pr).sort_stats("tottime").print_stats(22)
    rt.barrier(rt.world)
    d.finalize(rt)
    _ = np


if __name__ == "__main__":
    main()
