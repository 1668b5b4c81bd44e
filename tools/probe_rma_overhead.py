"""Host-side cost of one put/get (D2D, 8 B) through the public API:
2 thread-ranks (GPUs 0 and 1 when present), rank 0 issues N puts back to back, then fences.
Prints us/op and a cProfile of the put loop."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.getcwd())
import paper_2506_02486_b200 as d
from paper_2506_02486_b200.emulate import run_emulated

N = int(os.environ.get("N", "3000"))


def fn(rt):
    rec = rt.alloc_symmetric(1 << 20, 0)
    src = rt.alloc_symmetric(1 << 20, 0)
    out = {}
    if rt.rank == 0:
        dst = rt.translate(rec.addr, 1)
        local = d.GlobalAddress(0, 0, src.addr.offset)
        for _ in range(200):
            rt.put(dst, local, 8, d.TransferKind.D2D)
        rt.fence(rt.world)
        t0 = time.perf_counter()
        for _ in range(N):
            rt.put(dst, local, 8, d.TransferKind.D2D)
        t1 = time.perf_counter()
        rt.fence(rt.world)
        t2 = time.perf_counter()
        out["put_us"] = (t1 - t0) / N * 1e6
        out["fence_us"] = (t2 - t1) * 1e6
        t0 = time.perf_counter()
        for _ in range(500):
            rt.put(dst, local, 8, d.TransferKind.D2D)
            rt.fence(rt.world)
        out["put_fence_us"] = (time.perf_counter() - t0) / 500 * 1e6
        t0 = time.perf_counter()
        for _ in range(500):
            rt.get(dst, local, 8, d.TransferKind.D2D).wait()
        out["get_wait_us"] = (time.perf_counter() - t0) / 500 * 1e6
        pr = cProfile.Profile()
        pr.enable()
        for _ in range(N):
            rt.put(dst, local, 8, d.TransferKind.D2D)
        rt.fence(rt.world)
        pr.disable()
        pstats.Stats(pr).sort_stats("tottime").print_stats(18)
    rt.barrier(rt.world)
    return out


import torch
print(run_emulated(2, fn, segment_bytes=8 << 20,
                   gpus=[0, 1] if torch.cuda.device_count() >= 2 else [0])[0])
