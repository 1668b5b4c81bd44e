"""LL (flag-in-payload) vs handshake allreduce / bcast by size through the
public API, one process per GPU: per-call time back to back (enqueue-only,
drained at the end) and blocking.  torchrun --nproc-per-node 2
tools/probe_ll_cross.py; DIOMP_LL_MAX picks the LL ceiling (0 = off)."""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("DIOMP_GPUS", str(local))
    os.environ.setdefault("DIOMP_SEGMENT_BYTES", str(256 << 20))
    import paper_2506_02486_b200 as d
    from paper_2506_02486_b200 import collectives as coll
    rt = d.init()
    comm = coll.bootstrap(rt, rt.world)
    send = rt.alloc_symmetric(4 << 20, 0)
    recv = rt.alloc_symmetric(4 << 20, 0)
    op = coll.ReduceOp(coll.ReduceKind.Sum, coll.ElementType.f32)
    out = {"ll_max": coll.LL_MAX_BYTES, "slot": coll._ll_slot_bytes(comm)}
    for nbytes in (1 << 10, 8 << 10, 32 << 10, 64 << 10, 128 << 10, 256 << 10, 1 << 20):
        n = nbytes // 4
        for _ in range(50):
            coll.allreduce(comm, send.addr, recv.addr, n, op)
        rt.barrier(rt.world)
        t0 = time.perf_counter()
        for _ in range(500):
            coll.allreduce(comm, send.addr, recv.addr, n, op, blocking=False)
        coll.complete(comm)
        bb = (time.perf_counter() - t0) / 500 * 1e6
        rt.barrier(rt.world)
        t0 = time.perf_counter()
        for _ in range(200):
            coll.allreduce(comm, send.addr, recv.addr, n, op)
        bl = (time.perf_counter() - t0) / 200 * 1e6
        out[nbytes] = {"b2b_us": round(bb, 2), "blocking_us": round(bl, 2),
                       "ll": coll._ll_ok(comm, nbytes)}
    if rt.rank == 0:
        print(json.dumps(out), flush=True)
    d.finalize(rt)


if __name__ == "__main__":
    main()
