"""Multi-process parity check (one process per GPU over CUDA IPC), run as
    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/mp_check.py
Checks against the reference-generated golden fixtures: fused stencil
checksums (device-flag halo), allreduce/reduce/bcast bitwise, put/get
byte-exact, Cannon ring (both shift engines) vs host BLAS.  Prints one JSON line per rank-0 check; exit 1 on any failure.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)


def main():
    import paper_2506_02486_b200 as d
    from oracle import oracle as O
    from paper_2506_02486_b200 import collectives as coll
    from paper_2506_02486_b200.apps.stencil import StencilSpec, run_stencil

    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("DIOMP_GPUS", str(local))
    os.environ.setdefault("DIOMP_SEGMENT_BYTES", str(256 << 20))
    rt = d.init()
    ok = True
    gold = json.load(open(os.path.join(HERE, "tests", "golden", "stencil_golden.json")))
    for c in gold["cases"]:
        if c["nx"] % rt.nranks or c["nx"] // rt.nranks < 4 or c["nx"] > 128:
            continue
        res = run_stencil(rt, StencilSpec(c["nx"], c["ny"], c["nz"], steps=c["steps"],
                                          source_amplitude=c["amp"]))
        if rt.rank == 0:
            good = res.checksum == c["sha256"]
            ok &= good
            print(json.dumps({"check": "stencil", "case": [c["nx"], c["ny"], c["nz"], c["steps"]],
                              "ranks": rt.nranks, "ok": good, "seconds": res.seconds}), flush=True)

    comm = coll.bootstrap(rt, rt.world)
    k = rt.nranks
    for etype, kind, count in [("f64", "sum", 9001), ("f32", "sum", 1 << 20), ("i64", "max", 4099),
                               ("f32", "min", 100_003)]:
        dt = {"f32": np.float32, "f64": np.float64, "i32": np.int32, "i64": np.int64}[etype]
        op = coll.ReduceOp(coll.ReduceKind(kind), coll.ElementType(etype))
        isz = np.dtype(dt).itemsize
        send = rt.alloc_symmetric(count * isz, 0)
        recv = rt.alloc_symmetric(count * isz, 0)

        def contrib(r):
            rng = np.random.default_rng(77 + r)
            return (rng.uniform(-1, 1, count) if etype[0] == "f" else
                    rng.integers(-2**40, 2**40, count)).astype(dt)
        mine = contrib(rt.rank)
        rt.gm.view(0, send.addr.offset, mine.nbytes)[:] = mine.tobytes()
        coll.allreduce(comm, send.addr, recv.addr, count, op)
        got = bytes(rt.gm.view(0, recv.addr.offset, count * isz))
        want = O.allreduce_fold([contrib(r) for r in range(k)], kind).tobytes()
        good = got == want
        root = k - 1
        coll.reduce(comm, send.addr, recv.addr, count, op, root=root)
        if rt.rank == root:
            good &= bytes(rt.gm.view(0, recv.addr.offset, count * isz)) == \
                O.reduce_fold([contrib(r) for r in range(k)], kind, root).tobytes()
        coll.bcast(comm, send.addr, count * isz, root=1 % k)
        good &= bytes(rt.gm.view(0, send.addr.offset, count * isz)) == contrib(1 % k).tobytes()
        flags = rt.ctrl.allgather(tuple(range(k)), f"mp/{etype}{kind}", bytes([good]))
        allgood = all(b == b"\x01" for _, b in flags)
        ok &= allgood
        if rt.rank == 0:
            print(json.dumps({"check": "collectives", "etype": etype, "op": kind, "count": count,
                              "ranks": k, "ok": allgood}), flush=True)
        rt.free(recv)
        rt.free(send)

    # put/get byte-exact rank 0 -> every peer
    buf = rt.alloc_symmetric(8 << 20, 0)
    src = rt.alloc_symmetric(8 << 20, 0)
    good = True
    if rt.rank == 0:
        for peer in range(1, k):
            for n in (1, 37, 4096, (8 << 20) - 3):
                data = np.random.default_rng(n + peer).integers(0, 256, n, dtype=np.uint8).tobytes()
                rt.gm.view(0, src.addr.offset, n)[:] = data
                rt.put(d.GlobalAddress(peer, 0, buf.addr.offset), d.GlobalAddress(0, 0, src.addr.offset),
                       n, d.TransferKind.D2D)
                rt.fence(rt.world)
                back = bytearray(n)
                rt.get(d.GlobalAddress(peer, 0, buf.addr.offset), back, n, d.TransferKind.D2H).wait()
                good &= bytes(back) == data
        print(json.dumps({"check": "put_get", "ranks": k, "ok": good}), flush=True)
    ok &= good
    rt.barrier(rt.world)

    # Cannon ring over IPC-mapped stripes (copy-engine and fused shift), two
    # back-to-back runs: each rank's C stripe vs host BLAS, 2 A@B
    import pickle

    from paper_2506_02486_b200.apps.cannon import CannonRing, MatmulSpec, _fill_matrices
    n = 1024
    a, b = _fill_matrices(n, 0)
    ns = n // rt.nranks
    want = 2.0 * (a[rt.rank * ns:(rt.rank + 1) * ns] @ b)
    for shift in ("ce", "fused"):
        os.environ["DIOMP_CANNON_SHIFT"] = shift
        ring = CannonRing(rt, MatmulSpec(n, rt.nranks), a_full=a, b_full=b)
        rt.barrier(rt.world)
        ring.run()
        ring.run()
        rt.barrier(rt.world)
        got = ring.local[rt.rank]["c"].cpu().numpy()
        rel = float(np.linalg.norm(got - want) / np.linalg.norm(want))
        mode = ring.shift
        ring.release()
        res = [pickle.loads(x) for _, x in rt.ctrl.allgather(tuple(range(rt.nranks)), f"mpc/{shift}",
                                                              pickle.dumps((rel, mode)))]
        good = all(r <= 1e-14 for r, _ in res)
        ok &= good
        if rt.rank == 0:
            print(json.dumps({"check": "cannon", "n": n, "ranks": rt.nranks, "shift": [m for _, m in res],
                              "max_rel": max(r for r, _ in res), "ok": good}), flush=True)
    os.environ.pop("DIOMP_CANNON_SHIFT", None)
    rt.barrier(rt.world)
    d.finalize(rt)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
