"""Device-synchronised work of different kinds in flight at once.

Collectives, the fused stencil and the Cannon ring each signal on their own
bank of flag slots (runtime.py CHANNEL_*), so a blocking=False allreduce, a
stencil step on another stream and a ring step on a third -- all spinning on
per-pair counters at the same time -- cannot satisfy or rewind each other's
waits.  100 interleaved iterations, every result checked: allreduce bitwise
vs the ring-order fold, stencil sha256 vs the reference, ring vs host BLAS.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, need_gpus

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
MIB = 1 << 20


@need_gpus(2)
def test_interleaved_allreduce_stencil_ring_100_iterations():
    from oracle import oracle as O
    from paper_2506_02486_b200 import _native
    from paper_2506_02486_b200 import collectives as coll
    from paper_2506_02486_b200.apps.cannon import CannonRing, MatmulSpec, _fill_matrices
    from paper_2506_02486_b200.apps.stencil import (StencilRunner, StencilSpec, _gather_field,
                                                    dump_bytes)
    from paper_2506_02486_b200.emulate import run_emulated
    import hashlib

    iters = 100
    gold = {(c["nx"], c["steps"], c["amp"]): c["sha256"]
            for c in json.load(open(os.path.join(GOLDEN, "stencil_golden.json")))["cases"]}
    want_field = gold[(64, 100, 1.0)]
    count = 4096 + 3
    contribs = [np.random.default_rng(50 + r).uniform(-1, 1, count).astype(np.float32)
                for r in range(2)]
    want_ar = O.allreduce_fold(contribs, "sum")
    n = 256
    a, b = _fill_matrices(n, 4)
    op = coll.ReduceOp(coll.ReduceKind.Sum, coll.ElementType.f32)

    def fn(rt):
        comm = coll.bootstrap(rt, rt.world)
        send = rt.alloc_symmetric(count * 4, 0)
        recv = rt.alloc_symmetric(count * 4, 0)
        rt.gm.view(0, send.addr.offset, count * 4)[:] = contribs[rt.rank].tobytes()
        runner = StencilRunner(rt, StencilSpec(64, 64, 64, steps=iters))
        ring = CannonRing(rt, MatmulSpec(n, 2), a_full=a, b_full=b)
        assert runner.mode == "fused" and ring.sync
        side = _native.stream_create(rt.gpus[0])
        rt.barrier(rt.world)
        ar_ok = True
        for it in range(iters):
            coll.allreduce(comm, send.addr, recv.addr, count, op, blocking=False)
            runner.enqueue(1, stream_handle=side)
            ring.enqueue_step()
            if it % 10 == 9:
                coll.complete(comm)
                got = np.frombuffer(bytes(rt.gm.view(0, recv.addr.offset, count * 4)),
                                    dtype=np.float32)
                ar_ok = ar_ok and got.tobytes() == want_ar.tobytes()
        _native.call("diomp_stream_sync", side)
        ring.synchronize()
        coll.complete(comm)
        _native.check_device(rt.gpus[0], "interleaved")
        rt.barrier(rt.world)
        f = _gather_field(rt, runner.cur_rec, runner.spec, runner.nxl, runner.shape)
        sha = hashlib.sha256(dump_bytes(f)).hexdigest() if rt.rank == 0 else ""
        c = {e: st["c"].cpu().numpy() for e, st in ring.local.items()}
        ring.release()
        _native.call("diomp_stream_destroy", side)
        return ar_ok, sha, c

    res = run_emulated(2, fn, segment_bytes=64 * MIB, gpus=[0, 1])
    assert all(r[0] for r in res)
    assert res[0][1] == want_field
    got = np.concatenate([res[r][2][r] for r in range(2)])
    want = (iters // 2) * (a @ b)   # the stripes return home every P = 2 steps
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert rel <= 1e-13, rel
