"""Data-plane behaviour the reference's test_transport.py pins, on the NVLink
path: concurrent gets of one buffer from every rank agree byte for byte,
put/get issued from several host threads at once (the reference allows RMA
from any thread) land exactly, and handle states only move
forward (Pending -> RemoteDone, never back)."""

import threading

import numpy as np
import pytest

from conftest import NGPU

pytestmark = pytest.mark.gpu
MIB = 1 << 20


def _gpus(n):
    return list(range(min(NGPU, n))) or [0]


def test_concurrent_gets_from_all_ranks_agree():
    import paper_2506_02486_b200 as d
    from paper_2506_02486_b200.emulate import run_emulated
    size = 5 * MIB + 3
    data = np.random.default_rng(77).integers(0, 256, size, dtype=np.uint8)

    def fn(rt):
        rec = rt.alloc_symmetric(8 * MIB, 0)
        if rt.rank == 0:
            rt.gm.view(0, rec.addr.offset, size)[:] = data.tobytes()
        rt.barrier(rt.world)
        out = bytearray(size)
        handles = [rt.get(d.GlobalAddress(0, 0, rec.addr.offset), out, size, d.TransferKind.D2H)]
        stage = rt.alloc_symmetric(8 * MIB, 0)
        handles.append(rt.get(d.GlobalAddress(0, 0, rec.addr.offset),
                              d.GlobalAddress(rt.rank, 0, stage.addr.offset), size,
                              d.TransferKind.D2D))
        for h in handles:
            h.wait(30)
        rt.barrier(rt.world)
        return bytes(out), bytes(rt.gm.view(0, stage.addr.offset, size))

    res = run_emulated(4, fn, segment_bytes=64 * MIB, gpus=_gpus(4))
    want = data.tobytes()
    assert all(a == want and b == want for a, b in res)


def test_put_get_from_several_threads():
    import paper_2506_02486_b200 as d
    from paper_2506_02486_b200.emulate import run_emulated
    nthreads, size = 4, MIB + 7

    def fn(rt):
        dst = rt.alloc_symmetric(8 * MIB, 0)
        rt.barrier(rt.world)
        errors = []
        if rt.rank == 0:
            def worker(t):
                try:
                    data = np.random.default_rng(t).integers(0, 256, size, dtype=np.uint8)
                    at = d.GlobalAddress(1, 0, dst.addr.offset + t * (size + 9))
                    for _ in range(3):
                        rt.put(at, data, size, d.TransferKind.H2D).wait(30)
                        back = bytearray(size)
                        rt.get(at, back, size, d.TransferKind.D2H).wait(30)
                        if bytes(back) != data.tobytes():
                            errors.append(t)
                except Exception as e:  # surfaced below
                    errors.append(repr(e))
            ts = [threading.Thread(target=worker, args=(t,)) for t in range(nthreads)]
            for t in ts:
                t.start()
            for t in ts:
                t.join()
            rt.fence(rt.world)
        rt.barrier(rt.world)
        return errors

    assert run_emulated(2, fn, segment_bytes=32 * MIB, gpus=_gpus(2)) == [[], []]


def test_handle_states_only_move_forward():
    import paper_2506_02486_b200 as d
    from paper_2506_02486_b200.emulate import run_emulated
    from paper_2506_02486_b200.runtime import HandleState

    def fn(rt):
        rec = rt.alloc_symmetric(64 * MIB, 0)
        src = rt.alloc_symmetric(64 * MIB, 0)
        seen = []
        if rt.rank == 0:
            h = rt.put(d.GlobalAddress(1, 0, rec.addr.offset),
                       d.GlobalAddress(0, 0, src.addr.offset), 64 * MIB, d.TransferKind.D2D)
            seen.append(h.state)
            while not h.done():
                seen.append(h.state)
            seen.append(h.state)
            h.wait(30)
            seen.append(h.state)
            assert h.done()
            z = rt.put(d.GlobalAddress(1, 0, rec.addr.offset), b"", 0, d.TransferKind.H2D)
            assert z.state == HandleState.RemoteDone and z.done()
        rt.barrier(rt.world)
        return seen

    seen = run_emulated(2, fn, segment_bytes=256 * MIB, gpus=_gpus(2))[0]
    order = [HandleState.Pending, HandleState.RemoteDone]
    idx = [order.index(s) for s in seen]
    assert idx == sorted(idx) and seen[-1] == HandleState.RemoteDone
