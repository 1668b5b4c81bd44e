"""Full BASELINE sizes (configs[1] and [2] top end, 1 GiB): put/get payloads
byte-exact through every engine the size selects (copy engine for the remote
put, bulk-async TMA for the remote get), and a 1 GiB f32 allreduce bitwise
equal to the CPU oracle's ring-order fold -- checked on whole buffers, not
samples."""

import numpy as np
import pytest

from conftest import NGPU

pytestmark = pytest.mark.gpu
GIB = 1 << 30


def _ranks_gpus():
    # two ranks on distinct GPUs (device-flag collectives, NVLink engines) when
    # the box has them, else emulated on one GPU
    return [0, 1] if NGPU >= 2 else [0]


@pytest.mark.parametrize("force_remote", [False, True])
def test_put_get_1gib_byte_exact(force_remote, monkeypatch):
    """force_remote: DIOMP_FORCE_REMOTE=1 makes a one-GPU box take the remote
    engines too (copy-engine put, bulk-TMA get) -- the paths a peer GPU uses."""
    import paper_2506_02486_b200 as d
    from paper_2506_02486_b200.emulate import run_emulated
    if force_remote:
        monkeypatch.setenv("DIOMP_FORCE_REMOTE", "1")
    payload = np.random.default_rng(2024).integers(0, 256, GIB, dtype=np.uint8)

    def fn(rt):
        src = rt.alloc_symmetric(GIB, 0)
        dst = rt.alloc_symmetric(GIB, 0)
        ok = True
        if rt.rank == 0:
            rt.put(d.GlobalAddress(0, 0, src.addr.offset), payload, GIB, d.TransferKind.H2D)
            rt.fence(rt.world)
            # D2D put of the whole GiB to rank 1, then a D2D get of it back
            # into rank 0's dst
            rt.put(d.GlobalAddress(1, 0, dst.addr.offset), d.GlobalAddress(0, 0, src.addr.offset),
                   GIB, d.TransferKind.D2D)
            rt.fence(rt.world)
            rt.get(d.GlobalAddress(1, 0, dst.addr.offset), d.GlobalAddress(0, 0, dst.addr.offset),
                   GIB, d.TransferKind.D2D).wait(60)
            back = bytearray(GIB)
            rt.get(d.GlobalAddress(0, 0, dst.addr.offset), back, GIB, d.TransferKind.D2H).wait(60)
            ok = bytes(back) == payload.tobytes()
        rt.barrier(rt.world)
        return ok

    assert run_emulated(2, fn, segment_bytes=4 * GIB, gpus=_ranks_gpus()) == [True, True]


def test_allreduce_1gib_f32_bitwise_vs_oracle():
    from oracle import oracle as O
    from paper_2506_02486_b200 import collectives as coll
    from paper_2506_02486_b200.emulate import run_emulated
    count = GIB // 4
    contribs = [np.random.default_rng(1000 + r).uniform(-1, 1, count).astype(np.float32)
                for r in range(2)]
    want = O.allreduce_fold(contribs, "sum")
    op = coll.ReduceOp(coll.ReduceKind.Sum, coll.ElementType.f32)

    def fn(rt):
        comm = coll.bootstrap(rt, rt.world)
        send = rt.alloc_symmetric(GIB, 0)
        recv = rt.alloc_symmetric(GIB, 0)
        rt.gm.view(0, send.addr.offset, GIB)[:] = contribs[rt.rank].tobytes()
        coll.allreduce(comm, send.addr, recv.addr, count, op)
        return bytes(rt.gm.view(0, recv.addr.offset, GIB)) == want.tobytes()

    assert run_emulated(2, fn, segment_bytes=4 * GIB, gpus=_ranks_gpus()) == [True, True]
