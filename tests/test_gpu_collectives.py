"""Collectives parity on the GPU: the CUDA kernels against the reference's own
results (tests/golden/collectives_golden.npz, produced by running the
reference's bcast/reduce/allreduce) -- bitwise, every dtype x op x k."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, NGPU, need_gpus

pytestmark = pytest.mark.gpu
MIB = 1 << 20
DT = {"f32": np.float32, "f64": np.float64, "i32": np.int32, "i64": np.int64}


def contrib(rank, etype, count, seed):
    """Same generator as tests/golden/make_golden.py."""
    rng = np.random.default_rng(seed * 100 + rank)
    if etype.startswith("f"):
        v = rng.uniform(-1, 1, count).astype(DT[etype])
        if count > 8:
            v[3] = np.nan if rank == 1 else v[3]
            v[5] = -0.0 if rank % 2 else 0.0
        return v
    return rng.integers(-2**30, 2**30, count).astype(DT[etype])


G = np.load(os.path.join(GOLDEN, "collectives_golden.npz"))
KEYS = sorted(G.files)


def _write(rt, rec, arr, device=0):
    rt.gm.view(device, rec.addr.offset, arr.nbytes)[:] = arr.view(np.uint8).tobytes()


def _read(rt, rec, dtype, count, device=0):
    return np.frombuffer(bytes(rt.gm.view(device, rec.addr.offset,
                                          count * np.dtype(dtype).itemsize)), dtype=dtype)


@pytest.mark.parametrize("key", [k for k in KEYS if int(k.split("_")[1]) <= 4]
                         + [k for k in KEYS if int(k.split("_")[1]) == 8][:12])
def test_reduce_allreduce_match_reference(key):
    from paper_2506_02486_b200 import collectives as coll
    from paper_2506_02486_b200.emulate import run_emulated
    which, k, et, kind, count, root, seed = key.split("_")
    k, count, root, seed = int(k), int(count), int(root), int(seed)
    op = coll.ReduceOp(coll.ReduceKind(kind), coll.ElementType(et))
    isz = np.dtype(DT[et]).itemsize

    def fn(rt):
        comm = coll.bootstrap(rt, rt.world)
        send = rt.alloc_symmetric(max(count * isz, 64), 0)
        recv = rt.alloc_symmetric(max(count * isz, 64), 0)
        _write(rt, send, contrib(rt.rank, et, count, seed))
        if which == "allreduce":
            coll.allreduce(comm, send.addr, recv.addr, count, op)
        else:
            coll.reduce(comm, send.addr, recv.addr, count, op, root=root)
        return _read(rt, recv, DT[et], count).tobytes()

    out = run_emulated(k, fn, segment_bytes=2 * MIB)
    want = G[key].tobytes()
    if which == "allreduce":
        assert all(o == want for o in out)
    else:
        assert out[root] == want


def test_bcast_root_snapshot_sizes_and_roots():
    from paper_2506_02486_b200 import GlobalAddress
    from paper_2506_02486_b200 import collectives as coll
    from paper_2506_02486_b200.emulate import run_emulated
    sizes = [1, 100, 128 * 1024, MIB + 7, 4 * MIB + 13]
    roots = [0, 3, 1, 2, 1]

    def fn(rt):
        comm = coll.bootstrap(rt, rt.world)
        buf = rt.alloc_symmetric(8 * MIB, 0)
        out = []
        for size, root in zip(sizes, roots):
            mine = np.random.default_rng(1000 + size + rt.rank).integers(0, 256, size,
                                                                         dtype=np.uint8)
            rt.gm.view(0, buf.addr.offset + 3, size)[:] = mine.tobytes()
            coll.bcast(comm, GlobalAddress(rt.rank, 0, buf.addr.offset + 3), size, root=root)
            out.append((mine.tobytes() if rt.rank == root else None,
                        bytes(rt.gm.view(0, buf.addr.offset + 3, size))))
        return out

    res = run_emulated(4, fn, segment_bytes=32 * MIB)
    for i in range(len(sizes)):
        snap = next(r[i][0] for r in res if r[i][0] is not None)
        assert all(r[i][1] == snap for r in res)


def test_allreduce_in_place_and_big_count():
    from oracle import oracle as O
    from paper_2506_02486_b200 import collectives as coll
    from paper_2506_02486_b200.emulate import run_emulated
    count = 3 * MIB // 8 + 5
    op = coll.ReduceOp(coll.ReduceKind.Sum, coll.ElementType.f64)

    def fn(rt):
        comm = coll.bootstrap(rt, rt.world)
        buf = rt.alloc_symmetric(count * 8, 0)
        _write(rt, buf, np.random.default_rng(50 + rt.rank).uniform(-1, 1, count))
        coll.allreduce(comm, buf.addr, buf.addr, count, op)
        return _read(rt, buf, np.float64, count).tobytes()

    out = run_emulated(3, fn, segment_bytes=64 * MIB)
    want = O.allreduce_fold([np.random.default_rng(50 + r).uniform(-1, 1, count)
                             for r in range(3)], "sum").tobytes()
    assert all(o == want for o in out)


@need_gpus(2)
def test_device_flag_mode_back_to_back():
    """Ranks on distinct GPUs: entry/exit flags, many consecutive collectives
    (the reference deadlocks here without a barrier between reps)."""
    from oracle import oracle as O
    from paper_2506_02486_b200 import collectives as coll
    from paper_2506_02486_b200.emulate import run_emulated
    k = min(NGPU, 4)
    count = 100_003
    op = coll.ReduceOp(coll.ReduceKind.Sum, coll.ElementType.f32)

    def fn(rt):
        comm = coll.bootstrap(rt, rt.world)
        assert comm.device_sync
        send = rt.alloc_symmetric(count * 4, 0)
        recv = rt.alloc_symmetric(count * 4, 0)
        outs = []
        for rep in range(20):
            _write(rt, send, np.random.default_rng(rep * 10 + rt.rank).uniform(-1, 1, count)
                   .astype(np.float32))
            coll.allreduce(comm, send.addr, recv.addr, count, op)
            outs.append(_read(rt, recv, np.float32, count).tobytes())
            coll.bcast(comm, recv.addr, count * 4, root=rep % k)
        return outs

    res = run_emulated(k, fn, segment_bytes=8 * MIB)
    for rep in range(20):
        want = O.allreduce_fold([np.random.default_rng(rep * 10 + r).uniform(-1, 1, count)
                                 .astype(np.float32) for r in range(k)], "sum").tobytes()
        assert all(r[rep] == want for r in res)


@need_gpus(2)
def test_ll_bcast_root_never_overruns_a_slow_peer():
    """A bcast root gets no words back from its peers, so without the
    acknowledgement bank it could run two LL calls ahead and overwrite a
    parity slot a slow peer has not read yet (the peer would then wait on an
    epoch that no longer exists).  Rank 1 dawdles on the host between calls
    while rank 0 issues blocking small bcasts back to back; every payload
    must arrive intact, interleaved with LL allreduces."""
    import time

    from paper_2506_02486_b200 import collectives as coll
    from paper_2506_02486_b200.emulate import run_emulated
    op = coll.ReduceOp(coll.ReduceKind.Sum, coll.ElementType.i32)

    def fn(rt):
        comm = coll.bootstrap(rt, rt.world)
        assert comm.device_sync
        buf = rt.alloc_symmetric(64 * 1024, 0)
        acc = rt.alloc_symmetric(4096, 0)
        rng = np.random.default_rng(31)
        bad = 0
        for i in range(150):
            size = int(rng.integers(1, 40000))
            if rt.rank == 0:
                rt.gm.view(0, buf.addr.offset, size)[:] = bytes([(i * 7 + j) & 255 for j in range(64)]) * (size // 64) + bytes((i * 7 + j) & 255 for j in range(size % 64))
            elif i % 3 == 0:
                time.sleep(0.002)   # the peer falls behind the root
            coll.bcast(comm, buf.addr, size, root=0)
            want = bytes([(i * 7 + j) & 255 for j in range(64)]) * (size // 64) + bytes((i * 7 + j) & 255 for j in range(size % 64))
            if bytes(rt.gm.view(0, buf.addr.offset, size)) != want:
                bad += 1
            if i % 10 == 9:
                coll.allreduce(comm, acc.addr, acc.addr, 100, op)
        return bad

    assert run_emulated(2, fn, segment_bytes=16 * MIB) == [0, 0]


_EXPERIMENTS = pytest.mark.skipif(
    not __import__("paper_2506_02486_b200._native", fromlist=["x"]).has_experiments(),
    reason="experiments build only (-DDIOMP_EXPERIMENTS)")


@need_gpus(3)
@_EXPERIMENTS
@pytest.mark.parametrize("pull", [0, 1])
def test_bcast_chain_device_flags(pull):
    """Chain bcast (k >= 3, per-CTA progress flags), push and pull flavours:
    every member ends with
    the root's bytes -- odd sizes and offsets, every root, repeated, mixed with
    pull+push bcasts and allreduces so the progress-flag values must stay
    monotone across calls and algorithms."""
    from paper_2506_02486_b200 import GlobalAddress, _native
    from paper_2506_02486_b200 import collectives as coll
    from paper_2506_02486_b200.emulate import run_emulated
    k = min(NGPU, 4)
    plan = [(4096 + 5, 0, 0), (MIB + 7, 1, 0), (24 * MIB + 13, 2, 0), (777, 0, 1 << 62),
            (3 * MIB, k - 1, 0), (24 * MIB + 13, 0, 0), (5 * MIB + 1, 1, 1 << 62),
            (24 * MIB + 13, k - 1, 0)]
    op = coll.ReduceOp(coll.ReduceKind.Sum, coll.ElementType.i32)

    def fn(rt):
        comm = coll.bootstrap(rt, rt.world)
        assert comm.device_sync
        buf = rt.alloc_symmetric(32 * MIB, 0)
        acc = rt.alloc_symmetric(4096, 0)
        out = []
        for i, (size, root, chain_min) in enumerate(plan):
            _native.call("diomp_set_bcast_chain_min", chain_min)
            mine = np.random.default_rng(7000 + 13 * i + rt.rank).integers(0, 256, size,
                                                                           dtype=np.uint8)
            at = GlobalAddress(rt.rank, 0, buf.addr.offset + 3)
            rt.gm.view(0, at.offset, size)[:] = mine.tobytes()
            coll.bcast(comm, at, size, root=root)
            out.append((mine.tobytes() if rt.rank == root else None,
                        bytes(rt.gm.view(0, at.offset, size))))
            coll.allreduce(comm, acc.addr, acc.addr, 1000, op)
        return out

    _native.call("diomp_set_bcast_pullchain", pull)
    try:
        res = run_emulated(k, fn, segment_bytes=128 * MIB)
    finally:
        _native.call("diomp_set_bcast_chain_min", (1 << 64) - 1)
        _native.call("diomp_set_bcast_pullchain", 0)
    for i in range(len(plan)):
        snap = next(r[i][0] for r in res if r[i][0] is not None)
        assert all(r[i][1] == snap for r in res), i


@need_gpus(2)
@pytest.mark.parametrize("ce_min", [None, pytest.param(8 * MIB, marks=_EXPERIMENTS)])
def test_allreduce_device_flag_algorithms_bitwise(ce_min):
    """Device-flag rings, both allreduce algorithms (fused; fold + copy-engine
    push from ce_min bytes): bitwise equal to the reference fold order, odd
    counts, offsets that are not 16-byte aligned, in place and out of place,
    back to back."""
    from oracle import oracle as O
    from paper_2506_02486_b200 import GlobalAddress
    from paper_2506_02486_b200 import collectives as coll
    from paper_2506_02486_b200.emulate import run_emulated
    k = min(NGPU, 4)
    cases = [("f32", "sum", (16 * MIB) // 4 + 3, 4), ("f64", "sum", 3 * MIB + 1, 8),
             ("i32", "max", 4 * MIB + 5, 12), ("f32", "min", 1000, 0), ("i64", "sum", MIB + 7, 0)]

    def contrib(r, et, count, i):
        rng = np.random.default_rng(900 + 10 * i + r)
        if et[0] == "f":
            return rng.uniform(-1, 1, count).astype(DT[et])
        return rng.integers(-2**30, 2**30, count).astype(DT[et])

    def fn(rt):
        comm = coll.bootstrap(rt, rt.world)
        assert comm.device_sync
        send = rt.alloc_symmetric(25 * MIB, 0)
        recv = rt.alloc_symmetric(25 * MIB, 0)
        outs = []
        for i, (et, kind, count, delta) in enumerate(cases):
            op = coll.ReduceOp(coll.ReduceKind(kind), coll.ElementType(et))
            isz = np.dtype(DT[et]).itemsize
            s = GlobalAddress(rt.rank, 0, send.addr.offset + delta)
            for in_place in (False, True):
                r = s if in_place else GlobalAddress(rt.rank, 0, recv.addr.offset + delta)
                v = contrib(rt.rank, et, count, i)
                rt.gm.view(0, s.offset, v.nbytes)[:] = v.tobytes()
                coll.allreduce(comm, s, r, count, op)
                outs.append(bytes(rt.gm.view(0, r.offset, count * isz)))
        return outs

    from paper_2506_02486_b200 import _native
    if ce_min is not None:
        _native.call("diomp_set_allreduce_ce_min", ce_min)
    try:
        res = run_emulated(k, fn, segment_bytes=256 * MIB)
    finally:
        if ce_min is not None:
            _native.call("diomp_set_allreduce_ce_min", (1 << 64) - 1)
    j = 0
    for i, (et, kind, count, delta) in enumerate(cases):
        want = O.allreduce_fold([contrib(r, et, count, i) for r in range(k)], kind).tobytes()
        for _ in (False, True):
            assert all(out[j] == want for out in res), (et, kind, count, delta)
            j += 1


@need_gpus(2)
@_EXPERIMENTS
def test_allreduce_nvls_in_switch(monkeypatch):
    """NVSwitch multicast allreduce (algorithm="nvls"): integer sum/min/max
    bitwise equal to the reference fold, float sums within the north-star
    tolerance (rel-L2 1e-6 f32, 1e-12 f64); several rounds through a small
    window, in place, back to back with the exact algorithm; float min/max
    refused."""
    from oracle import oracle as O
    from paper_2506_02486_b200 import collectives as coll
    from paper_2506_02486_b200 import nvls
    from paper_2506_02486_b200.emulate import run_emulated
    import torch
    if not all(nvls.supported(g) for g in range(NGPU)):
        pytest.skip("no NVSwitch multicast on this box")
    monkeypatch.setenv("DIOMP_NVLS_WINDOW", str(2 * MIB))   # rounds of <= 2 MiB (+ header)
    k = min(NGPU, 4)
    cases = [("f32", "sum", 3 * MIB // 4 + 5), ("f64", "sum", MIB // 8 + 3),
             ("i32", "sum", MIB + 1), ("i32", "min", 1001), ("i64", "max", 70_001),
             ("i64", "sum", 3), ("f32", "sum", 1)]

    def contrib(r, et, count, i):
        rng = np.random.default_rng(700 + 10 * i + r)
        if et[0] == "f":
            return rng.uniform(-1, 1, count).astype(DT[et])
        return rng.integers(-2**28, 2**28, count).astype(DT[et])

    def fn(rt):
        comm = coll.bootstrap(rt, rt.world)
        buf = rt.alloc_symmetric(8 * MIB, 0)
        out = rt.alloc_symmetric(8 * MIB, 0)
        res = []
        for i, (et, kind, count) in enumerate(cases):
            op = coll.ReduceOp(coll.ReduceKind(kind), coll.ElementType(et))
            v = contrib(rt.rank, et, count, i)
            _write(rt, buf, v)
            in_place = i % 2 == 1
            dst = buf if in_place else out
            coll.allreduce(comm, buf.addr, dst.addr, count, op, algorithm="nvls")
            res.append(_read(rt, dst, DT[et], count).copy())
            _write(rt, buf, v)
            coll.allreduce(comm, buf.addr, out.addr, count, op)          # exact, same comm
            res.append(_read(rt, out, DT[et], count).copy())
        with pytest.raises(coll.TypeMismatch):
            coll.allreduce(comm, buf.addr, out.addr, 8,
                           coll.ReduceOp(coll.ReduceKind.Min, coll.ElementType.f32),
                           algorithm="nvls")
        return res

    got = run_emulated(k, fn, segment_bytes=64 * MIB)
    for i, (et, kind, count) in enumerate(cases):
        want = O.allreduce_fold([contrib(r, et, count, i) for r in range(k)], kind)
        for g in got:
            nv, ex = g[2 * i], g[2 * i + 1]
            assert ex.tobytes() == want.tobytes(), (et, kind, "exact")
            if et[0] == "i":
                assert nv.tobytes() == want.tobytes(), (et, kind, "nvls")
            else:
                tol = 1e-6 if et == "f32" else 1e-12
                w64 = want.astype(np.float64)
                err = np.linalg.norm(nv.astype(np.float64) - w64) / max(np.linalg.norm(w64), 1e-300)
                assert err <= tol, (et, kind, err)
    _ = torch


@need_gpus(2)
def test_absent_peer_surfaces_transport_failure_at_the_deadline():
    """Peer-failure analogue of the reference's test_transport.py:221-259 and
    its per-wait deadlines (config.py:20, 120): rank 1 never enters the
    collective, so rank 0's device-side entry wait gives up at its deadline
    and the call raises TransportFailure instead of hanging the GPU."""
    import time

    from paper_2506_02486_b200 import _native, errors
    from paper_2506_02486_b200 import collectives as coll
    from paper_2506_02486_b200.emulate import run_emulated
    op = coll.ReduceOp(coll.ReduceKind.Sum, coll.ElementType.f32)
    count = 1024

    def fn(rt):
        comm = coll.bootstrap(rt, rt.world)
        buf = rt.alloc_symmetric(count * 4, 0)
        out = None
        if rt.rank == 0:
            assert comm.device_sync
            _native.call("diomp_set_wait_timeout", rt.gpus[0], 0.5)
            t0 = time.perf_counter()
            try:
                coll.allreduce(comm, buf.addr, buf.addr, count, op)
                out = ("no error", 0.0)
            except errors.TransportFailure:
                out = ("TransportFailure", time.perf_counter() - t0)
            finally:
                _native.call("diomp_set_wait_timeout", rt.gpus[0], float(rt.cfg.timeout))
        rt.barrier(rt.world)   # rank 1's segment stays mapped until rank 0 is done
        return out

    res = run_emulated(2, fn, segment_bytes=64 * MIB, timeout=30.0)
    assert res[0][0] == "TransportFailure", res[0]
    assert 0.4 < res[0][1] < 10.0, res[0]


@need_gpus(2)
def test_small_message_ll_path_bitwise_back_to_back():
    """One-shot LL collectives (payload + flag in one 8-byte store, no
    handshakes) for small messages: bitwise equal to the reference fold for
    every dtype/op, in place and out of place, 300 back-to-back non-blocking
    calls interleaved with two-phase (large) allreduces and LL / two-phase
    bcasts -- the LL slot parities and the two-phase exit bookkeeping must
    never let a call see another call's bytes."""
    from oracle import oracle as O
    from paper_2506_02486_b200 import GlobalAddress
    from paper_2506_02486_b200 import collectives as coll
    from paper_2506_02486_b200.emulate import run_emulated
    k = min(NGPU, 4)
    plan = []
    for i in range(300):
        et = ("f32", "f64", "i32", "i64")[i % 4]
        kind = ("sum", "min", "max")[i % 3]
        count = (1, 3, 257, 1000, 4093, 300_001)[i % 6]
        plan.append((et, kind, count, i % 5 == 0))

    def contrib(r, et, count, i):
        rng = np.random.default_rng(4000 + 7 * i + r)
        if et[0] == "f":
            return rng.uniform(-1, 1, count).astype(DT[et])
        return rng.integers(-2**30, 2**30, count).astype(DT[et])

    def fn(rt):
        comm = coll.bootstrap(rt, rt.world)
        assert comm.device_sync
        bufs = [rt.alloc_symmetric(3 * MIB, 0) for _ in range(6)]
        bc = rt.alloc_symmetric(64 * 1024, 0)
        outs = []
        for i, (et, kind, count, in_place) in enumerate(plan):
            op = coll.ReduceOp(coll.ReduceKind(kind), coll.ElementType(et))
            isz = np.dtype(DT[et]).itemsize
            send = bufs[(2 * i) % 6]
            recv = send if in_place else bufs[(2 * i + 1) % 6]
            v = contrib(rt.rank, et, count, i)
            rt.gm.view(0, send.addr.offset, v.nbytes)[:] = v.tobytes()
            coll.allreduce(comm, send.addr, recv.addr, count, op, blocking=False)
            if i % 7 == 3:   # an LL-sized bcast from a rotating root
                nb = 1 + (i * 37) % 5000
                root = i % comm.size
                mine = np.random.default_rng(9000 + i + rt.rank).integers(
                    0, 256, nb, dtype=np.uint8)
                coll.complete(comm)
                rt.gm.view(0, bc.addr.offset, nb)[:] = mine.tobytes()
                coll.bcast(comm, bc.addr, nb, root=root)
                outs.append(("bc", i, mine.tobytes() if rt.rank == root else None,
                             bytes(rt.gm.view(0, bc.addr.offset, nb))))
            coll.complete(comm)
            outs.append(("ar", i, bytes(rt.gm.view(0, recv.addr.offset, count * isz))))
        return outs

    res = run_emulated(k, fn, segment_bytes=64 * MIB)
    for j, item in enumerate(res[0]):
        if item[0] == "ar":
            _, i, _ = item
            et, kind, count, _ = plan[i]
            want = O.allreduce_fold([contrib(r, et, count, i) for r in range(k)], kind).tobytes()
            assert all(r[j][2] == want for r in res), (i, et, kind, count)
        else:
            snap = next(r[j][2] for r in res if r[j][2] is not None)
            assert all(r[j][3] == snap for r in res), item[1]
