"""Runtime lifecycle, groups, barrier and fence semantics on the GPU runtime
(the properties of reference pkg/tests/test_runtime_groups.py; runtime.py:
186-238 groups, 493-556 barrier/fence, 558-583 finalize), run as thread-ranks
through emulate.run_emulated."""

import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
MIB = 1 << 20


def emu(n, fn, **kw):
    from paper_2506_02486_b200.emulate import run_emulated
    kw.setdefault("segment_bytes", 2 * MIB)
    return run_emulated(n, fn, **kw)


def test_world_members_per_device():
    got = emu(1, lambda rt: [(e.rank, e.device) for e in rt.world.members], devices_per_rank=4)
    assert got[0] == [(0, d) for d in range(4)]
    assert emu(3, lambda rt: len(rt.world.members)) == [3, 3, 3]


def test_finalize_is_idempotent_and_fences():
    import paper_2506_02486_b200 as d

    def fn(rt):
        rec = rt.alloc_symmetric(4096, 0)
        if rt.rank == 0:
            rt.put(rt.translate(rec.addr, 1), b"FINALBYTES", 10, d.TransferKind.H2D)
            rt.finalize()
            rt.finalize()
            return rt.finalized
        # rank 0's finalize fenced the put before blocking in its barrier,
        # which pairs with this rank's own finalize (run by the emulator)
        deadline = time.monotonic() + 20
        while bytes(rt.gm.view(0, rec.addr.offset, 10)) != b"FINALBYTES":
            assert time.monotonic() < deadline
            time.sleep(0.01)
        return bytes(rt.gm.view(0, rec.addr.offset, 10))

    out = emu(2, fn)
    assert out == [True, b"FINALBYTES"]


def test_group_create_ids_and_membership():
    from paper_2506_02486_b200.errors import CollectiveMismatch

    def fn(rt):
        everyone = rt.group_create([rt.endpoint(r, 0) for r in reversed(range(4))])
        assert [e.rank for e in everyone.members] == [0, 1, 2, 3]
        assert everyone.id not in (0, rt.world.id)
        lo = rt.rank < 2
        pair = rt.group_create([rt.endpoint(r, 0) for r in ((0, 1) if lo else (2, 3))])
        if rt.rank == 0:
            with pytest.raises(CollectiveMismatch):
                rt.group_create([rt.endpoint(3, 0)])
        return everyone.id, pair.id, tuple(e.rank for e in pair.members)

    out = emu(4, fn)
    assert len({o[0] for o in out}) == 1
    assert out[0][1] == out[1][1] != out[2][1] == out[3][1]
    assert out[1][2] == (0, 1) and out[3][2] == (2, 3)


def test_group_merge_is_local_set_union():
    def fn(rt):
        solo = rt.group_create([rt.endpoint(rt.rank, 0)])
        same = rt.group_merge(solo, solo)
        assert same.members == solo.members and same.id != solo.id
        assert rt.group_merge(solo, rt.world).members == rt.world.members
        eps = [rt.endpoint(r, 0) for r in range(4)]
        ab = rt.group_create(eps[:2]) if rt.rank < 2 else None
        bc = rt.group_create(eps[1:3]) if rt.rank in (1, 2) else None
        cd = rt.group_create(eps[2:]) if rt.rank >= 2 else None
        if rt.rank == 1:
            assert {e.rank for e in rt.group_merge(ab, bc).members} == {0, 1, 2}
        if rt.rank == 2:
            assert {e.rank for e in rt.group_merge(bc, cd).members} == {1, 2, 3}
        rt.barrier(rt.world)
        return True

    assert emu(4, fn) == [True] * 4


def test_freed_group_is_stale():
    from paper_2506_02486_b200.errors import StaleGroup

    def fn(rt):
        g = rt.group_create([rt.endpoint(rt.rank, 0)])
        rt.group_free(g)
        for op in (lambda: rt.group_merge(g, rt.world), lambda: rt.barrier(g),
                   lambda: rt.group_free(g)):
            with pytest.raises(StaleGroup):
                op()
        with pytest.raises(StaleGroup):
            rt.group_free(rt.world)
        return True

    assert emu(2, fn) == [True, True]


def test_group_split_matches_sort_oracle():
    rng = np.random.default_rng(7)
    cases = [(rng.integers(0, 3, 4).tolist(), rng.integers(-4, 4, 4).tolist())
             for _ in range(16)]

    def fn(rt):
        return [(g.id, tuple((e.rank, e.device) for e in g.members))
                for g in (rt.group_split(rt.world, c[rt.rank], k[rt.rank]) for c, k in cases)]

    res = emu(4, fn)
    for i, (colors, keys) in enumerate(cases):
        for r in range(4):
            peers = [q for q in range(4) if colors[q] == colors[r]]
            want = tuple((q, 0) for q in sorted(peers, key=lambda q: (keys[q], q)))
            assert res[r][i][1] == want
            assert len({res[q][i][0] for q in peers}) == 1


def test_group_tables_identical_across_ranks():
    rng = np.random.default_rng(3)
    layouts = [rng.integers(0, 2, 4).tolist() for _ in range(20)]

    def fn(rt):
        rows = []
        for devs in layouts:
            g = rt.group_create([rt.endpoint(r, dv) for r, dv in enumerate(devs)])
            rows.append((g.id, tuple(e.key() for e in g.members)))
        return repr(rows)

    assert len(set(emu(4, fn, devices_per_rank=2))) == 1


def test_barrier_and_fence_timing():
    def fn(rt):
        g = rt.group_create([rt.endpoint(rt.rank, 0)])
        t0 = time.perf_counter()
        rt.barrier(g)
        rt.fence(rt.world)
        quick = time.perf_counter() - t0
        time.sleep(0.2 if rt.rank == 2 else 0.0)
        t_in = time.perf_counter()
        rt.barrier(rt.world)
        return quick, t_in, time.perf_counter()

    out = emu(3, fn)
    assert max(o[0] for o in out) < 0.05
    last = max(o[1] for o in out)
    assert all(o[2] >= last - 1e-4 for o in out)


def test_fence_drains_plain_and_stream_bound_puts():
    import paper_2506_02486_b200 as d

    def fn(rt):
        pool = rt.pools[0]
        streams = [pool.acquire() for _ in range(4)]
        plain = rt.alloc_symmetric(64 * 1024, 0)
        bound = rt.alloc_symmetric(64 * 1024, 0, stream=streams[0])
        if rt.rank == 0:
            for i in range(48):
                off = 128 * i
                if i % 2:
                    dst = rt.translate(plain.addr, 1)
                    rt.put(d.GlobalAddress(1, 0, dst.offset + off), bytes([i]) * 128, 128,
                           d.TransferKind.H2D)
                else:
                    dst = rt.translate(bound.addr, 1)
                    rt.put(d.GlobalAddress(1, 0, dst.offset + off), bytes([i]) * 128, 128,
                           d.TransferKind.H2D, stream=streams[0])
                if i % 6 == 0:
                    streams[i % 4].submit(lambda: time.sleep(0.001))
            rt.fence(rt.world)
            assert rt.outstanding_rma(rt.world) == 0
            assert rt.outstanding_stream_events(rt.world) == 0
        rt.barrier(rt.world)
        ok = True
        if rt.rank == 1:
            for i in range(48):
                rec = plain if i % 2 else bound
                ok &= bytes(rt.gm.view(0, rec.addr.offset + 128 * i, 128)) == bytes([i]) * 128
        for s in streams:
            pool.release(s)
        return ok

    assert emu(2, fn, sim_task_us=200) == [True, True]


def test_stream_bound_allocation_requires_its_stream():
    import paper_2506_02486_b200 as d
    from paper_2506_02486_b200.errors import StreamMismatch

    def fn(rt):
        s, other = rt.pools[0].acquire(), rt.pools[0].acquire()
        rec = rt.alloc_symmetric(4096, 0, stream=s)
        dst = rt.translate(rec.addr, rt.rank)
        for wrong in (None, other):
            with pytest.raises(StreamMismatch):
                rt.put(dst, b"x" * 16, 16, d.TransferKind.H2D, stream=wrong)
        rt.put(dst, b"bound-stream-ok!", 16, d.TransferKind.H2D, stream=s).wait(10)
        got = bytes(rt.gm.view(0, rec.addr.offset, 16))
        rt.pools[0].release(s)
        rt.pools[0].release(other)
        return got

    assert emu(1, fn) == [b"bound-stream-ok!"]
