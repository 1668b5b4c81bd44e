"""App-level properties from the reference selftest (selftest.py:451-484) on
the GPU build: Cannon residual / identity / overlap, benchmark accounting,
collective isolation between disjoint communicators."""

import numpy as np
import pytest

from conftest import NGPU, need_gpus

pytestmark = pytest.mark.gpu
MIB = 1 << 20


@pytest.mark.parametrize("n,p", [(48, 1), (48, 2), (256, 2), (96, 3), (512, 4),
                                 (25, 1), (90, 2), (75, 3), (132, 4)])
def test_cannon_residual(n, p):
    from paper_2506_02486_b200.apps.cannon import MatmulSpec, cannon_matmul
    from paper_2506_02486_b200.emulate import run_emulated
    seg = 1 << max(23, (4 * (n // p) * n * 8 * 2).bit_length())
    res = run_emulated(p, lambda rt: cannon_matmul(rt, MatmulSpec(n, p), seed=1), segment_bytes=seg)
    assert max(r.residual for r in res) <= 1e-12
    assert all(r.overlap_observed() for r in res)


def test_cannon_identity_exact():
    from paper_2506_02486_b200.apps.cannon import MatmulSpec, cannon_matmul
    from paper_2506_02486_b200.emulate import run_emulated
    res = run_emulated(2, lambda rt: cannon_matmul(rt, MatmulSpec(64, 2), seed=3, identity_b=True),
                       segment_bytes=8 * MIB)
    assert all(r.identity_exact for r in res)


@pytest.mark.parametrize("shift,ranks", [("ce", 2), ("fused", 2), ("ce", 4), ("fused", 4)])
def test_cannon_matches_host_blas_at_1024(shift, ranks, monkeypatch):
    """GPU ring product vs numpy (OpenBLAS) on the reference's own inputs, both
    shift engines (copy engine on a side stream / fused into the DMMA kernel);
    two back-to-back runs (stripes return home after P steps), so C = 2 A@B."""
    import torch

    from paper_2506_02486_b200.apps.cannon import CannonRing, MatmulSpec, _fill_matrices
    from paper_2506_02486_b200.emulate import run_emulated
    monkeypatch.setenv("DIOMP_CANNON_SHIFT", shift)
    n = 1024
    a, b = _fill_matrices(n, 0)
    want = 2.0 * (a @ b)

    def fn(rt):
        ring = CannonRing(rt, MatmulSpec(n, rt.nranks), a_full=a, b_full=b)
        mode = ring.shift
        rt.barrier(rt.world)
        ring.run()
        ring.run()
        rt.barrier(rt.world)
        out = {e: st["c"].cpu().numpy() for e, st in ring.local.items()}
        ring.release()
        return out, mode

    res = run_emulated(ranks, fn, segment_bytes=64 * MIB)
    if NGPU >= ranks:
        assert all(m == shift for _, m in res)
    ns = n // ranks
    got = np.concatenate([res[r][0][r] for r in range(ranks)])
    assert got.shape == (n, n) and ns * ranks == n
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert rel <= 1e-14, rel


def test_benchmark_accounting_and_csv():
    from paper_2506_02486_b200.apps import bench as B
    from paper_2506_02486_b200.emulate import run_emulated

    def fn(rt):
        rows = B.run_p2p(rt, B.BenchSpec(B.BenchKind.PutLatency, (64, 1024), iters=5, warmup=1))
        if rt.rank == 0:
            for row in rows:
                assert row.wire_put_bytes == row.size_bytes * row.iters
        return B.to_csv(rows)

    out = run_emulated(2, fn, segment_bytes=4 * MIB)
    lines = out[0].strip().splitlines()
    assert lines[0] == "kind,size_bytes,iters,mean_us,bw_MiBs"
    assert len(lines) == 3 and lines[1].startswith("put,64,5,")


@pytest.mark.parametrize("kind", ["bw", "get_bw", "put", "get"])
def test_p2p_bench_asymmetric_target(kind):
    """configs[1] asymmetric leg: rank 0 reaches rank 1's asymmetric payload
    through resolve_cell (byte exactness of asymmetric puts/gets:
    test_gpu_rma.py)."""
    from paper_2506_02486_b200.apps import bench as B
    from paper_2506_02486_b200.emulate import run_emulated
    from paper_2506_02486_b200.global_memory import TransferKind

    def fn(rt):
        spec = B.BenchSpec(B.BenchKind(kind), (8, 4096, 65536), iters=3, warmup=1,
                           transfer=TransferKind.D2D, allocation="asymmetric")
        rows = B.run_p2p(rt, spec)
        return [(r.kind, r.size_bytes, r.iters) for r in rows]

    out = run_emulated(2, fn, segment_bytes=4 * MIB)
    assert out[0] == [(f"{kind}_d2d_asym", n, 3) for n in (8, 4096, 65536)]
    assert out[1] == []


def test_collective_bench_rows():
    from paper_2506_02486_b200.apps import bench as B
    from paper_2506_02486_b200.emulate import run_emulated

    def fn(rt):
        return B.run_collective(rt, B.BenchSpec(B.BenchKind.Allreduce, (4096, 65536), iters=3,
                                                warmup=1))

    out = run_emulated(2, fn, segment_bytes=4 * MIB)
    assert [r.size_bytes for r in out[0]] == [4096, 65536] and out[1] == []


def test_collective_isolation_disjoint_communicators():
    from paper_2506_02486_b200 import collectives as coll
    from paper_2506_02486_b200.emulate import run_emulated

    def fn(rt):
        pair = (0, 1) if rt.rank < 2 else (2, 3)
        g = rt.group_create([rt.endpoint(pair[0], 0), rt.endpoint(pair[1], 0)])
        comm = coll.bootstrap(rt, g)
        rec = rt.alloc_symmetric(8192, 0)
        fill = pair[0] + 1
        if rt.rank == pair[0]:
            rt.gm.view(0, rec.addr.offset, 8192)[:] = bytes([fill]) * 8192
        coll.bcast(comm, rec.addr, 8192, root=0)
        assert bytes(rt.gm.view(0, rec.addr.offset, 8192)) == bytes([fill]) * 8192
        return True

    assert run_emulated(4, fn, segment_bytes=2 * MIB) == [True] * 4


def test_device_bcast_caches_one_communicator():
    from paper_2506_02486_b200 import collectives as coll
    from paper_2506_02486_b200.emulate import run_emulated

    def fn(rt):
        rec = rt.alloc_symmetric(4096, 0)
        if rt.rank == 0:
            rt.gm.view(0, rec.addr.offset, 4096)[:] = b"\x07" * 4096
        for _ in range(3):
            coll.device_bcast(rt, rec.addr, 4096, rt.world)
        boots = rt.bootstrap_count
        assert bytes(rt.gm.view(0, rec.addr.offset, 4096)) == b"\x07" * 4096
        sub = rt.group_create([rt.endpoint(r, 0) for r in range(rt.nranks)])
        coll.device_bcast(rt, rec.addr, 4096, sub)
        rt.group_free(sub)
        assert sub.id not in rt.comm_cache
        return boots

    assert run_emulated(2, fn, segment_bytes=2 * MIB) == [1, 1]


def test_group_split_and_world_shapes():
    from paper_2506_02486_b200.emulate import run_emulated

    def fn(rt):
        g = rt.group_split(rt.world, color=rt.rank // 2, key=rt.rank)
        rev = rt.group_split(rt.world, color=0, key=-rt.rank)
        return (g.id, tuple(ep.rank for ep in g.members), rev.id,
                tuple(ep.rank for ep in rev.members), len(rt.world.members))

    out = run_emulated(4, fn, segment_bytes=2 * MIB)
    assert out[0][1] == out[1][1] == (0, 1) and out[2][1] == out[3][1] == (2, 3)
    assert out[0][0] == out[1][0] != out[2][0]
    assert out[0][3] == (3, 2, 1, 0) and len({o[2] for o in out}) == 1
    assert all(o[4] == 4 for o in out)


def test_public_init_singleton(monkeypatch):
    import paper_2506_02486_b200 as d
    monkeypatch.setenv("DIOMP_NRANKS", "1")
    monkeypatch.setenv("DIOMP_SEGMENT_BYTES", str(2 * MIB))
    monkeypatch.setenv("DIOMP_GPUS", "0")
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    rt = d.init()
    try:
        with pytest.raises(d.DiompError):
            d.init()
    finally:
        d.finalize()
    rt2 = d.init()
    d.finalize(rt2)
    assert rt2.finalized
