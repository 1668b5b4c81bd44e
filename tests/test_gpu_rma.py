"""One-sided put/get on the GPU: byte-exact round trips over every kind and
path (test_transport.py:28-70 pattern), asymmetric two-step access, and the
range checks."""

import numpy as np
import pytest

from conftest import NGPU

pytestmark = pytest.mark.gpu
MIB = 1 << 20
SIZES = [0, 1, 3, 4, 64, 4096, 8192, 65536 + 5, 3 * MIB + 17]


def roundtrip_worker(rt):
    import paper_2506_02486_b200 as d
    rec0 = rt.alloc_symmetric(4 * MIB, 0)
    stage = rt.alloc_symmetric(4 * MIB, 0)
    rt.barrier(rt.world)
    if rt.rank == 0:
        rng = np.random.default_rng(1)
        targets = [rt.translate(rec0.addr, 0), rt.translate(rec0.addr, 1)]
        for size in SIZES:
            data = rng.integers(0, 256, size, dtype=np.uint8).tobytes()
            for dst in targets:
                rt.put(dst, data, size, d.TransferKind.H2D)
                rt.fence(rt.world)
                back = bytearray(size)
                rt.get(dst, back, size, d.TransferKind.D2H).wait(20)
                assert bytes(back) == data, f"H2D/D2H {dst} size {size}"
                if size:
                    rt.gm.view(0, stage.addr.offset, size)[:] = data
                rt.put(dst, d.GlobalAddress(0, 0, stage.addr.offset), size, d.TransferKind.D2D)
                rt.fence(rt.world)
                if size:
                    rt.gm.view(0, stage.addr.offset, size)[:] = bytes(size)
                rt.get(dst, d.GlobalAddress(0, 0, stage.addr.offset), size,
                       d.TransferKind.D2D).wait(20)
                assert bytes(rt.gm.view(0, stage.addr.offset, size)) == data, \
                    f"D2D/D2D {dst} size {size}"
    rt.barrier(rt.world)
    return True


def test_roundtrips_two_ranks():
    from paper_2506_02486_b200.emulate import run_emulated
    assert run_emulated(2, roundtrip_worker, segment_bytes=32 * MIB) == [True, True]


@pytest.mark.parametrize("size", [65536 + 5, 16 * MIB + 3, 16 * MIB + 4096])
@pytest.mark.parametrize("offs", [(0, 0), (3, 3), (5, 9)])
def test_remote_engines_byte_exact(size, offs, monkeypatch):
    """The engines a peer GPU selects -- copy-engine put (>= 64 KiB) and the
    bulk-async TMA get (>= 16 MiB, same alignment mod 16) -- forced on this box
    (DIOMP_FORCE_REMOTE=1), byte-exact incl. unaligned heads/tails and the
    misaligned-pair fallback."""
    import torch

    import paper_2506_02486_b200 as d
    from paper_2506_02486_b200.emulate import run_emulated
    monkeypatch.setenv("DIOMP_FORCE_REMOTE", "1")
    so, do = offs

    def fn(rt):
        src = rt.alloc_symmetric(size + 64, 0)
        dst = rt.alloc_symmetric(size + 64, 0)
        back = rt.alloc_symmetric(size + 64, 0)
        ok = True
        if rt.rank == 0:
            arena = rt.gm.arena(0)
            g = torch.Generator(device=arena.device).manual_seed(size + so)
            data = torch.randint(0, 256, (size,), dtype=torch.uint8, device=arena.device,
                                 generator=g)
            arena[src.addr.offset + so:src.addr.offset + so + size] = data
            torch.cuda.synchronize(arena.device)
            rt.put(d.GlobalAddress(1, 0, dst.addr.offset + do),
                   d.GlobalAddress(0, 0, src.addr.offset + so), size, d.TransferKind.D2D)
            rt.fence(rt.world)
            rt.get(d.GlobalAddress(1, 0, dst.addr.offset + do),
                   d.GlobalAddress(0, 0, back.addr.offset + so), size, d.TransferKind.D2D).wait(30)
            got = arena[back.addr.offset + so:back.addr.offset + so + size]
            ok = bool(torch.equal(got, data))
        rt.barrier(rt.world)
        return ok

    assert run_emulated(2, fn, segment_bytes=256 * MIB) == [True, True]


def test_misaligned_offsets_byte_exact():
    import paper_2506_02486_b200 as d
    from paper_2506_02486_b200.emulate import run_emulated

    def fn(rt):
        rec = rt.alloc_symmetric(MIB, 0)
        if rt.rank == 0:
            src = rt.alloc_symmetric(MIB, 0)
        else:
            src = rt.alloc_symmetric(MIB, 0)
        if rt.rank == 0:
            data = np.random.default_rng(3).integers(0, 256, 100_001, dtype=np.uint8).tobytes()
            rt.gm.view(0, src.addr.offset + 5, len(data))[:] = data
            for so, do in [(5, 5), (5, 9), (5, 12)]:
                dst = d.GlobalAddress(1, 0, rec.addr.offset + do)
                rt.put(dst, d.GlobalAddress(0, 0, src.addr.offset + so), len(data),
                       d.TransferKind.D2D)
                rt.fence(rt.world)
                back = bytearray(len(data))
                rt.get(dst, back, len(data), d.TransferKind.D2H).wait()
                assert bytes(back) == data, (so, do)
        else:
            pass
        rt.barrier(rt.world)
        return True

    run_emulated(2, fn, segment_bytes=8 * MIB)


def test_asymmetric_two_step_access_and_checks():
    import paper_2506_02486_b200 as d
    from paper_2506_02486_b200.emulate import run_emulated

    def fn(rt):
        cell = rt.alloc_asymmetric(4096 * (rt.rank + 1), 0)
        if rt.rank == 0:
            addr = rt.resolve_cell(cell, 1)
            fetched = rt.engine.stats.cell_fetches
            assert rt.resolve_cell(cell, 1) == addr            # cache hit
            assert rt.engine.stats.cell_fetches == fetched
            payload = bytes(range(256)) * 32                    # 8192 B fits rank 1's payload
            rt.put(addr, payload, len(payload), d.TransferKind.H2D)
            rt.fence(rt.world)
            back = bytearray(len(payload))
            rt.get(addr, back, len(payload), d.TransferKind.D2H).wait()
            assert bytes(back) == payload
            with pytest.raises(d.InvalidAddress):              # straddles its end
                rt.put(d.GlobalAddress(1, 0, addr.offset + 8192 - 32), b"x" * 64, 64,
                       d.TransferKind.H2D)
            with pytest.raises(d.InvalidAddress):              # below its start
                rt.put(d.GlobalAddress(1, 0, addr.offset - 64), b"x" * 64, 64,
                       d.TransferKind.H2D)
        rt.barrier(rt.world)
        return True

    run_emulated(2, fn, segment_bytes=8 * MIB)


def test_invalid_and_kind_errors():
    import paper_2506_02486_b200 as d
    from paper_2506_02486_b200.emulate import run_emulated

    def fn(rt):
        rec = rt.alloc_symmetric(4096, 0)
        with pytest.raises(d.InvalidAddress):
            rt.put(d.GlobalAddress(1 - rt.rank, 0, rec.addr.offset + 4000), b"z" * 200, 200,
                   d.TransferKind.H2D)
        with pytest.raises(d.KindMismatch):
            rt.put(rec.addr, b"x", 1, d.TransferKind.D2H)
        with pytest.raises(d.KindMismatch):
            rt.get(rec.addr, bytearray(1), 1, d.TransferKind.H2D)
        rt.barrier(rt.world)
        return True

    run_emulated(2, fn, segment_bytes=2 * MIB)


def test_listing_pattern_halo_visibility():
    import paper_2506_02486_b200 as d
    from paper_2506_02486_b200.emulate import run_emulated

    def fn(rt):
        r, n = rt.rank, rt.nranks
        rec = rt.alloc_symmetric(4096, 0)
        me = bytes([65 + r]) * 16
        if r != 0:
            rt.put(d.GlobalAddress(r - 1, 0, rec.addr.offset + 2048), me, 16, d.TransferKind.H2D)
        if r != n - 1:
            rt.put(d.GlobalAddress(r + 1, 0, rec.addr.offset), me, 16, d.TransferKind.H2D)
        rt.fence(rt.world)
        rt.barrier(rt.world)
        left = bytes(rt.gm.view(0, rec.addr.offset, 16))
        right = bytes(rt.gm.view(0, rec.addr.offset + 2048, 16))
        if r != 0:
            assert left == bytes([65 + r - 1]) * 16
        if r != n - 1:
            assert right == bytes([65 + r + 1]) * 16
        return True

    run_emulated(4, fn, segment_bytes=2 * MIB)
