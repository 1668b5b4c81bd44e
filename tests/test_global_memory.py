"""Global-memory ledger (host state machine, no device backing needed):
offsets, cells, generations, translate, range checks -- the reference's
test_global_memory.py contracts, plus the reference-generated ledger traces."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2506_02486_b200.errors import (DoubleFree, InvalidAddress, NotSymmetric,
                                          NullPayload, StaleCell)
from paper_2506_02486_b200.global_memory import (CELL_BYTES, AllocatorKind, GlobalAddress,
                                                 GlobalMemory, SegmentConfig, pack_cell,
                                                 unpack_cell)

MIB = 1 << 20


def _gm(nbytes=4 * MIB, kind=AllocatorKind.Buddy, devices=1):
    return GlobalMemory(SegmentConfig(nbytes, kind), devices, backing=False)


def test_segment_config_invariants():
    for bad in (dict(segment_bytes=MIB - 1), dict(segment_bytes=3 * MIB),
                dict(segment_bytes=MIB, alignment=48), dict(segment_bytes=MIB, alignment=8192)):
        with pytest.raises(ValueError):
            SegmentConfig(**bad)


def test_global_address_order():
    a = GlobalAddress(0, 1, 100)
    assert GlobalAddress(0, 0, 500) < a < GlobalAddress(1, 0, 0)
    with pytest.raises(ValueError):
        GlobalAddress(-1, 0, 0)


def test_linear_s1_s2_layout():
    gm = _gm(kind=AllocatorKind.Linear)
    s1 = gm.local_alloc_symmetric(16 * 1024, 0)
    s2 = gm.local_alloc_symmetric(32 * 1024, 0)
    assert (s1.addr.offset, s2.addr.offset) == (0, 16384)


def test_symmetric_offsets_rank_invariant_under_asymmetric_interleave():
    a, b = _gm(), _gm()
    rng = np.random.default_rng(0)
    for _ in range(20):
        size = int(rng.integers(100, 40_000))
        a.local_alloc_symmetric(size, 0)
        b.local_alloc_symmetric(size, 0)
        a.local_alloc_asymmetric(int(rng.integers(0, 60_000)), 0)
        b.local_alloc_asymmetric(int(rng.integers(0, 60_000)), 0)
    assert a.symmetric_ledger(0) == b.symmetric_ledger(0)


def test_cell_layout_and_generation():
    gm = _gm()
    cell = gm.local_alloc_asymmetric(4096, 0)
    assert cell.cell_addr.offset % 32 == 0
    assert gm.read_local_cell(cell) == (cell.local_payload.offset, 4096, 1)
    assert cell.local_payload.offset >= gm.asym_base(0)
    gm.local_free_cell(cell)
    cell2 = gm.local_alloc_asymmetric(100, 0)
    assert cell2.cell_addr.offset == cell.cell_addr.offset
    assert cell2.generation == 3


def test_pack_unpack_and_resolve():
    raw = pack_cell(123456, 789, 42)
    assert len(raw) == CELL_BYTES and unpack_cell(raw) == (123456, 789, 42)
    gm = _gm()
    cell = gm.local_alloc_asymmetric(2048, 0)
    with pytest.raises(StaleCell):
        gm.resolve_from_bytes(cell, 1, pack_cell(999, 2048, cell.generation + 1))
    addr = gm.resolve_from_bytes(cell, 1, pack_cell(999, 2048, cell.generation))
    assert addr == GlobalAddress(1, 0, 999)
    assert gm.cache_lookup(cell, 1) == (addr, 2048, cell.generation)
    gm.local_free_cell(cell)
    assert gm.cache_lookup(cell, 1) is None
    z = gm.local_alloc_asymmetric(0, 0)
    assert z.local_payload is None
    with pytest.raises(NullPayload):
        gm.resolve_from_bytes(z, 0, pack_cell(0, 0, z.generation))
    with pytest.raises(DoubleFree):
        gm.local_free_cell(cell)


def test_translate_and_range_checks():
    gm = _gm()
    rec = gm.local_alloc_symmetric(4096, 0)
    assert gm.translate(rec.addr, 3) == GlobalAddress(3, 0, rec.addr.offset)
    assert gm.translate(GlobalAddress(0, 0, rec.addr.offset + 100), 2).offset == rec.addr.offset + 100
    cell = gm.local_alloc_asymmetric(4096, 0)
    with pytest.raises(NotSymmetric):
        gm.translate(cell.local_payload, 1)
    b = gm.local_alloc_symmetric(4096, 0)
    assert gm.check_rma_range(0, rec.addr.offset + 100, 100) is rec
    with pytest.raises(InvalidAddress):
        gm.check_rma_range(0, rec.addr.offset, 4096 + 1)
    with pytest.raises(InvalidAddress):
        gm.check_rma_range(0, gm.config.segment_bytes - 8, 64)
    assert gm.mirror_check(0, rec.addr.offset, 4096) is rec
    assert gm.mirror_check(0, gm.asym_base(0) + 64, 64) is None
    gm.local_free(rec)
    with pytest.raises(NotSymmetric):
        gm.translate(rec.addr, 1)
    with pytest.raises(InvalidAddress):
        gm.check_rma_range(0, rec.addr.offset, 16)
    assert gm.check_rma_range(0, b.addr.offset, 4096) is b


@pytest.mark.parametrize("kind", ["buddy", "linear"])
def test_ledger_replays_reference_trace(kind):
    gold = json.load(open(os.path.join(GOLDEN, "allocator_golden.json")))["global_memory"][kind]
    gm = _gm(kind=AllocatorKind(kind))
    cells, recs = [], {}
    for step in gold["seq"]:
        if step[0] == "sym":
            rec = gm.local_alloc_symmetric(step[1], 0)
            assert [rec.addr.offset, rec.size] == step[2:4]
            recs[rec.addr.offset] = rec
        elif step[0] == "asym":
            cell = gm.local_alloc_asymmetric(step[1], 0)
            cells.append(cell)
            pay = cell.local_payload.offset if cell.local_payload else None
            assert [cell.cell_addr.offset, cell.generation, pay] == step[2:5]
        elif step[0] == "free_cell":
            assert cells[0].cell_addr.offset == step[1]
            gm.local_free_cell(cells.pop(0))
        else:
            gm.local_free(recs.pop(step[1]))
    assert [list(x) for x in gm.full_ledger(0)] == gold["ledger"]
    assert not gm.live_ranges_overlap(0)
