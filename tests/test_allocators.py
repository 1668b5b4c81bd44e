"""Native heaps (csrc/heap.cuh via paper_2506_02486_b200.allocators) against
the reference's allocator tests (test_allocators.py known answers) and
reference-generated operation traces.  Host-only: no GPU needed."""

import json
import os

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from conftest import GOLDEN
from oracle import oracle as O
from paper_2506_02486_b200.allocators import (BuddyAllocator, LinearAllocator,
                                              ReverseBumpAllocator)
from paper_2506_02486_b200.errors import DoubleFree, OutOfSegment

MIB = 1 << 20


def test_linear_first_two_allocations_stack():
    lin = LinearAllocator(MIB)
    assert lin.alloc(16 * 1024) == 0
    assert lin.alloc(32 * 1024) == 16 * 1024


def test_linear_alignment_and_exact_reuse():
    lin = LinearAllocator(MIB, alignment=64)
    assert lin.alloc(1) == 0 and lin.alloc(1) == 64
    a = lin.alloc(4096)
    lin.free(a)
    assert lin.alloc(4096) == a
    assert lin.alloc(8192) != a


def test_linear_out_of_segment():
    lin = LinearAllocator(4096)
    lin.alloc(4096)
    with pytest.raises(OutOfSegment):
        lin.alloc(1)


def test_buddy_rounding_and_coalescing():
    b = BuddyAllocator(MIB)
    assert [b.block_size(s) for s in (1, 256, 257, 8192, 8193)] == [256, 256, 512, 8192, 16384]
    x, y = b.alloc(4096), b.alloc(4096)
    assert {x, y} == {0, 4096}
    blocker = b.alloc(512 * 1024)
    b.free(x)
    b.free(y)
    assert b.alloc(8192) == 0
    b.free(blocker)


def test_buddy_exhaustion_double_free_reserved_tail():
    b = BuddyAllocator(4096)
    offs = [b.alloc(256) for _ in range(16)]
    with pytest.raises(OutOfSegment):
        b.alloc(256)
    b.free(offs[0])
    with pytest.raises(DoubleFree):
        b.free(offs[0])
    r = BuddyAllocator(MIB, reserve_from=MIB - MIB // 4)
    assert r.alloc(MIB // 2) == 0
    assert r.alloc(MIB // 4) == MIB // 2
    with pytest.raises(OutOfSegment):
        r.alloc(MIB // 4)


def test_reverse_grows_downward_and_floor():
    rev = ReverseBumpAllocator(0, MIB)
    a, b = rev.alloc(4096), rev.alloc(4096)
    assert a == MIB - 4096 and b == a - 4096
    rev.free(a)
    assert rev.alloc(4096) == a
    f = ReverseBumpAllocator(MIB - 8192, MIB)
    f.alloc(8192)
    with pytest.raises(OutOfSegment):
        f.alloc(64)


def test_buddy_rejects_non_pow2():
    with pytest.raises(ValueError):
        BuddyAllocator(3 * MIB)


GOLD = json.load(open(os.path.join(GOLDEN, "allocator_golden.json")))


@pytest.mark.parametrize("name", ["buddy", "buddy_reserved", "linear", "reverse"])
def test_native_heaps_replay_reference_traces(name):
    make = {"buddy": lambda: BuddyAllocator(4 * MIB),
            "buddy_reserved": lambda: BuddyAllocator(4 * MIB, reserve_from=3 * MIB),
            "linear": lambda: LinearAllocator(4 * MIB),
            "reverse": lambda: ReverseBumpAllocator(3 * MIB, 4 * MIB)}[name]
    alloc, live, trace = make(), [], []
    for op in GOLD["allocators"][name]["ops"]:
        if op[0] == "free":
            off = live.pop(op[1])
            trace.append(["f", off, alloc.free(off)])
        else:
            try:
                off = alloc.alloc(op[1])
                live.append(off)
                trace.append(["a", off, alloc.block_size(op[1])])
            except OutOfSegment:
                trace.append(["oom"])
    assert trace == GOLD["allocators"][name]["trace"]


@st.composite
def _ops(draw):
    ops, live = [], 0
    for _ in range(draw(st.integers(1, 150))):
        if live and draw(st.booleans()):
            ops.append(("free", draw(st.integers(0, live - 1))))
            live -= 1
        else:
            ops.append(("alloc", draw(st.integers(0, 60_000))))
            live += 1
    return ops


@settings(max_examples=80, deadline=None)
@given(_ops(), st.sampled_from(["buddy", "linear", "reverse"]))
def test_fuzz_native_equals_oracle_and_never_overlaps(ops, kind):
    native = {"buddy": lambda: BuddyAllocator(4 * MIB, reserve_from=3 * MIB),
              "linear": lambda: LinearAllocator(3 * MIB),
              "reverse": lambda: ReverseBumpAllocator(3 * MIB, 4 * MIB)}[kind]()
    oracle = {"buddy": lambda: O.OracleBuddy(4 * MIB, reserve_from=3 * MIB),
              "linear": lambda: O.OracleLinear(3 * MIB),
              "reverse": lambda: O.OracleReverse(3 * MIB, 4 * MIB)}[kind]()
    live = []
    for op, arg in ops:
        if op == "alloc":
            try:
                a = native.alloc(arg)
            except OutOfSegment:
                a = None
            try:
                b = oracle.alloc(arg)
            except MemoryError:
                b = None
            assert a == b
            if a is not None:
                live.append(a)
        elif live:
            off = live.pop(arg % len(live))
            assert native.free(off) == oracle.free(off)
    assert native.live == oracle.live
    spans = sorted(native.live.items())
    for (o1, s1), (o2, _) in zip(spans, spans[1:]):
        assert o1 + s1 <= o2


def test_fault_injection_seam_creates_overlap(monkeypatch):
    monkeypatch.setenv("DIOMP_FAULT_INJECT", "alloc_overlap")
    lin = LinearAllocator(MIB)
    a = lin.alloc(4096)
    b = lin.alloc(4096)
    assert a == b  # the mutation makes the non-overlap property fail, as in the reference
