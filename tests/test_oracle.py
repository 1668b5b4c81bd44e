"""The oracle is pinned before it is trusted: every restatement in oracle/ is
checked against fixtures produced by running the reference itself
(tests/golden/make_golden.py)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle as O

GOLD = json.load(open(os.path.join(GOLDEN, "stencil_golden.json")))


def test_time_params_bit_identical_to_reference():
    dt, w = O.time_params(4)
    meta = GOLD["time_params"]
    assert dt.hex() == meta["dt"]
    assert [float(x).hex() for x in w] == meta["w"]
    assert float(3.0 * w[0]).hex() == meta["center"]


@pytest.mark.parametrize("case", [c for c in GOLD["cases"] if c["nx"] <= 64],
                         ids=lambda c: f"{c['nx']}x{c['ny']}x{c['nz']}x{c['steps']}a{c['amp']}")
def test_c_oracle_driver_matches_reference_checksums(case):
    f = O.stencil_run(case["nx"], case["ny"], case["nz"], case["steps"], case["amp"])
    assert O.checksum(f) == case["sha256"]


@pytest.mark.parametrize("ranks", [2, 3])
def test_slab_restatement_matches_reference(ranks):
    case = GOLD["cases"][1]  # 24x20x18, 7 steps
    f = O.stencil_run_slabs(case["nx"], case["ny"], case["nz"], case["steps"], ranks)
    assert O.checksum(f) == case["sha256"]


@pytest.mark.parametrize("name", ["s4", "s4b", "s2", "s3"])
def test_stencil_update_restatements_bitwise(name):
    g = np.load(os.path.join(GOLDEN, "kernels_golden.npz"))
    w = g[f"{name}_w"]
    r = w.shape[1] - 1
    for fn in (O.stencil_update_c, O.stencil_update_np):
        out = g[f"{name}_prev"].copy()
        fn(out, g[f"{name}_cur"], out, float(g[f"{name}_center"][0]), w[0], w[1], w[2], r)
        assert np.array_equal(out.view(np.uint64), g[f"{name}_out"].view(np.uint64)), fn


@pytest.mark.parametrize("name", ["m1", "m2", "m3"])
def test_matmul_oracle_bitwise(name):
    g = np.load(os.path.join(GOLDEN, "kernels_golden.npz"))
    got = O.matmul_f64(g[f"{name}_a"], g[f"{name}_b"])
    assert np.array_equal(got.view(np.uint64), g[f"{name}_c"].view(np.uint64))


def _contrib(rank, etype, count, seed):
    dt = {"f32": np.float32, "f64": np.float64, "i32": np.int32, "i64": np.int64}
    rng = np.random.default_rng(seed * 100 + rank)
    if etype.startswith("f"):
        v = rng.uniform(-1, 1, count).astype(dt[etype])
        if count > 8:
            v[3] = np.nan if rank == 1 else v[3]
            v[5] = -0.0 if rank % 2 else 0.0
        return v
    return rng.integers(-2**30, 2**30, count).astype(dt[etype])


def test_collective_fold_oracles_match_reference_runs():
    g = np.load(os.path.join(GOLDEN, "collectives_golden.npz"))
    assert len(g.files) == 96
    for key in g.files:
        which, k, et, kind, count, root, seed = key.split("_")
        k, count, root, seed = int(k), int(count), int(root), int(seed)
        cs = [_contrib(r, et, count, seed) for r in range(k)]
        want = O.allreduce_fold(cs, kind) if which == "allreduce" else O.reduce_fold(cs, kind, root)
        assert np.array_equal(want.view(np.uint8), g[key].view(np.uint8)), key


def test_numpy_min_max_semantics_pinned():
    """The device Min/Max follow numpy: NaN propagates, ties keep operand 2."""
    a = np.array([np.nan, 1.0, 0.0, -0.0])
    b = np.array([1.0, np.nan, -0.0, 0.0])
    mn, mx = np.minimum(a, b), np.maximum(a, b)
    assert np.isnan(mn[0]) and np.isnan(mn[1]) and np.isnan(mx[0]) and np.isnan(mx[1])
    assert np.signbit(mn[2]) and not np.signbit(mn[3])
    assert np.signbit(mx[2]) and not np.signbit(mx[3])


def test_allocator_restatements_match_reference_traces():
    gold = json.load(open(os.path.join(GOLDEN, "allocator_golden.json")))["allocators"]
    mib = 1 << 20
    makers = {"buddy": lambda: O.OracleBuddy(4 * mib),
              "buddy_reserved": lambda: O.OracleBuddy(4 * mib, reserve_from=3 * mib),
              "linear": lambda: O.OracleLinear(4 * mib),
              "reverse": lambda: O.OracleReverse(3 * mib, 4 * mib)}
    for name, make in makers.items():
        alloc, live, trace = make(), [], []
        for op in gold[name]["ops"]:
            if op[0] == "free":
                off = live.pop(op[1])
                trace.append(["f", off, alloc.free(off)])
            else:
                try:
                    off = alloc.alloc(op[1])
                    live.append(off)
                    trace.append(["a", off, alloc.block_size(op[1])])
                except MemoryError:
                    trace.append(["oom"])
        assert trace == gold[name]["trace"], name


def test_full_size_golden_recorded_with_provenance():
    """1024^3 x 3 steps: the reference's checksum was reproduced by
    the C oracle in 63 s when the fixture was recorded; the GPU suite checks the
    CUDA path against it (tests/test_gpu_edges.py)."""
    full = GOLD["full_size"][0]
    assert (full["nx"], full["steps"]) == (1024, 3)
    assert full["sha256"].startswith("3277fbcc")
