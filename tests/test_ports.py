"""The multi-process CPU restatements bench.py times as the reference CPU path
(oracle/ports.py) are pinned before their numbers are reported: run_stencil on
2 and 4 processes equals the reference's own checksums (tests/golden, from
running the reference), the ring allreduce equals the reference fold bitwise,
bcast delivers the root's bytes, the wire put/get round trip is byte-exact."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

GOLD = {(c["nx"], c["ny"], c["nz"], c["steps"], c["amp"]): c["sha256"]
        for c in json.load(open(os.path.join(GOLDEN, "stencil_golden.json")))["cases"]}


@pytest.mark.parametrize("key,ranks", [((64, 64, 64, 100, 1.0), 2), ((64, 64, 64, 100, 1.0), 4),
                                       ((24, 20, 18, 7, 1.0), 3),
                                       ((128, 128, 128, 100, 1.0), 2)])
def test_stencil_procs_matches_reference_checksum(key, ranks):
    from oracle import ports as P
    nx, ny, nz, steps, amp = key
    r = P.stencil_procs(nx, ny, nz, steps, ranks, amp)
    assert r["sha256"] == GOLD[key]
    assert r["seconds"] > 0 and r["ranks"] == ranks


@pytest.mark.parametrize("k", [2, 3, 4])
def test_ring_allreduce_port_equals_reference_fold(k):
    from oracle import oracle as O
    from oracle import ports as P
    count = 10_007
    r = P.ring_collective("allreduce", k, 4 * count, iters=1)
    contribs = [np.random.default_rng(1000 + q).uniform(-1, 1, count).astype(np.float32)
                for q in range(k)]
    assert r["result"] == O.allreduce_fold(contribs, "sum").tobytes()


@pytest.mark.parametrize("k", [2, 4])
def test_ring_bcast_port_delivers_root_bytes(k):
    import hashlib

    from oracle import ports as P
    n = 3 * (1 << 20) + 5
    r = P.ring_collective("bcast", k, n, iters=1)
    root = np.random.default_rng(77).integers(0, 256, n, dtype=np.uint8).tobytes()
    assert r["digests"] == [hashlib.sha256(root).hexdigest()] * k


def test_wire_put_get_port_byte_exact():
    from oracle import ports as P
    r = P.p2p_sample(bw_bytes=(1 << 20) + 13, bw_iters=2, lat_iters=5)
    assert r["byte_exact"]
    assert r["put_latency_us_8B"] > 0 and r["put_bandwidth_gbs"] > 0


def test_wire_fragments_above_the_64mib_cap():
    from oracle import ports as P
    n = (64 << 20) + 4099
    link = P.WirePair(n)
    try:
        data = np.random.default_rng(5).integers(0, 256, n, dtype=np.uint8)
        link.put(0, data)
        link.fence()
        back = bytearray(n)
        link.get(0, back)
        assert bytes(back) == data.tobytes()
    finally:
        link.close()
