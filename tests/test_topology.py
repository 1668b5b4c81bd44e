"""Endpoint / path classification (reference topology.py:1-89, its
test_topology.py cases): pure host logic on CPU, runtime discovery on GPU."""

import itertools

import pytest

from paper_2506_02486_b200.errors import UnknownEndpoint
from paper_2506_02486_b200.topology import (Endpoint, PathKind, TopologyMap, classify_path,
                                            empty_peer_matrix, full_peer_matrix)


def make_topo(nranks=4, devices=2, nodes=(0, 0, 1, 1), peers=True):
    matrix = (full_peer_matrix if peers else empty_peer_matrix)(devices)
    return TopologyMap(nranks, devices, tuple(nodes), tuple(500 + r for r in range(nranks)),
                       matrix)


@pytest.mark.parametrize("a,b,kind", [
    ((0, 0), (0, 1), PathKind.PeerFabric),     # same process, two GPUs with peer access
    ((1, 1), (1, 1), PathKind.IntraProcess),   # same endpoint
    ((1, 0), (3, 1), PathKind.InterNode),      # nodes 0 and 1
    ((2, 1), (3, 0), PathKind.IntraNodeIPC),   # two processes on node 1
])
def test_known_classifications(a, b, kind):
    topo = make_topo()
    assert classify_path(topo.endpoint(*a), topo.endpoint(*b), topo) is kind


def test_no_peer_access_means_intra_process_copy():
    topo = make_topo(peers=False)
    assert classify_path(topo.endpoint(2, 0), topo.endpoint(2, 1), topo) is PathKind.IntraProcess


def test_every_pair_classified_and_symmetric():
    topo = make_topo()
    eps = topo.endpoints()
    assert len(eps) == 8 and len(set(eps)) == 8
    for a, b in itertools.product(eps, eps):
        assert classify_path(a, b, topo) is classify_path(b, a, topo)


def test_out_of_range_endpoints_raise():
    topo = make_topo()
    for bad in ((4, 0), (-1, 0), (0, 2)):
        with pytest.raises(UnknownEndpoint):
            topo.endpoint(*bad)
    with pytest.raises(UnknownEndpoint):
        classify_path(Endpoint(0, 0, 0), Endpoint(1, 7, 0), topo)


def test_peer_matrices():
    full, none = full_peer_matrix(4), empty_peer_matrix(4)
    for a, b in itertools.product(range(4), range(4)):
        assert full[(a, b)] == (a != b)
        assert none[(a, b)] is False


def test_global_endpoint_index_is_rank_major():
    topo = make_topo(nranks=3, devices=2, nodes=(0, 0, 0))
    assert [topo.index(r, d) for r, d in itertools.product(range(3), range(2))] == list(range(6))


@pytest.mark.gpu
def test_discovery_digest_identical_on_every_rank():
    from paper_2506_02486_b200.emulate import run_emulated
    got = run_emulated(4, lambda rt: rt.topology.digest_bytes(), node_ids=[0, 0, 1, 1],
                       segment_bytes=2 << 20)
    assert len(set(got)) == 1


@pytest.mark.gpu
def test_single_process_multi_device_world():
    from conftest import NGPU
    from paper_2506_02486_b200.emulate import run_emulated
    if NGPU < 2:
        pytest.skip("needs 2 GPUs for two devices per rank")
    nd = min(NGPU, 4)
    members = run_emulated(1, lambda rt: [(ep.rank, ep.device) for ep in rt.world.members],
                           devices_per_rank=nd, segment_bytes=2 << 20)[0]
    assert members == [(0, d) for d in range(nd)]
