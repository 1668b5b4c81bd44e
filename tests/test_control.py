"""Multi-process control plane on CPU (gloo, world_size 2 and 3): rendezvous
through torch.distributed, tagged messages, allgather with digest matching,
dissemination barrier -- the host side of the N>1 path (runtime init,
allocation digests, IPC-handle exchange, bench max-over-ranks)."""

import os
import pickle
import time

import pytest
import torch.multiprocessing as mp

from paper_2506_02486_b200.emulate import free_port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    os.environ.pop("DIOMP_RENDEZVOUS", None)
    try:
        from paper_2506_02486_b200.config import resolve_from_env
        from paper_2506_02486_b200.control import ControlPlane, make_store
        from paper_2506_02486_b200.errors import CollectiveMismatch
        cfg = resolve_from_env()
        assert (cfg.rank, cfg.nranks, cfg.gpus) == (rank, world, (rank,))
        cp = ControlPlane(make_store(cfg), rank, world, timeout=30)
        got = cp.allgather(range(world), "t1", pickle.dumps(rank * 10))
        assert [pickle.loads(b) for _, b in got] == [r * 10 for r in range(world)]
        same = cp.allgather(range(world), "t2", b"same", must_match=True)
        assert len(same) == world
        try:
            cp.allgather(range(world), "t3", b"r%d" % rank, must_match=True)
            raise AssertionError("mismatch not detected")
        except CollectiveMismatch:
            pass
        # ring of tagged messages, tag reuse after consumption
        for it in range(3):
            cp.send((rank + 1) % world, "ring", b"%d:%d" % (rank, it))
            assert cp.recv("ring", (rank - 1) % world) == b"%d:%d" % ((rank - 1) % world, it)
        # barrier gates on the last entrant
        if rank == world - 1:
            time.sleep(0.3)
        t_in = time.time()
        cp.barrier(tuple(range(world)), "b0")
        q.put((rank, t_in, time.time()))
        sub = cp.allgather((0, world - 1), "pair", b"x") if rank in (0, world - 1) else None
        assert sub is None or len(sub) == 2
        import torch.distributed as dist
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "error", traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 3])
def test_control_plane_multiprocess_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    errs = [o for o in out if o[1] == "error"]
    assert not errs, errs[0][2]
    last_in = max(o[1] for o in out)
    assert all(o[2] >= last_in - 1e-3 for o in out)
