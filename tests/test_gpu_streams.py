"""Streams on real CUDA streams: the reference's pool policy and task-order
properties (reference pkg/tests/test_streams.py; streams.py:56-246), plus the
device-side half the reference cannot have -- host tasks and device work on
one CUDA stream are ordered both ways, without stalling other streams."""

import threading
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture
def pool_factory():
    from paper_2506_02486_b200.streams import StreamPool
    made = []

    def make(max_active):
        p = StreamPool(0, max_active=max_active)
        made.append(p)
        return p

    yield make
    for p in made:
        p.shutdown()


def test_streams_are_created_lazily_and_reused(pool_factory):
    pool = pool_factory(8)
    assert pool.created_count == 0
    first = pool.acquire()
    pool.release(first)
    again = pool.acquire()
    assert again.id == first.id and pool.created_count == 1
    pool.release(again)
    for _ in range(50):
        s = pool.acquire()
        s.submit(lambda: None)
        pool.release(s)
    assert pool.created_count == 1
    held = [pool.acquire() for _ in range(8)]
    assert pool.created_count == 8 and pool.active_count() == 8
    for s in held:
        pool.release(s)


def test_task_runs_and_events_are_monotone(pool_factory):
    pool = pool_factory(2)
    s = pool.acquire()
    src = np.arange(4096, dtype=np.uint8)
    dst = np.zeros_like(src)
    assert s.submit(lambda: dst.__setitem__(slice(None), src)).wait(5)
    assert np.array_equal(dst, src)
    gate, seen = threading.Event(), []
    first = s.submit(lambda: (gate.wait(5), seen.append("a")))
    second = s.submit(lambda: seen.append("b"))
    time.sleep(0.02)
    assert not first.completed and not second.completed
    gate.set()
    assert second.wait(5) and first.completed
    assert seen == ["a", "b"]


def test_per_stream_fifo_under_interleaving(pool_factory):
    pool = pool_factory(4)
    streams = [pool.acquire() for _ in range(3)]
    log, lock = [], threading.Lock()
    for step in range(12):
        for s in streams:
            s.submit(lambda sid=s.id, k=step: (lock.acquire(), log.append((sid, k)), lock.release()))
    pool.sync_all()
    assert len(log) == 36
    for s in streams:
        assert [k for sid, k in log if sid == s.id] == list(range(12))
    assert pool.active_count() == 0


def test_idle_stream_rejects_tasks(pool_factory):
    from paper_2506_02486_b200.errors import StreamClosed
    pool = pool_factory(2)
    s = pool.acquire()
    pool.release(s)
    with pytest.raises(StreamClosed):
        s.submit(lambda: None)


def test_task_error_is_kept_and_queue_continues(pool_factory):
    pool = pool_factory(1)
    s = pool.acquire()
    bad = s.submit(lambda: 1 / 0)
    good = s.submit(lambda: None)
    assert good.wait(5) and bad.completed
    assert isinstance(bad.error, ZeroDivisionError) and good.error is None


def _busy(pool, streams, n_busy, gate):
    for s in streams[:n_busy]:
        s.submit(lambda: gate.wait(10))
    for s in streams[n_busy:]:
        s.submit(lambda: None).wait(5)
    time.sleep(0.02)


@pytest.mark.parametrize("n_busy,want", [(4, (4, 2)), (7, (1, 1))])
def test_half_release_of_completed_streams(pool_factory, n_busy, want):
    pool = pool_factory(8)
    streams = [pool.acquire() for _ in range(8)]
    gate = threading.Event()
    _busy(pool, streams, n_busy, gate)
    released = pool.enforce_bound()
    assert pool.audit.enforcements[-1] == want and released == want[1]
    gate.set()


def test_enforce_blocks_on_oldest_when_nothing_completed(pool_factory):
    pool = pool_factory(4)
    streams = [pool.acquire() for _ in range(4)]
    gates = [threading.Event() for _ in streams]
    for s, g in zip(streams, gates):
        s.submit(lambda g=g: g.wait(10))
    t = threading.Thread(target=pool.enforce_bound)
    t.start()
    time.sleep(0.05)
    assert t.is_alive()
    gates[0].set()
    t.join(5)
    assert not t.is_alive() and pool.audit.enforcements[-1] == (0, 1)
    assert streams[0].state == "idle"
    for g in gates[1:]:
        g.set()


@pytest.mark.parametrize("max_active", [1, 3, 8])
def test_bound_holds_under_random_traffic(pool_factory, max_active):
    pool = pool_factory(max_active)
    rng = np.random.default_rng(100 + max_active)
    for _ in range(300):
        s = pool.acquire()
        delay = rng.random() * 1e-4 if rng.random() < 0.3 else 0.0
        s.submit(lambda d=delay: time.sleep(d))
        if rng.random() < 0.6:
            pool.release(s)
    assert pool.audit.max_active_seen <= max_active
    assert all(rel == max(1, -(-done // 2)) for done, rel in pool.audit.enforcements)


def test_host_task_orders_device_work_both_ways(pool_factory):
    """Device work issued before a host task is complete when the task runs;
    device work issued while the task is pending is held back (on the host)
    until it returns -- and other streams (torch's) are never blocked."""
    import torch

    from paper_2506_02486_b200 import _native
    pool = pool_factory(2)
    s = pool.acquire()
    n = 64 << 20
    src = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda:0")
    mid = torch.zeros(n, dtype=torch.uint8, device="cuda:0")
    dst = torch.zeros(n, dtype=torch.uint8, device="cuda:0")
    torch.cuda.synchronize()

    def copy(to, frm):
        return lambda: _native.call("diomp_copy", 0, to.data_ptr(), frm.data_ptr(), n, s.handle)

    first = s.enqueue(copy(mid, src))
    assert first.issued
    seen = {}
    gate = threading.Event()

    def task():
        seen["mid_ok"] = bool(torch.equal(mid, src))   # torch's stream, after `first`
        gate.wait(10)

    ev = s.submit(task)
    later = s.enqueue(copy(dst, mid))
    time.sleep(0.1)
    assert not later.issued and not later.completed and not s.is_quiescent()
    assert int(dst[:4096].sum().item()) == 0          # torch's stream runs freely
    gate.set()
    assert ev.wait(10) and later.wait(10)
    s.synchronize()
    assert ev.error is None and seen["mid_ok"] and torch.equal(dst, src)


def test_sync_all_drains_everything(pool_factory):
    pool = pool_factory(4)
    streams = [pool.acquire() for _ in range(4)]
    evs = [s.submit(lambda: time.sleep(0.003)) for s in streams for _ in range(3)]
    pool.sync_all()
    assert all(e.completed for e in evs) and pool.active_count() == 0
