"""Host control plane: rendezvous, tagged messages, allgather, barrier.

Replaces the reference's TCP mesh control traffic (transport.py:313-454,
591-655: ctrl_send/ctrl_recv, BOOTSTRAP and BARRIER frames) with a
torch.distributed key-value store: a TCPStore when ranks are processes
(torchrun / DIOMP_RENDEZVOUS), a HashStore shared by the threads of the
in-process emulation.  Only setup-time traffic uses it (allocation digests,
IPC handles, group tables, communicator ids, host barriers); the hot loops
synchronise on the device (csrc flags).
"""

from __future__ import annotations

import pickle
import struct
import threading
from datetime import timedelta

from .errors import CollectiveMismatch, HandshakeTimeout, PeerFailure


def _store_timeout(seconds: float):
    return timedelta(seconds=max(seconds, 1.0))


class ControlPlane:
    """Tagged point-to-point messages over a key-value store.

    Every (tag, src, dst) stream is FIFO: the key carries a per-stream
    sequence number kept on both sides, so a sender that runs ahead never
    overwrites a message its receiver has not consumed yet.  Keys are deleted
    by the receiver.
    """

    def __init__(self, store, rank: int, nranks: int, timeout: float = 60.0, prefix: str = "d"):
        self.store = store
        self.rank = rank
        self.nranks = nranks
        self.timeout = timeout
        self.prefix = prefix
        self._lock = threading.Lock()
        self._seq: dict = {}
        self._sent: dict = {}
        self._recvd: dict = {}

    # -- raw messaging ---------------------------------------------------------
    def _key(self, tag, src: int, dst: int, n: int) -> str:
        t = tag.decode() if isinstance(tag, bytes) else str(tag)
        return f"{self.prefix}/m/{t}/{src}>{dst}#{n}"

    def _bump(self, table: dict, k) -> int:
        with self._lock:
            n = table.get(k, 0)
            table[k] = n + 1
            return n

    def send(self, dst: int, tag, blob: bytes):
        n = self._bump(self._sent, (tag, dst))
        self.store.set(self._key(tag, self.rank, dst, n), blob)

    def recv(self, tag, src: int, timeout: float | None = None) -> bytes:
        key = self._key(tag, src, self.rank, self._bump(self._recvd, (tag, src)))
        try:
            self.store.wait([key], _store_timeout(timeout or self.timeout))
        except Exception as e:  # torch raises DistStoreError / RuntimeError
            raise PeerFailure(f"rank {src} never sent {key!r}: {e}") from e
        blob = self.store.get(key)
        self.store.delete_key(key)
        return blob

    # -- collectives over subsets of ranks -------------------------------------------
    def next_seq(self, scope) -> int:
        with self._lock:
            n = self._seq.get(scope, 0)
            self._seq[scope] = n + 1
            return n

    def allgather(self, ranks, tag, blob: bytes, must_match: bool = False):
        """Gather at the lowest rank, redistribute (runtime.py:244-266 shape)."""
        ranks = tuple(ranks)
        root = ranks[0]
        if self.rank == root:
            blobs = {root: blob}
            for r in ranks[1:]:
                blobs[r] = self.recv(tag, r)
            packed = pickle.dumps([blobs[r] for r in ranks])
            for r in ranks[1:]:
                self.send(r, f"{tag}/r", packed)
        else:
            self.send(root, tag, blob)
            packed = self.recv(f"{tag}/r", root)
        items = list(zip(ranks, pickle.loads(packed)))
        if must_match and any(b != blob for _, b in items):
            raise CollectiveMismatch(f"collective arguments disagree across ranks for {tag!r}")
        return items

    def barrier(self, ranks, tag):
        """Dissemination barrier: ceil(log2 k) rounds (runtime.py:493-513)."""
        ranks = tuple(ranks)
        k = len(ranks)
        if k <= 1:
            return
        me = ranks.index(self.rank)
        step, rnd = 1, 0
        while step < k:
            self.send(ranks[(me + step) % k], f"{tag}/{rnd}", b"")
            self.recv(f"{tag}/{rnd}", ranks[(me - step) % k])
            step <<= 1
            rnd += 1


def pack_blobs(blobs: list[bytes]) -> bytes:
    out = [struct.pack("<I", len(blobs))]
    for b in blobs:
        out += [struct.pack("<I", len(b)), b]
    return b"".join(out)


def make_store(cfg, shared=None):
    """Store for this rank: the emulator's shared HashStore, torch.distributed's
    default store when a process group exists, else a TCPStore at the
    rendezvous address (rank 0 hosts it)."""
    if shared is not None:
        return shared
    import os

    import torch.distributed as dist
    if cfg.nranks == 1:
        return dist.HashStore()
    if not dist.is_initialized() and "DIOMP_RENDEZVOUS" not in os.environ and \
            "MASTER_ADDR" in os.environ:
        # launched by torchrun: join its rendezvous (the agent owns MASTER_PORT)
        dist.init_process_group("gloo", rank=cfg.rank, world_size=cfg.nranks,
                                timeout=_store_timeout(cfg.timeout))
    if dist.is_initialized():
        from torch.distributed import distributed_c10d as c10d
        return dist.PrefixStore("diomp", c10d._get_default_store())
    host, port = cfg.rendezvous
    try:
        return dist.TCPStore(host, port, cfg.nranks, cfg.rank == 0,
                             timeout=_store_timeout(cfg.timeout), use_libuv=True)
    except Exception as e:
        raise HandshakeTimeout(f"control-plane rendezvous at {host}:{port} failed: {e}") from e
