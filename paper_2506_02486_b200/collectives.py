"""OMPCCL collectives over device endpoints (API of
reference/pkg/src/diomp/collectives.py:1-416).

A Communicator is a group plus a bootstrap-derived 128-bit id; its ring is
the member order rotated to the lowest participating rank.  The data path is
one libdiomp_b200 kernel per local ring position that reads and writes the
peers' symmetric buffers directly over NVLink (csrc/collectives.cuh), with
the reference's combination orders reproduced bit for bit:

  * reduce     root receives ((v_root op v_root+1) op ...) op v_root-1
  * allreduce  block b = [b*count//k, (b+1)*count//k) is left-folded starting
               at ring position b, and every member ends with all blocks.

Synchronisation: when every endpoint of the ring is on its own GPU the kernels
meet on system-scope flags (entry and exit) -- no host round trip.  When
endpoints share a GPU (the in-process emulation on a small box) the host
orders them with control-plane barriers instead, because kernels that spin on
each other must never share a GPU.
"""

from __future__ import annotations

import enum
import os
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import InvalidAddress, RootOutOfRange, StaleGroup, TypeMismatch, UsageError
from .global_memory import GlobalAddress
from .runtime import CHANNEL_COLL, COUNTER_COLL, COUNTER_OFF, Group, Runtime
from .topology import Endpoint


class ReduceKind(enum.Enum):
    Sum = "sum"
    Min = "min"
    Max = "max"


class ElementType(enum.Enum):
    f32 = "f32"
    f64 = "f64"
    i32 = "i32"
    i64 = "i64"

    @property
    def dtype(self) -> np.dtype:
        return np.dtype({"f32": "<f4", "f64": "<f8", "i32": "<i4", "i64": "<i8"}[self.value])

    @property
    def code(self) -> int:
        return {"f32": 0, "f64": 1, "i32": 2, "i64": 3}[self.value]


@dataclass(frozen=True)
class ReduceOp:
    kind: ReduceKind
    etype: ElementType

    @property
    def ufunc(self):
        return {ReduceKind.Sum: np.add, ReduceKind.Min: np.minimum,
                ReduceKind.Max: np.maximum}[self.kind]

    @property
    def code(self) -> int:
        return {ReduceKind.Sum: 0, ReduceKind.Min: 1, ReduceKind.Max: 2}[self.kind]


class UniqueId:
    """128-bit random token shared by the members of a communicator."""

    __slots__ = ("value",)

    def __init__(self, value: bytes):
        assert len(value) == 16
        self.value = value

    @classmethod
    def generate(cls) -> "UniqueId":
        return cls(os.urandom(16))

    def __eq__(self, other):
        return isinstance(other, UniqueId) and self.value == other.value

    def __hash__(self):
        return hash(self.value)


class Communicator:
    def __init__(self, rt: Runtime, group: Group, uid: UniqueId, ring: tuple):
        self.rt = rt
        self.group = group
        self.uid = uid
        self.ring = ring
        self.my_positions = tuple(i for i, ep in enumerate(ring) if ep.rank == rt.rank)
        self.device_sync = rt.distinct_gpus(ring)
        self._seq = 0

    @property
    def size(self) -> int:
        return len(self.ring)

    def _next_seq(self) -> int:
        self._seq += 1
        return self._seq


def bootstrap(rt: Runtime, group: Group) -> Communicator:
    """Collective over the group's ranks; a fresh UniqueId per call."""
    group = rt._check_group(group)
    ranks = group.ranks
    if rt.rank not in ranks:
        raise StaleGroup(f"rank {rt.rank} owns no endpoint in group {group.id:#x}")
    seq = rt._per_group_seq[("boot", group.id)]
    rt._per_group_seq[("boot", group.id)] += 1
    tag = f"uid/{group.id}/{seq}"
    root = ranks[0]
    if rt.rank == root:
        uid = UniqueId.generate()
        for r in ranks[1:]:
            rt.ctrl.send(r, tag, uid.value)
    else:
        uid = UniqueId(rt.ctrl.recv(tag, root))
    members = group.members
    rot = next(i for i, ep in enumerate(members) if ep.rank == root)
    rt.bootstrap_count += 1
    return Communicator(rt, group, uid, members[rot:] + members[:rot])


# ---------------------------------------------------------------------------
# launch plumbing
# ---------------------------------------------------------------------------

def _team(comm: Communicator, pos: int, sync: int) -> _native.Team:
    """Team descriptor of ring position `pos` (cached; epochs refreshed)."""
    rt = comm.rt
    cache = comm.__dict__.setdefault("_teams", {})
    t = cache.get((pos, sync))
    me_ep = comm.ring[pos]
    me = rt.endpoint_index(me_ep.rank, me_ep.device)
    if t is None:
        t = _native.Team()
        t.k, t.pos, t.sync = comm.size, pos, sync
        t.device = rt.gpus[me_ep.device]
        t.flag_off = rt.channel_flag_offset(CHANNEL_COLL)
        t.counter_off = rt.scratch_offset + COUNTER_OFF + 64 * COUNTER_COLL
        for q, ep in enumerate(comm.ring):
            t.base[q] = rt.peer_address(ep.rank, ep.device)
            t.slot[q] = rt.endpoint_index(ep.rank, ep.device)
        cache[(pos, sync)] = t
    for q in range(comm.size):
        if q != pos:
            t.epoch_to[q], t.epoch_from[q] = rt.pair_epochs(me, t.slot[q], CHANNEL_COLL)
    return t


def _after_torch(rt: Runtime, device: int):
    """Order our stream after pending torch work on the same GPU (arena writes
    made through torch run on torch's current stream)."""
    import torch
    gpu = rt.gpus[device]
    torch.cuda.current_stream(gpu).synchronize()


def _run(comm: Communicator, launch, blocking: bool = True, signals: int = 2):
    """launch(team, stream) for every local position, device- or host-synchronised.
    `signals` = device signals the call consumes per ordered pair (allreduce 3:
    entry, phase, exit; reduce / bcast 2: entry, exit).
    blocking=False (device-synchronised rings only) enqueues and returns: the
    result is ready once the rank's RMA stream of that device has drained."""
    rt = comm.rt
    sync = 1 if (comm.device_sync and comm.size > 1) else 0
    if not sync:
        blocking = True
    if blocking:
        for pos in comm.my_positions:
            _after_torch(rt, comm.ring[pos].device)
    if not sync and comm.size > 1:
        rt.barrier(comm.group)
    used = []
    for pos in comm.my_positions:
        ep = comm.ring[pos]
        s = rt._rma_streams[ep.device]
        _native.check(launch(_team(comm, pos, sync), s.handle), "collective launch")
        used.append((pos, s))
    if blocking:
        for pos, s in used:
            s.synchronize()
            _native.check_device(s.gpu, "collective")
    if sync:
        for pos in comm.my_positions:
            me_ep = comm.ring[pos]
            me = rt.endpoint_index(me_ep.rank, me_ep.device)
            for q, ep in enumerate(comm.ring):
                if q != pos:
                    rt.advance_pair(me, rt.endpoint_index(ep.rank, ep.device), signals,
                                    CHANNEL_COLL)
    elif comm.size > 1:
        rt.barrier(comm.group)


def _member_addr(ep: Endpoint, buffer: GlobalAddress, delta: int = 0) -> GlobalAddress:
    return GlobalAddress(ep.rank, ep.device, buffer.offset + delta)


def _check_typed(buffer: GlobalAddress, count: int, etype: ElementType):
    if buffer.offset % etype.dtype.itemsize:
        raise TypeMismatch(f"offset {buffer.offset} misaligned for {etype.value}")


# ---------------------------------------------------------------------------
# collectives
# ---------------------------------------------------------------------------

def bcast(comm: Communicator, buffer: GlobalAddress, nbytes: int, root: int = 0, *,
          blocking: bool = True):
    """Every member's buffer ends equal to the root member's buffer at entry."""
    rt, k = comm.rt, comm.size
    if not 0 <= root < k:
        raise RootOutOfRange(f"root index {root} outside communicator of size {k}")
    for ep in comm.ring:
        if ep.rank == rt.rank:
            rt.gm.check_rma_range(ep.device, buffer.offset, max(nbytes, 1))
    if k == 1 or nbytes == 0:
        return
    comm._next_seq()
    _run(comm, lambda t, s: _native.lib.diomp_bcast(t, buffer.offset, nbytes, root, s), blocking)


def reduce(comm: Communicator, send: GlobalAddress, recv: GlobalAddress, count: int,
           op: ReduceOp, root: int = 0, *, blocking: bool = True):
    """Ring-ordered reduction to the root member; non-root recv untouched."""
    rt, k = comm.rt, comm.size
    if not 0 <= root < k:
        raise RootOutOfRange(f"root index {root} outside communicator of size {k}")
    _check_typed(send, count, op.etype)
    _check_typed(recv, count, op.etype)
    nbytes = count * op.etype.dtype.itemsize
    for ep in comm.ring:
        if ep.rank == rt.rank:
            rt.gm.check_rma_range(ep.device, send.offset, max(nbytes, 1))
    if count == 0:
        return
    root_ep = comm.ring[root]
    if root_ep.rank == rt.rank:
        rt.gm.check_rma_range(root_ep.device, recv.offset, nbytes)
    if k == 1:
        if send.offset != recv.offset:
            _after_torch(rt, root_ep.device)
            base = rt.gm.base(root_ep.device)
            s = rt._rma_streams[root_ep.device]
            _native.call("diomp_copy", rt.gpus[root_ep.device], base + recv.offset,
                         base + send.offset, nbytes, s.handle)
            s.synchronize()
        return
    comm._next_seq()
    _run(comm, lambda t, s: _native.lib.diomp_reduce(t, send.offset, recv.offset, count,
                                                     op.etype.code, op.code, root, s), blocking)


def allreduce(comm: Communicator, send: GlobalAddress, recv: GlobalAddress, count: int,
              op: ReduceOp, *, blocking: bool = True, algorithm: str | None = None):
    """Reduce-scatter in ring-fold order + all-gather; in place works.

    algorithm "exact" (default; DIOMP_ALLREDUCE_ALGO overrides): the
    reference's fold order, bit-identical.  "nvls": the NVSwitch reduces
    (multimem.ld_reduce) -- integer results identical, float sums within
    rounding (rel-L2 1e-6 f32 / 1e-12 f64), float min/max refused."""
    rt, k = comm.rt, comm.size
    _check_typed(send, count, op.etype)
    _check_typed(recv, count, op.etype)
    nbytes = count * op.etype.dtype.itemsize
    for ep in comm.ring:
        if ep.rank == rt.rank:
            rt.gm.check_rma_range(ep.device, send.offset, max(nbytes, 1))
            rt.gm.check_rma_range(ep.device, recv.offset, max(nbytes, 1))
    if count == 0:
        return
    algo = algorithm or os.environ.get("DIOMP_ALLREDUCE_ALGO", "exact")
    if algo not in ("exact", "nvls"):
        raise UsageError(f"unknown allreduce algorithm {algo!r}")
    if algo == "nvls" and not _native.has_experiments():
        raise UsageError("allreduce algorithm 'nvls' is in the experiments build only "
                         "(python paper_2506_02486_b200/build.py -DDIOMP_EXPERIMENTS)")
    if k == 1:
        ep = comm.ring[0]
        if send.offset != recv.offset:
            _after_torch(rt, ep.device)
            base = rt.gm.base(ep.device)
            s = rt._rma_streams[ep.device]
            _native.call("diomp_copy", rt.gpus[ep.device], base + recv.offset,
                         base + send.offset, nbytes, s.handle)
            s.synchronize()
        return
    comm._next_seq()
    if algo == "nvls":
        _allreduce_nvls(comm, send, recv, count, op, blocking)
        return
    _run(comm, lambda t, s: _native.lib.diomp_allreduce(t, send.offset, recv.offset, count,
                                                        op.etype.code, op.code, s), blocking,
         signals=3)


def _allreduce_nvls(comm: Communicator, send: GlobalAddress, recv: GlobalAddress, count: int,
                    op: ReduceOp, blocking: bool):
    from .nvls import NvlsWindow
    rt = comm.rt
    if op.etype in (ElementType.f32, ElementType.f64) and op.kind is not ReduceKind.Sum:
        raise TypeMismatch("nvls allreduce: the switch's float min/max NaN rules are not "
                           "numpy's; use algorithm='exact'")
    if send.offset % 16 or recv.offset % 16:
        raise UsageError("nvls allreduce needs 16-byte aligned send/recv offsets")
    w = comm.__dict__.get("_nvls")
    if w is None:
        w = comm._nvls = NvlsWindow(comm)
    ep = comm.ring[w.pos]
    if blocking:
        _after_torch(rt, ep.device)
    base = rt.gm.base(ep.device)
    s = rt._rma_streams[ep.device]
    w.launch(base + send.offset, base + recv.offset, count, op.etype.code, op.code,
             rt.counter_address(ep.device, COUNTER_COLL), s.handle)
    if blocking:
        s.synchronize()
        _native.check_device(s.gpu, "allreduce_nvls")


def device_bcast(rt: Runtime, var: GlobalAddress, nbytes: int, group: Group):
    """Broadcast from the group's first endpoint with one cached communicator."""
    group = rt._check_group(group)
    comm = rt.comm_cache.get(group.id)
    if comm is None:
        comm = bootstrap(rt, group)
        rt.comm_cache[group.id] = comm
    bcast(comm, var, nbytes, root=0)


__all__ = ["ReduceKind", "ElementType", "ReduceOp", "UniqueId", "Communicator", "bootstrap",
           "bcast", "reduce", "allreduce", "device_bcast", "InvalidAddress"]
