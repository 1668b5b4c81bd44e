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
meet on system-scope flags -- an entry handshake per call, an exit handshake
only where the caller needs the result (blocking calls, complete()) -- no
host round trip.  When
endpoints share a GPU (the in-process emulation on a small box) the host
orders them with control-plane barriers instead, because kernels that spin on
each other must never share a GPU.
"""

from __future__ import annotations

import ctypes
import enum
import os
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import InvalidAddress, RootOutOfRange, StaleGroup, TypeMismatch, UsageError
from .global_memory import GlobalAddress
from .runtime import CHANNEL_COLL, COUNTER_COLL, COUNTER_OFF, LL_OFF, Group, Runtime
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
        return _ET_DTYPE[self.value]

    @property
    def code(self) -> int:
        return _ET_CODE[self.value]


_ET_DTYPE = {k: np.dtype(v) for k, v in
             {"f32": "<f4", "f64": "<f8", "i32": "<i4", "i64": "<i8"}.items()}
_ET_CODE = {"f32": 0, "f64": 1, "i32": 2, "i64": 3}


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
        return _RK_CODE[self.kind.value]


_RK_CODE = {"sum": 0, "min": 1, "max": 2}


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


_torch_ev: dict = {}


def _after_torch(rt: Runtime, device: int):
    """Order our RMA stream after pending torch work on the same GPU (arena
    writes made through torch run on torch's current stream): an event on
    torch's stream and a stream wait -- no host synchronisation."""
    gpu = rt.gpus[device]
    ev = _torch_ev.get(gpu)
    if ev is None:
        ev = _torch_ev[gpu] = _native.event_create(gpu, timing=False)
    rc = _native.lib.diomp_event_record(ev, _torch_stream(gpu))
    if not rc:
        rc = _native.lib.diomp_stream_wait_event(rt._rma_streams[device].handle, ev)
    if rc:
        _native.check(rc, "order after torch")


def _torch_stream(gpu: int) -> int:
    import torch
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    return raw(gpu) if raw is not None else torch.cuda.current_stream(gpu).cuda_stream


def _advance(comm: Communicator, n: int, channel: int = CHANNEL_COLL):
    rt = comm.rt
    for pos in comm.my_positions:
        me_ep = comm.ring[pos]
        me = rt.endpoint_index(me_ep.rank, me_ep.device)
        for q, ep in enumerate(comm.ring):
            if q != pos:
                rt.advance_pair(me, rt.endpoint_index(ep.rank, ep.device), n, channel)


# ---- one-shot low-latency (LL) path for small messages ---------------------
# Up to the slot capacity (half an LL slot: payload words travel with their
# flags) -- measured faster than the handshake path at every size that fits
# (2 B200, f32 allreduce, blocking: 1 KiB 21.3 vs 37.2 us, 128 KiB 23.7 vs
# 34.5 us; back to back 10.4 vs 11.8 us at 128 KiB; profiles/r02_ll_crossover.txt).
# The slot is 2*chunk/(2*endpoints) of the reference-sized scratch, so the
# ceiling is ~255 KiB at 2 endpoints, ~127 KiB at 4, ~63 KiB at 8.
LL_MAX_BYTES = int(os.environ.get("DIOMP_LL_MAX", str(1 << 20)))


def _ll_slot_bytes(comm: Communicator) -> int:
    """Bytes per (source endpoint, parity) LL slot in the runtime scratch, or 0
    when the LL path is unavailable for this communicator."""
    v = comm.__dict__.get("_ll_slot")
    if v is None:
        rt = comm.rt
        w = rt.nranks * rt.cfg.devices_per_rank
        avail = rt._scratch_bytes - LL_OFF
        v = (avail // (2 * w)) // 256 * 256 if avail > 0 else 0
        # the experiments build's chain-bcast flags share this scratch
        if not (comm.device_sync and 2 <= comm.size <= 8) or _native.has_experiments():
            v = 0
        comm._ll_slot = v
    return v


def _ll_ok(comm: Communicator, nbytes: int) -> bool:
    slot = _ll_slot_bytes(comm)
    return slot > 0 and nbytes <= LL_MAX_BYTES and (nbytes + 3) // 4 * 8 <= slot


def _ll_calls(comm: Communicator) -> list:
    """Per local position: (LLArgs, RMA stream, GPU) -- built once per
    communicator; the per-call work is one C call per position."""
    calls = comm.__dict__.get("_ll_calls")
    if calls is None:
        rt = comm.rt
        slot = _ll_slot_bytes(comm)
        calls = []
        for pos in comm.my_positions:
            me_ep = comm.ring[pos]
            x = _native.LLArgs()
            x.k, x.pos, x.device = comm.size, pos, rt.gpus[me_ep.device]
            for q, ep in enumerate(comm.ring):
                x.base[q] = rt.peer_address(ep.rank, ep.device)
                x.slot[q] = rt.endpoint_index(ep.rank, ep.device)
            x.ll_off = rt.scratch_offset + LL_OFF
            x.slot_bytes = slot
            calls.append((x, ctypes.byref(x), rt._rma_streams[me_ep.device], rt.gpus[me_ep.device]))
        comm._ll_calls = calls
    return calls


def _ll_run(comm: Communicator, mode: int, send_off: int, recv_off: int, count: int,
            dtype: int, op: int, root: int, blocking: bool):
    """One LL call: diomp_ll_call per local position does the epochs (kept in
    the native RMA context, per endpoint pair), the ordering after torch's
    stream, the launch and -- for a blocking call on one position -- the wait
    and the device error check."""
    rt = comm.rt
    if comm.__dict__.get("_pending"):
        _exit(comm)   # a two-phase call still owes its exit: its stores may be in flight
    calls = _ll_calls(comm)
    one = len(calls) == 1
    ll_call = _native.lib.diomp_ll_call
    for x, xref, s, gpu in calls:
        x.mode, x.dtype, x.op, x.root = mode, dtype, op, root
        x.send_off, x.recv_off, x.count = send_off, recv_off, count
        rc = ll_call(rt._rma_ctx, xref, s.handle, _torch_stream(gpu), 1 if (blocking and one) else 0)
        if rc:   # DIOMP_INTERNAL: a device-side wait timed out -> TransportFailure
            _native.check(rc, "collective")
    if blocking and not one:
        # every position's kernel is in flight before any wait (they wait on
        # each other's words)
        for _, _, s, gpu in calls:
            s.synchronize()
            _native.check_device(gpu, "collective")


def _exit(comm: Communicator):
    """The exit handshake of the calls enqueued so far: every local position
    signals its peers and waits for theirs (one-CTA diomp_team_barrier behind
    the collective kernels on the RMA stream).  Afterwards every member's
    stores into this position's buffers have landed."""
    rt = comm.rt
    for pos in comm.my_positions:
        ep = comm.ring[pos]
        _native.check(_native.lib.diomp_team_barrier(_team(comm, pos, 1),
                                                     rt._rma_streams[ep.device].handle),
                      "collective exit")
    _advance(comm, 1)
    comm._pending = False


def complete(comm: Communicator):
    """Collective over the communicator: results of every blocking=False call
    issued on it so far are in place (the reference's calls are blocking; this
    is the completion point of the non-blocking form)."""
    rt = comm.rt
    if comm.device_sync and comm.size > 1 and comm.__dict__.get("_pending"):
        _exit(comm)
    for pos in comm.my_positions:
        s = rt._rma_streams[comm.ring[pos].device]
        s.synchronize()
        _native.check_device(s.gpu, "collective")


def _run(comm: Communicator, launch, blocking: bool = True):
    """launch(team, stream) for every local position, device- or host-synchronised.

    Device-synchronised rings: every call costs one signal per ordered pair
    (the kernel's entry handshake); a blocking call adds the exit handshake
    (one more) and waits for it.  blocking=False enqueues and returns -- the
    next call's entry handshake certifies this one's completion toward each
    peer, and complete(comm) (or any blocking call) makes results visible.
    Members must agree on `blocking` call by call, as on the call itself."""
    rt = comm.rt
    sync = 1 if (comm.device_sync and comm.size > 1) else 0
    if not sync:
        blocking = True
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
    if sync:
        _advance(comm, 1)
        comm._pending = True
        if blocking:
            _exit(comm)
    if blocking:
        for pos, s in used:
            s.synchronize()
            _native.check_device(s.gpu, "collective")
    if not sync and comm.size > 1:
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
    if _ll_ok(comm, nbytes):
        _ll_run(comm, 1, buffer.offset, buffer.offset, nbytes, 0, 0, root, blocking)
        return
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
    algo = algorithm or os.environ.get("DIOMP_ALLREDUCE_ALGO", "exact")
    memo = comm.__dict__.setdefault("_memo", {})
    key = ("allreduce", send, recv, count, op, algo)
    if memo.get(key) == rt._ledger_gen and k > 1 and algo == "exact":
        # same call shape validated since the last allocation change
        comm._next_seq()
        _allreduce_exact(comm, send, recv, count, op, blocking)
        return
    _check_typed(send, count, op.etype)
    _check_typed(recv, count, op.etype)
    nbytes = count * op.etype.dtype.itemsize
    for ep in comm.ring:
        if ep.rank == rt.rank:
            rt.gm.check_rma_range(ep.device, send.offset, max(nbytes, 1))
            rt.gm.check_rma_range(ep.device, recv.offset, max(nbytes, 1))
    if count == 0:
        return
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
    memo[key] = rt._ledger_gen
    _allreduce_exact(comm, send, recv, count, op, blocking)


def _allreduce_exact(comm, send, recv, count, op, blocking):
    nbytes = count * op.etype.dtype.itemsize
    if _ll_ok(comm, nbytes):
        _ll_run(comm, 0, send.offset, recv.offset, count, op.etype.code, op.code, 0, blocking)
        return
    _run(comm, lambda t, s: _native.lib.diomp_allreduce(t, send.offset, recv.offset, count,
                                                        op.etype.code, op.code, s), blocking)


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
           "bcast", "reduce", "allreduce", "complete", "device_bcast", "InvalidAddress"]
