"""Minimod acoustic-isotropic wave propagation with one-sided halo exchange
(API of reference/pkg/src/diomp/apps/stencil.py:1-161).

Second-order leapfrog, order-8 space (R=4), v = 1500 m/s, unit spacing, dt at
half the CFL limit, zero exterior, a constant point source at the global
centre each step, x-slab decomposition (one slab per rank).  The field after
T steps is bitwise identical to the reference for any rank count.

B200 execution (StencilRunner):
  * fused (default when every rank has its own GPU, or one rank): one kernel
    per step does update + source + halo stores into the neighbours' ghost
    planes + neighbour flags (csrc/stencil.cuh); the whole loop is enqueued
    with no host involvement;
  * listing1 (ranks sharing a GPU): the reference's order -- exchange()
    puts + fence + barrier, then the update kernel -- host-synchronised;
  * fused_host: the fused kernel (halo stores from its epilogue straight
    into the neighbours' ghost planes) ordered by a host barrier per step
    instead of device flags -- valid for ranks sharing a GPU, and the way a
    one-GPU box exercises the fused epilogue's peer stores;
  * twosided (exchange="twosided"): the reference's mailbox send/recv
    comparison variant (apps/halo_twosided.py), host-synchronised.
"""

from __future__ import annotations

import hashlib
import math
import time
from dataclasses import dataclass

import numpy as np

from .. import _native
from ..errors import DecompositionError, UsageError
from ..global_memory import GlobalAddress, TransferKind
from ..runtime import CHANNEL_STENCIL, COUNTER_STENCIL, Runtime
from . import halo_onesided, halo_twosided

VELOCITY = 1500.0
_COEF = (-205.0 / 72.0, 8.0 / 5.0, -1.0 / 5.0, 8.0 / 315.0, -1.0 / 560.0)


@dataclass(frozen=True)
class StencilSpec:
    nx: int
    ny: int
    nz: int
    steps: int
    radius: int = 4
    source_amplitude: float = 1.0

    def __post_init__(self):
        if self.radius != len(_COEF) - 1:
            raise DecompositionError("only radius 4 coefficients are built in")


@dataclass
class StencilResult:
    checksum: str
    field: np.ndarray | None
    seconds: float


def rank_xmin_xmax(r: int, nranks: int, nx: int) -> tuple[int, int]:
    """Contiguous block decomposition of [0, nx)."""
    if not 0 <= r < nranks <= nx:
        raise DecompositionError(f"rank {r} of {nranks} over nx={nx}")
    return (r * nx) // nranks, ((r + 1) * nx) // nranks - 1


def _time_params(radius: int) -> tuple[float, np.ndarray]:
    """dt = half the CFL limit; weights = coef * (v dt)^2 (same float ops as
    the reference so the constants are bit-identical)."""
    per_axis = abs(_COEF[0]) + 2 * sum(abs(c) for c in _COEF[1:radius + 1])
    dt = 0.5 * 2.0 / (VELOCITY * math.sqrt(3.0 * per_axis))
    scale = (VELOCITY * dt) ** 2
    return dt, np.array(_COEF[:radius + 1]) * scale


class StencilRunner:
    """Allocates the two symmetric fields and enqueues steps on a CUDA stream."""

    def __init__(self, rt: Runtime, spec: StencilSpec, mode: str | None = None):
        nranks, r = rt.nranks, spec.radius
        if spec.nx % nranks:
            raise DecompositionError(f"nx={spec.nx} not divisible by {nranks} ranks")
        self.nxl = nxl = spec.nx // nranks
        if nxl < r:
            raise DecompositionError(f"local slab {nxl} thinner than radius {r}")
        self.rt, self.spec = rt, spec
        self.shape = (nxl + 2 * r, spec.ny + 2 * r, spec.nz + 2 * r)
        self.nbytes = int(np.prod(self.shape)) * 8
        self.plane_bytes = self.shape[1] * self.shape[2] * 8
        self.field_a = rt.alloc_symmetric(self.nbytes, 0)
        self.field_b = rt.alloc_symmetric(self.nbytes, 0)
        self.gpu = rt.gpus[0]
        self.stream = rt._rma_streams[0]
        base = rt.gm.base(0)
        for rec in (self.field_a, self.field_b):
            _native.call("diomp_memset_async", base + rec.addr.offset, 0, self.nbytes,
                         self.stream.handle)
        self.stream.synchronize()

        _, w = _time_params(r)
        self.w, self.center = w, 3.0 * w[0]
        gxmin, gxmax = rank_xmin_xmax(rt.rank, nranks, spec.nx)
        cx, cy, cz = spec.nx // 2, spec.ny // 2, spec.nz // 2
        own = gxmin <= cx <= gxmax and bool(spec.source_amplitude)
        self.src = (cx - gxmin + r, cy + r, cz + r) if own else (-1, -1, -1)

        if mode is None:
            mode = "fused" if (nranks == 1 or rt.distinct_gpus(rt.world.members)) else "listing1"
        if mode not in ("fused", "fused_host", "listing1", "twosided"):
            raise UsageError(f"unknown stencil mode {mode!r}")
        self.mode = mode
        self.mailbox = None
        if mode == "twosided":
            mb = halo_twosided.mailbox_bytes(r, self.plane_bytes)
            self.mailbox = rt.alloc_symmetric(mb, 0)
            _native.call("diomp_memset_async", base + self.mailbox.addr.offset, 0, mb,
                         self.stream.handle)
            self.stream.synchronize()
        self.step = 0
        self.left = rt.rank - 1 if rt.rank > 0 else None
        self.right = rt.rank + 1 if rt.rank < nranks - 1 else None
        self.me_idx = rt.endpoint_index(rt.rank, 0)

    # -- plan ----------------------------------------------------------------------
    def _plan(self) -> _native.StencilPlan:
        rt, r = self.rt, self.spec.radius
        p = _native.StencilPlan()
        p.device, p.radius = self.gpu, r
        p.NX, p.NY, p.NZ = self.shape
        offs = (self.field_a.addr.offset, self.field_b.addr.offset)
        p.field[0], p.field[1] = (rt.gm.base(0) + o for o in offs)
        fused = self.mode in ("fused", "fused_host")
        if fused and self.left is not None:
            p.left_field[0], p.left_field[1] = (rt.peer_address(self.left, 0, o) for o in offs)
        if fused and self.right is not None:
            p.right_field[0], p.right_field[1] = (rt.peer_address(self.right, 0, o) for o in offs)
        p.src_i, p.src_j, p.src_k = self.src
        p.amp = float(self.spec.source_amplitude)
        p.center = float(self.center)
        for t in range(r + 1):
            p.w[t] = float(self.w[t])
        p.sync = 1 if (self.mode == "fused" and rt.nranks > 1) else 0
        if p.sync:
            for side, nb in (("left", self.left), ("right", self.right)):
                if nb is None:
                    continue
                nb_idx = rt.endpoint_index(nb, 0)
                sent, recvd = rt.pair_epochs(self.me_idx, nb_idx, CHANNEL_STENCIL)
                setattr(p, f"wait_{side}", rt.flag_address(rt.rank, 0, nb_idx, CHANNEL_STENCIL))
                setattr(p, f"sig_{side}", rt.flag_address(nb, 0, self.me_idx, CHANNEL_STENCIL))
                setattr(p, f"from_{side}", recvd)
                setattr(p, f"to_{side}", sent)
            p.counter = rt.counter_address(0, COUNTER_STENCIL)
        return p

    def enqueue(self, nsteps: int, stream_handle: int | None = None):
        """Enqueue nsteps fused steps (no host synchronisation)."""
        if self.mode != "fused":
            raise UsageError("enqueue() needs the fused mode")
        plan = self._plan()
        s = self.stream.handle if stream_handle is None else stream_handle
        _native.check(_native.lib.diomp_stencil_run(plan, self.step, nsteps, s), "stencil_run")
        if plan.sync:
            for nb in (self.left, self.right):
                if nb is not None:
                    # nsteps + 1 signals per call: entry + one per step
                    self.rt.advance_pair(self.me_idx, self.rt.endpoint_index(nb, 0), nsteps + 1,
                                         CHANNEL_STENCIL)
        self.step += nsteps

    def run(self, nsteps: int):
        """Run nsteps to completion on this rank."""
        rt = self.rt
        if self.mode == "fused":
            self.enqueue(nsteps)
            self.stream.synchronize()
            _native.check_device(self.gpu, "stencil")
            return
        if self.mode == "fused_host":
            # step s writes the neighbours' ghost planes of field[s%2], which
            # they last read (as u_cur) in step s-1: a barrier after every
            # rank's step s-1 has drained orders the two
            for _ in range(nsteps):
                if rt.nranks > 1:
                    rt.barrier(rt.world)
                _native.check(_native.lib.diomp_stencil_run(self._plan(), self.step, 1,
                                                            self.stream.handle), "stencil_run")
                self.stream.synchronize()
                _native.check_device(self.gpu, "stencil")
                self.step += 1
            if rt.nranks > 1:
                rt.barrier(rt.world)
            return
        for _ in range(nsteps):
            cur = self.field_b if self.step % 2 == 0 else self.field_a
            if rt.nranks > 1 and self.mode == "twosided":
                halo_twosided.exchange(rt, rt.world, cur.addr, self.mailbox.addr,
                                       self.plane_bytes, self.spec.radius, self.nxl, rt.rank,
                                       rt.nranks, self.step)
            elif rt.nranks > 1:
                halo_onesided.exchange(rt, rt.world, cur.addr, self.plane_bytes,
                                       self.spec.radius, self.nxl, rt.rank, rt.nranks,
                                       stream=None)
            plan = self._plan()
            _native.check(_native.lib.diomp_stencil_run(plan, self.step, 1, self.stream.handle),
                          "stencil_run")
            self.stream.synchronize()
            self.step += 1

    @property
    def cur_rec(self):
        """Record holding u at the current time level (swap order of stencil.py:126)."""
        return self.field_b if self.step % 2 == 0 else self.field_a

    def free(self):
        if self.mailbox is not None:
            self.rt.free(self.mailbox)
        self.rt.free(self.field_b)
        self.rt.free(self.field_a)


def run_stencil(rt: Runtime, spec: StencilSpec, exchange: str = "onesided",
                gather: bool = True) -> StencilResult:
    if exchange not in ("onesided", "fused", "twosided"):
        raise UsageError(f"unknown exchange {exchange!r}")
    runner = StencilRunner(rt, spec, "twosided" if exchange == "twosided" else None)
    rt.barrier(rt.world)
    t0 = time.perf_counter()
    runner.run(spec.steps)
    rt.barrier(rt.world)
    seconds = time.perf_counter() - t0
    if not gather:
        return StencilResult("", None, seconds)
    field = _gather_field(rt, runner.cur_rec, spec, runner.nxl, runner.shape)
    checksum = hashlib.sha256(dump_bytes(field)).hexdigest() if rt.rank == 0 else ""
    return StencilResult(checksum, field, seconds)


def _gather_field(rt: Runtime, cur_rec, spec: StencilSpec, nxl: int, shape):
    r = spec.radius
    interior = (slice(r, r + nxl), slice(r, r + spec.ny), slice(r, r + spec.nz))
    if rt.rank != 0:
        rt.barrier(rt.world)
        return None
    field = np.empty((spec.nx, spec.ny, spec.nz))
    nbytes = int(np.prod(shape)) * 8
    for peer in range(rt.nranks):
        buf = np.empty(shape)
        rt.get(GlobalAddress(peer, 0, cur_rec.addr.offset), buf, nbytes,
               TransferKind.D2H).wait(rt.cfg.timeout)
        gxmin, _ = rank_xmin_xmax(peer, rt.nranks, spec.nx)
        field[gxmin:gxmin + nxl] = buf[interior]
    rt.barrier(rt.world)
    return field


def dump_bytes(field: np.ndarray) -> bytes:
    """--dump-field serialisation: f64, x fastest, little-endian."""
    return field.transpose(2, 1, 0).astype("<f8", copy=False).tobytes()
