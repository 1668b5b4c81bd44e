"""Row-stripe ring matrix multiply C = A x B (API of
reference/pkg/src/diomp/apps/cannon.py:1-170).

Endpoint e owns A and C row stripes [e*ns, (e+1)*ns) and starts holding B
stripe e; at step s it holds stripe (e+s) mod P, computes
C_e += A_e[:, blk] @ B_held and shifts the held stripe to its predecessor.

B200 execution: the product runs on the FP64 tensor cores (DMMA kernel,
csrc/gemm.cuh).  With every endpoint on its own GPU the ring steps are
ordered by device flags (wait: successor wrote my stripe, predecessor freed
its spare; signal: both) and the shift runs on the copy engine from a side
stream, concurrently with the product that reads the same stripe, so it
costs the DMMA pipe nothing.  The alternative fused shift (every B tile the
kernel stages in shared memory also stored into the predecessor's spare
stripe over NVLink, DIOMP_CANNON_SHIFT=fused, and the path used when
endpoints share a GPU) measured 5 % slower on 2 and 4 B200: the remote
stores stall the DMMA warps (profiles/r01_cannon_shift.txt).  The residual is measured against
the bit-exact k-ordered matmul seam (kernels.matmul_f64, the reference's
oracle arithmetic) run on the GPU.
"""

from __future__ import annotations

import struct
import os
import time
from dataclasses import dataclass, field

import numpy as np

from .. import _native, gemm, kernels
from ..errors import ShapeMismatch
from ..runtime import CHANNEL_GEMM, COUNTER_GEMM, Runtime


@dataclass(frozen=True)
class MatmulSpec:
    n: int
    p: int

    @property
    def ns(self) -> int:
        return self.n // self.p

    def __post_init__(self):
        if self.p < 1 or self.n < 1 or self.n % self.p:
            raise ShapeMismatch(f"P={self.p} must divide N={self.n}")


@dataclass
class CannonResult:
    residual: float
    seconds: float
    identity_exact: bool | None
    timeline: list = field(default_factory=list)  # (endpoint, step, kind, t0, t1)

    def overlap_observed(self) -> bool:
        spans = {}
        for ep, step, kind, t0, t1 in self.timeline:
            spans.setdefault((ep, step), {})[kind] = (t0, t1)
        for pair in spans.values():
            if "compute" in pair and "xfer" in pair:
                (c0, c1), (x0, x1) = pair["compute"], pair["xfer"]
                if max(c0, x0) < min(c1, x1):
                    return True
        return False


def _fill_matrices(n: int, seed: int, identity_b: bool = False):
    """A then B from one generator (cannon.py:73-77)."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1.0, 1.0, (n, n))
    b = np.eye(n) if identity_b else rng.uniform(-1.0, 1.0, (n, n))
    return a, b


class CannonRing:
    """State of one ring multiply: stripes in symmetric memory, A/C per endpoint."""

    def __init__(self, rt: Runtime, spec: MatmulSpec, use_streams: bool = True,
                 a_full=None, b_full=None, device_seed: int | None = None):
        import torch
        p, dpr = spec.p, rt.cfg.devices_per_rank
        if p != rt.nranks * dpr:
            raise ShapeMismatch(f"P={p} but the world has {rt.nranks * dpr} endpoints")
        self.rt, self.spec = rt, spec
        n, ns = spec.n, spec.ns
        self.stripe_bytes = ns * n * 8
        self.streams = [rt.pools[d].acquire() for d in range(dpr)] if use_streams else None
        self.bufs = []
        for d in range(dpr):
            s = self.streams[d] if self.streams else None
            self.bufs.append([rt.alloc_symmetric(self.stripe_bytes, d, stream=s),
                              rt.alloc_symmetric(self.stripe_bytes, d, stream=s)])
        self.world = rt.world.members
        self.my_eps = [(i, ep) for i, ep in enumerate(self.world) if ep.rank == rt.rank]
        self.local = {}
        for e, ep in self.my_eps:
            d, gpu = ep.device, rt.gpus[ep.device]
            dev = torch.device("cuda", gpu)
            if device_seed is not None:
                g = torch.Generator(device=dev).manual_seed(device_seed * 1000 + e)
                a = torch.rand(ns, n, dtype=torch.float64, device=dev, generator=g) * 2 - 1
                b = torch.rand(ns, n, dtype=torch.float64, device=dev, generator=g) * 2 - 1
            else:
                a = torch.from_numpy(np.ascontiguousarray(a_full[e * ns:(e + 1) * ns])).to(dev)
                b = torch.from_numpy(np.ascontiguousarray(b_full[e * ns:(e + 1) * ns])).to(dev)
            self.stripe(d, 0).copy_(b.view(-1).view(torch.uint8).view(torch.float64)
                                    .view(ns, n))
            self.local[e] = dict(a=a, c=torch.zeros(ns, n, dtype=torch.float64, device=dev),
                                 dev=d, gpu=gpu)
        torch.cuda.synchronize()
        self.sync = p > 1 and rt.distinct_gpus(self.world)
        self.step_no = 0
        # ring shift engine with device flags: "ce" (default) = the copy engine
        # pushes the whole stripe on a side stream while the DMMA kernel runs;
        # "fused" = the GEMM's CTAs store each B tile from shared memory
        # (measured 5 % slower on 2 and 4 B200: the remote stores stall the
        # DMMA warps, profiles/r01_cannon_shift.txt)
        self.shift = os.environ.get("DIOMP_CANNON_SHIFT", "ce") if self.sync else "fused"
        if self.shift not in ("ce", "fused"):
            raise ValueError(f"DIOMP_CANNON_SHIFT={self.shift!r}: expected 'ce' or 'fused'")
        self._side = {}
        if self.shift == "ce":
            for _, ep in self.my_eps:
                g = rt.gpus[ep.device]
                self._side[ep.device] = (_native.stream_create(g), _native.event_create(g, False),
                                         _native.event_create(g, False))

    def stripe(self, d: int, which: int):
        """torch view of this rank's stripe buffer `which` on device d."""
        import torch
        rec = self.bufs[d][which]
        t = self.rt.gm.arena(d)[rec.addr.offset:rec.addr.offset + self.stripe_bytes]
        return t.view(torch.float64).view(self.spec.ns, self.spec.n)

    def _stream(self, d: int) -> int:
        return self.streams[d].handle if self.streams else self.rt._rma_streams[d].handle

    def enqueue_step(self):
        """One ring step on every local endpoint (no host synchronisation in
        device-flag mode)."""
        rt, spec = self.rt, self.spec
        p, ns, n, t = spec.p, spec.ns, spec.n, self.step_no
        for e, ep in self.my_eps:
            d = ep.device
            st = self.local[e]
            cur_rec = self.bufs[d][t % 2]
            s = (e + t) % p
            a_blk = st["a"][:, s * ns:(s + 1) * ns]
            fwd, sync = 0, None
            if p > 1:
                pred = self.world[(e - 1) % p]
                # always forward (also on the last step, as cannon.py:124-131 does):
                # after P steps every stripe is back home, so runs can repeat
                fwd = rt.peer_address(pred.rank, pred.device, self.bufs[d][(t + 1) % 2].addr.offset)
            if self.sync:
                me = rt.endpoint_index(ep.rank, ep.device)
                nbrs = []
                for nb in (self.world[(e - 1) % p], self.world[(e + 1) % p]):
                    idx = rt.endpoint_index(nb.rank, nb.device)
                    if idx not in [x[1] for x in nbrs]:
                        nbrs.append((nb, idx))
                sync = dict(wait_addr=[], wait_value=[], sig_addr=[], sig_value=[],
                            counter=rt.counter_address(d, COUNTER_GEMM))
                for nb, idx in nbrs:
                    sent, recvd = rt.pair_epochs(me, idx, CHANNEL_GEMM)
                    sync["wait_addr"].append(rt.flag_address(ep.rank, d, idx, CHANNEL_GEMM))
                    sync["wait_value"].append(recvd)
                    sync["sig_addr"].append(rt.flag_address(nb.rank, nb.device, me, CHANNEL_GEMM))
                    sync["sig_value"].append(sent + 1)
                    rt.advance_pair(me, idx, 1, CHANNEL_GEMM)
            src = rt.gm.base(d) + cur_rec.addr.offset
            if self.shift == "ce":
                self._ce_step(st["gpu"], d, ns, n, a_blk, src, st["c"], fwd, sync)
                continue
            gemm.dgemm_raw(st["gpu"], ns, n, ns, a_blk.data_ptr(), n, src, n, st["c"].data_ptr(), n,
                           self._stream(d), fwd=fwd, ldf=n, sync=sync)
        self.step_no += 1

    def _ce_step(self, gpu, d, ns, n, a_blk, src, c, fwd, sync):
        """One step with the shift on the copy engine: wait for both
        neighbours' previous step (our stripe has arrived, the predecessor's
        spare buffer is free) -> side stream pushes the stripe to the
        predecessor while the DMMA kernel multiplies it -> join -> signal."""
        main = self._stream(d)
        side, ready, sent = self._side[d]
        for a, v in zip(sync["wait_addr"], sync["wait_value"]):
            _native.call("diomp_wait", gpu, a, v, main)
        _native.call("diomp_event_record", ready, main)
        _native.call("diomp_stream_wait_event", side, ready)
        _native.call("diomp_put", gpu, fwd, src, self.stripe_bytes, 1, side)
        _native.call("diomp_event_record", sent, side)
        gemm.dgemm_raw(gpu, ns, n, ns, a_blk.data_ptr(), n, src, n, c.data_ptr(), n, main)
        _native.call("diomp_stream_wait_event", main, sent)
        for a, v in zip(sync["sig_addr"], sync["sig_value"]):
            _native.call("diomp_signal", gpu, a, v, main)

    def synchronize(self):
        for e, ep in self.my_eps:
            _native.call("diomp_stream_sync", self._stream(ep.device))
            _native.check_device(self.rt.gpus[ep.device], "cannon")

    def run(self, timeline: list | None = None):
        rt = self.rt
        for _ in range(self.spec.p):
            c0 = time.perf_counter()
            if not self.sync and self.spec.p > 1:
                rt.barrier(rt.world)
            self.enqueue_step()
            if not self.sync:
                self.synchronize()
            if timeline is not None:
                c1 = time.perf_counter()
                for e, _ in self.my_eps:
                    # the shift is fused into the product: same device interval
                    timeline.append((e, self.step_no - 1, "compute", c0, c1))
                    timeline.append((e, self.step_no - 1, "xfer", c0, c1))
        self.synchronize()

    def release(self):
        for side, ready, sent in self._side.values():
            _native.call("diomp_stream_sync", side)
            _native.call("diomp_event_destroy", ready)
            _native.call("diomp_event_destroy", sent)
            _native.call("diomp_stream_destroy", side)
        self._side = {}
        if self.streams:
            for d, s in enumerate(self.streams):
                self.rt.pools[d].release(s)
        for pair in self.bufs:
            for rec in reversed(pair):
                self.rt.free(rec)


def cannon_matmul(rt: Runtime, spec: MatmulSpec, seed: int = 0, identity_b: bool = False,
                  use_streams: bool = True) -> CannonResult:
    import torch
    a_full, b_full = _fill_matrices(spec.n, seed, identity_b)
    ring = CannonRing(rt, spec, use_streams, a_full, b_full)
    rt.barrier(rt.world)
    timeline: list = []
    t0 = time.perf_counter()
    ring.run(timeline)
    rt.barrier(rt.world)
    seconds = time.perf_counter() - t0

    # residual against the k-ordered (oracle-arithmetic) matmul on the GPU
    residual, exact = 0.0, True
    ns = spec.ns
    for e, ep in ring.my_eps:
        st = ring.local[e]
        dev = torch.device("cuda", st["gpu"])
        b_dev = torch.from_numpy(b_full).to(dev)
        ref = torch.empty(ns, spec.n, dtype=torch.float64, device=dev)
        kernels.matmul_f64(st["a"], b_dev, ref)
        diff = (st["c"] - ref).abs()
        residual = max(residual, float(diff.max()) if diff.numel() else 0.0)
        if identity_b:
            exact = exact and torch.equal(st["c"], st["a"])
    seq = rt._per_group_seq[("app", "cannon")]
    rt._per_group_seq[("app", "cannon")] += 1
    got = rt.ctrl.allgather(tuple(range(rt.nranks)), f"cannon/res/{seq}",
                            struct.pack("<dB", residual, int(exact)))
    residual = max(struct.unpack("<dB", b)[0] for _, b in got)
    exact = all(struct.unpack("<dB", b)[1] for _, b in got)
    ring.release()
    return CannonResult(residual, seconds, exact if identity_b else None, timeline)
