"""Micro-benchmarks: point-to-point latency/bandwidth and collective sweeps
(API of reference/pkg/src/diomp/apps/bench.py:1-174; CSV columns
kind,size_bytes,iters,mean_us,bw_MiBs unchanged).

Timing is on the device (CUDA events on the RMA stream, max over ranks for
collectives) unless a row measures host-visible latency (put+fence, get+wait),
which -- like the reference -- includes the host round trip.  `transfer`
selects the reference's host-sourced payloads (None: H2D put / D2H get) or
GPU-resident D2D payloads (the NVLink sweep of BASELINE.json configs[1]).
"""

from __future__ import annotations

import enum
import json
import math
import os
import pickle
import time
from dataclasses import dataclass

import numpy as np

from .. import _native
from .. import collectives as coll
from ..errors import UsageError
from ..global_memory import GlobalAddress, TransferKind
from ..runtime import Runtime

CSV_HEADER = "kind,size_bytes,iters,mean_us,bw_MiBs"
MIB = 1024 * 1024
NVLINK_PEER_GBS = 770.0      # measured peer copy per direction (B200_PROFILING.md)
NVLINK_NOMINAL_GBS = 900.0


class BenchKind(enum.Enum):
    PutLatency = "put"
    GetLatency = "get"
    Bandwidth = "bw"
    Bcast = "bcast"
    Allreduce = "allreduce"
    GetBandwidth = "get_bw"


def latency_sizes() -> list[int]:
    return [4 << i for i in range(12)]


def collective_sizes() -> list[int]:
    return [(128 * 1024) << i for i in range(10)]


@dataclass(frozen=True)
class BenchSpec:
    kind: BenchKind
    sizes: tuple
    iters: int = 100
    warmup: int = 5
    transfer: TransferKind | None = None
    allocation: str = "symmetric"   # or "asymmetric": the target is a resolved cell payload

    def __post_init__(self):
        if self.iters < 1:
            raise UsageError("iters must be >= 1")
        if list(self.sizes) != sorted(self.sizes):
            raise UsageError("sizes must be ascending")
        if self.allocation not in ("symmetric", "asymmetric"):
            raise UsageError(f"unknown allocation {self.allocation!r}")


@dataclass
class BenchRow:
    kind: str
    size_bytes: int
    iters: int
    mean_us: float
    bw_mibs: float
    wire_put_bytes: int = 0
    ratio: float | None = None

    def csv(self) -> str:
        base = f"{self.kind},{self.size_bytes},{self.iters},{self.mean_us:.3f},{self.bw_mibs:.3f}"
        return base + (f",{self.ratio:.4f}" if self.ratio is not None else "")


def _pinned(src: np.ndarray | None = None, nbytes: int = 0) -> np.ndarray:
    """A page-locked host buffer (a numpy view of pinned torch memory), filled
    from `src` when given: host legs of the timed regions run from pinned
    memory, as a production caller's would (pageable copies are staged by
    the driver at a fraction of PCIe speed)."""
    import torch
    n = src.nbytes if src is not None else nbytes
    buf = torch.empty(max(n, 1), dtype=torch.uint8, pin_memory=True).numpy()[:n]
    if src is not None:
        buf[:] = src.view(np.uint8).reshape(-1)
        return buf.view(src.dtype)
    return buf


def bw_iters(size: int, base: int) -> int:
    """Repetitions of one bandwidth row: at least `base`, and enough that the
    timed region holds >= 2 GiB up to 32 reps (so a 64 MiB row is not
    dominated by the first launch and the closing fence / handshake)."""
    return max(base, min(32, (2 << 30) // max(size, 1)))


class _Timer:
    """CUDA-event timer on the rank's RMA stream of device 0."""

    def __init__(self, rt: Runtime):
        self.rt = rt
        self.gpu = rt.gpus[0]
        self.stream = rt._rma_streams[0].handle
        self.e0 = _native.event_create(self.gpu)
        self.e1 = _native.event_create(self.gpu)

    def start(self):
        _native.call("diomp_event_record", self.e0, self.stream)

    def stop_ms(self) -> float:
        _native.call("diomp_event_record", self.e1, self.stream)
        _native.call("diomp_event_sync", self.e1)
        return _native.event_elapsed_ms(self.e0, self.e1)


def run_p2p(rt: Runtime, spec: BenchSpec) -> list[BenchRow]:
    """Rank 0 drives transfers against rank 1; other ranks cooperate."""
    if rt.nranks < 2:
        raise UsageError("p2p benchmark needs at least 2 ranks")
    size_max = max(spec.sizes)
    asym = spec.allocation == "asymmetric"
    # asymmetric: every rank binds a size_max payload in its asymmetric region;
    # the initiator reaches rank 1's through the two-step access (one 32-byte
    # cell read, then cached per generation -- runtime.py:318-349)
    buf = rt.alloc_asymmetric(size_max, 0) if asym else rt.alloc_symmetric(size_max, 0)
    src = rt.alloc_symmetric(size_max, 0)
    rows: list[BenchRow] = []
    rt.barrier(rt.world)
    if rt.rank == 0:
        dst = rt.resolve_cell(buf, 1) if asym else rt.translate(buf.addr, 1)
        stats = rt.engine.stats
        timer = _Timer(rt)
        d2d = spec.transfer is TransferKind.D2D
        for size in spec.sizes:
            payload = np.random.default_rng(size).integers(0, 256, size, dtype=np.uint8)
            sink = bytearray(size)
            if not d2d:
                payload, sink = _pinned(payload), _pinned(nbytes=size)
            if d2d:
                rt.gm.view(0, src.addr.offset, size)[:] = payload.tobytes()
            for _ in range(spec.warmup):
                _one_rep(rt, spec.kind, dst, payload, sink, size, 1, d2d, src)
            wire0 = stats.put_bytes_total()
            t0 = time.perf_counter()
            if d2d and spec.kind in (BenchKind.Bandwidth, BenchKind.GetBandwidth):
                timer.start()
                reps = _one_rep(rt, spec.kind, dst, payload, sink, size, spec.iters, d2d, src,
                                fence=False)
                elapsed = timer.stop_ms() / 1e3
                rt.fence(rt.world)
            else:
                reps = _one_rep(rt, spec.kind, dst, payload, sink, size, spec.iters, d2d, src)
                elapsed = time.perf_counter() - t0
            wire = stats.put_bytes_total() - wire0
            rows.append(BenchRow(spec.kind.value + ("_d2d" if d2d else "") + ("_asym" if asym else ""),
                                 size, reps,
                                 elapsed / reps * 1e6, size * reps / elapsed / MIB, wire))
    rt.barrier(rt.world)
    rt.free(src)
    rt.free(buf)
    return rows


def _one_rep(rt, kind, dst, payload, sink, size, iters, d2d, src, fence=True) -> int:
    local = GlobalAddress(rt.rank, 0, src.addr.offset)
    if kind is BenchKind.PutLatency:
        for _ in range(iters):
            if d2d:
                rt.put(dst, local, size, TransferKind.D2D)
            else:
                rt.put(dst, payload, size, TransferKind.H2D)
            rt.fence(rt.world)
        return iters
    if kind is BenchKind.GetLatency:
        for _ in range(iters):
            if d2d:
                rt.get(dst, local, size, TransferKind.D2D).wait(rt.cfg.timeout)
            else:
                rt.get(dst, sink, size, TransferKind.D2H).wait(rt.cfg.timeout)
        return iters
    if kind in (BenchKind.Bandwidth, BenchKind.GetBandwidth):
        for _ in range(iters):
            if kind is BenchKind.GetBandwidth:
                rt.get(dst, local, size, TransferKind.D2D)
            elif d2d:
                rt.put(dst, local, size, TransferKind.D2D)
            else:
                rt.put(dst, payload, size, TransferKind.H2D)
        if fence:
            rt.fence(rt.world)
        return iters
    raise UsageError(f"{kind} is not a point-to-point benchmark")


def run_collective(rt: Runtime, spec: BenchSpec, comm=None) -> list[BenchRow]:
    """Warm-up then `iters` timed repetitions per size (device-timed, max over
    ranks); rank 0 reports.  No barrier is needed between repetitions."""
    if spec.kind not in (BenchKind.Bcast, BenchKind.Allreduce):
        raise UsageError(f"{spec.kind} is not a collective benchmark")
    if comm is None:
        comm = coll.bootstrap(rt, rt.world)
    if comm.size < 2:
        raise UsageError("collective benchmark needs at least 2 endpoints")
    max_size = max(spec.sizes)
    send = rt.alloc_symmetric(max_size, 0)
    recv = rt.alloc_symmetric(max_size, 0)
    op = coll.ReduceOp(coll.ReduceKind.Sum, coll.ElementType.f32)
    vals = np.random.default_rng(1000 + rt.rank).uniform(-1, 1, max_size // 4).astype(np.float32)
    rt.gm.view(0, send.addr.offset, vals.nbytes)[:] = vals.tobytes()
    rows: list[BenchRow] = []
    timer = _Timer(rt)
    device_timed = comm.device_sync

    def run_once(size, blocking):
        if spec.kind is BenchKind.Bcast:
            coll.bcast(comm, send.addr, size, root=0, blocking=blocking)
        else:
            coll.allreduce(comm, send.addr, recv.addr, size // 4, op, blocking=blocking)

    for size in spec.sizes:
        for _ in range(spec.warmup):
            run_once(size, True)
        rt.barrier(rt.world)
        if device_timed:
            # enqueue-only repetitions, CUDA events on the RMA stream (device
            # time); a device-side team barrier first, so the timed region
            # starts with every GPU in step (host barrier skew excluded)
            coll._exit(comm)
            timer.start()
            for _ in range(spec.iters):
                run_once(size, False)
            coll._exit(comm)   # the last call's results in place, inside the timed region
            elapsed = timer.stop_ms() / 1e3
            _native.check_device(rt.gpus[0], "collective bench")
        else:
            t0 = time.perf_counter()
            for _ in range(spec.iters):
                run_once(size, True)
            elapsed = time.perf_counter() - t0
        got = rt.ctrl.allgather(tuple(range(rt.nranks)), "collbench", pickle.dumps(elapsed))
        elapsed = max(pickle.loads(b) for _, b in got)
        if rt.rank == 0:
            rows.append(BenchRow(spec.kind.value, size, spec.iters, elapsed / spec.iters * 1e6,
                                 size * spec.iters / elapsed / MIB))
    rt.free(recv)
    rt.free(send)
    return rows


def apply_baseline(rows: list[BenchRow], baseline_csv: str):
    """ratio = log10(baseline_mean / measured_mean), matched by kind+size."""
    table = {}
    for line in baseline_csv.strip().splitlines():
        if line.startswith("kind,") or not line.strip():
            continue
        parts = line.split(",")
        table[(parts[0], int(parts[1]))] = float(parts[3])
    for row in rows:
        base = table.get((row.kind, row.size_bytes))
        if base is not None and row.mean_us > 0:
            row.ratio = math.log10(base / row.mean_us)


def to_csv(rows: list[BenchRow], with_ratio: bool = False) -> str:
    header = CSV_HEADER + (",log10_ratio" if with_ratio else "")
    return "\n".join([header] + [r.csv() for r in rows]) + "\n"


# ---------------------------------------------------------------------------
# bench.py --workload p2p | allreduce | bcast | dgemm  (secondary JSON lines)
# ---------------------------------------------------------------------------

def _cli_runtime(seg_bytes: int):
    from ..config import LaunchConfig, resolve_from_env
    from ..global_memory import AllocatorKind, SegmentConfig
    from ..runtime import Runtime
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("DIOMP_GPUS", str(local))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    cfg = resolve_from_env(LaunchConfig(nranks=world, segment=SegmentConfig(
        seg_bytes, AllocatorKind.Linear)))
    return Runtime(cfg)


_LINE_HOOK = None   # bench.py sets this to attach its cpu_baseline to the line


def _line(rt, metric, value, unit, args, config, extra):
    d = {"metric": metric, "value": value, "unit": unit, "n_gpus": rt.nranks,
         "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
         "scaling": "weak", "vs_baseline": None, "data": "synthetic", "config": config}
    d.update(extra)
    if _LINE_HOOK is not None:
        _LINE_HOOK(d)
    print(json.dumps(d), flush=True)


def _p2p_cli(args):
    rt = _cli_runtime(8 << 30)   # 2 GiB symmetric + a 1 GiB asymmetric payload
    if rt.nranks < 2:
        raise UsageError("--workload p2p needs 2 GPUs (torchrun --nproc-per-node 2)")
    sizes = tuple(8 << i for i in range(28))  # 8 B .. 1 GiB
    out = {}
    for kind in (BenchKind.Bandwidth, BenchKind.GetBandwidth, BenchKind.PutLatency,
                 BenchKind.GetLatency):
        szs = sizes if kind in (BenchKind.Bandwidth, BenchKind.GetBandwidth) else sizes[:11]
        rows = run_p2p(rt, BenchSpec(kind, szs, iters=max(args.steps, 5), warmup=args.warmup,
                                     transfer=TransferKind.D2D))
        out[kind.value] = [(r.size_bytes, round(r.mean_us, 3),
                            round(r.size_bytes / r.mean_us / 1e3, 2)) for r in rows]
    # the same sweep against an asymmetric allocation (configs[1]: "symmetric
    # and asymmetric allocations")
    for kind in (BenchKind.Bandwidth, BenchKind.GetBandwidth, BenchKind.PutLatency,
                 BenchKind.GetLatency):
        szs = sizes if kind in (BenchKind.Bandwidth, BenchKind.GetBandwidth) else sizes[:11]
        rows = run_p2p(rt, BenchSpec(kind, szs, iters=max(args.steps, 5), warmup=args.warmup,
                                     transfer=TransferKind.D2D, allocation="asymmetric"))
        out[kind.value + "_asym"] = [(r.size_bytes, round(r.mean_us, 3),
                                      round(r.size_bytes / r.mean_us / 1e3, 2)) for r in rows]
    # end to end: the same puts with a HOST payload (TransferKind.H2D, the
    # reference's default kind) -- the PCIe leg is inside every timed put
    e2e_rows = run_p2p(rt, BenchSpec(BenchKind.Bandwidth, (64 * MIB, 1 << 30), iters=3,
                                     warmup=1))
    if rt.rank == 0:
        big = [gbps for n, _, gbps in out["bw"] if n >= 64 * MIB]
        value = out["bw"][-1][2]
        _line(rt, "put_bandwidth_1GiB", value, "GB/s", args,
              {"workload": "p2p_d2d_sweep_8B_1GiB", "pair": "rank0->rank1",
               "allocations": ["symmetric", "asymmetric"]},
              {"roofline": {"bound": "nvlink", "achieved": value, "peak": NVLINK_PEER_GBS,
                            "unit": "GB/s", "frac": round(value / NVLINK_PEER_GBS, 4),
                            "nominal": NVLINK_NOMINAL_GBS},
               "min_bw_ge_64MiB": min(big) if big else None,
               "get_bandwidth_1GiB": out["get_bw"][-1][2],
               "put_latency_us_8B": out["put"][0][1], "get_latency_us_8B": out["get"][0][1],
               "asymmetric": {"put_bandwidth_1GiB": out["bw_asym"][-1][2],
                              "get_bandwidth_1GiB": out["get_bw_asym"][-1][2],
                              "min_put_bw_ge_64MiB": min(g for n, _, g in out["bw_asym"]
                                                         if n >= 64 * MIB),
                              "put_latency_us_8B": out["put_asym"][0][1],
                              "get_latency_us_8B": out["get_asym"][0][1]},
               "rows": out, "row_format": "[bytes, mean_us, GB/s]",
               "e2e": {"value": round(e2e_rows[-1].size_bytes / e2e_rows[-1].mean_us / 1e3, 2),
                       "unit": "GB/s", "h2d_bytes_per_step": e2e_rows[-1].size_bytes,
                       "d2h_bytes_per_step": 0,
                       "rows": [(r.size_bytes, round(r.size_bytes / r.mean_us / 1e3, 2))
                                for r in e2e_rows],
                       "note": "1 GiB puts from a host buffer (TransferKind.H2D) to rank 1"}})
    rt.finalize()
    return 0


def _coll_cli(args, kind):
    rt = _cli_runtime(8 << 30)
    if rt.nranks < 2:
        raise UsageError(f"--workload {kind} needs >= 2 GPUs")
    sizes = tuple(1024 << (2 * i) for i in range(11))  # 1 KiB .. 1 GiB (x4)
    bk = BenchKind.Allreduce if kind == "allreduce" else BenchKind.Bcast
    spec = BenchSpec(bk, sizes, iters=max(args.steps, 3), warmup=args.warmup)
    rows = run_collective(rt, spec)
    # the in-switch (NVLS) allreduce, where every GPU supports multicast:
    # float sums within rounding of the exact fold (collectives.allreduce)
    nvls_rows = None
    if kind == "allreduce" and os.environ.get("BENCH_NVLS", "1") != "0":
        from .. import nvls
        ok = rt.ctrl.allgather(tuple(range(rt.nranks)), "bench/nvls",
                               bytes([nvls.supported(rt.gpus[0])]))
        if all(b == b"\x01" for _, b in ok):
            prev = os.environ.get("DIOMP_ALLREDUCE_ALGO")
            os.environ["DIOMP_ALLREDUCE_ALGO"] = "nvls"
            try:
                nvls_rows = run_collective(rt, spec)
            finally:
                if prev is None:
                    os.environ.pop("DIOMP_ALLREDUCE_ALGO", None)
                else:
                    os.environ["DIOMP_ALLREDUCE_ALGO"] = prev
    e2e = _coll_e2e(rt, kind, 1 << 30)
    if rt.rank == 0:
        k = rt.nranks
        factor = 2 * (k - 1) / k if kind == "allreduce" else 1.0

        def tab(rs):
            return [(r.size_bytes, round(r.mean_us, 2),
                     round(factor * r.size_bytes / r.mean_us / 1e3, 2)) for r in rs]
        table = tab(rows)
        value = table[-1][2]
        extra = {"roofline": {"bound": "nvlink", "achieved": value, "peak": NVLINK_PEER_GBS,
                              "unit": "GB/s", "frac": round(value / NVLINK_PEER_GBS, 4)},
                 "rows": table, "row_format": "[bytes, mean_us, busBW GB/s]",
                 "algorithm": "exact (reference ring-fold order, bitwise)" if kind == "allreduce"
                 else "p2p"}
        extra["e2e"] = {"value": round(factor * e2e["bytes"] / e2e["seconds"] / 1e9, 2),
                        "unit": "GB/s (busBW)", "h2d_bytes_per_step": e2e["bytes"],
                        "d2h_bytes_per_step": e2e["bytes"], "seconds": round(e2e["seconds"], 5),
                        "note": "host buffer -> put (H2D) into the own send buffer, the "
                                "collective, get (D2H) of the result, on every rank; "
                                "wall clock, max over ranks"}
        if nvls_rows:
            nt = tab(nvls_rows)
            extra["nvls"] = {"busbw_1GiB": nt[-1][2], "rows": nt,
                             "algorithm": "NVSwitch multimem.ld_reduce + multimem.st "
                                          "(f32 sums within rounding of the exact fold)"}
        _line(rt, f"{kind}_busbw_1GiB", value, "GB/s", args,
              {"workload": f"{kind}_f32_sum_sweep_1KiB_1GiB", "endpoints": k}, extra)
    rt.finalize()
    return 0


def _coll_e2e(rt, kind: str, nbytes: int, reps: int = 3) -> dict:
    """One collective end to end through the public API with host buffers."""
    comm = coll.bootstrap(rt, rt.world)
    send = rt.alloc_symmetric(nbytes, 0)
    recv = rt.alloc_symmetric(nbytes, 0)
    host = _pinned(np.random.default_rng(2000 + rt.rank).uniform(-1, 1, nbytes // 4)
                   .astype(np.float32))
    out = _pinned(nbytes=nbytes).view(np.float32)
    op = coll.ReduceOp(coll.ReduceKind.Sum, coll.ElementType.f32)
    me = GlobalAddress(rt.rank, 0, send.addr.offset)
    res = GlobalAddress(rt.rank, 0, (recv if kind == "allreduce" else send).addr.offset)
    best = float("inf")
    for _ in range(reps):
        rt.barrier(rt.world)
        t0 = time.perf_counter()
        rt.put(me, host, nbytes, TransferKind.H2D)
        rt.fence(rt.world)
        if kind == "allreduce":
            coll.allreduce(comm, send.addr, recv.addr, nbytes // 4, op)
        else:
            coll.bcast(comm, send.addr, nbytes, root=0)
        rt.get(res, out, nbytes, TransferKind.D2H).wait(rt.cfg.timeout)
        best = min(best, time.perf_counter() - t0)
    rt.free(recv)
    rt.free(send)
    return {"bytes": nbytes, "seconds": _max_over_ranks(rt, f"e2e/{kind}", best)}


def _dgemm_cli(args):
    from .cannon import CannonRing, MatmulSpec
    n = int(os.environ.get("BENCH_GEMM_N", "16384"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    stripe = (n // world) * n * 8
    rt = _cli_runtime(1 << max(30, (4 * stripe + (64 << 20) - 1).bit_length()))
    spec = MatmulSpec(n, rt.nranks)
    ring = CannonRing(rt, spec, device_seed=0)
    timer = _Timer(rt)
    for _ in range(max(args.warmup, 1)):
        ring.run()
    rt.barrier(rt.world)
    ms = []
    for _ in range(max(args.steps, 1)):
        rt.barrier(rt.world)
        timer.stream = ring._stream(0)
        timer.start()
        for _ in range(spec.p):
            ring.enqueue_step() if ring.sync else ring.run()
        ms.append(timer.stop_ms())
        ring.synchronize()
    got = rt.ctrl.allgather(tuple(range(rt.nranks)), "gemmbench", pickle.dumps(min(ms)))
    t = max(pickle.loads(b) for _, b in got) / 1e3
    ring.release()
    ring = CannonRing(rt, spec, device_seed=0)
    e2e = _ring_e2e(rt, ring, n)
    ring.release()
    # library reference point: cuBLAS DGEMM (torch addmm, f64) over the same
    # per-endpoint shapes -- P products C(ns x n) += A(ns x ns) @ B(ns x n) --
    # without the stripe shift
    t_cublas = _cublas_same_shapes(rt, spec, args)
    got = rt.ctrl.allgather(tuple(range(rt.nranks)), "gemmbench/cublas", pickle.dumps(t_cublas))
    t_cublas = max(pickle.loads(b) for _, b in got)
    if rt.rank == 0:
        tflops = 2.0 * n ** 3 / t / 1e12
        extra = {"ms_per_multiply": round(t * 1e3, 3),
                 "cublas_same_shapes": {"tflops": round(2.0 * n ** 3 / t_cublas / 1e12, 3),
                                        "ms_per_multiply": round(t_cublas * 1e3, 3),
                                        "note": "torch.addmm f64 (cuBLAS DGEMM), P products "
                                                "per endpoint, no ring shift"},
                 "roofline": {"bound": "tensor (DMMA f64)", "achieved": round(tflops / rt.nranks, 3),
                              "peak": round(2.0 * n ** 3 / t_cublas / 1e12 / rt.nranks, 3),
                              "unit": "TFLOP/s per GPU",
                              "frac": round(t_cublas / t, 4),
                              "peak_source": "cuBLAS DGEMM on the same shapes, this run"}}
        extra["e2e"] = e2e
        if rt.nranks == 1 and os.environ.get("BENCH_GEMM_CPU", "1") != "0":
            extra["cpu_baseline"] = _cpu_dgemm_sample(n)
        _line(rt, "dgemm_ring_tflops", round(tflops, 3), "TFLOP/s", args,
              {"workload": f"cannon_ring_{n}^2_fp64", "endpoints": rt.nranks,
               "kernel": "DMMA m8n8k4", "shift": ring.shift if rt.nranks > 1 else None}, extra)
    rt.finalize()
    return 0


def _cublas_same_shapes(rt, spec, args) -> float:
    import torch
    ns, n = spec.ns, spec.n
    dev = torch.device("cuda", rt.gpus[0])
    a = torch.rand(ns, n, dtype=torch.float64, device=dev)
    b = torch.rand(ns, n, dtype=torch.float64, device=dev)
    c = torch.zeros(ns, n, dtype=torch.float64, device=dev)

    def one():
        for s in range(spec.p):
            c.addmm_(a[:, s * ns:(s + 1) * ns], b)
    one()
    torch.cuda.synchronize(dev)
    best = float("inf")
    for _ in range(max(args.steps, 1)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        one()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    del a, b, c
    torch.cuda.empty_cache()
    return best


def _cpu_dgemm_sample(n: int) -> dict:
    """The reference's compute (cannon.py:138, numpy @ -> OpenBLAS) on the
    host cores: one ring step of the P=16 split, C(1024 x n) += A(1024 x 1024)
    @ B(1024 x n), best of 3."""
    ns = 1024
    rng = np.random.default_rng(0)
    a = rng.uniform(-1, 1, (ns, ns))
    b = rng.uniform(-1, 1, (ns, n))
    c = np.zeros((ns, n))
    best = float("inf")
    for _ in range(3):
        t0 = time.perf_counter()
        c += a @ b
        best = min(best, time.perf_counter() - t0)
    return {"value": round(2.0 * ns * ns * n / best / 1e12, 4), "unit": "TFLOP/s",
            "cores": os.cpu_count(), "kind": "reference",
            "sample": f"numpy/OpenBLAS C += A @ B, {ns}x{ns} @ {ns}x{n} (one ring step "
                      f"at P=16), default BLAS threads"}


# ---------------------------------------------------------------------------
# secondary measurements (the other BASELINE configs, reported in the
# headline line of bench.py next to the Minimod 1024^3 number)
# ---------------------------------------------------------------------------

def _max_over_ranks(rt, tag: str, value: float) -> float:
    got = rt.ctrl.allgather(tuple(range(rt.nranks)), tag, pickle.dumps(value))
    return max(pickle.loads(b) for _, b in got)


def measure_stencil_config1(rt: Runtime, n: int = 128, steps: int = 100) -> dict:
    """BASELINE configs[0] (Minimod n^3, `steps` steps; the reference runs it on
    2 ranks) on this job's ranks through the public StencilRunner: device time
    of the whole run (CUDA events, max over ranks), the end-to-end time with
    the zero initial fields copied H2D from pinned host memory and the final
    field D2H inside the timed region, and the sha256 of the gathered field."""
    import hashlib

    import torch

    from .stencil import StencilRunner, StencilSpec, _gather_field, dump_bytes
    spec = StencilSpec(n, n, n, steps=steps)
    runner = StencilRunner(rt, spec)
    timer = _Timer(rt)
    # one untimed warm-up run (the first run pays the module / tensor-map /
    # launch-path warm-up), then zero fields again for the checksummed run
    runner.enqueue(steps) if runner.mode == "fused" else runner.run(steps)
    runner.stream.synchronize()
    rt.barrier(rt.world)   # every neighbour's last halo stores into our ghost planes landed
    base = rt.gm.base(0)
    for rec in (runner.field_a, runner.field_b):
        _native.call("diomp_memset_async", base + rec.addr.offset, 0, runner.nbytes,
                     runner.stream.handle)
    runner.stream.synchronize()
    runner.step = 0
    rt.barrier(rt.world)
    timer.stream = runner.stream.handle
    timer.start()
    runner.enqueue(steps) if runner.mode == "fused" else runner.run(steps)
    dev_s = _max_over_ranks(rt, "cfg1/dev", timer.stop_ms() / 1e3)
    _native.check_device(runner.gpu, "stencil config1")
    rt.barrier(rt.world)
    field = _gather_field(rt, runner.cur_rec, spec, runner.nxl, runner.shape)
    sha = hashlib.sha256(dump_bytes(field)).hexdigest() if rt.rank == 0 else ""
    # end to end: fresh fields from host, run, result back to host
    host_in = torch.zeros(runner.nbytes // 8, dtype=torch.float64).pin_memory()
    host_out = torch.empty(runner.nbytes // 8, dtype=torch.float64).pin_memory()
    base, s = rt.gm.base(0), runner.stream.handle
    runner.step = 0
    rt.barrier(rt.world)
    t0 = time.perf_counter()
    for rec in (runner.field_a, runner.field_b):
        _native.call("diomp_memcpy_async", base + rec.addr.offset, host_in.data_ptr(),
                     runner.nbytes, 1, s)
    runner.enqueue(steps) if runner.mode == "fused" else runner.run(steps)
    _native.call("diomp_memcpy_async", host_out.data_ptr(), base + runner.cur_rec.addr.offset,
                 runner.nbytes, 2, s)
    runner.stream.synchronize()
    rt.barrier(rt.world)
    e2e_s = _max_over_ranks(rt, "cfg1/e2e", time.perf_counter() - t0)
    mode = runner.mode
    runner.free()
    pts = float(n) ** 3 * steps
    return {"workload": f"minimod_{n}^3_{steps}steps", "ranks": rt.nranks, "mode": mode,
            "value": round(pts / dev_s / 1e9, 3), "unit": "Gpts/s",
            "seconds": round(dev_s, 6), "sha256": sha,
            "e2e": {"value": round(pts / e2e_s / 1e9, 3), "unit": "Gpts/s",
                    "seconds": round(e2e_s, 6),
                    "h2d_bytes": 2 * runner.nbytes * rt.nranks,
                    "d2h_bytes": runner.nbytes * rt.nranks}}


def _ring_e2e(rt: Runtime, ring, n: int) -> dict:
    """End to end on a fresh ring (step 0): every rank copies its A stripe and
    its B stripe from pinned host buffers, the ring multiplies, every rank
    copies its C stripe back; wall clock, max over ranks."""
    import torch
    spec = ring.spec
    (e, st), = ring.local.items()
    g = torch.Generator().manual_seed(4000 + e)
    ha = (torch.rand(spec.ns, n, dtype=torch.float64, generator=g) * 2 - 1).pin_memory()
    hb = (torch.rand(spec.ns, n, dtype=torch.float64, generator=g) * 2 - 1).pin_memory()
    hc = torch.empty(spec.ns, n, dtype=torch.float64).pin_memory()
    torch.cuda.synchronize()
    rt.barrier(rt.world)
    t0 = time.perf_counter()
    st["a"].copy_(ha, non_blocking=True)
    ring.stripe(st["dev"], 0).copy_(hb, non_blocking=True)
    st["c"].zero_()
    torch.cuda.synchronize()
    for _ in range(spec.p):
        ring.enqueue_step() if ring.sync else ring.run()
    ring.synchronize()
    hc.copy_(st["c"], non_blocking=True)
    torch.cuda.synchronize()
    sec = _max_over_ranks(rt, "gemm/e2e", time.perf_counter() - t0)
    nb = spec.ns * n * 8 * spec.p
    return {"value": round(2.0 * n ** 3 / sec / 1e12, 3), "unit": "TFLOP/s", "seconds": round(sec, 4),
            "h2d_bytes_per_step": 2 * nb, "d2h_bytes_per_step": nb,
            "note": "A and B stripes H2D from pinned host memory, the ring, C stripes D2H, every rank"}


def measure_dgemm_ring(rt: Runtime, n: int = 16384, reps: int = 3, host_check: bool = True):
    """BASELINE configs[3]: the n x n fp64 ring multiply on this job's
    endpoints.  Device time per multiply (best of `reps`, max over ranks), the
    cuBLAS DGEMM time of the same per-endpoint products without the shift,
    and -- at one rank with host_check -- the reference's inputs
    (_fill_matrices(n, 0)), the end-to-end time (A, B pinned H2D, the ring,
    C D2H) and rel-L2 of C against host BLAS (numpy a @ b, cannon.py:138)."""
    import torch

    from .cannon import CannonRing, MatmulSpec, _fill_matrices
    spec = MatmulSpec(n, rt.nranks)
    host = host_check and rt.nranks == 1
    a = b = None
    if host:
        a, b = _fill_matrices(n, 0)
        ring = CannonRing(rt, spec, a_full=a, b_full=b)
    else:
        ring = CannonRing(rt, spec, device_seed=0)
    timer = _Timer(rt)
    timer.stream = ring._stream(0)

    def one():
        for _ in range(spec.p):
            ring.enqueue_step() if ring.sync else ring.run()

    out = {"workload": f"cannon_ring_{n}^2_fp64", "endpoints": spec.p,
           "kernel": "DMMA m8n8k4", "shift": ring.shift if spec.p > 1 else None}
    if host:
        (e, st), = ring.local.items()
        pa = torch.from_numpy(a).pin_memory()
        pb = torch.from_numpy(b).pin_memory()
        pc = torch.empty(n, n, dtype=torch.float64).pin_memory()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st["a"].copy_(pa, non_blocking=True)
        ring.stripe(st["dev"], 0).copy_(pb, non_blocking=True)
        st["c"].zero_()
        torch.cuda.synchronize()
        ring.step_no = 0
        one()
        ring.synchronize()
        pc.copy_(st["c"], non_blocking=True)
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        got = pc.numpy()
        want = a @ b
        out["rel_l2_vs_host_blas"] = float(np.linalg.norm(got - want) / np.linalg.norm(want))
        out["e2e"] = {"value": round(2.0 * n ** 3 / e2e_s / 1e12, 3), "unit": "TFLOP/s",
                      "seconds": round(e2e_s, 4), "h2d_bytes": 2 * n * n * 8,
                      "d2h_bytes": n * n * 8}
        del pa, pb, pc, got, want
    elif spec.p > 1:
        out["e2e"] = _ring_e2e(rt, ring, n)
    ms = []
    rt.barrier(rt.world)
    for _ in range(reps):
        rt.barrier(rt.world)
        timer.start()
        one()
        ms.append(timer.stop_ms())
        ring.synchronize()
    t = _max_over_ranks(rt, "gemm/dev", min(ms)) / 1e3
    ring.release()

    class _A:
        steps = reps
    t_cublas = _max_over_ranks(rt, "gemm/cublas", _cublas_same_shapes(rt, spec, _A))
    tflops = 2.0 * n ** 3 / t / 1e12
    out.update({"value": round(tflops, 3), "unit": "TFLOP/s", "ms_per_multiply": round(t * 1e3, 3),
                "cublas_same_shapes_tflops": round(2.0 * n ** 3 / t_cublas / 1e12, 3),
                "frac_of_cublas": round(t_cublas / t, 4)})
    return out


def measure_p2p(rt: Runtime, sizes=(8, 64 * MIB, 1 << 30), iters: int = 5) -> dict | None:
    """BASELINE configs[1] legs between rank 0 and rank 1: D2D put / get
    bandwidth (device-timed), 8 B put+fence and get+wait latency (host API),
    and the end-to-end put with a HOST payload (kind H2D, the reference's
    default) at the largest size."""
    if rt.nranks < 2:
        return None
    big = [x for x in sizes if x >= MIB]
    res = {}
    for kind in (BenchKind.Bandwidth, BenchKind.GetBandwidth):
        res[kind.value] = {}
        for size in big:
            rows = run_p2p(rt, BenchSpec(kind, (size,), iters=bw_iters(size, iters), warmup=2,
                                         transfer=TransferKind.D2D))
            res[kind.value].update({r.size_bytes: round(r.size_bytes / r.mean_us / 1e3, 2)
                                    for r in rows})
    for kind in (BenchKind.PutLatency, BenchKind.GetLatency):
        rows = run_p2p(rt, BenchSpec(kind, (8,), iters=200, warmup=20, transfer=TransferKind.D2D))
        res[kind.value] = {r.size_bytes: round(r.mean_us, 2) for r in rows}
    rows = run_p2p(rt, BenchSpec(BenchKind.Bandwidth, (max(big),), iters=2, warmup=1))
    res["bw_h2d"] = {r.size_bytes: round(r.size_bytes / r.mean_us / 1e3, 2) for r in rows}
    if rt.rank != 0:
        return None
    top = max(big)
    return {"workload": "p2p_rank0_rank1", "unit": "GB/s",
            "put_bw": res["bw"], "get_bw": res["get_bw"],
            "put_latency_us_8B": res["put"].get(8), "get_latency_us_8B": res["get"].get(8),
            "value": res["bw"][top], "frac_of_peer_copy": round(res["bw"][top] / NVLINK_PEER_GBS, 4),
            "e2e": {"value": res["bw_h2d"][top], "unit": "GB/s", "h2d_bytes": top,
                    "d2h_bytes": 0, "note": "put with a host payload (TransferKind.H2D)"}}


def measure_collectives(rt: Runtime, sizes=(64 * MIB, 1 << 30), iters: int = 5) -> dict | None:
    """BASELINE configs[2] top sizes: allreduce (f32 sum, exact fold) and bcast
    busBW over every rank, device-timed, max over ranks."""
    if rt.nranks < 2:
        return None
    out = {}
    comm = coll.bootstrap(rt, rt.world)
    k = rt.nranks
    for kind in (BenchKind.Allreduce, BenchKind.Bcast):
        f = 2 * (k - 1) / k if kind is BenchKind.Allreduce else 1.0
        out[kind.value] = {}
        for size in sizes:
            rows = run_collective(rt, BenchSpec(kind, (size,), iters=bw_iters(size, iters),
                                                warmup=2), comm)
            out[kind.value].update({r.size_bytes: round(f * r.size_bytes / r.mean_us / 1e3, 2)
                                    for r in rows})
    if rt.rank != 0:
        return None
    return {"workload": f"collectives_k{k}", "unit": "GB/s (busBW)",
            "allreduce": out["allreduce"], "bcast": out["bcast"],
            "frac_of_peer_copy_64MiB": {kk: round(v[64 * MIB] / NVLINK_PEER_GBS, 4)
                                        for kk, v in out.items() if 64 * MIB in v}}


def cli_bench(args) -> int:
    if args.workload == "p2p":
        return _p2p_cli(args)
    if args.workload in ("allreduce", "bcast"):
        return _coll_cli(args, args.workload)
    if args.workload == "dgemm":
        return _dgemm_cli(args)
    raise UsageError(f"unknown workload {args.workload!r}")
