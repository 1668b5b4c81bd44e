"""Benchmark driver (one JSON line on rank 0).

Headline workload (BASELINE.json configs[4], "Minimod 1024^3 grid strong
scaling 1/2/4/8 GPUs with overlapped halo exchange"): one step = one leapfrog
time step of the 8th-order acoustic stencil over the whole 1024^3 grid,
x-slabs of 1024/N planes per GPU, halos stored straight into the neighbours'
ghost planes by the fused kernel.  metric = Gpts/s (interior points x steps /
max-over-ranks device time).  Fields are 8.8 GB each at N=1 (always > L2), so
no L2 flush is needed.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--workload stencil|p2p|allreduce|dgemm]

N>1 is launched by the driver as torchrun --nproc-per-node N; each rank
drives LOCAL_RANK's GPU.  --impl reference times the reference's own compiled
CPU kernel (oracle/_ref, built from reference/pkg/src/diomp/kernels/_core.c)
on the host cores, same metric and config.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

GRID = int(os.environ.get("BENCH_GRID", "1024"))
GEMM_N = int(os.environ.get("BENCH_GEMM_N", "16384"))
FALLBACK_HBM_GBS = 6650.0
E2E_MIN_STEPS = 100


def _env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _peaks():
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def _traffic_per_launch(key: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed
    ncu --set full capture summary (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(HERE, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(key)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int, interval_ms: int = 50):
        self.gpu, self.interval = gpu, interval_ms
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", f"-lms", str(self.interval)],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                    rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][2]),
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())
                if any(r[3].replace(".", "").isdigit() for r in rows) else None}


# ---------------------------------------------------------------------------
# CPU reference arm / baseline (oracle/_ref = the reference's compiled kernel)
# ---------------------------------------------------------------------------

_W = {}


def _cpu_init(kind, planes, ny, nz):
    import numpy as np
    sys.path.insert(0, HERE)
    from oracle import oracle as O
    _, w = O.time_params(4)
    shape = (planes + 8, ny + 8, nz + 8)
    u_cur = np.full(shape, 0.25)
    u_cur[1::3] = -0.5
    _W.update(u_cur=u_cur, u_prev=u_cur * 0.5, w=w, center=3.0 * w[0],
              pts=planes * ny * nz,
              fn=_load_ref_core().stencil_update if kind == "reference" else O.stencil_update_c)
    _cpu_step(0)  # warm


def _cpu_step(_):
    t0 = time.perf_counter()
    w = _W["w"]
    _W["fn"](_W["u_prev"], _W["u_cur"], _W["u_prev"], _W["center"], w, w, w, 4)
    return _W["pts"], time.perf_counter() - t0


def _load_ref_core():
    import importlib.util
    d = os.path.join(HERE, "oracle", "_ref")
    for f in sorted(os.listdir(d)):
        if f.startswith("_core") and f.endswith(".so"):
            spec = importlib.util.spec_from_file_location("_core", os.path.join(d, f))
            mod = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(mod)
            return mod
    raise ImportError("oracle/_ref/_core*.so not built")


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


class CpuReference:
    """The reference's compiled stencil_update (oracle/_ref, built from
    reference/pkg/src/diomp/kernels/_core.c with -O3 -ffp-contract=off) on
    the host cores: one x-slab per process, like the reference's
    one-single-threaded-rank-per-core layout.  kind = "port" when only the
    oracle restatement is available."""

    def __init__(self, grid: int, planes: int = 8, max_cores: int = 64):
        import multiprocessing as mp
        self.kind = "reference"
        try:
            _load_ref_core()
        except Exception:
            self.kind = "port"
        self.cores = min(os.cpu_count() or 1, max_cores)
        self.planes, self.grid = planes, grid
        self.pool = mp.get_context("fork").Pool(self.cores, initializer=_cpu_init,
                                                initargs=(self.kind, planes, grid, grid))

    def step(self) -> float:
        """One stencil step on every core's slab; aggregate Gpts/s."""
        res = self.pool.map(_cpu_step, range(self.cores), chunksize=1)
        return sum(r[0] for r in res) / max(r[1] for r in res) / 1e9

    def describe(self, value: float, steps: int) -> dict:
        return {"value": round(value, 4), "unit": "Gpts/s", "cores": self.cores, "kind": self.kind,
                "cpu_model": _cpu_model(),
                "sample": f"{self.cores} processes x {steps} steps of a "
                          f"{self.planes}x{self.grid}x{self.grid} slab each (reference "
                          f"stencil_update, aggregate over cores)"}

    def close(self):
        self.pool.terminate()


def cpu_baseline(grid: int, steps: int = 3) -> dict:
    ref = CpuReference(grid)
    try:
        vals = [ref.step() for _ in range(steps)]
        return ref.describe(statistics.median(vals), steps)
    finally:
        ref.close()


def _reference_whole_config(steps: int):
    """The reference's own run_stencil structure at the headline config:
    GRID^3 as x-slabs on a power-of-two number of host processes (one
    single-threaded rank per core, as the reference runs), one-sided halo
    copies + barrier every step, the reference's compiled stencil_update
    (oracle/ports.stencil_procs).  None when the host lacks the memory."""
    from oracle import ports as P
    cores = min(os.cpu_count() or 1, 64)
    nr = 1 << (cores.bit_length() - 1)
    while GRID % nr:
        nr //= 2
    need = 2 * nr * (GRID // nr + 8) * (GRID + 8) ** 2 * 8
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        avail = 0
    if avail and need > 0.6 * avail:
        return None
    r = P.stencil_procs(GRID, GRID, GRID, steps, nr, checksum=False)
    return r, nr


def run_reference_arm(args):
    rank, world, _ = _env_rank()
    if rank != 0:
        return 0
    steps = max(1, min(args.steps, 10))   # ~1 s of host time per step at 1024^3
    whole = None
    try:
        whole = _reference_whole_config(steps)
    except Exception as e:   # report below, fall back to the per-core slab sample
        sys.stderr.write(f"whole-config reference run failed: {e!r}\n")
    if whole is not None:
        r, nr = whole
        value, wall = r["gpts"], r["seconds"]
        cpu = {"value": round(value, 4), "unit": "Gpts/s", "cores": nr, "kind": r["kernel"],
               "cpu_model": _cpu_model(), "seconds": round(wall, 3),
               "sample": f"the whole config: run_stencil {GRID}^3 x {steps} steps on {nr} "
                         f"processes (x-slabs, one-sided halo copies + barrier per step, the "
                         f"reference's compiled stencil_update; oracle/ports.stencil_procs)"}
        steps_done = steps
    else:
        ref = CpuReference(GRID)
        try:
            for _ in range(args.warmup):
                ref.step()
            t0 = time.perf_counter()
            vals = [ref.step() for _ in range(args.steps)]
            wall = time.perf_counter() - t0
        finally:
            ref.close()
        value = statistics.median(vals)
        cpu = ref.describe(value, args.steps)
        steps_done = args.steps
    sec = {}
    if not args.no_secondary:
        sec = {"minimod_128": {"workload": "minimod_128^3_100steps", "ranks": 2}}
        if world >= 2:
            sec["p2p"] = {"value": 0.0}
            sec["collectives"] = {"allreduce": {}}
        if world == 1:
            sec["dgemm_ring"] = {"value": 0.0, "workload": f"cannon_ring_{GEMM_N}^2_fp64"}
        sec["minimod_128"]["value"] = 0.0
        _secondary_cpu(sec, world)
        for v in sec.values():   # the CPU arm's own numbers are the values
            if isinstance(v, dict) and "cpu_baseline" in v:
                v["value"] = v["cpu_baseline"]["value"]
                v["unit"] = v["cpu_baseline"]["unit"]
    line = {"metric": "minimod_gpts_per_s", "value": round(value, 4), "unit": "Gpts/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(wall / steps_done * 1e3, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"minimod_{GRID}^3_strong_scaling", "grid": [GRID] * 3,
                       "radius": 4},
            "impl": "reference", "cpu_baseline": cpu,
            "e2e": {"value": round(value, 4), "unit": "Gpts/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if sec:
        line["secondary"] = sec
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def _secondary_bytes(world: int) -> int:
    """Segment room for the secondary measurements (linear heap, no reuse
    across sizes): two DGEMM ring stripes + the 1 GiB p2p / collective pair."""
    ns = GEMM_N // world
    return 2 * ns * GEMM_N * 8 + (2 << 30) + (256 << 20)


def _make_runtime(world: int, rank: int, local: int, field_bytes: int):
    from paper_2506_02486_b200 import (AllocatorKind, LaunchConfig, SegmentConfig, runtime)
    from paper_2506_02486_b200.config import resolve_from_env
    need = (2 * field_bytes + (64 << 20) + _secondary_bytes(world)) * 4 // 3
    seg = 1 << max(24, (need - 1).bit_length())
    os.environ.setdefault("DIOMP_GPUS", str(local))
    cfg = resolve_from_env(LaunchConfig(nranks=world, segment=SegmentConfig(
        seg, AllocatorKind.Linear)))
    return runtime.Runtime(cfg)


def _max_over_ranks(rt, value: float) -> float:
    import pickle
    got = rt.ctrl.allgather(tuple(range(rt.nranks)), "bench/max", pickle.dumps(value))
    return max(pickle.loads(b) for _, b in got)


def run_stencil_bench(args):
    import numpy as np
    import torch

    from paper_2506_02486_b200 import _native
    from paper_2506_02486_b200.apps.stencil import StencilRunner, StencilSpec

    rank, world, local = _env_rank()
    torch.cuda.set_device(local)
    nxl = GRID // world
    shape = (nxl + 8, GRID + 8, GRID + 8)
    field_bytes = int(np.prod(shape)) * 8
    rt = _make_runtime(world, rank, local, field_bytes)
    spec = StencilSpec(GRID, GRID, GRID, steps=args.steps)
    runner = StencilRunner(rt, spec)
    gpu = runner.gpu
    stream = runner.stream.handle

    # warm-up (>= 3 steps), then K timed steps bracketed by barrier + sync
    runner.enqueue(max(args.warmup, 3))
    runner.stream.synchronize()
    ev0, ev1 = _native.event_create(gpu), _native.event_create(gpu)
    rt.barrier(rt.world)
    _native.call("diomp_device_sync", gpu)
    with ClockSampler(gpu) as clocks:
        _native.call("diomp_event_record", ev0, stream)
        runner.enqueue(args.steps)
        _native.call("diomp_event_record", ev1, stream)
        _native.call("diomp_event_sync", ev1)
    _native.check_device(gpu, "stencil bench")
    rt.barrier(rt.world)
    ms = _native.event_elapsed_ms(ev0, ev1)
    ms_max = _max_over_ranks(rt, ms)
    pts = float(GRID) ** 3 * args.steps
    value = pts / (ms_max / 1e3) / 1e9

    # roofline: 24 algorithmic bytes per interior point per step (read u_cur,
    # read u_prev, write u_next); one kernel launch per step per GPU
    local_pts = nxl * GRID * GRID
    per_launch_ms = ms / args.steps
    achieved = 24.0 * local_pts / (per_launch_ms / 1e3) / 1e9
    peak, peak_src = _peaks()
    traffic = _traffic_per_launch(f"stencil_{GRID}_n{world}")

    # end to end through the public driver class: host (pinned) initial fields
    # H2D, the steps, final interior D2H, all inside the timed region.  One
    # run of at least E2E_MIN_STEPS steps (the PCIe legs are per run, not per
    # step, so a short K would measure mostly the copies).
    runner.free()
    e2e = None
    if not args.no_e2e:
        e2e = _stencil_e2e(rt, spec, max(args.steps, E2E_MIN_STEPS), field_bytes)
    clk = clocks.summary()
    # one stencil kernel per step; with neighbours, one one-thread signal
    # kernel per neighbour after the last step (rank 0: right only)
    launches = args.steps + (1 if world > 1 else 0)
    secondary = None if args.no_secondary else _secondary(rt, rank, world)
    if rank == 0:
        line = {"metric": "minimod_gpts_per_s", "value": round(value, 3), "unit": "Gpts/s",
                "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
                "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (zero fields + point source, reference initial condition)",
                "config": {"workload": f"minimod_{GRID}^3_strong_scaling", "grid": [GRID] * 3,
                           "radius": 4, "decomposition": f"x-slabs of {nxl} planes",
                           "mode": runner.mode, "l2": "inputs larger than L2 (no flush)",
                           "parallelism": f"slab{world}"},
                "roofline": {"bound": "hbm", "achieved": round(achieved, 1),
                             "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                             "traffic": traffic, "peak_source": peak_src,
                             "bytes_per_point": 24, "points_per_launch": local_pts},
                "e2e": e2e, "gpu_launches": launches, "clocks": clk}
        if world == 1 and not args.no_cpu:
            try:
                line["cpu_baseline"] = cpu_baseline(GRID)
            except Exception as e:  # report, do not fail the GPU number
                line["cpu_baseline"] = {"error": str(e)[:200]}
        if secondary is not None:
            if not args.no_cpu:
                _secondary_cpu(secondary, world)
            line["secondary"] = secondary
        print(json.dumps(line), flush=True)
    rt.finalize()
    return 0


def _secondary(rt, rank, world):
    """The other BASELINE configs, measured in the same run on the same
    runtime (after the headline's fields are freed): configs[0] Minimod 128^3
    x 100 steps, configs[3] the 16384^2 fp64 ring (reference inputs and a
    host-BLAS rel-L2 at one GPU), and at >= 2 GPUs configs[1] put/get and
    configs[2] allreduce / bcast at 64 MiB and 1 GiB."""
    from paper_2506_02486_b200.apps import bench as appbench
    out = {}
    for name, fn in (("minimod_128", lambda: appbench.measure_stencil_config1(rt)),
                     ("dgemm_ring", lambda: appbench.measure_dgemm_ring(rt, GEMM_N)),
                     ("p2p", lambda: appbench.measure_p2p(rt)),
                     ("collectives", lambda: appbench.measure_collectives(rt))):
        try:
            v = fn()
        except Exception as e:   # report, do not lose the headline
            v = {"error": f"{type(e).__name__}: {str(e)[:300]}"}
        if v is not None and rank == 0:
            out[name] = v
    if rank == 0 and "minimod_128" in out and "sha256" in out["minimod_128"]:
        try:
            gold = json.load(open(os.path.join(HERE, "tests", "golden", "stencil_golden.json")))
            want = [c["sha256"] for c in gold["cases"]
                    if (c["nx"], c["steps"], c["amp"]) == (128, 100, 1.0)][0]
            out["minimod_128"]["matches_reference_sha256"] = out["minimod_128"]["sha256"] == want
        except Exception:
            pass
    return out if rank == 0 else None


def _secondary_cpu(sec, world):
    """cpu_baseline of each secondary entry: the oracle's multi-process
    restatements of the reference's drivers (oracle/ports.py) on the host."""
    from oracle import ports as P
    try:
        if "minimod_128" in sec and "value" in sec["minimod_128"]:
            r = P.stencil_procs(128, 128, 128, 100, 2, checksum=False)
            sec["minimod_128"]["cpu_baseline"] = {
                "value": round(r["gpts"], 4), "unit": "Gpts/s", "cores": 2, "kind": r["kernel"],
                "seconds": round(r["seconds"], 3),
                "sample": "the whole config: run_stencil 128^3 x 100 steps on 2 processes "
                          "(shared-memory halo puts + barrier, the reference's compiled "
                          "stencil_update)"}
        if "dgemm_ring" in sec and "value" in sec["dgemm_ring"] and world == 1:
            from paper_2506_02486_b200.apps import bench as appbench
            sec["dgemm_ring"]["cpu_baseline"] = appbench._cpu_dgemm_sample(GEMM_N)
        if sec.get("p2p") and "value" in sec["p2p"]:
            r = P.p2p_sample()
            sec["p2p"]["cpu_baseline"] = {
                "value": round(r["put_bandwidth_gbs"], 3), "unit": "GB/s", "cores": 2,
                "kind": "port", "put_latency_us_8B": round(r["put_latency_us_8B"], 2),
                "get_latency_us_8B": round(r["get_latency_us_8B"], 2),
                "get_bandwidth_gbs": round(r["get_bandwidth_gbs"], 3),
                "sample": "2 processes, loopback TCP with the reference's wire frames "
                          "(oracle/ports.WirePair): 8 x 64 MiB puts + fence, 200 x 8 B"}
        if sec.get("collectives") and "allreduce" in sec["collectives"]:
            cb = {}
            for op in ("allreduce", "bcast"):
                r = P.ring_collective(op, world, 64 << 20, iters=3, check=False)
                cb[op] = round(r["busbw_gbs"], 4)
            sec["collectives"]["cpu_baseline"] = {
                "value": cb["allreduce"], "unit": "GB/s (busBW)", "cores": world, "kind": "port",
                "bcast": cb["bcast"],
                "sample": f"{world} processes in a loopback-TCP ring (oracle/ports), 64 MiB, "
                          "3 reps each"}
    except Exception as e:
        sec["cpu_baseline_error"] = str(e)[:300]


def _stencil_e2e(rt, spec, steps, field_bytes):
    import numpy as np
    import torch

    from paper_2506_02486_b200 import _native
    from paper_2506_02486_b200.apps.stencil import StencilRunner

    runner = StencilRunner(rt, spec)
    host_in = torch.zeros(field_bytes // 8, dtype=torch.float64).pin_memory()
    host_out = torch.empty(field_bytes // 8, dtype=torch.float64).pin_memory()
    base = rt.gm.base(0)
    s = runner.stream.handle
    rt.barrier(rt.world)
    t0 = time.perf_counter()
    for rec in (runner.field_a, runner.field_b):
        _native.call("diomp_memcpy_async", base + rec.addr.offset, host_in.data_ptr(),
                     field_bytes, 1, s)
    runner.enqueue(steps)
    _native.call("diomp_memcpy_async", host_out.data_ptr(), base + runner.cur_rec.addr.offset,
                 field_bytes, 2, s)
    runner.stream.synchronize()
    rt.barrier(rt.world)
    dt = _max_over_ranks(rt, time.perf_counter() - t0)
    runner.free()
    return {"value": round(float(spec.nx) ** 3 * steps / dt / 1e9, 3), "unit": "Gpts/s",
            "h2d_bytes_per_step": int(2 * field_bytes * rt.nranks / steps),
            "d2h_bytes_per_step": int(field_bytes * rt.nranks / steps),
            "steps": steps,
            "note": "public StencilRunner, one run of `steps` steps; initial fields H2D from "
                    "pinned host, final field D2H, both inside the timed region"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="stencil")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.workload == "stencil":
        return run_stencil_bench(args)
    from paper_2506_02486_b200.apps import bench as appbench
    if not args.no_cpu:
        appbench._LINE_HOOK = _cli_cpu_hook
    return appbench.cli_bench(args)


def _cli_cpu_hook(d):
    """cpu_baseline for the --workload lines: the oracle's restatement of the
    reference's own CPU path for that config (oracle/ports.py), on rank 0."""
    from oracle import ports as P
    world = d.get("n_gpus", 1)
    try:
        if d["metric"].startswith("put_bandwidth"):
            r = P.p2p_sample()
            d["cpu_baseline"] = {"value": round(r["put_bandwidth_gbs"], 3), "unit": "GB/s",
                                 "cores": 2, "kind": "port",
                                 "put_latency_us_8B": round(r["put_latency_us_8B"], 2),
                                 "get_latency_us_8B": round(r["get_latency_us_8B"], 2),
                                 "get_bandwidth_gbs": round(r["get_bandwidth_gbs"], 3),
                                 "sample": "2 processes, loopback TCP, the reference's wire "
                                           "frames: 8 x 64 MiB puts + fence; 200 x 8 B"}
        elif d["metric"].startswith(("allreduce", "bcast")):
            op = "allreduce" if d["metric"].startswith("allreduce") else "bcast"
            rows = []
            for nbytes in (1 << 20, 64 << 20):
                r = P.ring_collective(op, world, nbytes, iters=3, check=False)
                rows.append((nbytes, round(r["seconds"] * 1e6, 1), round(r["busbw_gbs"], 4)))
            d["cpu_baseline"] = {"value": rows[-1][2], "unit": "GB/s (busBW)", "cores": world,
                                 "kind": "port", "rows": rows,
                                 "sample": f"{world} processes, loopback-TCP ring "
                                           "(oracle/ports.ring_collective), 1 MiB and 64 MiB"}
        elif d["metric"].startswith("dgemm") and world == 1:
            pass   # already attached (OpenBLAS sample) by the dgemm CLI
    except Exception as e:
        d["cpu_baseline"] = {"error": str(e)[:300]}


if __name__ == "__main__":
    sys.exit(main())
