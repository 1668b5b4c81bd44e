"""Generate golden fixtures by importing the REFERENCE package (read-only at
/root/reference/pkg/src) and running its own code paths.

Run here (not on the GPU box -- /root/reference does not exist there):

    python tests/golden/make_golden.py

Outputs (committed): tests/golden/stencil_golden.json, collectives_golden.npz,
allocator_golden.json, kernels_golden.npz.  The reference's compiled kernel
core is taken from oracle/_ref (built from the reference's own _core.c by
oracle/Makefile) when present, else its numpy backend (bitwise equal,
kernels/__init__.py:1-6).
"""

from __future__ import annotations

import hashlib
import importlib.util
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
MIB = 1024 * 1024


def _import_reference():
    core = None
    ref_dir = os.path.join(REPO, "oracle", "_ref")
    for f in os.listdir(ref_dir) if os.path.isdir(ref_dir) else []:
        if f.startswith("_core") and f.endswith(".so"):
            spec = importlib.util.spec_from_file_location("diomp.kernels._core",
                                                          os.path.join(ref_dir, f))
            core = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(core)
            sys.modules["diomp.kernels._core"] = core
    os.environ["DIOMP_KERNELS"] = "cy" if core is not None else "py"
    sys.path.insert(0, REF_SRC)
    import diomp  # noqa: F401
    return diomp


def stencil_cases(diomp):
    from diomp.apps.stencil import StencilSpec, run_stencil, _time_params
    from diomp.emulate import run_emulated

    cases = [
        # (nx, ny, nz, steps, amp, ranks)
        (16, 12, 12, 4, 1.0, (1, 2)),
        (24, 20, 18, 7, 1.0, (1, 2, 3)),
        (20, 15, 13, 5, 1.0, (1, 2)),          # odd ny/nz: generic-kernel path
        (64, 64, 64, 100, 1.0, (1, 2, 4)),
        (64, 64, 64, 100, 0.0, (1,)),
        (128, 128, 128, 100, 1.0, (2,)),       # BASELINE config 1
    ]
    out = []
    for nx, ny, nz, steps, amp, ranks in cases:
        sums = {}
        for p in ranks:
            seg = 1 << max(21, (2 * 8 * (nx // p + 8) * (ny + 8) * (nz + 8) * 4 - 1).bit_length())
            spec = StencilSpec(nx, ny, nz, steps=steps, source_amplitude=amp)
            res = run_emulated(p, lambda rt: run_stencil(rt, spec).checksum,
                               segment_bytes=seg, timeout=600.0)
            sums[p] = res[0]
            print(f"stencil {nx}x{ny}x{nz} steps={steps} amp={amp} ranks={p}: {res[0]}",
                  flush=True)
        assert len(set(sums.values())) == 1, sums
        out.append(dict(nx=nx, ny=ny, nz=nz, steps=steps, amp=amp,
                        ranks=list(ranks), sha256=next(iter(sums.values()))))
    dt, w = _time_params(4)
    meta = dict(dt=dt.hex(), w=[float(x).hex() for x in w], center=float(3.0 * w[0]).hex())
    return dict(cases=out, time_params=meta)


def kernel_fixtures(diomp):
    from diomp.kernels import reference as kref
    arrays = {}
    # stencil_update seam: random fields, distinct per-axis weights, R=4 and R=2
    for name, shape, r in [("s4", (14, 13, 12), 4), ("s4b", (11, 17, 20), 4),
                           ("s2", (9, 8, 7), 2), ("s3", (10, 12, 16), 3)]:
        rng = np.random.default_rng(len(name) * 97 + r)
        u_cur = rng.uniform(-1, 1, shape)
        u_prev = rng.uniform(-1, 1, shape)
        wx, wy, wz = (rng.uniform(-0.1, 0.1, r + 1) for _ in range(3))
        center = float(rng.uniform(-0.5, 0.5))
        u_next = u_prev.copy()
        kref.stencil_update(u_next, u_cur, u_next, center, wx, wy, wz, r)
        arrays[f"{name}_cur"] = u_cur
        arrays[f"{name}_prev"] = u_prev
        arrays[f"{name}_w"] = np.stack([wx, wy, wz])
        arrays[f"{name}_center"] = np.array([center])
        arrays[f"{name}_out"] = u_next
    # matmul_f64 seam
    for name, (n, k, m) in [("m1", (13, 7, 9)), ("m2", (33, 65, 17)), ("m3", (64, 64, 64))]:
        rng = np.random.default_rng(n * 1000 + k * 10 + m)
        a = rng.uniform(-1, 1, (n, k))
        b = rng.uniform(-1, 1, (k, m))
        c = np.empty((n, m))
        kref.matmul_f64(a, b, c)
        arrays[f"{name}_a"], arrays[f"{name}_b"], arrays[f"{name}_c"] = a, b, c
    return arrays


def collective_fixtures(diomp):
    """Run the reference's own bcast/reduce/allreduce in its emulated runtime."""
    from diomp import collectives as coll
    from diomp.emulate import run_emulated

    arrays = {}
    dtypes = {"f32": np.float32, "f64": np.float64, "i32": np.int32, "i64": np.int64}

    def contrib(rank, etype, count, seed):
        rng = np.random.default_rng(seed * 100 + rank)
        if etype.startswith("f"):
            v = rng.uniform(-1, 1, count).astype(dtypes[etype])
            if count > 8:
                v[3] = np.nan if rank == 1 else v[3]
                v[5] = -0.0 if rank % 2 else 0.0
            return v
        return rng.integers(-2**30, 2**30, count).astype(dtypes[etype])

    cases = []
    seed = 0
    for k in (2, 3, 4, 8):
        for etype in ("f32", "f64", "i32", "i64"):
            for kind in ("sum", "min", "max"):
                for which in ("allreduce", "reduce"):
                    seed += 1
                    count = [1, 7, 1000, 4099][seed % 4]
                    root = seed % k
                    cases.append((k, etype, kind, which, count, root, seed))

    for (k, etype, kind, which, count, root, seed) in cases:
        op = coll.ReduceOp(coll.ReduceKind(kind), coll.ElementType(etype))
        isz = np.dtype(dtypes[etype]).itemsize

        def fn(rt, k=k, etype=etype, which=which, count=count, root=root, seed=seed, op=op,
               isz=isz):
            comm = coll.bootstrap(rt, rt.world)
            send = rt.alloc_symmetric(max(count * isz, 64), 0)
            recv = rt.alloc_symmetric(max(count * isz, 64), 0)
            v = contrib(rt.rank, etype, count, seed)
            rt.gm.arena(0)[send.addr.offset:send.addr.offset + v.nbytes] = v.view(np.uint8)
            if which == "allreduce":
                coll.allreduce(comm, send.addr, recv.addr, count, op)
            else:
                coll.reduce(comm, send.addr, recv.addr, count, op, root=root)
            return bytes(rt.gm.view(0, recv.addr.offset, count * isz))

        res = run_emulated(k, fn, segment_bytes=2 * MIB, timeout=120.0)
        key = f"{which}_{k}_{etype}_{kind}_{count}_{root}_{seed}"
        if which == "allreduce":
            assert len(set(res)) == 1
            arrays[key] = np.frombuffer(res[0], dtype=dtypes[etype])
        else:
            arrays[key] = np.frombuffer(res[root], dtype=dtypes[etype])
        print("collective", key, flush=True)
    return arrays


def allocator_fixtures(diomp):
    from diomp.allocators import BuddyAllocator, LinearAllocator, ReverseBumpAllocator
    from diomp.errors import OutOfSegment
    from diomp.global_memory import (AllocatorKind, GlobalMemory, SegmentConfig)

    traces = {}
    rng = np.random.default_rng(7)
    for name, make in [("buddy", lambda: BuddyAllocator(4 * MIB)),
                       ("buddy_reserved", lambda: BuddyAllocator(4 * MIB, reserve_from=3 * MIB)),
                       ("linear", lambda: LinearAllocator(4 * MIB)),
                       ("reverse", lambda: ReverseBumpAllocator(3 * MIB, 4 * MIB))]:
        alloc = make()
        live, ops, trace = [], [], []
        for _ in range(400):
            if live and rng.random() < 0.45:
                i = int(rng.integers(0, len(live)))
                off = live.pop(i)
                ops.append(["free", i])
                trace.append(["f", off, alloc.free(off)])
            else:
                size = int(rng.integers(1, 70_000))
                ops.append(["alloc", size])
                try:
                    off = alloc.alloc(size)
                    live.append(off)
                    trace.append(["a", off, alloc.block_size(size)])
                except OutOfSegment:
                    trace.append(["oom"])
        traces[name] = dict(ops=ops, trace=trace)

    # global-memory ledger: interleaved symmetric / asymmetric allocations
    gm_cases = {}
    for kind in (AllocatorKind.Buddy, AllocatorKind.Linear):
        gm = GlobalMemory(SegmentConfig(4 * MIB, kind), 1)
        seq = []
        rng2 = np.random.default_rng(11)
        cells = []
        for i in range(30):
            size = int(rng2.integers(100, 40_000))
            rec = gm.local_alloc_symmetric(size, 0)
            seq.append(["sym", size, rec.addr.offset, rec.size])
            asz = int(rng2.integers(0, 60_000)) if i % 5 else 0
            cell = gm.local_alloc_asymmetric(asz, 0)
            cells.append(cell)
            seq.append(["asym", asz, cell.cell_addr.offset, cell.generation,
                        cell.local_payload.offset if cell.local_payload else None])
            if i % 7 == 3:
                gm.local_free_cell(cells[0])
                seq.append(["free_cell", cells[0].cell_addr.offset])
                cells.pop(0)
            if i % 9 == 4:
                gm.local_free(rec)
                seq.append(["free", rec.addr.offset])
        gm_cases[kind.value] = dict(seq=seq, ledger=[list(x) for x in gm.full_ledger(0)])
    return dict(allocators=traces, global_memory=gm_cases)


def main():
    diomp = _import_reference()
    print("reference kernels backend:", diomp.kernels.BACKEND)
    with open(os.path.join(HERE, "allocator_golden.json"), "w") as f:
        json.dump(allocator_fixtures(diomp), f)
    np.savez_compressed(os.path.join(HERE, "kernels_golden.npz"), **kernel_fixtures(diomp))
    np.savez_compressed(os.path.join(HERE, "collectives_golden.npz"),
                        **collective_fixtures(diomp))
    with open(os.path.join(HERE, "stencil_golden.json"), "w") as f:
        json.dump(stencil_cases(diomp), f, indent=1)
    h = hashlib.sha256()
    for fn in sorted(os.listdir(HERE)):
        if fn.endswith((".json", ".npz")):
            h.update(open(os.path.join(HERE, fn), "rb").read())
    print("golden digest", h.hexdigest())


if __name__ == "__main__":
    main()
