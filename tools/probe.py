"""Kernel-level timing probes (CUDA events, warm-up, inputs > L2).

    python tools/probe.py dgemm [N]      DMMA DGEMM vs cuBLAS (torch.matmul f64)
    python tools/probe.py copy           SM copy kernel (local D2D), 8 B .. 1 GiB
    python tools/probe.py stencil [G [NX]] stencil_update seam on a G^3 field / NX x G x G slab
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)


def _time(fn, iters=10, warm=3):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def dgemm(n=8192, nn=None, k=None):
    """C(n x nn) += A(n x k) @ B(k x nn); square when only n is given."""
    import torch

    from paper_2506_02486_b200 import gemm
    nn, k = nn or n, k or n
    A = torch.rand(n, k, dtype=torch.float64, device="cuda")
    B = torch.rand(k, nn, dtype=torch.float64, device="cuda")
    C = torch.zeros(n, nn, dtype=torch.float64, device="cuda")
    ms = _time(lambda: gemm.dgemm_accumulate(A, B, C), iters=5, warm=2)
    ms_cublas = _time(lambda: C.addmm_(A, B), iters=5, warm=2)
    fl = 2.0 * n * nn * k
    return {"probe": "dgemm", "m_n_k": [n, nn, k], "dmma_ms": ms, "dmma_tflops": fl / ms / 1e9,
            "cublas_ms": ms_cublas, "cublas_tflops": fl / ms_cublas / 1e9,
            "frac_of_cublas": ms_cublas / ms}


def copy():
    import torch

    from paper_2506_02486_b200 import _native
    out = []
    buf = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
    src, dst = buf.data_ptr(), buf.data_ptr() + (1 << 30)
    s = torch.cuda.current_stream().cuda_stream
    for p in range(3, 31, 3):
        n = 1 << p
        ms = _time(lambda: _native.call("diomp_copy", 0, dst, src, n, s), iters=20)
        out.append({"bytes": n, "us": ms * 1e3, "GBps_rw": 2 * n / ms / 1e6})
    return {"probe": "copy_local", "rows": out}


def stencil(g=512, nx=None):
    """stencil_update seam on a g^3 grid, or an nx x g x g slab (the per-GPU
    share of a g^3 grid over g/nx GPUs, without the halo exchange)."""
    import torch

    from paper_2506_02486_b200 import kernels
    from paper_2506_02486_b200.apps.stencil import _time_params
    _, w = _time_params(4)
    nx = g if nx is None else nx
    shape = (nx + 8, g + 8, g + 8)
    a = torch.rand(shape, dtype=torch.float64, device="cuda")
    b = torch.rand(shape, dtype=torch.float64, device="cuda")
    iters = int(os.environ.get("PROBE_ITERS", "10"))
    ms = _time(lambda: kernels.stencil_update(b, a, b, 3 * w[0], w, w, w, 4), iters=iters,
               warm=max(3, iters // 10))
    pts = nx * g * g
    return {"probe": "stencil_update", "grid": [nx, g, g], "ms": ms, "gpts": pts / ms / 1e6,
            "GBps_24B": 24 * pts / ms / 1e6}


def triad(n_gb=8):
    """STREAM-style reference for the stencil's access pattern: c = a + b
    (2 reads + 1 write = 24 B per f64 element) with torch's own kernel."""
    import torch
    n = int(n_gb * 2**30 // 8)
    a = torch.rand(n, dtype=torch.float64, device="cuda")
    b = torch.rand(n, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    ms = _time(lambda: torch.add(a, b, out=c), iters=10)
    ms_copy = _time(lambda: c.copy_(a), iters=10)
    ms_read = _time(lambda: a.sum(), iters=10)
    return {"probe": "triad", "elements": n, "triad_ms": ms, "triad_GBps": 24 * n / ms / 1e6,
            "copy_GBps": 16 * n / ms_copy / 1e6, "read_GBps": 8 * n / ms_read / 1e6}


if __name__ == "__main__":
    what = sys.argv[1]
    arg = [int(x) for x in sys.argv[2:]]
    print(json.dumps({"dgemm": dgemm, "copy": copy, "stencil": stencil, "triad": triad}[what](*arg)),
          flush=True)
