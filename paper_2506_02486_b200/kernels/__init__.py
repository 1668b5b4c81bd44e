"""Kernel seam (reference/pkg/src/diomp/kernels/__init__.py:15-31).

`stencil_update` and `matmul_f64` keep the reference signatures and its
bitwise results, but operate on float64 CUDA tensors and run the sm_100a
kernels of libdiomp_b200 on the caller's current torch stream.  There is one
backend and no CPU fallback: host arrays are rejected.
"""

from __future__ import annotations

import ctypes

from .. import _native

BACKEND = "cuda"


def _check(t, name: str, ndim: int):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != torch.float64 or t.dim() != ndim or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous {ndim}-D float64 tensor")


def _weights(w, radius: int):
    vals = [float(x) for x in (w.tolist() if hasattr(w, "tolist") else w)]
    if len(vals) < radius + 1:
        raise ValueError(f"need {radius + 1} weights, got {len(vals)}")
    return (ctypes.c_double * 9)(*(vals[:radius + 1] + [0.0] * (9 - radius - 1)))


def stencil_update(u_next, u_cur, u_prev, center: float, wx, wy, wz, radius: int):
    """u_next = 2*u_cur - u_prev + lap(u_cur) on the interior (ghost width
    `radius`), reference order, no FMA; u_next may alias u_prev."""
    import torch
    for n, t in (("u_next", u_next), ("u_cur", u_cur), ("u_prev", u_prev)):
        _check(t, n, 3)
    if not (u_next.shape == u_cur.shape == u_prev.shape):
        raise ValueError("u_next, u_cur and u_prev must share one shape")
    if not (u_next.device == u_cur.device == u_prev.device):
        raise ValueError("all fields must live on one GPU")
    if not 0 <= radius <= 8:
        raise ValueError("radius must be in [0, 8]")
    a = _native.StencilArgs()
    a.u_next, a.u_cur, a.u_prev = u_next.data_ptr(), u_cur.data_ptr(), u_prev.data_ptr()
    a.NX, a.NY, a.NZ = u_cur.shape
    a.radius = radius
    a.center = float(center)
    a.wx, a.wy, a.wz = _weights(wx, radius), _weights(wy, radius), _weights(wz, radius)
    dev = u_cur.device.index
    stream = torch.cuda.current_stream(dev).cuda_stream
    _native.check(_native.lib.diomp_stencil_update(dev, ctypes.byref(a), stream), "stencil_update")


def matmul_f64(a, b, c):
    """c = a @ b with a k-ordered left fold per element (bit-exact oracle order)."""
    import torch
    for n, t in (("a", a), ("b", b), ("c", c)):
        _check(t, n, 2)
    n_, k_ = a.shape
    k2, m_ = b.shape
    if k2 != k_ or tuple(c.shape) != (n_, m_):
        raise ValueError(f"shape mismatch {tuple(a.shape)} @ {tuple(b.shape)} -> {tuple(c.shape)}")
    dev = a.device.index
    stream = torch.cuda.current_stream(dev).cuda_stream
    _native.check(_native.lib.diomp_matmul_f64(dev, n_, k_, m_, a.data_ptr(), b.data_ptr(),
                                               c.data_ptr(), stream), "matmul_f64")


def backends() -> dict[str, object]:
    import sys
    return {"cuda": sys.modules[__name__]}
