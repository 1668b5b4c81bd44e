"""DIOMP_KERNELS=b200 backend for the reference package's kernel seam.

This is the file a maintainer drops into the reference as
`pkg/src/diomp/kernels/_b200.py` and selects from `kernels/__init__.py:15-31`
(INTEGRATION.md section 2).  It keeps the seam's contract exactly --
`stencil_update(u_next, u_cur, u_prev, center, wx, wy, wz, radius)` in place
(u_next may alias u_prev) and `matmul_f64(a, b, c)`, numpy float64 in and out
(kernels/__init__.py:30-31, _core.pyx:9-46) -- and reaches the B200 kernels
through the C ABI only (include/diomp_b200.h): device buffers come from
`diomp_seg_create`, copies from `diomp_memcpy_sync`, no torch and no package
import.  Results are bit-identical to the reference's `_core` / `reference.py`
(tests/test_gpu_integration.py against tests/golden/kernels_golden.npz).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_LIB_PATH = os.environ.get("DIOMP_B200_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "..", "paper_2506_02486_b200",
    "libdiomp_b200.so")
_lib = ctypes.CDLL(_LIB_PATH)
_DEVICE = int(os.environ.get("DIOMP_B200_DEVICE", "0"))

u64, i64, i32 = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32
H2D, D2H = 1, 2


class _StencilArgs(ctypes.Structure):   # diomp_stencil_args
    _fields_ = [("u_next", u64), ("u_cur", u64), ("u_prev", u64),
                ("NX", i64), ("NY", i64), ("NZ", i64),
                ("radius", i32), ("_pad", i32), ("center", ctypes.c_double),
                ("wx", ctypes.c_double * 9), ("wy", ctypes.c_double * 9),
                ("wz", ctypes.c_double * 9)]


_lib.diomp_seg_create.argtypes = [ctypes.c_int, u64, ctypes.POINTER(u64)]
_lib.diomp_seg_destroy.argtypes = [ctypes.c_int, u64]
_lib.diomp_memcpy_sync.argtypes = [ctypes.c_int, u64, u64, u64, ctypes.c_int]
_lib.diomp_stencil_update.argtypes = [ctypes.c_int, ctypes.POINTER(_StencilArgs), ctypes.c_void_p]
_lib.diomp_matmul_f64.argtypes = [ctypes.c_int, i64, i64, i64, u64, u64, u64, ctypes.c_void_p]
_lib.diomp_device_sync.argtypes = [ctypes.c_int]
_lib.diomp_status_string.argtypes = [ctypes.c_int]
_lib.diomp_status_string.restype = ctypes.c_char_p


def _check(rc: int, what: str):
    if rc:
        raise RuntimeError(f"{what}: {_lib.diomp_status_string(rc).decode()} (status {rc})")


class _DeviceBuffers:
    """Device scratch reused across calls (grown on demand, freed at exit)."""

    def __init__(self):
        self.bufs: dict[str, tuple[int, int]] = {}

    def get(self, name: str, nbytes: int) -> int:
        ptr, size = self.bufs.get(name, (0, 0))
        if size < nbytes:
            if ptr:
                _check(_lib.diomp_seg_destroy(_DEVICE, ptr), "seg_destroy")
            out = u64(0)
            _check(_lib.diomp_seg_create(_DEVICE, max(nbytes, 256), ctypes.byref(out)),
                   "seg_create")
            ptr, size = out.value, max(nbytes, 256)
            self.bufs[name] = (ptr, size)
        return ptr

    def close(self):
        for ptr, _ in self.bufs.values():
            _lib.diomp_seg_destroy(_DEVICE, ptr)
        self.bufs.clear()


_bufs = _DeviceBuffers()


def _h2d(name: str, arr: np.ndarray) -> int:
    arr = np.ascontiguousarray(arr, dtype=np.float64)
    dev = _bufs.get(name, arr.nbytes)
    if arr.nbytes:
        _check(_lib.diomp_memcpy_sync(_DEVICE, dev, arr.ctypes.data, arr.nbytes, H2D), "H2D")
    return dev


def _d2h(dev: int, out: np.ndarray):
    host = np.empty(out.shape, dtype=np.float64)
    if host.nbytes:
        _check(_lib.diomp_memcpy_sync(_DEVICE, host.ctypes.data, dev, host.nbytes, D2H), "D2H")
    out[...] = host


def stencil_update(u_next, u_cur, u_prev, center, wx, wy, wz, radius):
    """kernels/__init__.py:30 seam: one interior update, in place in u_next."""
    if u_cur.ndim != 3 or u_cur.dtype != np.float64:
        raise TypeError("stencil_update expects 3-D float64 arrays")
    cur = _h2d("cur", u_cur)
    prev = _h2d("prev", u_prev)
    nxt = prev
    if u_next is not u_prev:   # distinct output: start from its current bytes
        nxt = _h2d("next", u_next)
    w = [(ctypes.c_double * 9)(*[float(x) for x in v][:radius + 1]) for v in (wx, wy, wz)]
    a = _StencilArgs(nxt, cur, prev, *u_cur.shape, int(radius), 0, float(center), *w)
    _check(_lib.diomp_stencil_update(_DEVICE, ctypes.byref(a), None), "stencil_update")
    _check(_lib.diomp_device_sync(_DEVICE), "sync")
    _d2h(nxt, u_next)


def matmul_f64(a, b, c):
    """kernels/__init__.py:31 seam: c = a @ b, k-ordered fold, no FMA."""
    n, k = a.shape
    k2, m = b.shape
    if k2 != k or c.shape != (n, m):
        raise ValueError("shape mismatch")
    da, db = _h2d("a", a), _h2d("b", b)
    dc = _bufs.get("c", n * m * 8)
    _check(_lib.diomp_matmul_f64(_DEVICE, n, k, m, da, db, dc, None), "matmul_f64")
    _check(_lib.diomp_device_sync(_DEVICE), "sync")
    _d2h(dc, c)
