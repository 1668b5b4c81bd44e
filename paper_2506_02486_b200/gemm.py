"""Host wrapper of the FP64 tensor-core GEMM (csrc/gemm.cuh, DMMA m8n8k4).

dgemm_accumulate(A, B, C) computes C += A @ B on float64 CUDA tensors (row
major, any leading dimension with unit column stride); the kernel of the
Cannon block product (apps/cannon.py:138).  Accumulation uses FMA on the
tensor cores, so results match host BLAS within rounding (rel-L2 ~1e-16),
not bit-for-bit -- exactly the reference's own contract for this product.
"""

from __future__ import annotations

import ctypes

from . import _native


def _ld(t) -> int:
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError("matrices must be row-major with unit column stride")
    return t.stride(0)


def dgemm_accumulate(A, B, C, *, fwd=None, stream=None, sync=None) -> None:
    """C += A @ B.  fwd: optional tensor (e.g. a peer-mapped stripe view) that
    receives a copy of B from inside the kernel.  sync: optional dict with
    wait_addr/wait_value/sig_addr/sig_value/counter for ring-step flags."""
    import torch
    for name, t in (("A", A), ("B", B), ("C", C)):
        if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64:
            raise TypeError(f"{name} must be a float64 CUDA tensor (no CPU fallback)")
    M, K = A.shape
    K2, N = B.shape
    if K2 != K or tuple(C.shape) != (M, N):
        raise ValueError(f"shape mismatch {tuple(A.shape)} @ {tuple(B.shape)} -> {tuple(C.shape)}")
    x = _native.DgemmArgs()
    x.device = A.device.index
    x.M, x.N, x.K = M, N, K
    x.A, x.B, x.C = A.data_ptr(), B.data_ptr(), C.data_ptr()
    x.lda, x.ldb, x.ldc = _ld(A), _ld(B), _ld(C)
    if fwd is not None:
        x.fwd, x.ldf = (fwd.data_ptr(), _ld(fwd)) if hasattr(fwd, "data_ptr") else fwd
    if sync:
        x.sync = 1
        for i, (a, v) in enumerate(zip(sync.get("wait_addr", []), sync.get("wait_value", []))):
            x.wait_addr[i], x.wait_value[i] = a, v
        for i, (a, v) in enumerate(zip(sync.get("sig_addr", []), sync.get("sig_value", []))):
            x.sig_addr[i], x.sig_value[i] = a, v
        x.counter = sync["counter"]
    s = stream if stream is not None else torch.cuda.current_stream(x.device).cuda_stream
    _native.check(_native.lib.diomp_dgemm(ctypes.byref(x), s), "dgemm")


def dgemm_raw(device: int, M: int, N: int, K: int, A: int, lda: int, B: int, ldb: int, C: int,
              ldc: int, stream: int, fwd: int = 0, ldf: int = 0, sync: dict | None = None):
    """Pointer-level form used by the ring driver."""
    x = _native.DgemmArgs()
    x.device, x.M, x.N, x.K = device, M, N, K
    x.A, x.B, x.C, x.lda, x.ldb, x.ldc = A, B, C, lda, ldb, ldc
    x.fwd, x.ldf = fwd, ldf
    if sync:
        x.sync = 1
        for i, (a, v) in enumerate(zip(sync.get("wait_addr", []), sync.get("wait_value", []))):
            x.wait_addr[i], x.wait_value[i] = a, v
        for i, (a, v) in enumerate(zip(sync.get("sig_addr", []), sync.get("sig_value", []))):
            x.sig_addr[i], x.sig_value[i] = a, v
        x.counter = sync["counter"]
    _native.check(_native.lib.diomp_dgemm(ctypes.byref(x), stream), "dgemm")
