"""ctypes binding of libdiomp_b200.so (include/diomp_b200.h).

There is no fallback: importing this module on a machine where the library
is missing raises ImportError, and every call's status is checked and raised
through errors.raise_for_status.  The library itself needs a GPU only for the
calls that touch one; loading it and the heap entry points work anywhere.
"""

from __future__ import annotations

import ctypes
import os

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DIOMP_B200_LIB") or os.path.join(HERE, "libdiomp_b200.so")

MAX_TEAM = 64
c_u64, c_i64, c_i32, c_u32, c_vp = (ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32,
                                    ctypes.c_uint32, ctypes.c_void_p)


class Team(ctypes.Structure):
    _fields_ = [("k", c_i32), ("pos", c_i32), ("device", c_i32), ("sync", c_i32),
                ("flag_off", c_u64), ("counter_off", c_u64),
                ("base", c_u64 * MAX_TEAM), ("slot", c_u32 * MAX_TEAM),
                ("epoch_to", c_u64 * MAX_TEAM), ("epoch_from", c_u64 * MAX_TEAM)]


class NvlsArgs(ctypes.Structure):
    _fields_ = [("device", c_i32), ("k", c_i32), ("pos", c_i32), ("dtype", c_i32),
                ("op", c_i32), ("_pad", c_i32), ("uc", c_u64), ("mc", c_u64),
                ("window", c_u64), ("send", c_u64), ("recv", c_u64), ("count", c_u64),
                ("epoch", c_u64), ("counter", c_u64)]


class LLArgs(ctypes.Structure):
    _fields_ = [("k", c_i32), ("pos", c_i32), ("device", c_i32), ("dtype", c_i32),
                ("op", c_i32), ("root", c_i32), ("mode", c_i32), ("_pad", c_i32),
                ("base", c_u64 * MAX_TEAM), ("slot", c_u32 * MAX_TEAM),
                ("epoch_to", c_u32 * MAX_TEAM), ("epoch_from", c_u32 * MAX_TEAM),
                ("ll_off", c_u64), ("slot_bytes", c_u64),
                ("send_off", c_u64), ("recv_off", c_u64), ("count", c_u64)]


class StencilArgs(ctypes.Structure):
    _fields_ = [("u_next", c_u64), ("u_cur", c_u64), ("u_prev", c_u64),
                ("NX", c_i64), ("NY", c_i64), ("NZ", c_i64),
                ("radius", c_i32), ("_pad", c_i32), ("center", ctypes.c_double),
                ("wx", ctypes.c_double * 9), ("wy", ctypes.c_double * 9),
                ("wz", ctypes.c_double * 9)]


class StencilPlan(ctypes.Structure):
    _fields_ = [("device", c_i32), ("radius", c_i32),
                ("NX", c_i64), ("NY", c_i64), ("NZ", c_i64),
                ("field", c_u64 * 2), ("left_field", c_u64 * 2), ("right_field", c_u64 * 2),
                ("src_i", c_i64), ("src_j", c_i64), ("src_k", c_i64),
                ("amp", ctypes.c_double), ("center", ctypes.c_double),
                ("w", ctypes.c_double * 5),
                ("sync", c_i32), ("_pad", c_i32),
                ("wait_left", c_u64), ("wait_right", c_u64),
                ("sig_left", c_u64), ("sig_right", c_u64),
                ("from_left", c_u64), ("from_right", c_u64),
                ("to_left", c_u64), ("to_right", c_u64),
                ("counter", c_u64)]


class DgemmArgs(ctypes.Structure):
    _fields_ = [("device", c_i32), ("sync", c_i32),
                ("M", c_i64), ("N", c_i64), ("K", c_i64),
                ("A", c_u64), ("B", c_u64), ("C", c_u64), ("fwd", c_u64),
                ("lda", c_i64), ("ldb", c_i64), ("ldc", c_i64), ("ldf", c_i64),
                ("wait_addr", c_u64 * 2), ("wait_value", c_u64 * 2),
                ("sig_addr", c_u64 * 2), ("sig_value", c_u64 * 2),
                ("counter", c_u64)]


_PROTOS = {
    "diomp_version": [],
    "diomp_device_count": [ctypes.POINTER(ctypes.c_int)],
    "diomp_device_sync": [ctypes.c_int],
    "diomp_device_error": [ctypes.c_int],
    "diomp_set_wait_timeout": [ctypes.c_int, ctypes.c_double],
    "diomp_seg_create": [ctypes.c_int, c_u64, ctypes.POINTER(c_u64)],
    "diomp_seg_destroy": [ctypes.c_int, c_u64],
    "diomp_seg_ipc_export": [ctypes.c_int, c_u64, ctypes.c_char_p],
    "diomp_seg_ipc_import": [ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(c_u64)],
    "diomp_seg_ipc_close": [ctypes.c_int, c_u64],
    "diomp_peer_enable": [ctypes.c_int, ctypes.c_int],
    "diomp_heap_create": [ctypes.c_int, c_u64, c_u64, c_u64, ctypes.POINTER(c_vp)],
    "diomp_heap_destroy": [c_vp],
    "diomp_heap_alloc": [c_vp, c_u64, ctypes.POINTER(c_u64)],
    "diomp_heap_free": [c_vp, c_u64, ctypes.POINTER(c_u64)],
    "diomp_heap_block_size": [c_vp, c_u64, ctypes.POINTER(c_u64)],
    "diomp_heap_live": [c_vp, ctypes.POINTER(c_u64), ctypes.POINTER(c_u64), ctypes.POINTER(c_u64)],
    "diomp_stream_create": [ctypes.c_int, ctypes.POINTER(c_vp)],
    "diomp_stream_destroy": [c_vp],
    "diomp_stream_sync": [c_vp],
    "diomp_event_create": [ctypes.c_int, ctypes.POINTER(c_vp)],
    "diomp_event_create_sync": [ctypes.c_int, ctypes.POINTER(c_vp)],
    "diomp_event_record": [c_vp, c_vp],
    "diomp_event_query": [c_vp],
    "diomp_event_sync": [c_vp],
    "diomp_event_destroy": [c_vp],
    "diomp_event_elapsed_ms": [c_vp, c_vp, ctypes.POINTER(ctypes.c_float)],
    "diomp_stream_wait_event": [c_vp, c_vp],
    "diomp_stream_query": [c_vp],
    "diomp_rma_ctx_create": [c_i32, c_i32, ctypes.POINTER(c_vp)],
    "diomp_rma_ctx_destroy": [c_vp],
    "diomp_rma_set_local": [c_vp, c_i32, c_i32, c_i32],
    "diomp_rma_set_force_remote": [c_vp, c_i32],
    "diomp_peer_table_set": [c_vp, c_i32, c_i32, c_u64, c_u64, c_i32],
    "diomp_rma_put": [c_vp, c_i32, c_i32, c_u64, c_u64, c_u64, c_i32, c_i32, c_vp,
                      ctypes.POINTER(c_u64)],
    "diomp_rma_get": [c_vp, c_i32, c_i32, c_u64, c_u64, c_u64, c_i32, c_i32, c_vp,
                      ctypes.POINTER(c_u64)],
    "diomp_op_query": [c_vp, c_u64],
    "diomp_op_wait": [c_vp, c_u64, ctypes.c_double],
    "diomp_fence_group": [c_vp, c_u64],
    "diomp_rma_outstanding": [c_vp, c_u64, ctypes.POINTER(c_u64)],
    "diomp_copy": [ctypes.c_int, c_u64, c_u64, c_u64, c_vp],
    "diomp_put": [ctypes.c_int, c_u64, c_u64, c_u64, ctypes.c_int, c_vp],
    "diomp_get": [ctypes.c_int, c_u64, c_u64, c_u64, ctypes.c_int, c_vp],
    "diomp_memcpy_async": [c_u64, c_u64, c_u64, ctypes.c_int, c_vp],
    "diomp_memset_async": [c_u64, ctypes.c_int, c_u64, c_vp],
    "diomp_memcpy_sync": [ctypes.c_int, c_u64, c_u64, c_u64, ctypes.c_int],
    "diomp_signal": [ctypes.c_int, c_u64, c_u64, c_vp],
    "diomp_wait": [ctypes.c_int, c_u64, c_u64, c_vp],
    "diomp_team_barrier": [ctypes.POINTER(Team), c_vp],
    "diomp_bcast": [ctypes.POINTER(Team), c_u64, c_u64, c_i32, c_vp],
    "diomp_reduce": [ctypes.POINTER(Team), c_u64, c_u64, c_u64, c_i32, c_i32, c_i32, c_vp],
    "diomp_allreduce": [ctypes.POINTER(Team), c_u64, c_u64, c_u64, c_i32, c_i32, c_vp],
    "diomp_ll_collective": [ctypes.POINTER(LLArgs), c_vp],
    "diomp_ll_call": [c_vp, ctypes.POINTER(LLArgs), c_vp, c_vp, c_i32],
    "diomp_stencil_update": [ctypes.c_int, ctypes.POINTER(StencilArgs), c_vp],
    "diomp_stencil_run": [ctypes.POINTER(StencilPlan), c_i64, c_i64, c_vp],
    "diomp_matmul_f64": [ctypes.c_int, c_i64, c_i64, c_i64, c_u64, c_u64, c_u64, c_vp],
    "diomp_dgemm": [ctypes.POINTER(DgemmArgs), c_vp],
}

# experiments build only (-DDIOMP_EXPERIMENTS, include/diomp_b200.h): bound
# when the loaded library has them
_EXPERIMENTAL_PROTOS = {
    "diomp_set_bcast_chain_min": [c_u64],
    "diomp_set_bcast_pullchain": [c_i32],
    "diomp_set_allreduce_ce_min": [c_u64],
    "diomp_mc_supported": [ctypes.c_int, ctypes.POINTER(ctypes.c_int)],
    "diomp_mc_window_bytes": [ctypes.c_int, c_u64, ctypes.POINTER(c_u64)],
    "diomp_mc_create": [ctypes.c_int, c_u64, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(c_u64)],
    "diomp_mc_import": [ctypes.c_int, ctypes.POINTER(c_u64)],
    "diomp_mc_add_device": [c_u64, ctypes.c_int],
    "diomp_mc_bind": [c_u64, ctypes.c_int, c_u64, ctypes.POINTER(c_u64), ctypes.POINTER(c_u64),
                      ctypes.POINTER(c_u64)],
    "diomp_mc_release": [c_u64, ctypes.c_int, c_u64, c_u64, c_u64, c_u64],
    "diomp_allreduce_nvls": [ctypes.POINTER(NvlsArgs), c_vp],
    "diomp_nvls_rounds": [c_u64, ctypes.c_int, c_u64, ctypes.POINTER(c_u64)],
}

# symbols declared in include/diomp_b200.h outside DIOMP_EXPERIMENTS (checked
# by tests/test_native_abi.py)
EXPORTS = sorted(list(_PROTOS) + ["diomp_status_string"])


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_2506_02486_b200/build.py` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name, args in _PROTOS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    for name, args in _EXPERIMENTAL_PROTOS.items():
        fn = getattr(lib, name, None)
        if fn is not None:
            fn.argtypes = args
            fn.restype = ctypes.c_int
    lib.diomp_status_string.argtypes = [ctypes.c_int]
    lib.diomp_status_string.restype = ctypes.c_char_p
    return lib


lib = _load()


def has_experiments() -> bool:
    """True when the loaded library is an experiments build."""
    return hasattr(lib, "diomp_allreduce_nvls")


def describe(status: int) -> str:
    return lib.diomp_status_string(status).decode()


def check(status: int, what: str):
    if status != 0:
        errors.raise_for_status(status, what, describe)


def call(name: str, *args):
    rc = getattr(lib, name)(*args)
    check(rc, name)
    return rc


# ---- small typed helpers ----------------------------------------------------

def device_count() -> int:
    n = ctypes.c_int(0)
    rc = lib.diomp_device_count(ctypes.byref(n))
    return n.value if rc == 0 else 0


def seg_create(device: int, nbytes: int) -> int:
    out = c_u64(0)
    call("diomp_seg_create", device, nbytes, ctypes.byref(out))
    return out.value


def seg_ipc_export(device: int, base: int) -> bytes:
    buf = ctypes.create_string_buffer(64)
    call("diomp_seg_ipc_export", device, base, buf)
    return buf.raw


def seg_ipc_import(device: int, handle: bytes) -> int:
    out = c_u64(0)
    call("diomp_seg_ipc_import", device, handle, ctypes.byref(out))
    return out.value


def stream_create(device: int) -> int:
    out = c_vp()
    call("diomp_stream_create", device, ctypes.byref(out))
    return out.value or 0


def event_create(device: int, timing: bool = True) -> int:
    out = c_vp()
    call("diomp_event_create" if timing else "diomp_event_create_sync", device, ctypes.byref(out))
    return out.value


def event_elapsed_ms(start: int, stop: int) -> float:
    ms = ctypes.c_float(0.0)
    call("diomp_event_elapsed_ms", start, stop, ctypes.byref(ms))
    return float(ms.value)


def check_device(device: int, what: str):
    rc = lib.diomp_device_error(device)
    if rc:
        raise errors.TransportFailure(f"{what}: a device-side wait timed out on GPU {device}")
