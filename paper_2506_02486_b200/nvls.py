"""NVSwitch multicast (NVLS) window for the in-switch allreduce.

`collectives.allreduce(..., algorithm="nvls")` (or DIOMP_ALLREDUCE_ALGO=nvls)
runs collectives.py:326-405 with the reduction done by the NVSwitch
(multimem.ld_reduce) instead of the reference's ring fold; see
csrc/nvls.cuh for the kernels and the round protocol.  Float sums match the
exact path within rounding only; integer sum/min/max are bit-identical.

Setup is collective over the communicator (every member is inside the same
allreduce call): position 0 creates the multicast object and exports it as a
POSIX file descriptor, which reaches the other processes over an abstract Unix
socket (SCM_RIGHTS); every member imports it and adds its GPU; after a
barrier each binds a window of its own HBM.  Windows are released at
Runtime.finalize.
"""

from __future__ import annotations

import os
import socket
import threading

from . import _native
from .errors import UsageError

DEFAULT_WINDOW = 256 << 20


def supported(gpu: int) -> bool:
    if not _native.has_experiments():   # NVLS lives in the experiments build only
        return False
    v = _native.ctypes.c_int(0)
    _native.call("diomp_mc_supported", gpu, _native.ctypes.byref(v))
    return bool(v.value)


class NvlsWindow:
    """One communicator's multicast window on this process's position."""

    def __init__(self, comm, window: int | None = None):
        rt = comm.rt
        if len(comm.my_positions) != 1:
            raise UsageError("nvls allreduce needs exactly one communicator position per rank")
        if not comm.device_sync:
            raise UsageError("nvls allreduce needs every member on its own GPU")
        self.comm = comm
        self.pos = comm.my_positions[0]
        ep = comm.ring[self.pos]
        self.gpu = rt.gpus[ep.device]
        k = comm.size
        ranks = tuple(e.rank for e in comm.ring)
        tag = f"nvls/{comm.uid.value.hex()}"
        ok = rt.ctrl.allgather(ranks, f"{tag}/ok", bytes([supported(self.gpu)]))
        if not all(b == b"\x01" for _, b in ok):
            raise UsageError("NVSwitch multicast is not available on every member GPU")
        want = int(window or os.environ.get("DIOMP_NVLS_WINDOW", DEFAULT_WINDOW))
        total = _native.ctypes.c_uint64(0)
        _native.call("diomp_mc_window_bytes", k, want, _native.ctypes.byref(total))
        self.total = total.value
        self.window = self.total - (2 << 20)
        mc = _native.ctypes.c_uint64(0)
        root_rank = comm.ring[0].rank
        name = b"\0diomp-nvls-" + comm.uid.value.hex().encode()
        if self.pos == 0:
            fd = _native.ctypes.c_int(-1)
            _native.call("diomp_mc_create", k, self.total, _native.ctypes.byref(fd),
                         _native.ctypes.byref(mc))
            server = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            server.bind(name)
            server.listen(k)
            peers = [e.rank for e in comm.ring[1:]]

            def serve():
                for _ in peers:
                    conn, _addr = server.accept()
                    with conn:
                        socket.send_fds(conn, [b"m"], [fd.value])
            th = threading.Thread(target=serve, daemon=True)
            th.start()
            for r in peers:
                rt.ctrl.send(r, f"{tag}/listen", b"")
            th.join(rt.cfg.timeout)
            server.close()
            os.close(fd.value)
            if th.is_alive():
                raise UsageError("nvls window: a member never fetched the multicast handle")
        else:
            rt.ctrl.recv(f"{tag}/listen", root_rank)
            with socket.socket(socket.AF_UNIX, socket.SOCK_STREAM) as c:
                c.connect(name)
                _msg, fds, _flags, _addr = socket.recv_fds(c, 16, 1)
            _native.call("diomp_mc_import", fds[0], _native.ctypes.byref(mc))
            os.close(fds[0])
        self.mc_handle = mc.value
        _native.call("diomp_mc_add_device", self.mc_handle, self.gpu)
        rt.ctrl.barrier(ranks, f"{tag}/added")
        uc, mva, phys = (_native.ctypes.c_uint64(0) for _ in range(3))
        _native.call("diomp_mc_bind", self.mc_handle, self.gpu, self.total,
                     _native.ctypes.byref(uc), _native.ctypes.byref(mva),
                     _native.ctypes.byref(phys))
        self.uc, self.mc, self.phys = uc.value, mva.value, phys.value
        rt.ctrl.barrier(ranks, f"{tag}/bound")
        self.epoch = 0
        self.args = _native.NvlsArgs()
        self.args.device, self.args.k, self.args.pos = self.gpu, k, self.pos
        self.args.uc, self.args.mc, self.args.window = self.uc, self.mc, self.window
        rt._cleanup.append(self.release)
        self._released = False

    def rounds(self, count: int, dtype: int) -> int:
        n = _native.ctypes.c_uint64(0)
        _native.call("diomp_nvls_rounds", count, dtype, self.window, _native.ctypes.byref(n))
        return n.value

    def launch(self, send_ptr: int, recv_ptr: int, count: int, dtype: int, op: int,
               counter: int, stream) -> None:
        a = self.args
        a.send, a.recv, a.count, a.dtype, a.op = send_ptr, recv_ptr, count, dtype, op
        a.epoch, a.counter = self.epoch, counter
        _native.check(_native.lib.diomp_allreduce_nvls(a, stream), "allreduce_nvls")
        self.epoch += self.rounds(count, dtype)

    def release(self):
        if self._released:
            return
        self._released = True
        _native.lib.diomp_mc_release(self.mc_handle, self.gpu, self.total, self.uc, self.mc,
                                     self.phys)
