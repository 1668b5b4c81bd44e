"""TEST INFRASTRUCTURE / CPU BASELINE ONLY -- multi-process CPU restatements of
the reference's distributed drivers, used as the checker in tests/ and timed
by bench.py as `cpu_baseline` / the `--impl reference` arm.  The product
package never imports this module.

The reference (reference/pkg/src/diomp/) runs every rank as a host process
over numpy arenas, a loopback-TCP mesh and a progress thread.  Its pure-Python
package cannot travel to the GPU box (/root/reference is absent there), so the
timed CPU paths are restated here with the same data movement:

  stencil_procs   run_stencil (apps/stencil.py:70-136) on `nranks` processes:
                  x-slabs in shared memory, the one-sided halo exchange of
                  apps/halo_onesided.py:12-25 (4-plane copies into the
                  neighbours' ghost planes, then fence + barrier), the update
                  through the reference's own compiled kernel core
                  (oracle/_ref/_core*.so, kernels/_core.pyx:9-32; the C oracle
                  if it is absent), the point source, the swap.
  WirePair        rma_put / rma_get (transport.py:508-566) between two
                  processes over loopback TCP: 40-byte wire.py header
                  (wire.py:1-30, "<4sBBQIIHQQ"), fragments <= 64 MiB, an ACK
                  per PUT fragment (fence = all ACKs back), GET_REQ/GET_RESP.
  ring_collective allreduce / bcast (collectives.py:232-258, 326-405) on `k`
                  processes in a TCP ring: reduce-scatter folding
                  `incoming op mine` so block b is left-folded from position b
                  (collectives.py:381), then the all-gather; bcast relayed
                  root -> root+1 -> ... in 1 MiB chunks (collectives.py:146-215
                  chunk size).

These are restatements (a little leaner than the reference: no progress
thread, no frame copies), so the CPU numbers they give are, if anything,
optimistic for the reference.
"""

from __future__ import annotations

import hashlib
import importlib.util
import multiprocessing as mp
import os
import socket
import struct
import threading
import time

import numpy as np

from . import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))

# ---------------------------------------------------------------------------
# kernel core: the reference's own compiled stencil_update, else the C oracle
# ---------------------------------------------------------------------------


def load_ref_core():
    d = os.path.join(HERE, "_ref")
    for f in sorted(os.listdir(d)) if os.path.isdir(d) else []:
        if f.startswith("_core") and f.endswith(".so"):
            spec = importlib.util.spec_from_file_location("_core", os.path.join(d, f))
            mod = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(mod)
            return mod
    return None


def stencil_kernel():
    """(callable stencil_update(u_next, u_cur, u_prev, center, wx, wy, wz, r), kind)."""
    core = load_ref_core()
    if core is not None:
        return core.stencil_update, "reference"
    return O.stencil_update_c, "port"


# ---------------------------------------------------------------------------
# run_stencil on nranks processes
# ---------------------------------------------------------------------------

def _stencil_rank(q, nranks, nx, ny, nz, steps, amp, raw, shape, barrier, out):
    r = 4
    nxl = nx // nranks
    allf = np.frombuffer(raw, dtype=np.float64).reshape((nranks, 2) + shape)
    fields = [allf[q, 0], allf[q, 1]]
    fn, _ = stencil_kernel()
    _, w = O.time_params(r)
    center = 3.0 * w[0]
    g0, g1 = O.rank_xmin_xmax(q, nranks, nx)
    cx, cy, cz = nx // 2, ny // 2, nz // 2
    own = g0 <= cx <= g1 and amp
    src = (cx - g0 + r, cy + r, cz + r)
    prev, cur = 0, 1
    barrier.wait()
    t0 = time.perf_counter()
    for _ in range(steps):
        if nranks > 1:   # halo_onesided.exchange: D2D puts, fence, barrier
            if q != 0:
                allf[q - 1, cur][r + nxl:2 * r + nxl] = fields[cur][r:2 * r]
            if q != nranks - 1:
                allf[q + 1, cur][0:r] = fields[cur][nxl:nxl + r]
            barrier.wait()
        fn(fields[prev], fields[cur], fields[prev], center, w, w, w, r)
        if own:
            fields[prev][src] += amp
        prev, cur = cur, prev
    barrier.wait()
    out.put((q, time.perf_counter() - t0, cur))


def stencil_procs(nx: int, ny: int, nz: int, steps: int, nranks: int, amp: float = 1.0,
                  checksum: bool = True) -> dict:
    """Returns {"seconds": timed loop (max over ranks, stencil.py:111-128),
    "gpts": nx*ny*nz*steps/seconds/1e9, "sha256", "kernel": reference|port}.
    The fields live in one fork-inherited shared mapping (every rank's slab
    addressable by its neighbours, as the reference's arenas are through
    the transport)."""
    if nx % nranks:
        raise ValueError("nx must divide by nranks")
    r = 4
    nxl = nx // nranks
    shape = (nxl + 2 * r, ny + 2 * r, nz + 2 * r)
    ctx = mp.get_context("fork")
    raw = ctx.RawArray("d", nranks * 2 * int(np.prod(shape)))   # zero-filled
    barrier = ctx.Barrier(nranks)
    out = ctx.Queue()
    procs = [ctx.Process(target=_stencil_rank,
                         args=(q, nranks, nx, ny, nz, steps, amp, raw, shape, barrier, out))
             for q in range(nranks)]
    for p in procs:
        p.start()
    res = [out.get(timeout=3600) for _ in procs]
    for p in procs:
        p.join()
    secs = max(t for _, t, _ in res)
    cur = res[0][2]
    sha = None
    if checksum:
        allf = np.frombuffer(raw, dtype=np.float64).reshape((nranks, 2) + shape)
        field = np.empty((nx, ny, nz))
        for q in range(nranks):
            field[q * nxl:(q + 1) * nxl] = allf[q, cur][r:r + nxl, r:r + ny, r:r + nz]
        sha = hashlib.sha256(O.dump_bytes(field)).hexdigest()
    return {"seconds": secs, "gpts": nx * ny * nz * steps / secs / 1e9, "sha256": sha,
            "kernel": stencil_kernel()[1], "ranks": nranks}


# ---------------------------------------------------------------------------
# wire transport: one-sided put/get over loopback TCP
# ---------------------------------------------------------------------------

_HDR = struct.Struct("<4sBBQIIHQQ")          # wire.py: 40-byte header
MAGIC, VERSION, MAX_FRAGMENT = b"DOMP", 1, 64 << 20
PUT, GET_REQ, GET_RESP, ACK, BYE = 1, 2, 3, 7, 0
_GETREQ = struct.Struct("<Q")


def _recv_exact(sock, view):
    got = 0
    n = len(view)
    while got < n:
        k = sock.recv_into(view[got:], n - got)
        if k == 0:
            raise ConnectionError("peer closed")
        got += k


def _target(port_q, arena_bytes):
    """The target rank: serves PUT / GET_REQ frames against its arena (the
    reference's progress thread handling of transport.py:591-655)."""
    srv = socket.socket()
    srv.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
    srv.bind(("127.0.0.1", 0))
    srv.listen(1)
    port_q.put(srv.getsockname()[1])
    conn, _ = srv.accept()
    conn.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
    arena = bytearray(arena_bytes)
    av = memoryview(arena)
    hdr = bytearray(_HDR.size)
    hv = memoryview(hdr)
    greq = bytearray(_GETREQ.size)
    while True:
        _recv_exact(conn, hv)
        magic, ver, op, mid, src, dst, dev, off, ln = _HDR.unpack(hdr)
        if op == BYE:
            break
        if op == PUT:
            _recv_exact(conn, av[off:off + ln])
            conn.sendall(_HDR.pack(MAGIC, VERSION, ACK, mid, dst, src, dev, 0, 0))
        elif op == GET_REQ:
            _recv_exact(conn, memoryview(greq))
            (fsize,) = _GETREQ.unpack(greq)
            conn.sendall(_HDR.pack(MAGIC, VERSION, GET_RESP, mid, dst, src, dev, 0, fsize))
            conn.sendall(av[off:off + fsize])
    conn.close()
    srv.close()


class WirePair:
    """Initiator side of a two-process wire link (rank 0 -> rank 1)."""

    def __init__(self, arena_bytes: int):
        ctx = mp.get_context("fork")
        q = ctx.Queue()
        self.proc = ctx.Process(target=_target, args=(q, arena_bytes), daemon=True)
        self.proc.start()
        port = q.get(timeout=60)
        self.sock = socket.create_connection(("127.0.0.1", port))
        self.sock.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
        self.mid = 0
        self.pending = 0
        self._hdr = bytearray(_HDR.size)

    def _frags(self, n):
        pos = 0
        while pos < n:
            f = min(MAX_FRAGMENT, n - pos)
            yield pos, f
            pos += f

    def put(self, offset: int, src) -> None:
        """rma_put: fragments sent, LocalDone; RemoteDone at the ACK (fence)."""
        view = memoryview(src).cast("B")
        for pos, f in self._frags(len(view)):
            self.mid += 1
            self.sock.sendall(_HDR.pack(MAGIC, VERSION, PUT, self.mid, 0, 1, 0, offset + pos, f))
            self.sock.sendall(view[pos:pos + f])
            self.pending += 1

    def fence(self) -> None:
        hv = memoryview(self._hdr)
        while self.pending:
            _recv_exact(self.sock, hv)
            if _HDR.unpack(self._hdr)[2] != ACK:
                raise ConnectionError("unexpected frame")
            self.pending -= 1

    def get(self, offset: int, dst) -> None:
        """rma_get + wait: GET_REQ per fragment, GET_RESP payloads into dst."""
        self.fence()
        view = memoryview(dst).cast("B")
        frags = list(self._frags(len(view)))
        for pos, f in frags:
            self.mid += 1
            self.sock.sendall(_HDR.pack(MAGIC, VERSION, GET_REQ, self.mid, 0, 1, 0,
                                        offset + pos, _GETREQ.size) + _GETREQ.pack(f))
        hv = memoryview(self._hdr)
        for pos, f in frags:
            _recv_exact(self.sock, hv)
            _recv_exact(self.sock, view[pos:pos + f])

    def close(self):
        try:
            self.sock.sendall(_HDR.pack(MAGIC, VERSION, BYE, 0, 0, 1, 0, 0, 0))
            self.sock.close()
        finally:
            self.proc.join(timeout=30)


def p2p_sample(bw_bytes: int = 64 << 20, bw_iters: int = 8, lat_iters: int = 200) -> dict:
    """The reference's p2p harness legs (apps/bench.py:78-121): put = put+fence,
    get = get+wait, bw = iters puts + one fence; MiB-free units (GB/s, us)."""
    link = WirePair(bw_bytes + 4096)
    try:
        small = np.arange(8, dtype=np.uint8)
        sink = bytearray(8)
        for _ in range(20):
            link.put(0, small)
            link.fence()
            link.get(0, sink)
        t0 = time.perf_counter()
        for _ in range(lat_iters):
            link.put(0, small)
            link.fence()
        put_lat = (time.perf_counter() - t0) / lat_iters
        t0 = time.perf_counter()
        for _ in range(lat_iters):
            link.get(0, sink)
        get_lat = (time.perf_counter() - t0) / lat_iters
        payload = np.random.default_rng(bw_bytes).integers(0, 256, bw_bytes, dtype=np.uint8)
        back = bytearray(bw_bytes)
        link.put(0, payload)
        link.fence()
        t0 = time.perf_counter()
        for _ in range(bw_iters):
            link.put(0, payload)
        link.fence()
        put_bw = bw_bytes * bw_iters / (time.perf_counter() - t0) / 1e9
        t0 = time.perf_counter()
        for _ in range(bw_iters):
            link.get(0, back)
        get_bw = bw_bytes * bw_iters / (time.perf_counter() - t0) / 1e9
        exact = bytes(back) == payload.tobytes()
    finally:
        link.close()
    return {"put_latency_us_8B": put_lat * 1e6, "get_latency_us_8B": get_lat * 1e6,
            "put_bandwidth_gbs": put_bw, "get_bandwidth_gbs": get_bw, "bytes": bw_bytes,
            "byte_exact": exact}


# ---------------------------------------------------------------------------
# ring collectives over TCP
# ---------------------------------------------------------------------------

_CHUNK = 1 << 20


def _ring_sockets(p, k, ports, ready):
    """Listen for the predecessor, connect to the successor."""
    srv = socket.socket()
    srv.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
    srv.bind(("127.0.0.1", 0))
    srv.listen(1)
    ports[p] = srv.getsockname()[1]
    ready.wait()
    nxt = socket.create_connection(("127.0.0.1", ports[(p + 1) % k]))
    prv, _ = srv.accept()
    srv.close()
    for s in (nxt, prv):
        s.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
    return nxt, prv


def _exchange(nxt, prv, out_bytes, in_view):
    t = threading.Thread(target=nxt.sendall, args=(out_bytes,))
    t.start()
    _recv_exact(prv, in_view)
    t.join()


def _allreduce_once(p, k, nxt, prv, vec, ufunc):
    count = len(vec)
    bounds = [(b * count // k, (b + 1) * count // k) for b in range(k)]
    acc = vec.copy()
    # reduce-scatter: at step s position p forwards its partial of block
    # (p - s) and folds block (p - s - 1): incoming op mine
    for s in range(k - 1):
        sb = (p - s) % k
        rb = (p - s - 1) % k
        lo, hi = bounds[rb]
        inc = np.empty(hi - lo, dtype=vec.dtype)
        slo, shi = bounds[sb]
        _exchange(nxt, prv, acc[slo:shi].tobytes(), memoryview(inc).cast("B"))
        acc[lo:hi] = ufunc(inc, acc[lo:hi])
    # all-gather: position p owns the full fold of block (p + 1)
    for s in range(k - 1):
        sb = (p + 1 - s) % k
        rb = (p - s) % k
        lo, hi = bounds[rb]
        slo, shi = bounds[sb]
        _exchange(nxt, prv, acc[slo:shi].tobytes(), memoryview(acc[lo:hi]).cast("B"))
    return acc


def _bcast_once(p, k, root, nxt, prv, buf):
    h = (p - root) % k
    view = memoryview(buf).cast("B")
    n = len(view)
    for pos in range(0, n, _CHUNK):
        seg = view[pos:min(n, pos + _CHUNK)]
        if h > 0:
            _recv_exact(prv, seg)
        if h < k - 1:
            nxt.sendall(seg)


def _coll_rank(p, k, op, count, iters, ports, ready, out, check):
    nxt, prv = _ring_sockets(p, k, ports, ready)
    try:
        if op == "allreduce":
            vec = np.random.default_rng(1000 + p).uniform(-1, 1, count).astype(np.float32)
            res = _allreduce_once(p, k, nxt, prv, vec, np.add)   # warm / checked result
            t0 = time.perf_counter()
            for _ in range(iters):
                _allreduce_once(p, k, nxt, prv, vec, np.add)
            dt = time.perf_counter() - t0
            out.put((p, dt, res.tobytes() if (p == 0 and check) else None))
        else:
            buf = np.random.default_rng(77).integers(0, 256, count, dtype=np.uint8) if p == 0 \
                else np.zeros(count, dtype=np.uint8)
            _bcast_once(p, k, 0, nxt, prv, buf)
            t0 = time.perf_counter()
            for _ in range(iters):
                _bcast_once(p, k, 0, nxt, prv, buf)
            dt = time.perf_counter() - t0
            out.put((p, dt, hashlib.sha256(buf.tobytes()).hexdigest()))
    finally:
        nxt.close()
        prv.close()


def ring_collective(op: str, k: int, nbytes: int, iters: int = 3, check: bool = True) -> dict:
    """Time `iters` allreduce (f32 sum, count = nbytes/4) or bcast (nbytes) on
    k processes.  Returns mean seconds (max over ranks), busBW and a result
    check (allreduce bytes of position 0 / bcast digests of every member)."""
    if op not in ("allreduce", "bcast"):
        raise ValueError(op)
    ctx = mp.get_context("fork")
    mgr_ports = ctx.Array("i", k)
    ready = ctx.Event()
    out = ctx.Queue()
    count = nbytes // 4 if op == "allreduce" else nbytes
    procs = [ctx.Process(target=_coll_rank, args=(p, k, op, count, iters, mgr_ports, ready, out, check))
             for p in range(k)]
    for pr in procs:
        pr.start()
    deadline = time.time() + 60
    while any(mgr_ports[i] == 0 for i in range(k)):
        if time.time() > deadline:
            raise TimeoutError("ring sockets")
        time.sleep(0.01)
    ready.set()
    res = [out.get(timeout=3600) for _ in procs]
    for pr in procs:
        pr.join()
    t = max(r[1] for r in res) / iters
    factor = 2 * (k - 1) / k if op == "allreduce" else 1.0
    d = {"seconds": t, "busbw_gbs": factor * nbytes / t / 1e9, "k": k, "bytes": nbytes}
    if op == "allreduce":
        d["result"] = next(r[2] for r in res if r[0] == 0)
    else:
        d["digests"] = [r[2] for r in sorted(res)]
    return d
