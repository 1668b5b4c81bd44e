"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the DiOMP-Offloading hot path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module, and only as the checker or the timed CPU
baseline.  The product package (paper_2506_02486_b200) never imports it.

Each function restates the reference algorithm and cites the reference
file:line it follows (paths relative to reference/pkg/src/diomp/).  The
restatements are pinned against fixtures produced by importing the reference
itself (tests/golden/make_golden.py -> tests/golden/*.json / *.npz).
"""

from __future__ import annotations

import ctypes
import hashlib
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

# apps/stencil.py:28-30
VELOCITY = 1500.0
COEF = (-205.0 / 72.0, 8.0 / 5.0, -1.0 / 5.0, 8.0 / 315.0, -1.0 / 560.0)


def _lib():
    """Load (building on first use if needed) oracle/liboracle.so."""
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            subprocess.check_call(["make", "-s", "liboracle.so"], cwd=HERE)
        lib = ctypes.CDLL(path)
        dp = ctypes.POINTER(ctypes.c_double)
        lib.oracle_stencil_update.argtypes = [dp, dp, dp, ctypes.c_long, ctypes.c_long,
                                              ctypes.c_long, ctypes.c_double, dp, dp, dp,
                                              ctypes.c_int]
        lib.oracle_stencil_run.argtypes = [ctypes.c_long] * 4 + [ctypes.c_int, dp,
                                                                 ctypes.c_double, dp]
        lib.oracle_stencil_run.restype = ctypes.c_int
        lib.oracle_matmul_f64.argtypes = [dp, dp, dp, ctypes.c_long, ctypes.c_long,
                                          ctypes.c_long]
        _LIB = lib
    return _LIB


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


# ---------------------------------------------------------------------------
# stencil
# ---------------------------------------------------------------------------

def time_params(radius: int = 4) -> tuple[float, np.ndarray]:
    """dt at half the CFL limit and the scaled weights (apps/stencil.py:61-67)."""
    per_axis = abs(COEF[0]) + 2 * sum(abs(c) for c in COEF[1:radius + 1])
    dt = 0.5 * 2.0 / (VELOCITY * math.sqrt(3.0 * per_axis))
    scale = (VELOCITY * dt) ** 2
    return dt, np.array(COEF[:radius + 1]) * scale


def rank_xmin_xmax(r: int, nranks: int, nx: int) -> tuple[int, int]:
    """Contiguous block decomposition (apps/stencil.py:54-58)."""
    return (r * nx) // nranks, ((r + 1) * nx) // nranks - 1


def stencil_update_c(u_next, u_cur, u_prev, center, wx, wy, wz, radius):
    """One interior update through the C restatement (kernels/_core.pyx:9-32)."""
    nx, ny, nz = u_cur.shape
    wx, wy, wz = (np.ascontiguousarray(w, dtype=np.float64) for w in (wx, wy, wz))
    _lib().oracle_stencil_update(_dp(u_next), _dp(u_cur), _dp(u_prev), nx, ny, nz,
                                 float(center), _dp(wx), _dp(wy), _dp(wz), int(radius))


def stencil_update_np(u_next, u_cur, u_prev, center, wx, wy, wz, radius):
    """Pure-numpy restatement, axis-by-axis in the same IEEE order
    (kernels/reference.py:14-31): acc = center*u, then += w[t]*(u[+t]+u[-t])
    for x, y, z taps in ascending t, then (2u - u_prev) + acc."""
    r = radius
    X, Y, Z = u_cur.shape
    u = u_cur[r:X - r, r:Y - r, r:Z - r]
    acc = center * u
    for t in range(1, r + 1):
        acc = acc + wx[t] * (u_cur[r + t:X - r + t, r:Y - r, r:Z - r]
                             + u_cur[r - t:X - r - t, r:Y - r, r:Z - r])
    for t in range(1, r + 1):
        acc = acc + wy[t] * (u_cur[r:X - r, r + t:Y - r + t, r:Z - r]
                             + u_cur[r:X - r, r - t:Y - r - t, r:Z - r])
    for t in range(1, r + 1):
        acc = acc + wz[t] * (u_cur[r:X - r, r:Y - r, r + t:Z - r + t]
                             + u_cur[r:X - r, r:Y - r, r - t:Z - r - t])
    u_next[r:X - r, r:Y - r, r:Z - r] = (2.0 * u - u_prev[r:X - r, r:Y - r, r:Z - r]) + acc


def stencil_run(nx: int, ny: int, nz: int, steps: int, amp: float = 1.0,
                radius: int = 4) -> np.ndarray:
    """Whole driver on one slab (apps/stencil.py:70-136); returns the interior."""
    _, w = time_params(radius)
    out = np.empty((nx, ny, nz), dtype=np.float64)
    rc = _lib().oracle_stencil_run(nx, ny, nz, steps, radius, _dp(np.ascontiguousarray(w)),
                                   float(amp), _dp(out))
    if rc != 0:
        raise MemoryError("oracle_stencil_run could not allocate")
    return out


def stencil_run_slabs(nx: int, ny: int, nz: int, steps: int, nranks: int,
                      amp: float = 1.0, radius: int = 4) -> np.ndarray:
    """Multi-slab restatement: x-slabs per rank, Listing-1 halo copies each step
    (apps/halo_onesided.py:12-25) then the update (stencil.py:113-126)."""
    r = radius
    nxl = nx // nranks
    _, w = time_params(r)
    center = 3.0 * w[0]
    shape = (nxl + 2 * r, ny + 2 * r, nz + 2 * r)
    prev = [np.zeros(shape) for _ in range(nranks)]
    cur = [np.zeros(shape) for _ in range(nranks)]
    cx, cy, cz = nx // 2, ny // 2, nz // 2
    for _ in range(steps):
        for q in range(nranks):
            if q != 0:
                cur[q - 1][r + nxl:2 * r + nxl] = cur[q][r:2 * r]
            if q != nranks - 1:
                cur[q + 1][0:r] = cur[q][nxl:nxl + r]
        for q in range(nranks):
            stencil_update_c(prev[q], cur[q], prev[q], center, w, w, w, r)
            g0, g1 = rank_xmin_xmax(q, nranks, nx)
            if amp and g0 <= cx <= g1:
                prev[q][cx - g0 + r, cy + r, cz + r] += amp
        prev, cur = cur, prev
    field = np.empty((nx, ny, nz))
    for q in range(nranks):
        field[q * nxl:(q + 1) * nxl] = cur[q][r:r + nxl, r:r + ny, r:r + nz]
    return field


def dump_bytes(field: np.ndarray) -> bytes:
    """f64 little-endian, x fastest (apps/stencil.py:159-161)."""
    return field.transpose(2, 1, 0).astype("<f8", copy=False).tobytes()


def checksum(field: np.ndarray) -> str:
    return hashlib.sha256(dump_bytes(field)).hexdigest()


# ---------------------------------------------------------------------------
# matmul
# ---------------------------------------------------------------------------

def matmul_f64(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """k-ordered left fold per element, no FMA (kernels/_core.pyx:35-46)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    c = np.empty((a.shape[0], b.shape[1]))
    _lib().oracle_matmul_f64(_dp(a), _dp(b), _dp(c), a.shape[0], a.shape[1], b.shape[1])
    return c


def fill_matrices(n: int, seed: int, identity_b: bool = False):
    """A then B from one generator (apps/cannon.py:73-77)."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1.0, 1.0, (n, n))
    b = np.eye(n) if identity_b else rng.uniform(-1.0, 1.0, (n, n))
    return a, b


# ---------------------------------------------------------------------------
# collectives
# ---------------------------------------------------------------------------

def np_op(kind: str):
    """numpy ufuncs of collectives.py:76-79 (Sum/Min/Max)."""
    return {"sum": np.add, "min": np.minimum, "max": np.maximum}[kind]


def reduce_fold(contribs, kind: str, root: int = 0) -> np.ndarray:
    """Root result of reduce: left fold in ring order starting at the root
    (collectives.py:19-21, 270-323; test_collectives.py:26-31)."""
    k = len(contribs)
    f = np_op(kind)
    acc = contribs[root].copy()
    for t in range(1, k):
        acc = f(acc, contribs[(root + t) % k])
    return acc


def allreduce_fold(contribs, kind: str) -> np.ndarray:
    """Ring reduce-scatter block folds (collectives.py:22-24, 349-350, 361-382;
    test_collectives.py:34-45): block b = [b*count//k, (b+1)*count//k) is
    left-folded starting at ring position b."""
    k = len(contribs)
    f = np_op(kind)
    count = len(contribs[0])
    out = np.empty_like(contribs[0])
    for b in range(k):
        lo, hi = b * count // k, (b + 1) * count // k
        acc = contribs[b][lo:hi].copy()
        for t in range(1, k):
            acc = f(acc, contribs[(b + t) % k][lo:hi])
        out[lo:hi] = acc
    return out


def bcast_payload(root_bytes: bytes, k: int) -> list[bytes]:
    """bcast: every member ends equal to the root's entry snapshot (collectives.py:232-258)."""
    return [root_bytes] * k


# ---------------------------------------------------------------------------
# allocators (host state machines; offsets must match exactly)
# ---------------------------------------------------------------------------

MIN_BUDDY_BLOCK = 256


def _ceil_log2(n: int) -> int:
    return (n - 1).bit_length() if n > 1 else 0


def _align_up(v: int, a: int) -> int:
    return (v + a - 1) & ~(a - 1)


class OracleLinear:
    """Bump + exact-size LIFO reuse (allocators.py:36-72)."""

    def __init__(self, capacity: int, alignment: int = 64):
        self.capacity, self.alignment = capacity, alignment
        self.top, self.free_lists, self.live = 0, {}, {}

    def block_size(self, size):
        return _align_up(max(size, 1), self.alignment)

    def alloc(self, size):
        rounded = self.block_size(size)
        lst = self.free_lists.get(rounded)
        if lst:
            off = lst.pop()
        else:
            if self.top + rounded > self.capacity:
                raise MemoryError("oom")
            off, self.top = self.top, self.top + rounded
        self.live[off] = rounded
        return off

    def free(self, off):
        rounded = self.live.pop(off)
        self.free_lists.setdefault(rounded, []).append(off)
        return rounded


class OracleBuddy:
    """Power-of-two buddy, lowest-address choice, reserved tail (allocators.py:75-150)."""

    def __init__(self, capacity: int, reserve_from: int | None = None):
        self.capacity = capacity
        self.min_order = _ceil_log2(MIN_BUDDY_BLOCK)
        self.max_order = _ceil_log2(capacity)
        self.free_sets = {o: set() for o in range(self.min_order, self.max_order + 1)}
        self.live = {}
        self.order_of = {}
        if reserve_from is None:
            self.free_sets[self.max_order].add(0)
        else:
            off, rest, order = 0, reserve_from, self.max_order
            while rest > 0:
                blk = 1 << order
                if blk <= rest and off % blk == 0:
                    self.free_sets[order].add(off)
                    off += blk
                    rest -= blk
                else:
                    order -= 1

    def block_size(self, size):
        return 1 << max(_ceil_log2(max(size, 1)), self.min_order)

    def alloc(self, size):
        if size > self.capacity:
            raise MemoryError("oom")
        order = max(_ceil_log2(max(size, 1)), self.min_order)
        src = order
        while src <= self.max_order and not self.free_sets[src]:
            src += 1
        if src > self.max_order:
            raise MemoryError("oom")
        off = min(self.free_sets[src])
        self.free_sets[src].discard(off)
        while src > order:
            src -= 1
            self.free_sets[src].add(off + (1 << src))
        self.live[off] = 1 << order
        self.order_of[off] = order
        return off

    def free(self, off):
        size = self.live.pop(off)
        order = self.order_of.pop(off)
        while order < self.max_order:
            buddy = off ^ (1 << order)
            if buddy not in self.free_sets[order]:
                break
            self.free_sets[order].discard(buddy)
            off = min(off, buddy)
            order += 1
        self.free_sets[order].add(off)
        return size


class OracleReverse:
    """Downward bump with exact-size reuse (allocators.py:153-190)."""

    def __init__(self, floor: int, capacity: int, alignment: int = 64):
        self.floor, self.capacity, self.alignment = floor, capacity, alignment
        self.bottom, self.free_lists, self.live = capacity, {}, {}

    def block_size(self, size):
        return _align_up(max(size, 1), self.alignment)

    def alloc(self, size):
        rounded = self.block_size(size)
        lst = self.free_lists.get(rounded)
        if lst:
            off = lst.pop()
        else:
            off = (self.bottom - rounded) & ~(self.alignment - 1)
            if off < self.floor:
                raise MemoryError("oom")
            self.bottom = off
        self.live[off] = rounded
        return off

    def free(self, off):
        rounded = self.live.pop(off)
        self.free_lists.setdefault(rounded, []).append(off)
        return rounded
