"""Segment heaps: Python face of the native heaps in libdiomp_b200
(csrc/heap.cuh), with the class names and methods of
reference/pkg/src/diomp/allocators.py:36-190.

The state machines run in C++; offsets, rounding, reuse order, the reserved
buddy tail and the DIOMP_FAULT_INJECT=alloc_overlap seam are bit-for-bit the
reference's (pinned by tests/test_allocators.py against reference-generated
traces in tests/golden/allocator_golden.json).
"""

from __future__ import annotations

import ctypes

from . import _native
from .errors import DoubleFree, OutOfSegment

MIN_BUDDY_BLOCK = 256
_NONE = (1 << 64) - 1


def is_pow2(n: int) -> bool:
    return n > 0 and not (n & (n - 1))


def align_up(value: int, align: int) -> int:
    return (value + align - 1) & ~(align - 1)


def ceil_log2(n: int) -> int:
    return (n - 1).bit_length() if n > 1 else 0


class _NativeHeap:
    kind = ""
    _code = -1

    def __init__(self, capacity: int, arg: int, alignment: int):
        self.capacity = capacity
        self.alignment = alignment
        h = ctypes.c_void_p()
        rc = _native.lib.diomp_heap_create(self._code, capacity, arg, alignment, ctypes.byref(h))
        if rc != 0:
            raise ValueError(f"invalid {self.kind} heap parameters "
                             f"(capacity={capacity}, arg={arg}, alignment={alignment})")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _native.lib.diomp_heap_destroy(h)
            self._h = None

    def block_size(self, size: int) -> int:
        out = ctypes.c_uint64()
        _native.lib.diomp_heap_block_size(self._h, max(int(size), 0), ctypes.byref(out))
        return out.value

    def alloc(self, size: int) -> int:
        if size > _NONE - 4096:
            raise OutOfSegment(f"{self.kind}: {size} bytes do not fit")
        out = ctypes.c_uint64()
        rc = _native.lib.diomp_heap_alloc(self._h, max(int(size), 0), ctypes.byref(out))
        if rc == 10:
            raise OutOfSegment(f"{self.kind}: no room for {size} bytes "
                               f"(capacity {self.capacity})")
        _native.check(rc, f"{self.kind}.alloc")
        return out.value

    def free(self, offset: int) -> int:
        out = ctypes.c_uint64()
        rc = _native.lib.diomp_heap_free(self._h, int(offset), ctypes.byref(out))
        if rc == 11:
            raise DoubleFree(f"{self.kind}: offset {offset} is not live")
        _native.check(rc, f"{self.kind}.free")
        return out.value

    @property
    def live(self) -> dict[int, int]:
        """offset -> block size, in allocation order (a snapshot)."""
        n = ctypes.c_uint64(0)
        _native.lib.diomp_heap_live(self._h, None, None, ctypes.byref(n))
        cap = n.value
        offs = (ctypes.c_uint64 * max(cap, 1))()
        sizes = (ctypes.c_uint64 * max(cap, 1))()
        n = ctypes.c_uint64(cap)
        _native.lib.diomp_heap_live(self._h, offs, sizes, ctypes.byref(n))
        return {offs[i]: sizes[i] for i in range(n.value)}


class LinearAllocator(_NativeHeap):
    """Bump over [0, capacity) with exact-size LIFO reuse."""

    kind = "linear"
    _code = 0

    def __init__(self, capacity: int, alignment: int = 64):
        super().__init__(capacity, 0, alignment)


class BuddyAllocator(_NativeHeap):
    """2^k blocks (min 256 B), lowest-address choice, optional reserved tail."""

    kind = "buddy"
    _code = 1

    def __init__(self, capacity: int, reserve_from: int | None = None):
        if not is_pow2(capacity):
            raise ValueError("buddy capacity must be a power of two")
        super().__init__(capacity, _NONE if reserve_from is None else reserve_from, 64)
        self.min_order = ceil_log2(MIN_BUDDY_BLOCK)
        self.max_order = ceil_log2(capacity)


class ReverseBumpAllocator(_NativeHeap):
    """Downward bump over [floor, capacity) with exact-size reuse."""

    kind = "reverse"
    _code = 2

    def __init__(self, floor: int, capacity: int, alignment: int = 64):
        self.floor = floor
        super().__init__(capacity, floor, alignment)
