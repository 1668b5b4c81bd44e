"""The C-ABI library loads and exports every symbol include/diomp_b200.h
declares (no compute call -- this runs without a GPU)."""

import ctypes
import os
import re
import subprocess

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "diomp_b200.h")
LIB = os.path.join(ROOT, "paper_2506_02486_b200", "libdiomp_b200.so")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    # the experiments block is not part of the product library
    text = re.sub(r"#ifdef DIOMP_EXPERIMENTS.*?#endif", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(diomp_[a-z0-9_]+)\s*\(", text)))


def test_header_declarations_exported():
    lib = ctypes.CDLL(LIB)
    declared = _declared()
    assert len(declared) >= 40
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_covers_header():
    from paper_2506_02486_b200 import _native
    assert set(_native.EXPORTS) == set(_declared())


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_struct_layouts_match_header():
    """ctypes mirrors of the header structs have the C sizes (checked by
    compiling a tiny C program against the header)."""
    from paper_2506_02486_b200 import _native
    src = ('#include <stdio.h>\n#include "diomp_b200.h"\nint main(){printf("%zu %zu %zu %zu\\n",'
           'sizeof(diomp_team),sizeof(diomp_stencil_args),sizeof(diomp_stencil_plan),'
           'sizeof(diomp_dgemm_args));printf("%zu\\n",sizeof(diomp_ll_args));return 0;}\n')
    tmp = os.path.join(ROOT, "build")
    os.makedirs(tmp, exist_ok=True)
    c, exe = os.path.join(tmp, "sz.c"), os.path.join(tmp, "sz")
    open(c, "w").write(src)
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
    got = [int(x) for x in subprocess.check_output([exe]).split()]
    want = [ctypes.sizeof(t) for t in (_native.Team, _native.StencilArgs, _native.StencilPlan,
                                        _native.DgemmArgs, _native.LLArgs)]
    assert got == want


def test_status_strings_and_heap_roundtrip_without_gpu():
    from paper_2506_02486_b200 import _native
    assert _native.describe(0) == "ok"
    assert "segment" in _native.describe(10)
    h = ctypes.c_void_p()
    assert _native.lib.diomp_heap_create(1, 1 << 20, (1 << 64) - 1, 64, ctypes.byref(h)) == 0
    off = ctypes.c_uint64()
    assert _native.lib.diomp_heap_alloc(h, 300, ctypes.byref(off)) == 0 and off.value == 0
    assert _native.lib.diomp_heap_free(h, 0, None) == 0
    assert _native.lib.diomp_heap_free(h, 0, None) == 11
    _native.lib.diomp_heap_destroy(h)


def test_product_path_has_no_oracle_dependency():
    """The package never imports or links the oracle (test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_2506_02486_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle|liboracle|oracle/", text,
                                     flags=re.M), f


def test_wire_status_codes_match_the_c_abi():
    """wire.Status (reference wire.py:46-52) = the library's status codes."""
    import re
    from paper_2506_02486_b200 import Status
    hdr = open(os.path.join(ROOT, "include", "diomp_b200.h")).read()
    for name in ("OK", "INVALID_ADDRESS", "BAD_REQUEST", "INTERNAL"):
        m = re.search(rf"#define DIOMP_{name} (\d+)", hdr)
        assert m and int(m.group(1)) == Status[name].value
