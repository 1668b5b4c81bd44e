"""The reference-side bindings of INTEGRATION.md, run for real:

* integration/_b200.py -- the DIOMP_KERNELS=b200 backend a maintainer drops
  into the reference's kernel seam (kernels/__init__.py:15-31): numpy in,
  numpy out, through the C ABI only; bitwise equal to the reference's own
  outputs (tests/golden/kernels_golden.npz, produced by running the reference);
* tests/c/rma_abi.c -- a C program that reaches the global address space
  through the rank-addressed RMA context (peer table, put/get -> op,
  op_query/op_wait, fence_group), compiled with gcc against
  include/diomp_b200.h and libdiomp_b200.so;
* tests/c/coll_abi.c -- two host threads driving the collectives (allreduce,
  bcast, the LL path through diomp_ll_call) on two GPUs from C.
"""

import importlib.util
import os
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN, NGPU, ROOT, need_gpus

pytestmark = pytest.mark.gpu


def _backend():
    spec = importlib.util.spec_from_file_location(
        "diomp_kernels_b200", os.path.join(ROOT, "integration", "_b200.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("case", ["s2", "s3", "s4", "s4b"])
def test_reference_seam_backend_stencil_bitwise(case):
    g = np.load(os.path.join(GOLDEN, "kernels_golden.npz"))
    if f"{case}_cur" not in g:
        pytest.skip(f"no {case} fixture")
    b = _backend()
    w = g[f"{case}_w"]
    u_prev = g[f"{case}_prev"].copy()
    b.stencil_update(u_prev, g[f"{case}_cur"], u_prev, float(g[f"{case}_center"][0]),
                     w[0], w[1], w[2], len(w[0]) - 1)
    assert np.array_equal(u_prev.view(np.uint64), g[f"{case}_out"].view(np.uint64))


@pytest.mark.parametrize("name", ["m1", "m2", "m3"])
def test_reference_seam_backend_matmul_bitwise(name):
    g = np.load(os.path.join(GOLDEN, "kernels_golden.npz"))
    b = _backend()
    a, bb = g[f"{name}_a"], g[f"{name}_b"]
    c = np.empty((a.shape[0], bb.shape[1]))
    b.matmul_f64(a, bb, c)
    assert np.array_equal(c.view(np.uint64), g[f"{name}_c"].view(np.uint64))


def test_c_caller_reaches_global_memory_through_the_rma_context(tmp_path):
    exe = tmp_path / "rma_abi"
    libdir = os.path.join(ROOT, "paper_2506_02486_b200")
    subprocess.check_call(["gcc", "-O2", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "c", "rma_abi.c"), "-o", str(exe),
                           "-L", libdir, "-l:libdiomp_b200.so", f"-Wl,-rpath,{libdir}"])
    gpus = ["0", "1"] if NGPU >= 2 else ["0", "0"]
    out = subprocess.run([str(exe), *gpus], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "all ok" in out.stdout


@need_gpus(2)
def test_c_caller_drives_collectives(tmp_path):
    exe = tmp_path / "coll_abi"
    libdir = os.path.join(ROOT, "paper_2506_02486_b200")
    subprocess.check_call(["gcc", "-O2", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "c", "coll_abi.c"), "-o", str(exe),
                           "-L", libdir, "-l:libdiomp_b200.so", "-lpthread",
                           f"-Wl,-rpath,{libdir}"])
    out = subprocess.run([str(exe), "0", "1"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "all ok" in out.stdout
