"""Build libdiomp_b200.so in-tree (sm_100a only).

    python paper_2506_02486_b200/build.py   (does not import the package)

The library is one translation unit (csrc/diomp_b200.cu) compiled with nvcc
for compute_100a/sm_100a, cudart linked statically so the .so carries no
dependency on torch's bundled runtime.  The built file sits next to this
module, travels to the GPU box with the repo snapshot, and is what
paper_2506_02486_b200._native loads (there is no fallback).
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdiomp_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
    "-cudart", "static",
    "-shared",
]


def sources() -> list[str]:
    out = [os.path.join(HERE, "..", "include", "diomp_b200.h")]
    for f in sorted(os.listdir(CSRC)):
        if f.endswith((".cu", ".cuh")):
            out.append(os.path.join(CSRC, f))
    return out


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force: bool = False, verbose: bool = False, defines: list[str] | None = None,
          out: str | None = None) -> str:
    """defines/out: experiment builds (e.g. -DDIOMP_STENCIL_NCW=16 into another
    file, loaded with DIOMP_B200_LIB); the default build is the product."""
    lib = out or LIB
    if not force and not defines and lib == LIB and up_to_date():
        return LIB
    tmp = lib + ".tmp"
    cmd = [NVCC, *NVCC_FLAGS, *(defines or []), os.path.join(CSRC, "diomp_b200.cu"), "-o", tmp]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    os.replace(tmp, lib)
    if verbose:
        sys.stdout.write(res.stderr)
    return lib


if __name__ == "__main__":
    defs = [a for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[len("--out="):] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose=not defs, defines=defs,
                out=outs[0] if outs else None))
