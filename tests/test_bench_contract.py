"""bench.py contract checks that run without a GPU: the reference arm (the
reference's compiled CPU kernel on the host cores) prints one well-formed JSON
line with the keys the driver reads."""

import json
import os
import subprocess
import sys

from conftest import ROOT


def _run(args, env_extra):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "2", "--warmup", "1"], {"BENCH_GRID": "128"})
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["metric"] == "minimod_gpts_per_s"
    assert d["unit"] == "Gpts/s" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]
    # the other BASELINE configs' CPU paths, timed in the same run
    sec = d["secondary"]
    assert sec["minimod_128"]["cpu_baseline"]["value"] > 0
    assert sec["minimod_128"]["cpu_baseline"]["cores"] == 2
    assert sec["dgemm_ring"]["cpu_baseline"]["unit"] == "TFLOP/s"


def test_reference_arm_non_zero_ranks_exit_quietly():
    env = dict(os.environ, BENCH_GRID="128", RANK="1", WORLD_SIZE="2")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0"], env=env, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0 and not out.stdout.strip()
