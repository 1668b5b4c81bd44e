"""Launcher (reference cli.py:1-327): argument validation, rank/node/GPU
assignment, environment mapping, CSV merge and exit codes -- on CPU -- and on
the GPU the reference's north-star config 1 end to end through the launcher
(`-n 2 stencil --grid 128 --steps 100`, checksum equal to the reference)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import GOLDEN, ROOT

from paper_2506_02486_b200 import cli
from paper_2506_02486_b200.errors import UsageError


def test_plan_for_stencil_and_env_mapping():
    plan = cli.parse_args(["-n", "2", "--segment-bytes", "268435456", "--allocator", "linear",
                           "--sim-task-us", "0", "--timeout", "30", "stencil", "--grid", "128",
                           "--steps", "100"])
    assert (plan.nranks, plan.devices_per_rank, plan.subcommand) == (2, 1, "stencil")
    assert plan.node_ids == [0, 1]
    assert plan.opts == dict(grid=[128, 128, 128], steps=100, exchange="onesided", source=True,
                             dump_field=None)
    assert plan.env == {"DIOMP_SEGMENT_BYTES": "268435456", "DIOMP_ALLOCATOR": "linear",
                        "DIOMP_SIM_TASK_US": "0", "DIOMP_TIMEOUT": "30.0"}


@pytest.mark.parametrize("argv", [
    ["-n", "0", "stencil", "--grid", "8"],
    ["-n", "3", "stencil", "--grid", "16"],              # nx not divisible by n
    ["-n", "2", "stencil", "--grid", "8", "8"],          # 1 or 3 extents
    ["-n", "1", "p2p"],                                  # p2p needs 2 ranks
    ["-n", "1", "collective"],
    ["-n", "2", "matmul", "--n", "9"],                   # P must divide N
    ["-n", "2", "matmul", "--n", "8", "--p", "4"],       # P = nranks * devices
    ["-n", "4", "--nodes", "5", "p2p"],
    ["-n", "2", "--node-map", "0", "p2p"],
    ["-n", "3", "stencil", "--grid", "8", "--exchange", "twosided"],  # 3 does not divide 8
])
def test_usage_errors(argv):
    with pytest.raises(UsageError):
        cli.parse_args(argv)
    assert cli.main(argv) == cli.EXIT_USAGE


def test_twosided_exchange_accepted():
    plan = cli.parse_args(["-n", "2", "stencil", "--grid", "8", "--exchange", "twosided"])
    assert plan.opts["exchange"] == "twosided"


def test_halo_loc_report():
    """apps/loc.py (reference loc.py): effective lines of each exchange body;
    the one-sided routine is the shorter one."""
    from paper_2506_02486_b200.apps import loc
    rep = loc.halo_loc_report()
    assert 0 < rep["onesided"] < rep["twosided"]
    src = "def exchange(a):\n    '''doc'''\n    # c\n\n    x = 1\n    return x\n"
    assert loc.loc_metric(src) == 2
    assert loc.effective_lines("a = 1\n# c\n\nb = 2\n") == 2
    assert loc.effective_lines("") == 0


def test_argparse_errors_exit_2(capsys):
    assert cli.main(["-n", "2", "nosuchcommand"]) == 2
    assert cli.main(["-n", "2", "p2p", "--sizes", "8,4"]) == 2


def test_node_blocks_and_gpu_assignment():
    assert cli.parse_args(["-n", "4", "--nodes", "2", "p2p"]).node_ids == [0, 0, 1, 1]
    assert cli.parse_args(["-n", "3", "--node-map", "1,0,1", "p2p"]).node_ids == [1, 0, 1]
    assert [cli.gpu_assignment(r, 1, 8) for r in range(4)] == ["0", "1", "2", "3"]
    assert [cli.gpu_assignment(r, 2, 8) for r in range(4)] == ["0,1", "2,3", "4,5", "6,7"]
    assert [cli.gpu_assignment(r, 1, 1) for r in range(3)] == ["0", "0", "0"]
    assert cli.gpu_assignment(3, 2, 4) == "2,3"


def test_merge_csv_rank_order_and_baseline(tmp_path, capsys):
    plan = cli.RunPlan(3, 1, [0, 1, 2], "p2p", out=None)
    (tmp_path / "rank1.csv").write_text("kind,size_bytes,iters,mean_us,bw_MiBs\n"
                                        "put,8,10,2.000,3.000\n")
    (tmp_path / "rank0.csv").write_text("kind,size_bytes,iters,mean_us,bw_MiBs\n"
                                        "put,4,10,1.000,2.000\n")
    cli._merge_csv(plan, str(tmp_path))
    out = capsys.readouterr().out.splitlines()
    assert out == ["kind,size_bytes,iters,mean_us,bw_MiBs", "put,4,10,1.000,2.000",
                   "put,8,10,2.000,3.000"]
    base = tmp_path / "base.csv"
    base.write_text("kind,size_bytes,iters,mean_us,bw_MiBs\nput,4,10,10.000,1.0\n")
    plan.baseline, plan.out = str(base), str(tmp_path / "merged.csv")
    cli._merge_csv(plan, str(tmp_path))
    merged = (tmp_path / "merged.csv").read_text().splitlines()
    assert merged[0].endswith("log10_ratio") and merged[1] == "put,4,10,1.000,2.000,1.0000"


@pytest.mark.gpu
def test_launcher_runs_north_star_config_1():
    gold = {(c["nx"], c["steps"]): c["sha256"]
            for c in json.load(open(os.path.join(GOLDEN, "stencil_golden.json")))["cases"]}
    env = dict(os.environ, PYTHONPATH=ROOT)
    out = subprocess.run([sys.executable, "-m", "paper_2506_02486_b200", "-n", "2",
                          "--segment-bytes", str(256 << 20), "stencil", "--grid", "128",
                          "--steps", "100"], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    header, row = out.stdout.strip().splitlines()[-2:]
    assert header == "kind,nx,ny,nz,steps,checksum,seconds"
    fields = row.split(",")
    assert fields[:5] == ["stencil", "128", "128", "128", "100"]
    assert fields[5] == gold[(128, 100)]


@pytest.mark.gpu
def test_launcher_child_failure_exit_3(tmp_path):
    env = dict(os.environ, PYTHONPATH=ROOT)
    # a segment too small for the fields: every rank fails inside the run
    out = subprocess.run([sys.executable, "-m", "paper_2506_02486_b200", "-n", "2",
                          "--segment-bytes", str(1 << 20), "stencil", "--grid", "64",
                          "--steps", "1"], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == cli.EXIT_CHILD, (out.returncode, out.stderr[-2000:])
