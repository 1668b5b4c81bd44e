"""configs[0] (Minimod 128^3 x 100 steps) on this job's ranks through the
public runner, REPS times: device Gpts/s per run (rank 0 prints).
torchrun --nproc-per-node N tools/cfg0_probe.py [REPS]"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("DIOMP_GPUS", str(local))
    os.environ.setdefault("DIOMP_SEGMENT_BYTES", str(256 << 20))
    import paper_2506_02486_b200 as d
    from paper_2506_02486_b200.apps import bench as B
    rt = d.init()
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    vals = [B.measure_stencil_config1(rt)["value"] for _ in range(reps)]
    if rt.rank == 0:
        print(json.dumps({"ranks": rt.nranks, "pdl": os.environ.get("DIOMP_STENCIL_PDL", "auto"),
                          "gpts": vals}), flush=True)
    d.finalize(rt)


if __name__ == "__main__":
    main()
