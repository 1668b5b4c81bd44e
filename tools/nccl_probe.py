"""NCCL reference point for the collective sweeps (not part of the product).

torch.distributed (NCCL 2.28, torch-bundled) all_reduce / broadcast of f32
buffers on this box, CUDA-event timed on the NCCL stream's caller stream,
max over ranks.  busBW as in the bench: allreduce 2(k-1)/k*S/t, bcast S/t.
Launch: python -m torch.distributed.run --nproc-per-node N tools/nccl_probe.py
Env NCCL_ALGO / NCCL_NVLS_ENABLE pass through to NCCL.
"""
import json
import os

import torch
import torch.distributed as dist


def main():
    rank = int(os.environ["RANK"])
    k = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl")
    rows = {"allreduce": [], "bcast": []}
    for op in ("allreduce", "bcast"):
        for sz in (1 << 20, 16 << 20, 64 << 20, 256 << 20, 1 << 30):
            x = torch.ones(sz // 4, dtype=torch.float32, device="cuda")
            iters = 20 if sz >= (256 << 20) else 50

            def run():
                if op == "allreduce":
                    dist.all_reduce(x)
                else:
                    dist.broadcast(x, 0)
            for _ in range(5):
                run()
            torch.cuda.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(iters):
                run()
            b.record()
            torch.cuda.synchronize()
            t = torch.tensor([a.elapsed_time(b) / iters / 1e3], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sec = t.item()
            bw = (2 * (k - 1) / k if op == "allreduce" else 1.0) * sz / sec / 1e9
            rows[op].append([sz, round(sec * 1e6, 2), round(bw, 1)])
    if rank == 0:
        print(json.dumps({"nccl": torch.cuda.nccl.version(), "k": k, "algo": os.environ.get("NCCL_ALGO"),
                          "nvls": os.environ.get("NCCL_NVLS_ENABLE"), "rows": rows,
                          "row_format": "[bytes, us, busBW GB/s]"}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
