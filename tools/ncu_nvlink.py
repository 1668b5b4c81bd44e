"""NVLink-counter capture of the one-sided and collective kernels (one process,
GPUs 0 and 1 with peer access, no cross-GPU spin waits so ncu can replay each
kernel on its own).  Run under

    ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,\
nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,\
dram__bytes_write.sum --csv python tools/ncu_nvlink.py

Kernels (256 MiB payload each):
  put  copy16_kernel on GPU0 storing into GPU1   (DIOMP_PUT_ENGINE=sm path)
  get  bulk_copy_kernel on GPU1 reading GPU0     (diomp_get, TMA engine)
  allreduce reduce_kernel<f32,Sum> position 0 on GPU0 (team of 2, host-synced mode)
  bcast bcast_kernel position 1 on GPU1 (root 0)
The copy-engine put is not a kernel; its rate is in profiles/r01_nvlink_probe.txt.
"""

from __future__ import annotations

import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)


def main():
    import torch

    from paper_2506_02486_b200 import _native
    n = 256 << 20
    _native.call("diomp_peer_enable", 0, 1)
    _native.call("diomp_peer_enable", 1, 0)
    bufs = []
    for d in (0, 1):
        seg = torch.zeros(3 * n, dtype=torch.uint8, device=f"cuda:{d}")
        seg[:n].copy_(torch.randint(0, 256, (n,), dtype=torch.uint8, device=f"cuda:{d}"))
        bufs.append(seg)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    base = [b.data_ptr() for b in bufs]
    s0 = torch.cuda.Stream(0).cuda_stream
    s1 = torch.cuda.Stream(1).cuda_stream
    # put: GPU0 SM kernel, local src -> peer dst
    _native.call("diomp_copy", 0, base[1] + n, base[0], n, s0)
    # get: GPU1 bulk-async kernel, peer src -> local dst
    _native.call("diomp_get", 1, base[1] + 2 * n, base[0], n, 1, s1)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    ok = bool(torch.equal(bufs[1][n:2 * n].cpu(), bufs[0][:n].cpu())) and \
        bool(torch.equal(bufs[1][2 * n:3 * n].cpu(), bufs[0][:n].cpu()))
    # allreduce position 0 (sync=0: no flags; reads both sends, stores block 0 to both recvs)
    t = _native.Team()
    t.k, t.pos, t.device, t.sync = 2, 0, 0, 0
    t.flag_off, t.counter_off = 0, 0
    t.base[0], t.base[1] = base[0], base[1]
    _native.call("diomp_allreduce", t, 0, n, n // 4, 0, 0, s0)
    torch.cuda.synchronize(0)
    # bcast position 1 from root 0 (pulls its block from the root)
    tb = _native.Team()
    tb.k, tb.pos, tb.device, tb.sync = 2, 1, 1, 0
    tb.base[0], tb.base[1] = base[0], base[1]
    _native.call("diomp_bcast", tb, 0, n, 0, s1)
    torch.cuda.synchronize(1)
    print("ncu_nvlink: done, put/get bytes ok =", ok)


if __name__ == "__main__":
    main()
