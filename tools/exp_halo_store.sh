# halo stores by TMA vs plain stores (DIOMP_STENCIL_HALO=st), 4 GPUs: stencil parity tests, then headline at N=2/4
O=gpurun_out/htma; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_edges.py tests/test_gpu_apps.py tests/test_gpu_concurrency.py tests/test_gpu_fullsize.py -x -q > $O/tests.txt 2>&1
for r in 1 2; do for n in 4 2; do for h in tma st; do
  echo "N=$n $h $(DIOMP_STENCIL_HALO=$h timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n bench.py --gpus $n --steps 30 --no-e2e --no-cpu --no-secondary 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"])')"
done; done; done > $O/perf.txt 2>&1
for h in tma st; do echo "cfg0 N=2 $h $(DIOMP_STENCIL_HALO=$h timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29619 tools/cfg0_probe.py 4 2>/dev/null | tail -1)"; done >> $O/perf.txt 2>&1
