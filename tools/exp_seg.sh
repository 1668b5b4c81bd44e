# halo-free bulk of the x-walk (step_plane<..., HALO=false> between the boundary segments):
# stencil parity tests, headline at N = 1 / 2 / 4
O=gpurun_out/seg; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_edges.py tests/test_gpu_apps.py tests/test_gpu_concurrency.py tests/test_gpu_fullsize.py -x -q > $O/tests.txt 2>&1
for r in 1 2; do
  echo "N=1 $(python bench.py --steps 20 --no-e2e --no-cpu --no-secondary 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"])')"
  for n in 2 4; do echo "N=$n $(timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2972$n bench.py --gpus $n --steps 30 --no-e2e --no-cpu --no-secondary 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"])')"; done
done > $O/perf.txt 2>&1
