# multi-GPU stencil knobs at N=2/4 (bench headline only) and the per-GPU slab probe
for nx in 1024 512 256; do echo "slab nx=$nx $(python tools/probe.py stencil 1024 $nx)"; done > gpurun_out/exp_scale.txt 2>&1
for n in 4 2; do for ef in 0 1; do
  echo "N=$n edge_first=$ef $(DIOMP_STENCIL_EDGE_FIRST=$ef timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n bench.py --gpus $n --steps 30 --no-e2e --no-cpu --no-secondary 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"])')" >> gpurun_out/exp_scale.txt 2>&1
done; done
