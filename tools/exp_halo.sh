# split of the multi-GPU stencil overhead: experiment builds without the halo stores /
# without the neighbour waits / without both (timing only, results not valid)
for r in 1 2; do for n in 4 2; do for v in prod nohalo nowait none; do
  if [ $v = prod ]; then L=""; else L=exp/$v.so; fi
  echo "N=$n $v $(DIOMP_B200_LIB=$L timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n bench.py --gpus $n --steps 30 --no-e2e --no-cpu --no-secondary 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"])')"
done; done; done > gpurun_out/exp_halo.txt 2>&1
