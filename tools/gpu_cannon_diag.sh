# Cannon ring shift engine: copy engine on a side stream (default) vs fused into the DMMA kernel
mkdir -p gpurun_out; O=gpurun_out/cannon_shift.txt; : > $O
timeout 900 python -m pytest tests/test_gpu_apps.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/cannon_pt.log 2>&1; echo "pytest rc=$?" >> $O; tail -2 gpurun_out/cannon_pt.log >> $O
for rep in 1 2; do for sh in ce fused; do for n in 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n"
  DIOMP_CANNON_SHIFT=$sh timeout 600 $TR bench.py --gpus $n --workload dgemm --steps 3 --warmup 1 > gpurun_out/cannon_${sh}_n$n.log 2>&1
  echo "shift=$sh n=$n rc=$? $(tail -1 gpurun_out/cannon_${sh}_n$n.log | cut -c1-400)" >> $O
done; done; done
cat $O
