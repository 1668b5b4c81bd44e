# Cannon ring 16384^2 fp64 at N = 1, 2, 4 with the cuBLAS same-shape reference point
mkdir -p gpurun_out
for n in 1 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n"
  timeout 900 $TR bench.py --gpus $n --workload dgemm --steps 3 --warmup 1 > gpurun_out/dgemm_n$n.log 2>&1; echo "dgemm n$n rc=$?"; tail -1 gpurun_out/dgemm_n$n.log
done
