# stencil halo-order A/B at N GPUs
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
for ef in 0 1 0 1; do
DIOMP_STENCIL_EDGE_FIRST=$ef timeout 600 $TR bench.py --gpus $N --steps 50 --warmup 3 --no-e2e --no-cpu > gpurun_out/edge_${ef}_$N.log 2>&1; echo "edge_first=$ef rc=$? $(tail -1 gpurun_out/edge_${ef}_$N.log | cut -c1-160)"
done
