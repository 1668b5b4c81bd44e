# after the spin-then-sleep flag wait: multi-GPU tests, N-GPU stencil bench, collective sweeps
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29563"
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider -k "collectives or stencil or apps or rma or groups" > gpurun_out/spin_pt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/spin_pt.log
timeout 900 $TR bench.py --gpus $N --no-e2e > gpurun_out/spin_bench_n$N.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/spin_bench_n$N.log | cut -c1-400
timeout 120 ./tools/coll_probe.bin allreduce > gpurun_out/spin_collprobe_$N.txt 2>&1; timeout 120 ./tools/coll_probe.bin bcast >> gpurun_out/spin_collprobe_$N.txt 2>&1; cat gpurun_out/spin_collprobe_$N.txt
for w in allreduce bcast; do
timeout 600 $TR bench.py --gpus $N --workload $w --steps 20 --warmup 3 > gpurun_out/spin_${w}_$N.log 2>&1; echo "$w rc=$?"; tail -1 gpurun_out/spin_${w}_$N.log | cut -c1-300
done
