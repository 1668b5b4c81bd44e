# rehearsal on a 4-GPU box: full GPU suite (multi-GPU tests included), smoke,
# N=1 bench + reference arm, N=4 bench, launch list of the N=1 bench
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29561"
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/reh_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/reh_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/reh_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/reh_smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/reh_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/reh_bench.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference > gpurun_out/reh_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/reh_ref.log
timeout 900 $TR bench.py --gpus $N > gpurun_out/reh_bench_n$N.log 2>&1; echo "bench n$N rc=$?"; tail -1 gpurun_out/reh_bench_n$N.log
B="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu"
CUDA_VISIBLE_DEVICES=0 timeout 300 $B > gpurun_out/reh_plain.log 2>&1 && CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/reh_launches.csv $B > gpurun_out/reh_ncu.log 2>&1; echo "ncu rc=$?"
