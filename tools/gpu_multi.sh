# Multi-GPU validation + secondary benchmarks (run with gpurun --gpus N).
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -k "fused or device_flag or multi_rank or baseline" > gpurun_out/mg_pytest_$N.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/mg_pytest_$N.log
timeout 600 $TR tools/mp_check.py > gpurun_out/mg_mpcheck_$N.log 2>&1; echo "mp_check rc=$?"; grep '"check"' gpurun_out/mg_mpcheck_$N.log
timeout 600 $TR bench.py --gpus $N --steps 50 --warmup 3 > gpurun_out/mg_bench_$N.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/mg_bench_$N.log | cut -c1-600
timeout 600 $TR bench.py --gpus $N --workload p2p --steps 20 --warmup 3 > gpurun_out/mg_p2p_$N.log 2>&1; echo "p2p rc=$?"; tail -1 gpurun_out/mg_p2p_$N.log | cut -c1-700
timeout 600 $TR bench.py --gpus $N --workload allreduce --steps 20 --warmup 3 > gpurun_out/mg_ar_$N.log 2>&1; echo "ar rc=$?"; tail -1 gpurun_out/mg_ar_$N.log | cut -c1-900
timeout 600 $TR bench.py --gpus $N --workload bcast --steps 20 --warmup 3 > gpurun_out/mg_bc_$N.log 2>&1; echo "bc rc=$?"; tail -1 gpurun_out/mg_bc_$N.log | cut -c1-900
timeout 900 $TR bench.py --gpus $N --workload dgemm --steps 2 --warmup 1 > gpurun_out/mg_dgemm_$N.log 2>&1; echo "dgemm rc=$?"; tail -1 gpurun_out/mg_dgemm_$N.log
