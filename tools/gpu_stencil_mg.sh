# multi-GPU stencil: parity (fused tests + mp_check) then bench x2
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -k "stencil or fused or device_flag" > gpurun_out/smg_pytest_$N.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/smg_pytest_$N.log
timeout 600 $TR tools/mp_check.py > gpurun_out/smg_mpcheck_$N.log 2>&1; echo "mp_check rc=$? $(grep -c '"ok": true' gpurun_out/smg_mpcheck_$N.log) ok / $(grep -c '"check"' gpurun_out/smg_mpcheck_$N.log)"
for rep in 1 2; do
timeout 600 $TR bench.py --gpus $N --steps 50 --warmup 3 --no-e2e --no-cpu > gpurun_out/smg_bench_$N.log 2>&1; echo "bench rc=$? $(tail -1 gpurun_out/smg_bench_$N.log | cut -c1-160)"
done
