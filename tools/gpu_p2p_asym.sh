# N GPUs: app/rma/collective GPU tests, p2p sweep (sym + asym), allreduce/bcast sweeps
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider -k "apps or rma or collectives or twosided" > gpurun_out/pt_$N.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_$N.log
timeout 600 $TR bench.py --gpus $N --workload p2p --steps 20 --warmup 3 > gpurun_out/p2p_$N.log 2>&1; echo "p2p rc=$?"; tail -1 gpurun_out/p2p_$N.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); d.pop('rows'); print(json.dumps(d))"
for w in allreduce bcast; do
timeout 600 $TR bench.py --gpus $N --workload $w --steps 20 --warmup 3 > gpurun_out/${w}_$N.log 2>&1; echo "$w rc=$?"; tail -1 gpurun_out/${w}_$N.log | cut -c1-900
done
