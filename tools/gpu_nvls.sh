# NVLS allreduce: parity test, then the allreduce sweep (exact + nvls)
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
timeout 600 python -m pytest tests/test_gpu_collectives.py -q --timeout 300 -p no:cacheprovider -x > gpurun_out/nvls_pytest_$N.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/nvls_pytest_$N.log
timeout 600 $TR bench.py --gpus $N --workload allreduce --steps 20 --warmup 3 > gpurun_out/nvls_ar_$N.log 2>&1; echo "ar rc=$?"; tail -1 gpurun_out/nvls_ar_$N.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('exact', [(r[0]>>10, r[2]) for r in d['rows']][-6:])
n=d.get('nvls'); print('nvls', [(r[0]>>10, r[2]) for r in n['rows']][-6:] if n else None)"
