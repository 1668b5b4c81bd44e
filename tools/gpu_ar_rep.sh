# allreduce algorithm A/B, repeated (variance check)
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
for rep in 1 2 3; do
for algo in ce fused; do
DIOMP_AR_ALGO=$algo timeout 600 $TR bench.py --gpus $N --workload allreduce --steps 20 --warmup 3 > gpurun_out/arrep_${algo}_$rep.log 2>&1
python - "$algo" gpurun_out/arrep_${algo}_$rep.log <<'PY'
import json,sys
d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print(sys.argv[1], [(r[0]>>20, r[2]) for r in d["rows"] if r[0] >= 1<<22])
PY
done; done
