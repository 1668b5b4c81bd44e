# halo-store cost split (experiment builds, timing only): product vs stores duplicated locally
# (localdup) vs no halo stores (nohalo), at N = 1 (code generation only) and N = 2 / 4
b() { DIOMP_B200_LIB=$2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 2971$1 bench.py --gpus $1 --steps 30 --no-e2e --no-cpu --no-secondary 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])'; }
for r in 1 2; do for v in prod nohalo localdup; do
  if [ $v = prod ]; then L=""; else L=exp/$v.so; fi
  echo "N=1 $v $(DIOMP_B200_LIB=$L python bench.py --steps 20 --no-e2e --no-cpu --no-secondary 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])')"
done; done > gpurun_out/exp_ld1.txt 2>&1
