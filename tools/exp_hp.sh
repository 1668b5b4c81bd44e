# HALO=true kernel with the halo addresses derived from the parameters (exp/hp.so) vs the
# product (per-plane pointer bookkeeping), N = 2 / 4; stencil tests on the variant
b() { DIOMP_B200_LIB=$2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 2974$1 bench.py --gpus $1 --steps 30 --no-e2e --no-cpu --no-secondary 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])'; }
for r in 1 2; do for n in 2 4; do for v in prod hp; do
  if [ $v = prod ]; then L=""; else L=exp/$v.so; fi
  echo "N=$n $v $(b $n $L)"
done; done; done > gpurun_out/exp_hp.txt 2>&1
DIOMP_B200_LIB=exp/hp.so timeout 900 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_edges.py tests/test_gpu_apps.py -x -q 2>&1 | tail -1 >> gpurun_out/exp_hp.txt
