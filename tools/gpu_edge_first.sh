# stencil N = all GPUs: edge-last (default) vs edge-first unit order, repeated
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29565"
for rep in 1 2; do for ef in 0 1; do
  DIOMP_STENCIL_EDGE_FIRST=$ef timeout 600 $TR bench.py --gpus $N --no-e2e > /tmp/ef.log 2>&1
  echo "edge_first=$ef rep=$rep $(tail -1 /tmp/ef.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])')"
done; done
