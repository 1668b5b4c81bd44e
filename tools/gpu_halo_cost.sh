# N-GPU stencil: cost of the halo stores and of the neighbour flags (timing-only knobs)
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29567"
for rep in 1 2; do for v in none XNOHALO XNOSYNC both; do
  case $v in none) E="";; XNOHALO) E="DIOMP_STENCIL_XNOHALO=1";; XNOSYNC) E="DIOMP_STENCIL_XNOSYNC=1";; both) E="DIOMP_STENCIL_XNOHALO=1 DIOMP_STENCIL_XNOSYNC=1";; esac
  env $E timeout 600 $TR bench.py --gpus $N --no-e2e > /tmp/h.log 2>&1
  echo "$v $(tail -1 /tmp/h.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])' 2>&1 | tail -1)"
done; done
