# stencil multi-GPU after moving the step-completion signal to the next kernel's start
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29569"
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider -k "stencil or edges or cli or fused or apps" > /tmp/pt.log 2>&1; echo "pytest rc=$?"; tail -2 /tmp/pt.log
for rep in 1 2; do for v in none XNOHALO EF; do
  case $v in none) E="";; XNOHALO) E="DIOMP_STENCIL_XNOHALO=1";; EF) E="DIOMP_STENCIL_EDGE_FIRST=1";; esac
  env $E timeout 600 $TR bench.py --gpus $N --no-e2e > /tmp/h.log 2>&1
  echo "$v $(tail -1 /tmp/h.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])' 2>&1 | tail -1)"
done; done
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR2 bench.py --gpus 2 --no-e2e > /tmp/h2.log 2>&1; echo "N=2 $(tail -1 /tmp/h2.log | cut -c1-200)"
