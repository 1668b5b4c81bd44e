# multi-GPU stencil: x-chunking with the edge chunks first (their halo stores drain under the
# interior chunks) vs the default single chunk; N=4 (256 planes) and N=2 (512 planes)
b() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 2965$1 bench.py --gpus $1 --steps 30 --no-e2e --no-cpu --no-secondary 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])'; }
for r in 1 2; do
  echo "N=4 default $(b 4)"
  for ch in 128 86 64 32; do for ef in 1 0; do echo "N=4 chunk=$ch edge_first=$ef $(DIOMP_STENCIL_CHUNK=$ch DIOMP_STENCIL_EDGE_FIRST=$ef b 4)"; done; done
  echo "N=2 default $(b 2)"
  for ch in 256 171 128; do echo "N=2 chunk=$ch edge_first=1 $(DIOMP_STENCIL_CHUNK=$ch DIOMP_STENCIL_EDGE_FIRST=1 b 2)"; done
done > gpurun_out/exp_edge.txt 2>&1
