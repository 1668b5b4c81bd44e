# headline stencil (1024^3, 1 GPU) under runtime knobs: L2 promotion of the TMA fills, x-chunk length
b() { python bench.py --steps 20 --no-e2e --no-cpu --no-secondary 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"])'; }
for r in 1 2; do
  echo "default $(b)"
  for v in 0 64 128; do echo "L2PROMO=$v $(DIOMP_STENCIL_L2PROMO=$v b)"; done
  for ch in 1024 512 342 256 205; do echo "CHUNK=$ch $(DIOMP_STENCIL_CHUNK=$ch b)"; done
done > gpurun_out/exp_knobs.txt 2>&1
