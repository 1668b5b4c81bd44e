# y-neighbour drift throttle experiment (DIOMP_STENCIL_THROTTLE planes), headline stencil, 1 GPU
b() { python bench.py --steps 20 --no-e2e --no-cpu --no-secondary 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"])'; }
for r in 1 2; do for t in 0 8 16 32 64; do echo "throttle=$t $(DIOMP_STENCIL_THROTTLE=$t b)"; done; done > gpurun_out/exp_throttle.txt 2>&1
for t in 0 16; do DIOMP_STENCIL_THROTTLE=$t timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k stencil_tma_kernel -s 3 -c 1 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --no-secondary > gpurun_out/exp_throttle_ncu_$t.txt 2>&1; done
