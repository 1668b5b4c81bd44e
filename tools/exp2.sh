# stencil tile-shape experiment: bench-only Gpts/s for experiment builds
for r in 1 2; do
for n in ${VARIANTS:-prod wz2}; do
  if [ $n = prod ]; then L=""; else L=exp/$n.so; fi
  echo "$n bench $(DIOMP_B200_LIB=$L python bench.py --steps 20 --no-e2e --no-cpu --no-secondary 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["roofline"]["frac"])')"
done; done > gpurun_out/exp2.txt 2>&1
