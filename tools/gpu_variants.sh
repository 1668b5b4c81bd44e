# stencil variant builds (DIOMP_B200_LIB), bench value / ms per step, two passes
for rep in 1 2; do for lib in "$@"; do
  DIOMP_B200_LIB=$PWD/paper_2506_02486_b200/$lib timeout 300 python bench.py --steps 20 --no-e2e --no-cpu > /tmp/v.log 2>&1
  echo "$lib $(tail -1 /tmp/v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])' 2>&1 | tail -1)"
done; done
