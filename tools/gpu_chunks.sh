# stencil x-chunk length sweep at 1024^3 (DIOMP_STENCIL_CHUNK; unset = list-schedule choice)
for ch in auto 1016 600 512 480 400 342 300 256 205 171 128; do
  if [ $ch = auto ]; then unset DIOMP_STENCIL_CHUNK; else export DIOMP_STENCIL_CHUNK=$ch; fi
  timeout 300 python bench.py --steps 20 --no-e2e --no-cpu > /tmp/v.log 2>&1
  echo "chunk=$ch $(tail -1 /tmp/v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])' 2>&1 | tail -1)"
done
