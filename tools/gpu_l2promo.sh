for rep in 1 2; do for v in 256 128 64 0; do
  DIOMP_STENCIL_L2PROMO=$v timeout 300 python bench.py --steps 20 --no-e2e --no-cpu > /tmp/v.log 2>&1
  echo "promo=$v $(tail -1 /tmp/v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])' 2>&1 | tail -1)"
done; done
