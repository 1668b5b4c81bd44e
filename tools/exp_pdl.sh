# programmatic dependent launch for the stencil steps: parity tests, then configs[0] and the
# headline with DIOMP_STENCIL_PDL=1/0 (1 and 2 GPUs)
O=gpurun_out/pdl; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_edges.py tests/test_gpu_apps.py tests/test_gpu_concurrency.py -x -q > $O/tests.txt 2>&1
for r in 1 2; do for v in 1 0; do
  echo "pdl=$v $(DIOMP_STENCIL_PDL=$v DIOMP_SEGMENT_BYTES=268435456 python -c '
import json,sys,os
sys.path.insert(0,".")
os.environ.setdefault("DIOMP_GPUS","0")
import paper_2506_02486_b200 as d
from paper_2506_02486_b200.apps import bench as B
rt=d.init(d.LaunchConfig(nranks=1))
r=B.measure_stencil_config1(rt)
print(json.dumps({k:r[k] for k in ("value","seconds","sha256")}))
d.finalize(rt)
' 2>&1 | tail -1)"
  echo "pdl=$v 128 probe $(DIOMP_STENCIL_PDL=$v PROBE_ITERS=200 python tools/probe.py stencil 128)"
  echo "pdl=$v bench1024 $(DIOMP_STENCIL_PDL=$v python bench.py --steps 20 --no-e2e --no-cpu --no-secondary 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"])')"
  echo "pdl=$v bench1024 N=2 $(DIOMP_STENCIL_PDL=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 2 --steps 30 --no-e2e --no-cpu --no-secondary 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["secondary"] if "secondary" in d else "")')"
done; done > $O/perf.txt 2>&1
