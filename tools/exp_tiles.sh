# Big vs Small stencil tiles per grid size (DIOMP_STENCIL_TILES), 1 GPU; stencil parity tests
O=gpurun_out/tiles; mkdir -p $O
[ -n "$TESTS" ] && timeout 900 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_edges.py tests/test_gpu_apps.py -x -q > $O/tests.txt 2>&1
for r in 1 2; do for g in 128 192 256 384 512; do for t in big small; do
  echo "g=$g tiles=$t $(PROBE_ITERS=200 DIOMP_STENCIL_TILES=$t python tools/probe.py stencil $g)"
done; done; done > $O/probe.txt 2>&1
for t in auto big small; do
  echo "tiles=$t $(DIOMP_STENCIL_TILES=$t python -c '
import json,sys
sys.path.insert(0,".")
import paper_2506_02486_b200 as d
from paper_2506_02486_b200.apps import bench as B
import os
os.environ.setdefault("DIOMP_GPUS","0")
rt=d.init(d.LaunchConfig(nranks=1))
r=B.measure_stencil_config1(rt)
print(json.dumps({k:r[k] for k in ("value","seconds","sha256")}))
d.finalize(rt)
' 2>&1 | tail -1)"
done > $O/cfg0.txt 2>&1
