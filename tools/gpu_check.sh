#!/bin/bash
# One GPU-box pass at HEAD: GPU tests, smoke, bench (N=1 and, with NGPU>=2,
# N=NGPU under torchrun), the ncu launch list of the bench and one
# `ncu --set full` capture of the stencil.  Usage (from the repo root):
#   NGPU=2 TAG=r02x bash tools/gpu_check.sh        [SKIP=tests,ncu,...]
set -u
NGPU=${NGPU:-1}; TAG=${TAG:-run}; SKIP=${SKIP:-}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpus.txt
if [[ $SKIP != *tests* ]]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
fi
if [[ $SKIP != *bench* ]]; then
  timeout 900 python bench.py > $O/bench_n1.jsonl 2> $O/bench_n1.err
  if [ $NGPU -ge 2 ]; then
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NGPU --master-addr 127.0.0.1 \
      --master-port 29531 bench.py --gpus $NGPU > $O/bench_n$NGPU.jsonl 2> $O/bench_n$NGPU.err
  fi
fi
if [[ $SKIP != *ncu* ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 > $O/ncu_launch.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k stencil_tma_kernel -s 3 -c 1 \
    -o $O/stencil_full python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --no-secondary > $O/ncu_full.log 2>&1
fi
tail -2 $O/pytest.txt 2>/dev/null; cat $O/smoke.txt 2>/dev/null | tail -2
