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
  for n in 2 4; do
    [ $NGPU -ge $n ] || continue
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 2953$n bench.py --gpus $n > $O/bench_n$n.jsonl 2> $O/bench_n$n.err
  done
  timeout 900 python bench.py --impl reference > $O/reference_n1.jsonl 2> $O/reference_n1.err
fi
if [[ $SKIP != *coll* ]] && [ $NGPU -ge 2 ]; then
  g++ -O2 -std=c++20 tools/coll_probe.cpp -o tools/coll_probe.bin paper_2506_02486_b200/libdiomp_b200.so \
    -Wl,-rpath,'$ORIGIN/../paper_2506_02486_b200' > $O/coll_build.log 2>&1
  for k in 2 4; do
    [ $NGPU -ge $k ] || continue
    for op in allreduce bcast; do timeout 300 ./tools/coll_probe.bin $op $k > $O/collprobe_${op}_k$k.txt 2>&1; done
  done
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29539 bench.py --gpus 2 --workload p2p --steps 20 > $O/p2p_n2.jsonl 2> $O/p2p_n2.err
fi
if [[ $SKIP != *ncu* ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 > $O/ncu_launch.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k stencil_tma_kernel -s 3 -c 1 \
    -o $O/stencil_full python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --no-secondary > $O/ncu_full.log 2>&1
fi
tail -2 $O/pytest.txt 2>/dev/null; cat $O/smoke.txt 2>/dev/null | tail -2
