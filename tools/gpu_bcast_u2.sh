# confirm the bcast U default (2) against the previous one (4), every size, k = 2, 3, 4, two passes
mkdir -p gpurun_out
O=gpurun_out/bcast_u2.txt; : > $O
for r in 1 2; do for k in 4 3 2; do
  echo "== k=$k U=2 (default) pass $r" >> $O; timeout 60 ./tools/coll_probe.bin bcast $k 2>&1 | grep -E "KiB|wrong|error" >> $O
  echo "== k=$k U=4 pass $r" >> $O; DIOMP_BCAST_U=4 timeout 60 ./tools/coll_probe.bin bcast $k 2>&1 | grep -E "KiB|wrong|error" >> $O
done; done
cat $O
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "bcast or collective" > gpurun_out/bcast_u2_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/bcast_u2_pytest.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571"
timeout 600 $TR bench.py --gpus 4 --workload bcast > gpurun_out/bcast_u2_bench4.jsonl 2> gpurun_out/bcast_u2_bench4.err; echo "bench rc=$?"; tail -1 gpurun_out/bcast_u2_bench4.jsonl | cut -c1-400
