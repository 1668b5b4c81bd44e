# allreduce exit-handshake placement: last CTA of the fold (default) vs a trailing one-CTA kernel
mkdir -p gpurun_out
O=gpurun_out/arexit.txt; : > $O
for k in 2 4; do for r in 1 2; do
  echo "== k=$k default (run $r)" >> $O; timeout 60 ./tools/coll_probe.bin allreduce $k >> $O 2>&1
  echo "== k=$k DIOMP_AR_EXIT=kernel (run $r)" >> $O; DIOMP_AR_EXIT=kernel timeout 60 ./tools/coll_probe.bin allreduce $k >> $O 2>&1
done; done
cat $O
DIOMP_AR_EXIT=kernel timeout 600 python -m pytest tests/test_gpu_collectives.py -m gpu -q -x -p no:cacheprovider > gpurun_out/arexit_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/arexit_pytest.log
