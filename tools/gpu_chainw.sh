# warp-unit chain bcast: GPU collective tests (incl. the forced-chain test),
# then the C-ABI probe: pull+push default vs chain at several unit shapes
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
O=gpurun_out/chainw_$N.txt; : > $O
timeout 600 python -m pytest tests/test_gpu_collectives.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/chainw_pt_$N.log 2>&1; echo "pytest rc=$?" >> $O; tail -3 gpurun_out/chainw_pt_$N.log >> $O
echo "== pull" >> $O; DIOMP_BCAST_ALGO=pull timeout 120 ./tools/coll_probe.bin bcast >> $O 2>&1
for gw in "64 4" "128 2" "32 8" "16 16" "256 1"; do set -- $gw
  echo "== chain G=$1 W=$2" >> $O
  DIOMP_BCAST_ALGO=chain DIOMP_BCAST_CHAIN_G=$1 DIOMP_BCAST_CHAIN_W=$2 timeout 120 ./tools/coll_probe.bin bcast >> $O 2>&1
done
for c in 16384 32768 131072; do
  echo "== chain G=64 W=4 CHUNK=$c" >> $O
  DIOMP_BCAST_ALGO=chain DIOMP_BCAST_CHAIN_CHUNK=$c timeout 120 ./tools/coll_probe.bin bcast >> $O 2>&1
done
cat $O
