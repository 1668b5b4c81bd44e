# collective kernel probe through the C ABI, all GPUs of the box, knob sweep
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
O=gpurun_out/collprobe_$N.txt
: > $O
for c in 4 2 1; do
  echo "== DIOMP_COLL_CTAS_PER_SM=$c" >> $O
  DIOMP_COLL_CTAS_PER_SM=$c timeout 120 ./tools/coll_probe.bin allreduce >> $O 2>&1
  DIOMP_COLL_CTAS_PER_SM=$c timeout 120 ./tools/coll_probe.bin bcast >> $O 2>&1
done
echo "== NOSYNC" >> $O
NOSYNC=1 timeout 120 ./tools/coll_probe.bin allreduce >> $O 2>&1
NOSYNC=1 timeout 120 ./tools/coll_probe.bin bcast >> $O 2>&1
cat $O
