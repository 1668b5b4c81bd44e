# k=4: collective probe (CTA caps 4 / 2) + NCCL reference point; twosided stencil tests
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
O=gpurun_out/collprobe_$N.txt
: > $O
for c in 4 2; do
  echo "== DIOMP_COLL_CTAS_PER_SM=$c" >> $O
  DIOMP_COLL_CTAS_PER_SM=$c timeout 120 ./tools/coll_probe.bin allreduce >> $O 2>&1
  DIOMP_COLL_CTAS_PER_SM=$c timeout 120 ./tools/coll_probe.bin bcast >> $O 2>&1
done
cat $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541"
timeout 300 $TR tools/nccl_probe.py > gpurun_out/nccl_$N.txt 2>&1; echo "nccl rc=$?"; tail -1 gpurun_out/nccl_$N.txt
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "twosided" > gpurun_out/twosided_$N.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/twosided_$N.log
