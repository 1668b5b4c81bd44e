# multi-process parity (one process per GPU, CUDA IPC) at N = 2 and 4
mkdir -p gpurun_out
for n in 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n"
  timeout 900 $TR tools/mp_check.py > gpurun_out/mpcheck_$n.log 2>&1; echo "mp_check n=$n rc=$?"; grep '"check"' gpurun_out/mpcheck_$n.log | grep -E "cannon|false" | cut -c1-250; grep -c '"ok": true' gpurun_out/mpcheck_$n.log
done
