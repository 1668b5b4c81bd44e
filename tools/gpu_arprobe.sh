# allreduce engine probe + NCCL reference point on all GPUs of the box
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > gpurun_out/topo_$N.txt 2>&1
timeout 300 ./tools/ar_probe.bin $N > gpurun_out/ar_probe_$N.txt 2>&1; echo "ar_probe rc=$?"; cat gpurun_out/ar_probe_$N.txt
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541"
: timeout 300 $TR tools/nccl_probe.py > gpurun_out/nccl_$N.txt 2>&1; echo "nccl rc=$?"; tail -1 gpurun_out/nccl_$N.txt
: NCCL_NVLS_ENABLE=0 timeout 300 $TR tools/nccl_probe.py > gpurun_out/nccl_nonvls_$N.txt 2>&1; echo "nccl nonvls rc=$?"; tail -1 gpurun_out/nccl_nonvls_$N.txt
