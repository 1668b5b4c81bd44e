# collectives on N GPUs: GPU collective tests, multi-process parity, allreduce sweep (auto vs fused), p2p.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -k "collective or rma" > gpurun_out/coll_pytest_$N.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/coll_pytest_$N.log
timeout 600 $TR tools/mp_check.py > gpurun_out/coll_mpcheck_$N.log 2>&1; echo "mp_check rc=$?"; grep '"check"' gpurun_out/coll_mpcheck_$N.log | cut -c1-200
timeout 600 $TR bench.py --gpus $N --workload allreduce --steps 20 --warmup 3 > gpurun_out/coll_ar_$N.log 2>&1; echo "ar rc=$?"; tail -1 gpurun_out/coll_ar_$N.log | cut -c1-1200
timeout 600 $TR bench.py --gpus $N --workload bcast --steps 20 --warmup 3 > gpurun_out/coll_bc_$N.log 2>&1; echo "bc rc=$?"; tail -1 gpurun_out/coll_bc_$N.log | cut -c1-300
timeout 600 $TR bench.py --gpus $N --workload p2p --steps 20 --warmup 3 > gpurun_out/coll_p2p_$N.log 2>&1; echo "p2p rc=$?"; tail -1 gpurun_out/coll_p2p_$N.log | cut -c1-600
