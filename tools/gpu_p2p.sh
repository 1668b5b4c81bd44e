# put/get engines on N GPUs: GPU RMA tests, then the p2p sweep through the public API.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
timeout 600 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -k "rma or edges or p2p" > gpurun_out/p2p_pytest_$N.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/p2p_pytest_$N.log
timeout 600 $TR bench.py --gpus $N --workload p2p --steps 20 --warmup 3 > gpurun_out/p2p_$N.log 2>&1; echo "p2p rc=$?"; tail -1 gpurun_out/p2p_$N.log | cut -c1-700
DIOMP_PUT_ENGINE=sm DIOMP_GET_ENGINE=sm timeout 600 $TR bench.py --gpus $N --workload p2p --steps 20 --warmup 3 > gpurun_out/p2p_sm_$N.log 2>&1; echo "p2p sm rc=$?"; tail -1 gpurun_out/p2p_sm_$N.log | cut -c1-700
