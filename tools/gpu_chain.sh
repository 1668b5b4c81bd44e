# chain bcast: GPU collective tests, then the C-ABI probe with pull vs chain
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
: timeout 600 python -m pytest tests/test_gpu_collectives.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/coll_pt_$N.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/coll_pt_$N.log
for a in pull chain; do DIOMP_BCAST_ALGO=$a timeout 120 ./tools/coll_probe.bin bcast; done
