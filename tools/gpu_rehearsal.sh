mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/reh_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/reh_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/reh_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/reh_smoke.log
timeout 900 python bench.py > gpurun_out/reh_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/reh_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/reh_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/reh_ref.log
B="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu"
timeout 300 $B > gpurun_out/reh_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/reh_launches.csv $B > gpurun_out/reh_ncu.log 2>&1; echo "ncu rc=$?"
