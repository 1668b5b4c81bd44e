mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_collectives.py -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_coll.log 2>&1; echo coll_rc=$?
timeout 300 python tools/probe.py dgemm 8192 > gpurun_out/probe_dgemm.log 2>&1; echo dg_rc=$?
timeout 300 python tools/probe.py copy > gpurun_out/probe_copy.log 2>&1; echo cp_rc=$?
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_tma -s 3 -c 1 -o gpurun_out/stencil_r1 $B > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
tail -2 gpurun_out/plain.log
