mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stencil.py -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_stencil.log 2>&1; echo st_rc=$?
tail -3 gpurun_out/pytest_stencil.log
timeout 300 python tools/probe.py stencil 512 > gpurun_out/probe_stencil.log 2>&1; echo pr_rc=$?
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
timeout 300 $B > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_tma -s 3 -c 1 -o gpurun_out/stencil_r1b $B > gpurun_out/ncu_full2.log 2>&1; echo ncu_rc=$?
timeout 600 python bench.py --steps 100 --warmup 3 --no-cpu > gpurun_out/bench2.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench2.log
