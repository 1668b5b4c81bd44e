mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stencil.py -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_stencil4.log 2>&1; echo st_rc=$?; tail -2 gpurun_out/pytest_stencil4.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for c in 1 0; do
  export DIOMP_STENCIL_CACHE=$c
  timeout 300 python tools/probe.py stencil 1024 > gpurun_out/v4_$c.log 2>&1 && \
  timeout 300 ncu --metrics $M --clock-control none -k regex:stencil_tma -s 3 -c 1 --csv python tools/probe.py stencil 1024 > gpurun_out/v4_ncu_$c.csv 2>&1
  echo "cache=$c rc=$?"; cat gpurun_out/v4_$c.log
done
unset DIOMP_STENCIL_CACHE
timeout 600 python bench.py --steps 100 --warmup 3 --no-cpu > gpurun_out/bench4.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/bench4.log | cut -c1-700
