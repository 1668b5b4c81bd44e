# NVLink counters for put/get/allreduce/bcast kernels (1 process, 2 GPUs) and DMMA pipe use of the DGEMM vs cuBLAS
mkdir -p gpurun_out
timeout 300 python tools/ncu_nvlink.py > gpurun_out/nvl_plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/nvl_plain.log
M=gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/nvl_ncu.csv python tools/ncu_nvlink.py > gpurun_out/nvl_ncu.log 2>&1; echo "ncu nvl rc=$?"
timeout 300 python tools/probe.py dgemm 8192 > gpurun_out/dg_plain.log 2>&1; echo "dgemm rc=$?"; tail -1 gpurun_out/dg_plain.log
D=gpu__time_duration.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second
timeout 600 ncu --metrics $D --clock-control none --csv --log-file gpurun_out/dg_ncu.csv python tools/probe.py dgemm 8192 > gpurun_out/dg_ncu.log 2>&1; echo "ncu dgemm rc=$?"
