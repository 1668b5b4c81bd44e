# DGEMM B-tile pitch: BN+2 (paired-k conflict-free, product) vs BN+4 (previous), vs cuBLAS
mkdir -p gpurun_out
O=gpurun_out/bpad.txt; : > $O
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/bpad_pt.log 2>&1; echo "pytest rc=$?" >> $O; tail -2 gpurun_out/bpad_pt.log >> $O
for rep in 1 2; do for lib in "" paper_2506_02486_b200/libdiomp_b200_bp4.so; do for shape in "8192 8192 8192" "16384 16384 16384" "4096 16384 4096"; do
  echo "lib=${lib:-product} $(DIOMP_B200_LIB=$lib timeout 300 python tools/probe.py dgemm $shape | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["m_n_k"], round(d["dmma_tflops"],2), round(d["cublas_tflops"],2), round(d["frac_of_cublas"],3))')" >> $O
done; done; done
M=gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active
for lib in "" paper_2506_02486_b200/libdiomp_b200_bp4.so; do
  echo "ncu lib=${lib:-product}" >> $O
  DIOMP_B200_LIB=$lib timeout 300 ncu --metrics $M --clock-control none -k regex:dgemm_dmma -c 1 --csv python tools/probe.py dgemm 8192 2>&1 | grep -E "bank|dmma_cycles|time_duration" | awk -F'","' '{print "   ", $(NF-2), $NF}' | tr -d '"' >> $O
done
cat $O
