# DGEMM experiment builds: probe 8192^3 / 16384^3 and the GEMM tests per build
for n in ${VARIANTS:-prod}; do
  if [ $n = prod ]; then L=""; else L=exp/$n.so; fi
  for sz in 8192 16384; do echo "$n $(DIOMP_B200_LIB=$L python tools/probe.py dgemm $sz)"; done
  DIOMP_B200_LIB=$L timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -1 | sed "s/^/$n tests: /"
done > gpurun_out/exp_dgemm.txt 2>&1
