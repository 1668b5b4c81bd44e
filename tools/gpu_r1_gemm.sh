mkdir -p gpurun_out
for c in 0 1 2; do DIOMP_DGEMM_CFG=$c timeout 300 python tools/probe.py dgemm 8192 > gpurun_out/g_$c.log 2>&1; echo cfg=$c; cat gpurun_out/g_$c.log; done
for c in 0 1 2; do DIOMP_DGEMM_CFG=$c timeout 300 python -m pytest tests/test_gpu_gemm.py -q -p no:cacheprovider 2>&1 | tail -1; done
