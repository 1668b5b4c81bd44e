mkdir -p gpurun_out
for c in 0 1 2; do DIOMP_DGEMM_CFG=$c timeout 300 python tools/probe.py dgemm 8192 > gpurun_out/g2_$c.log 2>&1; echo cfg=$c; cat gpurun_out/g2_$c.log; done
bash tools/gpu_r1_variants2.sh
