# round-end rehearsal (what the driver runs) + ncu --set full of the top kernels
mkdir -p gpurun_out
bash tools/gpu_rehearsal.sh
B="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_tma -s 3 -c 1 -o gpurun_out/stencil_v6 $B > gpurun_out/fin_ncu_s.log 2>&1; echo "ncu stencil rc=$?"
G="python tools/probe.py dgemm 8192"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm_dmma -s 2 -c 1 -o gpurun_out/dgemm_v2 $G > gpurun_out/fin_ncu_g.log 2>&1; echo "ncu dgemm rc=$?"
