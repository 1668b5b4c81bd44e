mkdir -p gpurun_out
S="python tools/probe.py stencil 1024"
G="python tools/probe.py dgemm 8192"
timeout 300 $S > gpurun_out/p3_s.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_tma -s 3 -c 1 -o gpurun_out/stencil_v4 $S > gpurun_out/p3_ncu_s.log 2>&1; echo s_rc=$?
timeout 300 $G > gpurun_out/p3_g.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm_dmma -s 2 -c 1 -o gpurun_out/dgemm_v1 $G > gpurun_out/p3_ncu_g.log 2>&1; echo g_rc=$?
cat gpurun_out/p3_s.log gpurun_out/p3_g.log
