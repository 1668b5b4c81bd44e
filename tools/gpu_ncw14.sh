mkdir -p gpurun_out
export DIOMP_B200_LIB=$PWD/build/lib_ncw14.so; echo "ncw14 $(timeout 300 python tools/probe.py stencil 1024)"
timeout 600 python -m pytest tests/test_gpu_stencil.py -q --timeout 300 -p no:cacheprovider 2>&1 | tail -1
unset DIOMP_B200_LIB
S="python tools/probe.py stencil 1024"
timeout 300 $S > gpurun_out/p5_s.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_tma -s 3 -c 1 -o gpurun_out/stencil_v5 $S > gpurun_out/p5_ncu.log 2>&1; echo ncu_rc=$?; cat gpurun_out/p5_s.log
