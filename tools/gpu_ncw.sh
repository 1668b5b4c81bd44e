mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stencil.py -q --timeout 300 -p no:cacheprovider 2>&1 | tail -1
for v in ncw8 ncw16 default; do
  if [ $v = default ]; then unset DIOMP_B200_LIB; else export DIOMP_B200_LIB=$PWD/build/lib_$v.so; fi
  echo "$v $(timeout 300 python tools/probe.py stencil 1024)"
done
unset DIOMP_B200_LIB
export DIOMP_B200_LIB=$PWD/build/lib_ncw16.so
timeout 600 python -m pytest tests/test_gpu_stencil.py -q --timeout 300 -p no:cacheprovider 2>&1 | tail -1
