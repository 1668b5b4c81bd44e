for v in s9_p4 s9_p3 s7_p7 s10_p2; do export DIOMP_B200_LIB=$PWD/build/lib_$v.so; echo "$v $(timeout 300 python tools/probe.py stencil 1024)"; done
unset DIOMP_B200_LIB; echo "default $(timeout 300 python tools/probe.py stencil 1024)"
