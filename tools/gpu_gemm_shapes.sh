# DGEMM tile configs on the Cannon per-step shapes (N=16384 at P=1/2/4) vs cuBLAS
for shape in "16384 16384 16384" "8192 16384 8192" "4096 16384 4096"; do
  for c in default 0 1 3; do
    if [ $c = default ]; then unset DIOMP_DGEMM_CFG; else export DIOMP_DGEMM_CFG=$c; fi
    echo "cfg=$c $(timeout 300 python tools/probe.py dgemm $shape | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["m_n_k"], round(d["dmma_tflops"],2), round(d["cublas_tflops"],2), round(d["frac_of_cublas"],3))')"
  done
done
