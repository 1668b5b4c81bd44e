mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for v in "3 0" "2 0" "0 0" "3 4" "3 8" "3 12" "2 12"; do
  set -- $v
  export DIOMP_STENCIL_PROMO=$1 DIOMP_STENCIL_CACHE=$2
  timeout 300 python tools/probe.py stencil 1024 > gpurun_out/w_$1_$2.log 2>&1 && \
  timeout 300 ncu --metrics $M --clock-control none -k regex:stencil_tma -s 3 -c 1 --csv python tools/probe.py stencil 1024 > gpurun_out/w_ncu_$1_$2.csv 2>&1
  echo "promo=$1 cache=$2 rc=$? $(cat gpurun_out/w_$1_$2.log)"
  grep -E "dram__bytes_read|gpu__time" gpurun_out/w_ncu_$1_$2.csv | awk -F'","' '{print "   ", $(NF-2), $NF}' | tr -d '"'
done
