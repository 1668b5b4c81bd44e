M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed
for c in 0 16; do
  export DIOMP_STENCIL_CACHE=$c
  timeout 300 python tools/probe.py stencil 1024 > gpurun_out/d_$c.log 2>&1 && timeout 300 ncu --metrics $M --clock-control none -k regex:stencil_tma -s 3 -c 1 --csv python tools/probe.py stencil 1024 > gpurun_out/d_ncu_$c.csv 2>&1
  echo "cache=$c $(cat gpurun_out/d_$c.log)"; grep -E "dram__|gpu__time" gpurun_out/d_ncu_$c.csv | awk -F'","' '{print "   ", $(NF-2), $NF}' | tr -d '"'
done
