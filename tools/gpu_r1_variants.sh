mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum
for v in "4 0" "0 0" "4 1" "4 2" "4 3" "12 3" "0 1"; do
  set -- $v
  export DIOMP_STENCIL_PREVPF=$1 DIOMP_STENCIL_CACHE=$2
  timeout 300 python tools/probe.py stencil 1024 > gpurun_out/var_$1_$2.log 2>&1 && \
  timeout 300 ncu --metrics $M --clock-control none -k regex:stencil_tma -s 3 -c 1 --csv python tools/probe.py stencil 1024 > gpurun_out/var_ncu_$1_$2.csv 2>&1
  echo "variant $1 $2 rc=$?"; cat gpurun_out/var_$1_$2.log
done
