# ncu of the memory-only stencil build vs torch's triad add (DRAM behaviour)
mkdir -p gpurun_out
M="dram__bytes_read.sum,dram__bytes_write.sum,dram__cycles_active.avg.pct_of_peak_sustained_elapsed,dram__cycles_active.max.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__d_sectors_fill_device.sum,dram__sectors_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_write_lookup_miss.sum,lts__average_t_sector_hit_rate_srcunit_tex_op_read.pct"
DIOMP_B200_LIB=$PWD/paper_2506_02486_b200/libdiomp_b200_memonly.so timeout 600 ncu --clock-control none --metrics $M -k regex:stencil_tma -s 3 -c 1 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_memonly.txt 2>&1; echo "memonly rc=$?"
timeout 600 ncu --clock-control none --metrics $M -k regex:stencil_tma -s 3 -c 1 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_real.txt 2>&1; echo "real rc=$?"
timeout 600 ncu --clock-control none --metrics $M -k regex:vectorized_elementwise -c 2 python tools/probe.py triad 8 > gpurun_out/ncu_triad.txt 2>&1; echo "triad rc=$?"
for f in memonly real triad; do echo "== $f"; grep -E "^\s+(dram|gpu__|lts)" gpurun_out/ncu_$f.txt | head -16; done
