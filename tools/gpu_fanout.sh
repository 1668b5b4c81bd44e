# root fan-out probe + collective probe at the library defaults
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 200 ./tools/fanout_probe.bin > gpurun_out/fanout_$N.txt 2>&1; echo "fanout rc=$?"; cat gpurun_out/fanout_$N.txt
timeout 120 ./tools/coll_probe.bin allreduce > gpurun_out/collprobe_def_$N.txt 2>&1
timeout 120 ./tools/coll_probe.bin bcast >> gpurun_out/collprobe_def_$N.txt 2>&1; cat gpurun_out/collprobe_def_$N.txt
