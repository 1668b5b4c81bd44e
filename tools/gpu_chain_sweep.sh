# chain bcast knob sweep through the C-ABI probe (k = all GPUs)
mkdir -p gpurun_out
O=gpurun_out/chain_sweep.txt; : > $O
for g in 64 128 256; do for c in 524288 1048576 2097152; do
  echo "== G=$g CHUNK=$c" >> $O
  DIOMP_BCAST_ALGO=chain DIOMP_BCAST_CHAIN_G=$g DIOMP_BCAST_CHAIN_CHUNK=$c timeout 60 ./tools/coll_probe.bin bcast 2>&1 | grep -E "65536|262144|1048576|wrong|error" >> $O
done; done
cat $O
