# pull-chain bcast knob sweep through the C-ABI probe (k = all GPUs), pull+push default first
mkdir -p gpurun_out
O=gpurun_out/pullchain_sweep.txt; : > $O
echo "== default (pull+push)" >> $O
timeout 60 ./tools/coll_probe.bin bcast >> $O 2>&1
for g in 74 148 256; do for c in 131072 524288 2097152; do
  echo "== pullchain G=$g CHUNK=$c" >> $O
  DIOMP_BCAST_ALGO=pullchain DIOMP_BCAST_CHAIN_G=$g DIOMP_BCAST_CHAIN_CHUNK=$c timeout 60 ./tools/coll_probe.bin bcast >> $O 2>&1
done; done
echo "== pullchain G=148 CHUNK=524288, k=3" >> $O
DIOMP_BCAST_ALGO=pullchain DIOMP_BCAST_CHAIN_G=148 DIOMP_BCAST_CHAIN_CHUNK=524288 timeout 60 ./tools/coll_probe.bin bcast 3 >> $O 2>&1
cat $O
