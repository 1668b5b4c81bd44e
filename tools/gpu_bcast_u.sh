# pull+push bcast: vectors in flight per thread (DIOMP_BCAST_U) x CTAs per SM, k = 4 and 3
mkdir -p gpurun_out
O=gpurun_out/bcast_u.txt; : > $O
for k in 4 3; do for u in 4 2 8; do for c in 2 1 4; do
  echo "== k=$k U=$u CTAS_PER_SM=$c" >> $O
  DIOMP_BCAST_U=$u DIOMP_COLL_CTAS_PER_SM=$c timeout 60 ./tools/coll_probe.bin bcast $k 2>&1 | grep -E "65536|262144|1048576 |wrong|error" >> $O
done; done; done
cat $O
