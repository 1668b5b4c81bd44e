# small-grid stencil: step time vs x-chunk length (DIOMP_STENCIL_CHUNK) at 128^3 / 256^3
for g in 128 256; do for ch in 0 4 6 8 10 12 16 24 32 64; do
  if [ $ch = 0 ]; then E=""; else E="DIOMP_STENCIL_CHUNK=$ch"; fi
  echo "g=$g chunk=$ch $(env $E python tools/probe.py stencil $g)"
done; done > gpurun_out/exp_small.txt 2>&1
