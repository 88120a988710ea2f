#!/bin/bash
# the fused last layer on top of the row gather; and the layer-1 gather on the sampler with it
out=gpurun_out/r3w; mkdir -p $out
for rep in 1 2; do
for v in "GS_LAST_FUSED=0" "GS_LAST_FUSED=1" "GS_L1_ON_SAMPLER=1"; do
  env $v python bench.py --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_products.json 2>>$out/err; echo "products $v" >> $out/bench_products.tags
done
done
for v in "GS_LAST_FUSED=0" "GS_LAST_FUSED=1"; do
  env $v python bench.py --config reddit --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_reddit.json 2>>$out/err; echo "reddit $v" >> $out/bench_reddit.tags
  env $v python tools/timeline.py products 30 > "$out/timeline_$(echo $v | tr ' =' '__').txt" 2>&1
done
