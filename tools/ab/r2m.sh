#!/bin/bash
out=gpurun_out/r2m; mkdir -p $out
for rep in 1 2; do
for c in reddit products_gcn; do
for v in "GS_SAMPLE_COOP=1" "GS_SAMPLE_COOP=0" "GS_SAMPLE_AFTER_L1=1"; do
  env $v python bench.py --config $c --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_ab.json 2>>$out/bench.err; echo "$c $v" >> $out/bench_ab.tags
done
done
for v in "GS_TC_BN256=0" "GS_TC_BN256=1"; do
  env $v python bench.py --steps 400 --warmup 20 --no-cpu-baseline --epochs 3 >> $out/bench_ab.json 2>>$out/bench.err; echo "products $v" >> $out/bench_ab.tags
done
done
