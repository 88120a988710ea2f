#!/bin/bash
out=gpurun_out/r2p; mkdir -p $out
for rep in 1 2; do
for v in "GS_AGG_FORCE_SH=0" "GS_AGG_FORCE_SH=1"; do
  env $v python bench.py --config reddit --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_ab.json 2>>$out/bench.err; echo "reddit $v" >> $out/bench_ab.tags
done
for v in "GS_SAMPLE_AFTER_L1=0" "GS_SAMPLE_AFTER_L1=1"; do
  env $v python bench.py --config products_shadow --steps 40 --warmup 5 --no-cpu-baseline --epochs 0 >> $out/bench_ab.json 2>>$out/bench.err; echo "shadow $v" >> $out/bench_ab.tags
done
done
