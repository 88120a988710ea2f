#!/bin/bash
out=gpurun_out/r2g; mkdir -p $out
for rep in 1 2; do
for v in "GS_L1_BULK=0" "GS_L1_BPS=3" "GS_L1_BPS=3 GS_SAMPLE_CARVE=100" "GS_L1_BPS=4" "GS_L1_BPS=3 GS_L1_CARVE=-1" "GS_L1_BULK=0 GS_SAMPLE_CARVE=100"; do
  env $v python bench.py --steps 400 --warmup 20 --no-cpu-baseline --epochs 3 >> $out/bench_ab.json 2>>$out/bench.err; echo "$v" >> $out/bench_ab.tags
done
done
for v in "" "GS_BAL_PANEL_CH=32" "GS_BAL_PANEL_CH=16" "GS_BAL_PANEL_CH=13"; do
  env $v python bench.py --config products_shadow --steps 30 --warmup 5 --no-cpu-baseline --epochs 0 >> $out/bench_shadow.json 2>>$out/bench.err; echo "$v" >> $out/bench_shadow.tags
done
