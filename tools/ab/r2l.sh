#!/bin/bash
out=gpurun_out/r2l; mkdir -p $out
GS_L1_BPS=3 GS_SAMPLE_AFTER_L1=1 python tools/timeline.py products 30 > $out/timeline_bulk_after.txt 2>&1
GS_L1_BULK=0 GS_SAMPLE_AFTER_L1=1 python tools/timeline.py products 30 > $out/timeline_old_after.txt 2>&1
for rep in 1 2; do
for v in "GS_L1_BULK=0" "GS_L1_BPS=3" "GS_L1_BULK=0 GS_SAMPLE_AFTER_L1=1" "GS_L1_BPS=3 GS_SAMPLE_AFTER_L1=1"; do
  env $v python bench.py --steps 400 --warmup 20 --no-cpu-baseline --epochs 3 >> $out/bench_ab.json 2>>$out/bench.err; echo "$v" >> $out/bench_ab.tags
done
done
