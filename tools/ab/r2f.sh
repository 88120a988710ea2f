#!/bin/bash
out=gpurun_out/r2f; mkdir -p $out
for rep in 1 2; do
for v in "GS_L1_BULK=0" "GS_L1_BPS=3" "GS_L1_BULK=0 GS_SERIAL=1" "GS_L1_BPS=3 GS_SERIAL=1" "GS_L1_BULK=0 GS_CARVEOUT=100" "GS_L1_BPS=3 GS_CARVEOUT=100" "GS_L1_BPS=3 GS_SAMPLE_COOP=0" "GS_L1_BULK=0 GS_SAMPLE_COOP=0"; do
  env $v python bench.py --steps 400 --warmup 20 --no-cpu-baseline --epochs 3 >> $out/bench_ab.json 2>>$out/bench.err; echo "$v" >> $out/bench_ab.tags
done
done
python bench.py --config papers100m --steps 200 --warmup 10 --epochs 1 > $out/bench_papers.json 2> $out/bench_papers.err
