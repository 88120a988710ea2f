#!/bin/bash
out=gpurun_out/r2t; mkdir -p $out
GS_LIB=paper_2403_17092_b200/libgnnstep_st23.so python tools/timeline.py products 30 > $out/timeline_st23.txt 2>&1
python tools/timeline.py products 30 > $out/timeline_default.txt 2>&1
for rep in 1 2 3; do
for v in "GS_LIB=paper_2403_17092_b200/libgnnstep.so" "GS_LIB=paper_2403_17092_b200/libgnnstep_st23.so"; do
  env $v python bench.py --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_ab.json 2>>$out/bench.err; echo "products $v" >> $out/bench_ab.tags
done
done
for v in "GS_LIB=paper_2403_17092_b200/libgnnstep.so" "GS_LIB=paper_2403_17092_b200/libgnnstep_st23.so"; do
  env $v python bench.py --config reddit --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_ab.json 2>>$out/bench.err; echo "reddit $v" >> $out/bench_ab.tags
done
