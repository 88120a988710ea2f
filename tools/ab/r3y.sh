#!/bin/bash
# GEMM pipelines small enough (2 wide / 3 narrow stages, <= 164 KB) to share an SM with a sampling block
out=gpurun_out/r3y; mkdir -p $out
for rep in 1 2; do
for v in "GS_LIB=paper_2403_17092_b200/libgnnstep.so" "GS_LIB=paper_2403_17092_b200/libgnnstep_st2.so"; do
  env $v python bench.py --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_products.json 2>>$out/err; echo "products $v" >> $out/bench_products.tags
  env $v python bench.py --config reddit --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_reddit.json 2>>$out/err; echo "reddit $v" >> $out/bench_reddit.tags
done
done
for v in "GS_LIB=paper_2403_17092_b200/libgnnstep.so" "GS_LIB=paper_2403_17092_b200/libgnnstep_st2.so"; do
  env $v python tools/timeline.py products 30 > "$out/timeline_$(basename ${v#GS_LIB=} .so).txt" 2>&1
done
