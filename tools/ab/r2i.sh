#!/bin/bash
out=gpurun_out/r2i; mkdir -p $out
timeout 300 compute-sanitizer --tool memcheck python tools/debug_shadow.py tiny_sage_shadow > $out/memcheck.log 2>&1
for rep in 1 2; do
for v in "GS_L1_BULK=0" "GS_L1_BPS=3" "GS_L1_BULK=0 GS_LIB=paper_2403_17092_b200/libgnnstep_st2.so" "GS_L1_BPS=3 GS_LIB=paper_2403_17092_b200/libgnnstep_st2.so"; do
  env $v python bench.py --steps 400 --warmup 20 --no-cpu-baseline --epochs 3 >> $out/bench_ab.json 2>>$out/bench.err; echo "$v" >> $out/bench_ab.tags
done
done
