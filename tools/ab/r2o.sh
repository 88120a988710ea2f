#!/bin/bash
# GEMM diagnostics: per-launch durations with parts of the GEMM disabled (GS_GEMM_DIAG bits:
# 1 skip C stores, 2 skip MMAs, 4 skip loads, 8 skip the CE epilogue, 16 skip the loss sum)
out=gpurun_out/r2o; mkdir -p $out
for d in 0 1 2 4 6 7; do
  GS_GEMM_DIAG=$d ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_gemm_tc --csv --log-file $out/gemm_diag$d.csv python tools/profile_step.py --config products --steps 2 --graph > $out/diag$d.log 2>&1
done
for c in reddit products_shadow; do
  python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline --epochs 1 >> $out/bench.json 2>>$out/bench.err; echo "$c" >> $out/bench.tags
done
