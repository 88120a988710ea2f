#!/bin/bash
out=gpurun_out/r2r; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_sharded.py -x -q -s -k "reddit" > $out/parity.log 2>&1; echo rc=$? >> $out/parity.log
for rep in 1 2; do
for v in "GS_L1_STREAM=0 GS_SAMPLE_AFTER_L1=0" "GS_L1_STREAM=1 GS_SAMPLE_AFTER_L1=0" "GS_L1_STREAM=1 GS_SAMPLE_AFTER_L1=1"; do
  env $v python bench.py --config reddit --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_ab.json 2>>$out/bench.err; echo "$v" >> $out/bench_ab.tags
done
done
