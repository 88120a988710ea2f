#!/bin/bash
out=gpurun_out/r3q; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "fused or determinism" > $out/parity.log 2>&1; echo "rc=$?" >> $out/parity.log
GS_LAST_FUSED=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -m gpu -k "training_parity and (products or reddit) and not gcn and not shadow" > $out/parity_full.log 2>&1; echo "rc=$?" >> $out/parity_full.log
for rep in 1 2; do
for v in 0 1; do
  GS_LAST_FUSED=$v python bench.py --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_products.json 2>>$out/err; echo "products fused=$v" >> $out/bench_products.tags
done
done
for v in 0 1; do
  GS_LAST_FUSED=$v python bench.py --config reddit --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_reddit.json 2>>$out/err; echo "reddit fused=$v" >> $out/bench_reddit.tags
done
GS_LAST_FUSED=1 ncu --nvtx --nvtx-include "steps/" -k regex:k_last_layer --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file $out/last.csv python tools/profile_step.py --config products --steps 3 --graph > $out/ncu.log 2>&1
