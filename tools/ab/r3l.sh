#!/bin/bash
out=gpurun_out/r3l; mkdir -p $out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_hub_rows.py -q -x -m gpu -k "not shadow and not bf16" > $out/parity.log 2>&1; echo "rc=$?" >> $out/parity.log
for rep in 1 2; do
for v in 0 1; do
  GS_LAST_FUSED=$v python bench.py --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_products.json 2>>$out/err; echo "products fused=$v" >> $out/bench_products.tags
  GS_LAST_FUSED=$v python bench.py --config reddit --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_reddit.json 2>>$out/err; echo "reddit fused=$v" >> $out/bench_reddit.tags
done
done
ncu --nvtx --nvtx-include "steps/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --cache-control none --clock-control none --csv --log-file $out/launches_warm.csv python tools/profile_step.py --config products --steps 3 --graph > $out/ncu.log 2>&1
ncu --nvtx --nvtx-include "steps/" -k regex:k_last_layer --launch-count 1 --set full --import-source on \
    --cache-control none --clock-control none -o $out/last_layer python tools/profile_step.py --config products --steps 1 --graph > $out/ncu_last.log 2>&1
