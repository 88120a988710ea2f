#!/bin/bash
# the fused last layer (k_last_layer) vs the tensor-core GEMM + CE epilogue + dgrad GEMM
out=gpurun_out/r3k; mkdir -p $out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_hub_rows.py tests/test_gpu_unified.py tests/test_gpu_exchange.py -q -x -m gpu > $out/parity.log 2>&1; echo "rc=$?" >> $out/parity.log
for rep in 1 2; do
for v in 0 1; do
  GS_LAST_FUSED=$v python bench.py --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_products.json 2>>$out/err; echo "products fused=$v" >> $out/bench_products.tags
  GS_LAST_FUSED=$v python bench.py --config reddit --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_reddit.json 2>>$out/err; echo "reddit fused=$v" >> $out/bench_reddit.tags
done
done
GS_LAST_FUSED=1 python bench.py --config products_shadow --steps 20 --warmup 5 --no-cpu-baseline --epochs 1 > $out/bench_shadow.json 2>>$out/err
ncu --nvtx --nvtx-include "steps/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --cache-control none --clock-control none --csv --log-file $out/launches_warm.csv python tools/profile_step.py --config products --steps 3 --graph > $out/ncu.log 2>&1
