#!/bin/bash
# spmm_bwd hoisted loads, CE tile partials, 16-deep split reduce, stale-error clearing; ShaDow store policy
out=gpurun_out/r3d; mkdir -p $out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -m gpu > $out/parity.log 2>&1; echo "rc=$?" >> $out/parity.log
for rep in 1 2 3; do
  python bench.py --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_products.json 2>>$out/err; echo "products" >> $out/bench_products.tags
  GS_LIB=paper_2403_17092_b200/libgnnstep_base.so python bench.py --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_products.json 2>>$out/err; echo "products base" >> $out/bench_products.tags
done
for v in 0 1; do
  GS_BAL_SPOL=$v python bench.py --config products_shadow --steps 20 --warmup 5 --no-cpu-baseline --epochs 1 >> $out/bench_shadow.json 2>>$out/err; echo "shadow spol=$v" >> $out/bench_shadow.tags
done
ncu --nvtx --nvtx-include "steps/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --cache-control none --clock-control none --csv --log-file $out/launches_products_warm.csv python tools/profile_step.py --config products --steps 2 --graph > $out/ncu_warm.log 2>&1
