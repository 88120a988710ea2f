#!/bin/bash
# dead-plane discard (GS_DISCARD) and bulk-copy gathers for every layer (GS_AGG_BULK_ALL)
out=gpurun_out/r3i; mkdir -p $out
GS_DISCARD=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -m gpu -k "tiny or products" > $out/parity_discard.log 2>&1; echo "rc=$?" >> $out/parity_discard.log
for rep in 1 2; do
for v in "GS_DISCARD=0" "GS_DISCARD=1" "GS_AGG_BULK_ALL=1"; do
  env $v python bench.py --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_products.json 2>>$out/err; echo "products $v" >> $out/bench_products.tags
  env $v python bench.py --config reddit --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_reddit.json 2>>$out/err; echo "reddit $v" >> $out/bench_reddit.tags
done
done
for v in 0 1; do
GS_DISCARD=$v ncu --nvtx --nvtx-include "steps/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --cache-control none --clock-control none --csv --log-file $out/launches_warm_discard$v.csv python tools/profile_step.py --config products --steps 3 --graph > $out/ncu_warm$v.log 2>&1
done
