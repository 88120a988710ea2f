#!/bin/bash
# source-range passes of the layer-1 gather (GS_L1_PASSES), CE tile partials, 16-deep split reduce
out=gpurun_out/r3c; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -m gpu > $out/parity.log 2>&1; echo "rc=$?" >> $out/parity.log
for rep in 1 2; do
for v in 1 2 3 4; do
  GS_L1_PASSES=$v python bench.py --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_products.json 2>>$out/err; echo "products passes=$v" >> $out/bench_products.tags
done
done
for v in 1 3; do
  GS_L1_PASSES=$v python bench.py --config papers100m --steps 100 --warmup 10 --no-cpu-baseline --epochs 1 >> $out/bench_papers.json 2>>$out/err; echo "papers passes=$v" >> $out/bench_papers.tags
done
python bench.py --config products_shadow --steps 10 --warmup 3 --no-cpu-baseline --epochs 0 > $out/bench_shadow.json 2>>$out/err
for v in 1 2 3 4; do
  GS_L1_PASSES=$v ncu --nvtx --nvtx-include "steps/" -k regex:k_agg_l1 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
     --cache-control none --clock-control none --csv --log-file $out/ncu_l1_p$v.csv python tools/profile_step.py --config products --steps 3 --graph > $out/ncu_l1_$v.log 2>&1
done
ncu --nvtx --nvtx-include "steps/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --cache-control none --clock-control none --csv --log-file $out/launches_products_warm.csv python tools/profile_step.py --config products --steps 2 --graph > $out/ncu_warm.log 2>&1
