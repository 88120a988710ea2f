#!/bin/bash
# layer-1 gather on the sampling stream (GS_L1_ON_SAMPLER): parity + A/B
out=gpurun_out/r3e; mkdir -p $out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -m gpu -k "l1_on_sampler or tiny_epoch" > $out/parity.log 2>&1; echo "rc=$?" >> $out/parity.log
for rep in 1 2; do
for v in 0 1; do
  GS_L1_ON_SAMPLER=$v python bench.py --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_products.json 2>>$out/err; echo "products l1s=$v" >> $out/bench_products.tags
  GS_L1_ON_SAMPLER=$v python bench.py --config reddit --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_reddit.json 2>>$out/err; echo "reddit l1s=$v" >> $out/bench_reddit.tags
done
done
for v in 0 1; do
  GS_L1_ON_SAMPLER=$v python bench.py --config papers100m --steps 100 --warmup 10 --no-cpu-baseline --epochs 1 >> $out/bench_papers.json 2>>$out/err; echo "papers l1s=$v" >> $out/bench_papers.tags
  GS_L1_ON_SAMPLER=$v GS_TIMELINE=1 python tools/timeline.py products 30 > $out/timeline_l1s$v.txt 2>&1
done
