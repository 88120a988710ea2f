#!/bin/bash
# dynamic GEMM tile scheduler (GS_GEMM_DYN) x layer-1 gather on the sampler (GS_L1_ON_SAMPLER)
out=gpurun_out/r3g; mkdir -p $out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -m gpu -k "not bf16 and not shadow" > $out/parity.log 2>&1; echo "rc=$?" >> $out/parity.log
for rep in 1 2; do
for dyn in 0 1; do
for l1s in 0 1; do
  GS_GEMM_DYN=$dyn GS_L1_ON_SAMPLER=$l1s python bench.py --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_products.json 2>>$out/err; echo "products dyn=$dyn l1s=$l1s" >> $out/bench_products.tags
done
done
done
for dyn in 0 1; do
for l1s in 0 1; do
  GS_GEMM_DYN=$dyn GS_L1_ON_SAMPLER=$l1s python bench.py --config reddit --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_reddit.json 2>>$out/err; echo "reddit dyn=$dyn l1s=$l1s" >> $out/bench_reddit.tags
done
done
GS_GEMM_DYN=1 GS_L1_ON_SAMPLER=1 python tools/timeline.py products 30 > $out/timeline_dyn_l1s.txt 2>&1
bash tools/r3f.sh
