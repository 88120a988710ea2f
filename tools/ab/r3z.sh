#!/bin/bash
# GEMM tiles by cluster launch control (GS_GEMM_CLC=1), with the sampler on all / half the SMs
out=gpurun_out/r3z; mkdir -p $out
GS_GEMM_CLC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "tiny_epoch_training or determinism" > $out/parity.log 2>&1; echo "rc=$?" >> $out/parity.log
GS_GEMM_CLC=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -m gpu -k "training_parity and (products or reddit) and not gcn and not shadow" > $out/parity_full.log 2>&1; echo "rc=$?" >> $out/parity_full.log
for rep in 1 2; do
for v in "GS_GEMM_CLC=0" "GS_GEMM_CLC=1" "GS_GEMM_CLC=1 GS_SAMPLE_GRID=74" "GS_GEMM_CLC=1 GS_SAMPLE_GRID=111"; do
  env $v timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_products.json 2>>$out/err; echo "products $v" >> $out/bench_products.tags
done
done
for v in "GS_GEMM_CLC=0" "GS_GEMM_CLC=1"; do
  env $v timeout 300 python bench.py --config reddit --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_reddit.json 2>>$out/err; echo "reddit $v" >> $out/bench_reddit.tags
  env $v timeout 300 python tools/timeline.py products 30 > "$out/timeline_$(echo $v | tr ' =' '__').txt" 2>&1
done
