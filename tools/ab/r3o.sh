#!/bin/bash
# sampling kernel on fewer SMs (GS_SAMPLE_GRID) x dynamic GEMM tiles (GS_GEMM_DYN)
out=gpurun_out/r3o; mkdir -p $out
GS_SAMPLE_GRID=74 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -m gpu -k "tiny or sampling" > $out/parity.log 2>&1; echo "rc=$?" >> $out/parity.log
for rep in 1 2; do
for v in "GS_SAMPLE_GRID=148" "GS_SAMPLE_GRID=74" "GS_SAMPLE_GRID=74 GS_GEMM_DYN=1" "GS_SAMPLE_GRID=111 GS_GEMM_DYN=1" "GS_SAMPLE_GRID=37 GS_GEMM_DYN=1"; do
  env $v python bench.py --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_products.json 2>>$out/err; echo "products $v" >> $out/bench_products.tags
done
done
for v in "GS_SAMPLE_GRID=148" "GS_SAMPLE_GRID=74 GS_GEMM_DYN=1"; do
  env $v python bench.py --config reddit --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_reddit.json 2>>$out/err; echo "reddit $v" >> $out/bench_reddit.tags
  env $v python tools/timeline.py products 30 > "$out/timeline_$(echo $v | tr ' =' '__').txt" 2>&1
done
