#!/bin/bash
# A/B: layer-1 gather L2 policy by row multiplicity (GS_L1_MPOL), ShaDow hub-row hint (GS_BAL_HOT)
out=gpurun_out/r3b; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > $out/parity.log 2>&1; echo "rc=$?" >> $out/parity.log
for rep in 1 2; do
for v in 0 1 2 3; do
  GS_L1_MPOL=$v python bench.py --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_products.json 2>>$out/err; echo "products mpol=$v" >> $out/bench_products.tags
  GS_L1_MPOL=$v python bench.py --config reddit --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_reddit.json 2>>$out/err; echo "reddit mpol=$v" >> $out/bench_reddit.tags
done
done
for v in 0 64 128 256 512; do
  GS_BAL_HOT=$v python bench.py --config products_shadow --steps 20 --warmup 5 --no-cpu-baseline --epochs 1 >> $out/bench_shadow.json 2>>$out/err; echo "shadow hot=$v" >> $out/bench_shadow.tags
done
for v in 0 1 2; do
  GS_L1_MPOL=$v ncu --nvtx --nvtx-include "steps/" -k regex:k_agg_l1 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
     --cache-control none --clock-control none --csv --log-file $out/ncu_l1_mpol$v.csv python tools/profile_step.py --config products --steps 4 --graph > $out/ncu_l1_$v.log 2>&1
done
# GEMM component diagnostics (timings only; results are wrong under diag): 1 no C stores, 2 no MMAs, 4 no loads
for d in 0 1 2 4 6 7; do
  GS_GEMM_DIAG=$d ncu --nvtx --nvtx-include "steps/" -k regex:k_gemm --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum \
     --cache-control none --clock-control none --csv --log-file $out/ncu_gemm_diag$d.csv python tools/profile_step.py --config products --steps 1 --graph > $out/ncu_gemm_$d.log 2>&1
done
