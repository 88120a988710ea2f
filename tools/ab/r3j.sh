#!/bin/bash
# L2 residency of the operand planes the next GEMM reads: A1 stores evict_last (GS_L1_APOL=2),
# dPre stores of the backward aggregation evict_last (GS_SPMM_SPOL=1)
out=gpurun_out/r3j; mkdir -p $out
for rep in 1 2; do
for v in "GS_L1_APOL=0" "GS_L1_APOL=2" "GS_SPMM_SPOL=1" "GS_L1_APOL=2 GS_SPMM_SPOL=1"; do
  env $v python bench.py --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_products.json 2>>$out/err; echo "products $v" >> $out/bench_products.tags
done
done
for v in "GS_L1_APOL=0" "GS_L1_APOL=2 GS_SPMM_SPOL=1"; do
env $v ncu --nvtx --nvtx-include "steps/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --cache-control none --clock-control none --csv --log-file "$out/launches_warm_$(echo $v | tr ' =' '__').csv" python tools/profile_step.py --config products --steps 3 --graph > $out/ncu.log 2>&1
done
