#!/bin/bash
# source-level ncu captures of the GEMM launches of a products step (fwd layer 1, CE, wgrad layer 1)
out=gpurun_out/r3f; mkdir -p $out
for k in 0 2 7; do
  ncu --nvtx --nvtx-include "steps/" -k regex:k_gemm_tc --launch-skip $k --launch-count 1 --set full --import-source on \
      --cache-control none --clock-control none -o $out/gemm_$k python tools/profile_step.py --config products --steps 1 --graph > $out/ncu_$k.log 2>&1
done
ncu --nvtx --nvtx-include "steps/" -k regex:k_agg_l1 --launch-count 1 --set full --import-source on \
    --cache-control none --clock-control none -o $out/agg_l1 python tools/profile_step.py --config products --steps 1 --graph > $out/ncu_l1.log 2>&1
