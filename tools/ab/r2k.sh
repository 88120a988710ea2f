#!/bin/bash
out=gpurun_out/r2k; mkdir -p $out
GS_L1_BULK=0 python tools/timeline.py products 30 > $out/timeline_old.txt 2>&1
GS_L1_BPS=3 python tools/timeline.py products 30 > $out/timeline_bulk.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 24 -c 8 -o $out/gemm python tools/profile_step.py --config products --steps 2 --graph > $out/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_spmm_bwd -s 6 -c 2 -o $out/spmm python tools/profile_step.py --config products --steps 2 --graph > $out/ncu_spmm.log 2>&1
