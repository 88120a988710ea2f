#!/bin/bash
out=gpurun_out/r2e; mkdir -p $out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "tiny_epoch_training or hub_row" > $out/parity.log 2>&1; echo rc=$? >> $out/parity.log
for rep in 1 2; do
for v in "GS_L1_BULK=0" "GS_L1_BULK=0 GS_AGG_DUMMY_SMEM=59000" "GS_L1_BPS=3" "GS_L1_BPS=3 GS_L1_PDL=0" "GS_L1_BPS=4 GS_L1_PDL=0" "GS_L1_BPS=3 GS_L1_APOL=1"; do
  env $v python bench.py --steps 400 --warmup 20 --no-cpu-baseline --epochs 3 --no-overlap >> $out/bench_ab.json 2>>$out/bench.err; echo "$v no-overlap" >> $out/bench_ab.tags
done
done
for v in "GS_L1_BULK=0" "GS_L1_BPS=3" "GS_L1_BPS=3 GS_L1_PDL=0"; do
  env $v python bench.py --steps 400 --warmup 20 --no-cpu-baseline --epochs 3 >> $out/bench_ab.json 2>>$out/bench.err; echo "$v overlap" >> $out/bench_ab.tags
done
