#!/bin/bash
out=gpurun_out/r2c; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_exchange.py -x -q -s > $out/exchange.log 2>&1; echo rc=$? >> $out/exchange.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "train_epoch or host_seeds or prefetched or drops_schedule or exchange or hub_row" > $out/parity_tiny.log 2>&1; echo rc=$? >> $out/parity_tiny.log
for v in "GS_L1_BULK=0" "GS_L1_BPS=3" "GS_L1_BPS=4" "GS_L1_BPS=2" "GS_L1_BPS=0"; do
  env $v python bench.py --steps 60 --no-cpu-baseline --epochs 3 >> $out/bench_ab.json 2>>$out/bench.err; echo "$v" >> $out/bench_ab.tags
done
for v in "GS_L1_BULK=0" "GS_L1_BPS=3"; do
  env $v python bench.py --steps 60 --no-cpu-baseline --epochs 0 --no-overlap >> $out/bench_ab.json 2>>$out/bench.err; echo "$v no-overlap" >> $out/bench_ab.tags
done
ncu --set full --clock-control none --import-source on -k regex:k_agg_l1_bulk -s 2 -c 1 -o $out/l1bulk python tools/profile_step.py --config products --steps 2 --graph > $out/ncu.log 2>&1
