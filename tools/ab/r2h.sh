#!/bin/bash
out=gpurun_out/r2h; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "grid or tiny_epoch_training or hub" > $out/parity.log 2>&1; echo rc=$? >> $out/parity.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -s -k "shadow or products" > $out/parity_full.log 2>&1; echo rc=$? >> $out/parity_full.log
for rep in 1 2; do
for v in "GS_L1_BULK=0" "GS_L1_BPS=3" "GS_L1_BPS=3 GS_L1_DYN=0" "GS_L1_BPS=4"; do
  env $v python bench.py --steps 400 --warmup 20 --no-cpu-baseline --epochs 3 >> $out/bench_ab.json 2>>$out/bench.err; echo "$v" >> $out/bench_ab.tags
done
done
for v in "" "GS_RF_COMPACT=0"; do
  env $v python bench.py --config products_shadow --steps 30 --warmup 5 --no-cpu-baseline --epochs 0 >> $out/bench_shadow.json 2>>$out/bench.err; echo "$v" >> $out/bench_shadow.tags
done
