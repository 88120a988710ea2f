#!/bin/bash
# gather4 variants: 4 gather blocks per SM (GS_L1_BPS=4), later layers by gather4 (GS_AGG_G4=1)
out=gpurun_out/r3t; mkdir -p $out
GS_AGG_G4=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "tiny_epoch or determinism" > $out/parity.log 2>&1; echo "rc=$?" >> $out/parity.log
for rep in 1 2; do
for v in "GS_L1_G4=1" "GS_L1_BPS=4" "GS_AGG_G4=1" "GS_L1_BPS=4 GS_AGG_G4=1"; do
  env $v python bench.py --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_products.json 2>>$out/err; echo "products $v" >> $out/bench_products.tags
done
done
for v in "GS_L1_G4=1" "GS_AGG_G4=1"; do
  env $v python bench.py --config reddit --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_reddit.json 2>>$out/err; echo "reddit $v" >> $out/bench_reddit.tags
done
