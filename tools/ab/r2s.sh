#!/bin/bash
out=gpurun_out/r2s; mkdir -p $out
GS_AGG_BULK_ALL=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "tiny_epoch_training or (training_parity and products) or (training_parity and reddit)" > $out/parity_all.log 2>&1; echo rc=$? >> $out/parity_all.log
for rep in 1 2; do
for c in products reddit; do
for v in "GS_AGG_BULK_ALL=0" "GS_AGG_BULK_ALL=1"; do
  env $v python bench.py --config $c --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_ab.json 2>>$out/bench.err; echo "$c $v" >> $out/bench_ab.tags
done
done
done
