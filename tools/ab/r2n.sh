#!/bin/bash
out=gpurun_out/r2n; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q -k "tiny_epoch_training or sharded" > $out/parity.log 2>&1; echo rc=$? >> $out/parity.log
for rep in 1 2; do
for c in reddit products_gcn products; do
for v in "GS_SAMPLE_PRIO=default" "GS_SAMPLE_PRIO=low"; do
  env $v python bench.py --config $c --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_ab.json 2>>$out/bench.err; echo "$c $v" >> $out/bench_ab.tags
done
done
done
