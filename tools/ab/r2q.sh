#!/bin/bash
out=gpurun_out/r2q; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -s -k "gcn" > $out/parity.log 2>&1; echo rc=$? >> $out/parity.log
for rep in 1 2; do
  python bench.py --config products_gcn --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench.json 2>>$out/bench.err; echo "gcn" >> $out/bench.tags
done
python tools/phase_times.py products_gcn > $out/phases_gcn.txt 2>&1
