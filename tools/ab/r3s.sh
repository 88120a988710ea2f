#!/bin/bash
# layer-1 gather with TMA tile::gather4 (GS_L1_G4=1)
out=gpurun_out/r3s; mkdir -p $out
GS_L1_G4=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -m gpu -k "tiny_epoch or determinism or (training_parity and (products or papers_small) and not gcn and not shadow)" > $out/parity.log 2>&1; echo "rc=$?" >> $out/parity.log
for rep in 1 2; do
for v in 0 1; do
  GS_L1_G4=$v python bench.py --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_products.json 2>>$out/err; echo "products g4=$v" >> $out/bench_products.tags
done
done
for v in 0 1; do
  GS_L1_G4=$v python bench.py --config papers100m --steps 100 --warmup 10 --no-cpu-baseline --epochs 1 >> $out/bench_papers.json 2>>$out/err; echo "papers g4=$v" >> $out/bench_papers.tags
  GS_L1_G4=$v ncu --nvtx --nvtx-include "steps/" -k regex:k_agg_l1 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
     --cache-control none --clock-control none --csv --log-file $out/l1_g4$v.csv python tools/profile_step.py --config products --steps 3 --graph > $out/ncu$v.log 2>&1
done
