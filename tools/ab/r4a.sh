#!/bin/bash
# the self row inside the first gather4 group (4 copy instructions per 15-neighbour row instead of 5)
out=gpurun_out/r4a; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -m gpu -k "tiny_epoch or determinism or (training_parity and (products or papers_small) and not gcn and not shadow)" > $out/parity.log 2>&1; echo "rc=$?" >> $out/parity.log
for rep in 1 2 3; do
for v in "GS_LIB=paper_2403_17092_b200/libgnnstep_g4a.so" "GS_LIB=paper_2403_17092_b200/libgnnstep.so"; do
  env $v python bench.py --steps 300 --warmup 20 --no-cpu-baseline --epochs 2 >> $out/bench_products.json 2>>$out/err; echo "products $v" >> $out/bench_products.tags
done
done
for v in "GS_LIB=paper_2403_17092_b200/libgnnstep_g4a.so" "GS_LIB=paper_2403_17092_b200/libgnnstep.so"; do
  env $v ncu --nvtx --nvtx-include "steps/" -k regex:k_agg_l1 --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file $out/l1_$(basename ${v#GS_LIB=} .so).csv python tools/profile_step.py --config products --steps 3 --graph > $out/ncu.log 2>&1
done
