#!/bin/bash
out=gpurun_out/r2d; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_exchange.py -x -q -s > $out/exchange.log 2>&1; echo rc=$? >> $out/exchange.log
for rep in 1 2; do
for v in "GS_L1_BULK=0" "GS_L1_BPS=3" "GS_L1_BPS=4"; do
  env $v python bench.py --steps 400 --warmup 20 --no-cpu-baseline --epochs 5 >> $out/bench_ab.json 2>>$out/bench.err; echo "$v" >> $out/bench_ab.tags
done
done
python bench.py --config products_gcn --steps 200 --warmup 20 --no-cpu-baseline --epochs 2 > $out/bench_gcn.json 2>>$out/bench.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $out/launches_shadow.csv python tools/profile_step.py --config products_shadow --steps 1 --graph > $out/ncu_l.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_papers100m.py -x -q -s > $out/papers.log 2>&1; echo rc=$? >> $out/papers.log
