#!/bin/bash
# bulk-copy layer-1 gather: parity + A/B + one ncu capture
out=gpurun_out/r2b; mkdir -p $out
free -g > $out/host.txt; nproc >> $out/host.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "tiny_epoch_training or bf16 or train_epoch or host_seeds or prefetched or drops_schedule or exchange" > $out/parity_tiny.log 2>&1; echo rc=$? >> $out/parity_tiny.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -s -k "products or papers_small" > $out/parity_full.log 2>&1; echo rc=$? >> $out/parity_full.log
for v in "GS_L1_BULK=1 GS_L1_NB=2" "GS_L1_BULK=0" "GS_L1_BULK=1 GS_L1_NB=3" "GS_L1_BULK=1 GS_L1_NB=2"; do
  env $v python bench.py --steps 60 --no-cpu-baseline --epochs 0 >> $out/bench_ab.json 2>>$out/bench.err; echo "$v" >> $out/bench_ab.tags
done
ncu --set full --clock-control none --import-source on -k regex:k_agg_l1_bulk -s 6 -c 1 -o $out/l1bulk python tools/profile_step.py --config products --steps 2 > $out/ncu.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $out/launches.csv python tools/profile_step.py --config products --steps 2 --graph > $out/ncu_l.log 2>&1
