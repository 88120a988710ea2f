#!/bin/bash
# One round-end measurement pass on a GPU box: the ncu launch list of the bench workload (and the
# per-class DRAM traffic it implies, read by bench.py), bench lines for every workload, one
# --set full capture of a step, sampling phase times and the random-gather ceiling.
set -u
out=${1:-gpurun_out/final}
mkdir -p "$out"
for c in products reddit products_shadow; do
    ncu --nvtx --nvtx-include "steps/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file "$out/launches_$c.csv" python tools/profile_step.py --config $c --steps 2 --graph \
        > "$out/ncu_l_$c.log" 2>&1
    python tools/ncu_traffic.py "$out/launches_$c.csv" $c > /dev/null
done
cp profiles/ncu_traffic.json "$out/ncu_traffic.json"
python bench.py > "$out/bench_products.json" 2> "$out/bench_products.err"
for c in reddit products_shadow products_gcn products_sage_shadow products_shadow_l5 tiny; do
    python bench.py --config $c --no-cpu-baseline > "$out/bench_$c.json" 2> "$out/bench_$c.err"
done
python bench.py --precision bf16 --no-cpu-baseline > "$out/bench_products_bf16.json" 2> "$out/bench_products_bf16.err"
python bench.py --impl reference --steps 2 --warmup 0 > "$out/bench_reference.json" 2> "$out/bench_reference.err"
ncu --nvtx --nvtx-include "steps/" --set full --import-source on --clock-control none -o "$out/step_full" \
    python tools/profile_step.py --config products --steps 1 --graph > "$out/ncu_full.log" 2>&1
python tools/phase_times.py products > "$out/phases_products.txt" 2>&1
python tools/phase_times.py products_shadow > "$out/phases_products_shadow.txt" 2>&1
python tools/gather_ceiling.py > "$out/gather_ceiling.txt" 2>&1
python bench.py --optimizer adam --no-cpu-baseline > "$out/bench_products_adam.json" 2> "$out/bench_products_adam.err"
