#!/bin/bash
# Round-2b measurement pass on one B200: full -m gpu suite, smoke, ncu launch lists (cold and
# warm), bench lines for every workload, the reference arm, the Unified protocol, a --set full
# capture of a products step, sampling phases, timeline, gather ceiling.
set -u
out=${1:-gpurun_out/final3}
mkdir -p "$out"
timeout 2400 python -m pytest tests -m gpu -q > "$out/gpu_tests.log" 2>&1; echo "rc=$?" >> "$out/gpu_tests.log"
python -c "import __graft_entry__ as g; g.smoke()" > "$out/smoke.log" 2>&1
for c in products reddit products_shadow; do
    ncu --nvtx --nvtx-include "steps/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file "$out/launches_$c.csv" python tools/profile_step.py --config $c --steps 2 --graph \
        > "$out/ncu_l_$c.log" 2>&1
    python tools/ncu_traffic.py "$out/launches_$c.csv" $c > /dev/null
done
ncu --nvtx --nvtx-include "steps/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --cache-control none --clock-control none --csv --log-file "$out/launches_products_warm.csv" \
    python tools/profile_step.py --config products --steps 2 --graph > "$out/ncu_warm.log" 2>&1
cp profiles/ncu_traffic.json "$out/ncu_traffic.json"
python bench.py > "$out/bench_products.json" 2> "$out/bench_products.err"
python bench.py --steps 400 --warmup 20 > "$out/bench_products_long.json" 2> "$out/bench_products_long.err"
for c in reddit products_shadow products_gcn products_sage_shadow products_shadow_l5 tiny papers100m; do
    python bench.py --config $c --no-cpu-baseline > "$out/bench_$c.json" 2> "$out/bench_$c.err"
done
python bench.py --precision bf16 --no-cpu-baseline > "$out/bench_products_bf16.json" 2> "$out/bench_products_bf16.err"
python bench.py --optimizer adam --no-cpu-baseline > "$out/bench_products_adam.json" 2> "$out/bench_products_adam.err"
python bench.py --impl reference --steps 2 --warmup 0 > "$out/bench_reference.json" 2> "$out/bench_reference.err"
timeout 900 python tools/unified_bench.py products 10 > "$out/unified_products.json" 2> "$out/unified_products.err"
ncu --nvtx --nvtx-include "steps/" --set full --import-source on --clock-control none -o "$out/step_full" \
    python tools/profile_step.py --config products --steps 1 --graph > "$out/ncu_full.log" 2>&1
python tools/phase_times.py products > "$out/phases_products.txt" 2>&1
python tools/timeline.py products 30 > "$out/timeline_products.txt" 2>&1
python tools/gather_ceiling.py > "$out/gather_ceiling.txt" 2>&1
# compute-sanitizer is closed on this pool since round 2's pass (profiles/r2/sanitize_*.log hold
# the memcheck / racecheck / synccheck runs of tools/sanitize.py)
