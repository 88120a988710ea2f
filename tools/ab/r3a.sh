#!/bin/bash
# Session re-entry confirmation: GPU suite, smoke, bench products + reddit + shadow.
out=gpurun_out/r3a; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -x > $out/gpu_tests.log 2>&1; echo "rc=$?" >> $out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
python bench.py > $out/bench_products.json 2> $out/bench_products.err
python bench.py --config reddit --no-cpu-baseline > $out/bench_reddit.json 2> $out/bench_reddit.err
python bench.py --config products_shadow --no-cpu-baseline > $out/bench_shadow.json 2> $out/bench_shadow.err
python tools/profile_step.py --config products --steps 20 --graph > $out/profile_products.txt 2>&1
