#!/bin/bash
out=gpurun_out/r3h; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_unified.py -q -x -m gpu > $out/unified_test.log 2>&1; echo "rc=$?" >> $out/unified_test.log
timeout 900 python tools/unified_bench.py products 10 > $out/unified_products.json 2> $out/unified_products.err
timeout 600 python tools/unified_bench.py tiny 50 > $out/unified_tiny.json 2> $out/unified_tiny.err
