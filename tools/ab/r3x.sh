#!/bin/bash
out=gpurun_out/r3x; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_hub_rows.py tests/test_gpu_papers100m.py -q -x -m gpu > $out/hub_then_papers.log 2>&1; echo "rc=$?" >> $out/hub_then_papers.log
timeout 2400 python -m pytest tests -m gpu -q > $out/gpu_tests.log 2>&1; echo "rc=$?" >> $out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
bash tools/ab/r3w.sh
