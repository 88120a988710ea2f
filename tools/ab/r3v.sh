#!/bin/bash
out=gpurun_out/r3v; mkdir -p $out
timeout 2400 python -m pytest tests -m gpu -q > $out/gpu_tests.log 2>&1; echo "rc=$?" >> $out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
