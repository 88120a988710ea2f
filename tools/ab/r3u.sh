#!/bin/bash
out=gpurun_out/r3u; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_papers100m.py -q -x -m gpu > $out/papers_g4.log 2>&1; echo "rc=$?" >> $out/papers_g4.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_papers100m.py -q -x -m gpu -k "papers" > $out/papers_seq.log 2>&1; echo "rc=$?" >> $out/papers_seq.log
