# A/B: sampling-kernel block size (1024: the whole register file, nothing co-resides; 512: half,
# so training kernels can share the SMs while the next batch is sampled)
mkdir -p gpurun_out/abs
for t in 1024 512; do
  python paper_2403_17092_b200/build.py --out /tmp/abs_$t/libgnnstep.so -DGS_SAMPLE_THREADS=$t > /dev/null
done
for rep in 1 2; do
for t in 1024 512; do
  GS_LIB=/tmp/abs_$t/libgnnstep.so python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/abs/products_${t}_$rep.json 2>/dev/null
  GS_LIB=/tmp/abs_$t/libgnnstep.so python bench.py --config products_shadow --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/abs/shadow_${t}_$rep.json 2>/dev/null
done
done
GS_LIB=/tmp/abs_512/libgnnstep.so timeout 900 python -m pytest tests -m gpu -x -q -k "tiny_sampling or fullsize_sampling" > gpurun_out/abs/pytest_512.log 2>&1
