mkdir -p gpurun_out/abs2
for t in 512 384 256; do
  python paper_2403_17092_b200/build.py --out /tmp/abs_$t/libgnnstep.so -DGS_SAMPLE_THREADS=$t > /dev/null
done
for rep in 1 2; do
for t in 512 384 256; do
  GS_LIB=/tmp/abs_$t/libgnnstep.so python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/abs2/products_${t}_$rep.json 2>/dev/null
done
GS_LIB=/tmp/abs_$t/libgnnstep.so python bench.py --config reddit --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/abs2/reddit_256_$rep.json 2>/dev/null
GS_LIB=/tmp/abs_512/libgnnstep.so python bench.py --config reddit --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/abs2/reddit_512_$rep.json 2>/dev/null
done
