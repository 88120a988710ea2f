mkdir -p gpurun_out/abr
for m in 2 3 4; do
  python paper_2403_17092_b200/build.py --out /tmp/abr_$m/libgnnstep.so -DGS_SAMPLE_MINB=$m > /dev/null
done
for rep in 1 2; do
for m in 2 3 4; do
  GS_LIB=/tmp/abr_$m/libgnnstep.so python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/abr/products_${m}_$rep.json 2>/dev/null
  GS_LIB=/tmp/abr_$m/libgnnstep.so python bench.py --config reddit --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/abr/reddit_${m}_$rep.json 2>/dev/null
done
done
