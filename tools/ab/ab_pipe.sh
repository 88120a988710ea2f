mkdir -p gpurun_out/abpipe
for rep in 1 2; do
for v in old new; do
  GS_LIB=abx/$v/libgnnstep.so python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/abpipe/products_${v}_$rep.json 2>/dev/null
  GS_LIB=abx/$v/libgnnstep.so python bench.py --config reddit --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/abpipe/reddit_${v}_$rep.json 2>/dev/null
done
done
