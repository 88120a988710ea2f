mkdir -p gpurun_out/aba
for m in 1 4 6; do
  python paper_2403_17092_b200/build.py --out /tmp/aba_$m/libgnnstep.so -DGS_AGG_MINB=$m > /dev/null
done
for rep in 1 2; do
for m in 1 4 6; do
  GS_LIB=/tmp/aba_$m/libgnnstep.so python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/aba/products_${m}_$rep.json 2>/dev/null
  GS_LIB=/tmp/aba_$m/libgnnstep.so python bench.py --config reddit --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/aba/reddit_${m}_$rep.json 2>/dev/null
done
done
