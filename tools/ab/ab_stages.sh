mkdir -p gpurun_out/abg2
for st in 3 2; do
  python paper_2403_17092_b200/build.py --out /tmp/abg_$st/libgnnstep.so -DGS_TC_STAGES_WIDE=$st > /dev/null
done
for rep in 1 2; do
for st in 3 2; do
  GS_LIB=/tmp/abg_$st/libgnnstep.so python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/abg2/products_${st}_$rep.json 2>/dev/null
  GS_LIB=/tmp/abg_$st/libgnnstep.so python bench.py --config reddit --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/abg2/reddit_${st}_$rep.json 2>/dev/null
done
done
