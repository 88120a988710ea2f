# A/B: neighbour rows in flight per warp in the layer-1 gather (k_agg_sage, CPL = 1)
mkdir -p gpurun_out/ab
for u in 4 8 16; do
  python paper_2403_17092_b200/build.py --out /tmp/ab_$u/libgnnstep.so -DGS_AGGU1=$u > /dev/null
done
for rep in 1 2; do
for u in 4 8 16; do
  GS_LIB=/tmp/ab_$u/libgnnstep.so python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab/aggu_${u}_$rep.json 2>/dev/null
done
done
