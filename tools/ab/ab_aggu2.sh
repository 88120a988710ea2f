mkdir -p gpurun_out/ab2
for u in 4 2 6; do
  python paper_2403_17092_b200/build.py --out /tmp/ab2_$u/libgnnstep.so -DGS_AGGU2=$u > /dev/null
done
for rep in 1 2; do
for u in 4 2 6; do
  GS_LIB=/tmp/ab2_$u/libgnnstep.so python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/ab2/products_${u}_$rep.json 2>/dev/null
done
done
