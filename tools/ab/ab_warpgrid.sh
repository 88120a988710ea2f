mkdir -p gpurun_out/abw
for w in 16 6 4 3; do
  python paper_2403_17092_b200/build.py --out /tmp/abw_$w/libgnnstep.so -DGS_WARP_GRID_PER_SM=$w > /dev/null
done
for rep in 1 2; do
for w in 16 6 4 3; do
  GS_LIB=/tmp/abw_$w/libgnnstep.so python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/abw/products_${w}_$rep.json 2>/dev/null
  GS_LIB=/tmp/abw_$w/libgnnstep.so python bench.py --config reddit --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/abw/reddit_${w}_$rep.json 2>/dev/null
done
done
GS_LIB=/tmp/abw_16/libgnnstep.so python bench.py --config products_shadow --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/abw/shadow_16.json 2>/dev/null
GS_LIB=/tmp/abw_4/libgnnstep.so python bench.py --config products_shadow --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/abw/shadow_4.json 2>/dev/null
