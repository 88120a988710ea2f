mkdir -p gpurun_out/abb
python paper_2403_17092_b200/build.py --out /tmp/abb_d/libgnnstep.so > /dev/null
for m in 3 4; do
  python paper_2403_17092_b200/build.py --out /tmp/abb_$m/libgnnstep.so -DGS_BAL_MINB=$m > /dev/null
done
for v in d 3 4; do
  GS_LIB=/tmp/abb_$v/libgnnstep.so python bench.py --config products_shadow --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/abb/shadow_$v.json 2>/dev/null
  GS_LIB=/tmp/abb_$v/libgnnstep.so python bench.py --config products_sage_shadow --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/abb/sage_shadow_$v.json 2>/dev/null
done
