mkdir -p gpurun_out/abp
for rep in 1 2; do
for p in default low high; do
  GS_SAMPLE_PRIO=$p python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/abp/products_${p}_$rep.json 2>/dev/null
  GS_SAMPLE_PRIO=$p python bench.py --config reddit --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/abp/reddit_${p}_$rep.json 2>/dev/null
done
done
