mkdir -p gpurun_out/cediag
for d in 0 1 2 4 8 16 31; do
  GS_GEMM_DIAG=$d ncu --nvtx --nvtx-include "steps/" -k regex:k_gemm_tc --metrics gpu__time_duration.sum,sm__cycles_active.max --clock-control none --csv --log-file gpurun_out/cediag/l_$d.csv python tools/profile_step.py --config products --steps 1 --graph > /dev/null 2>&1
done
for d in 0 31; do
  GS_GEMM_DIAG=$d ncu --nvtx --nvtx-include "steps/" -k regex:k_gemm_tc --cache-control none --metrics gpu__time_duration.sum,sm__cycles_active.max --clock-control none --csv --log-file gpurun_out/cediag/w_$d.csv python tools/profile_step.py --config products --steps 1 --graph > /dev/null 2>&1
done
