mkdir -p gpurun_out/diag
for d in 0 1 2 4 7; do
  GS_GEMM_DIAG=$d ncu --nvtx --nvtx-include "steps/" --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/diag/l_$d.csv python tools/profile_step.py --config products --steps 1 --graph > gpurun_out/diag/log_$d.txt 2>&1
done
GS_GEMM_DIAG=0 ncu --nvtx --nvtx-include "steps/" --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/diag/l_warm.csv python tools/profile_step.py --config products --steps 1 --graph > gpurun_out/diag/log_warm.txt 2>&1
