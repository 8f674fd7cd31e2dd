# A/B at batch 1: split-K cap of the transposed residual GEMMs (RC_GEMM_T_SPLITS)
set -x
for sp in 16 2 1; do
  RC_GEMM_T_SPLITS=$sp timeout 300 python bench.py --batch 1 --steps 30 --no-baselines --no-cpu-baseline > gpurun_out/ab_sp$sp.log 2>&1; echo sp$sp=$?
done
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
B="python bench.py --profile-only --batch 1 --steps 1 --warmup 1 --no-baselines --no-cpu-baseline --pools random"
for sp in 16 2 1; do
  RC_GEMM_T_SPLITS=$sp timeout 900 ncu --metrics $M --clock-control none -k "regex:k_gemm_t" --csv --log-file gpurun_out/launches_tsp$sp.csv $B > /dev/null 2>&1; echo l$sp=$?
done
