# A/B at batch 1: every eligible small-M GEMM on the transposed pair kernel (RC_GEMM_T=2) vs the default
set -x
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
B="python bench.py --profile-only --batch 1 --steps 1 --warmup 1 --no-baselines --no-cpu-baseline --pools random"
RC_GEMM_T=2 timeout 1500 ncu --metrics $M --clock-control none -k "regex:k_gemm" --csv --log-file gpurun_out/launches_b1_t2.csv $B > /dev/null 2>&1; echo l2=$?
timeout 1500 ncu --metrics $M --clock-control none -k "regex:k_gemm" --csv --log-file gpurun_out/launches_b1_t0.csv $B > /dev/null 2>&1; echo l0=$?
timeout 300 python bench.py --batch 1 --steps 30 --no-baselines --no-cpu-baseline > gpurun_out/ab_t_def.log 2>&1; echo d=$?
RC_GEMM_T=2 timeout 300 python bench.py --batch 1 --steps 30 --no-baselines --no-cpu-baseline > gpurun_out/ab_t_2.log 2>&1; echo t2=$?
