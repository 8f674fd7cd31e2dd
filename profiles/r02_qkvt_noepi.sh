# transposed QKV / SwiGLU at batch 1 (RC_GEMM_T=2): launch times with and without the epilogue
# (RC_GEMM_NOEPI=1, diagnostics: outputs not written) to split main loop from epilogue cost
set -x
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
B="python bench.py --profile-only --batch 1 --steps 1 --warmup 1 --no-baselines --no-cpu-baseline --pools random"
RC_GEMM_T=2 timeout 600 ncu --metrics $M --clock-control none -k "regex:k_gemm" --csv --log-file gpurun_out/ne_t2.csv $B > /dev/null 2>&1; echo a=$?
RC_GEMM_T=2 RC_GEMM_NOEPI=1 timeout 600 ncu --metrics $M --clock-control none -k "regex:k_gemm" --csv --log-file gpurun_out/ne_t2_noepi.csv $B > /dev/null 2>&1; echo b=$?
