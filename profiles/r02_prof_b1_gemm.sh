# full ncu captures of the batch-1 selective-layer GEMMs (default: single-CTA SwiGLU / QKV, transposed
# residuals; RC_GEMM_T=2: transposed SwiGLU / QKV) for the stall / pipe analysis (outputs in gpurun_out/)
set -x
B="python bench.py --profile-only --batch 1 --steps 1 --warmup 1 --no-baselines --no-cpu-baseline --pools random"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm --launch-skip 24 --launch-count 8 -f -o gpurun_out/prof_gemm_b1 $B > /dev/null 2>&1; echo d=$?
RC_GEMM_T=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm --launch-skip 24 --launch-count 8 -f -o gpurun_out/prof_gemm_b1_t2 $B > /dev/null 2>&1; echo t2=$?
