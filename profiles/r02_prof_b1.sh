# full ncu captures of the batch-1 selective-layer kernels (outputs in gpurun_out/)
set -x
B="python bench.py --profile-only --batch 1 --steps 1 --warmup 1 --no-baselines --no-cpu-baseline"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm_t --launch-skip 20 --launch-count 2 -f -o gpurun_out/prof_t2_b1 $B > /dev/null 2>&1; echo t2=$?
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_gemm<" --launch-skip 30 --launch-count 2 -f -o gpurun_out/prof_single_b1 $B > /dev/null 2>&1; echo s=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_attn_tc --launch-skip 10 --launch-count 1 -f -o gpurun_out/prof_attn_b1 $B > /dev/null 2>&1; echo a=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_rmsnorm --launch-skip 20 --launch-count 1 -f -o gpurun_out/prof_norm_b1 $B > /dev/null 2>&1; echo n=$?
