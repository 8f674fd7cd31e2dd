# ncu --set full of one selective-layer attention launch at batch 32 (paired) and batch 1 (single tile), random
# pools (no materialisation launches before the steps); plus the full-size GPU tests on materialised pools
set -x
B="python bench.py --profile-only --steps 1 --warmup 1 --no-baselines --no-cpu-baseline --pools random"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_attn_pair --launch-skip 40 --launch-count 1 -f -o gpurun_out/prof_attn_pair_b32 $B > /dev/null 2>&1; echo a32=$?
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_attn_tc --launch-skip 40 --launch-count 1 -f -o gpurun_out/prof_attn_tc_b1 $B --batch 1 > /dev/null 2>&1; echo a1=$?
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_gemm_t --launch-skip 80 --launch-count 2 -f -o gpurun_out/prof_gemm_t_b1 $B --batch 1 > /dev/null 2>&1; echo gt1=$?
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s > gpurun_out/t_fullsize.log 2>&1; echo tf=$?
