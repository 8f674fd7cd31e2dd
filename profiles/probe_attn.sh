set -x
timeout 300 env RC_GEMM_PAIR=1 python bench.py --batch 1 --steps 30 --no-baselines --no-cpu-baseline > gpurun_out/b1_pair1.log 2>&1; echo p1=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attn_pair --launch-skip 5 --launch-count 1 -f -o gpurun_out/attn_pair_b32 python bench.py --profile-only --steps 1 --warmup 1 --no-baselines --no-cpu-baseline > gpurun_out/ncu1.log 2>&1; echo n1=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attn_tc --launch-skip 5 --launch-count 1 -f -o gpurun_out/attn_tc_b1 python bench.py --profile-only --batch 1 --steps 1 --warmup 1 --no-baselines --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo n2=$?
