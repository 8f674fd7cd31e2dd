# (ncu captures use --pools random: the materialised-pool setup runs full prefills whose launches would
#  otherwise be counted by --launch-skip; the timed steps are the same kernels either way)
# round-2 evidence: default bench lines (b32, b1), cfg5-mixed, ncu launch lists of one step at b32 and b1,
# ncu --set full of the dominant kernels and of the gather (outputs in gpurun_out/)
set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "semlib" > gpurun_out/t_semlib.log 2>&1; echo tsem=$?
tail -3 gpurun_out/t_semlib.log
timeout 900 python bench.py > gpurun_out/final_b32.log 2>&1; echo b32=$?
timeout 600 python bench.py --batch 1 --steps 30 > gpurun_out/final_b1.log 2>&1; echo b1=$?
timeout 900 python bench.py --config cfg5-mixed --steps 5 > gpurun_out/final_cfg5_mixed.log 2>&1; echo mixed=$?
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
B="python bench.py --profile-only --steps 1 --warmup 1 --no-baselines --no-cpu-baseline --pools random"
timeout 1500 ncu --metrics $M --clock-control none -k "regex:^k_|k_gemm|k_attn" --csv --log-file gpurun_out/launches_b32.csv $B > /dev/null 2>&1; echo l32=$?
timeout 1500 ncu --metrics $M --clock-control none -k "regex:^k_|k_gemm|k_attn" --csv --log-file gpurun_out/launches_b1.csv $B --batch 1 > /dev/null 2>&1; echo l1=$?
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_gather[^_]" --launch-skip 1 --launch-count 1 -f -o gpurun_out/prof_gather_b32 $B > /dev/null 2>&1; echo g=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_attn_pair --launch-skip 5 --launch-count 1 -f -o gpurun_out/prof_attn_pair_b32 $B > /dev/null 2>&1; echo a32=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm_pair --launch-skip 7 --launch-count 1 -f -o gpurun_out/prof_gemm_pair_b32 $B > /dev/null 2>&1; echo g32=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm_t --launch-skip 21 --launch-count 1 -f -o gpurun_out/prof_gemm_t_b1 $B --batch 1 > /dev/null 2>&1; echo gt1=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_attn_tc --launch-skip 5 --launch-count 1 -f -o gpurun_out/prof_attn_tc_b1 $B --batch 1 > /dev/null 2>&1; echo a1=$?
