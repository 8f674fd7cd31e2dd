# Profile capture used for profiles/ (run on the GPU box from the repo root; outputs go to gpurun_out/)
set -x
timeout 600 python bench.py > gpurun_out/final_b32.log 2>&1; echo b32=$?
timeout 600 python bench.py --batch 1 --steps 30 > gpurun_out/final_b1.log 2>&1; echo b1=$?
python profiles/summ.py gpurun_out/final_b32.log gpurun_out/final_b1.log
# launch list of one cfg3 step (our kernels only; ncu serialises launches and runs them cold)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
timeout 900 ncu --metrics $M --clock-control none -k "regex:^k_|k_gemm|k_attn" --csv --log-file gpurun_out/launches_b32.csv python bench.py --profile-only --steps 1 --warmup 1 --no-baselines --no-cpu-baseline > /dev/null 2>&1; echo l32=$?
timeout 900 ncu --metrics $M --clock-control none -k "regex:^k_|k_gemm|k_attn" --csv --log-file gpurun_out/launches_b1.csv python bench.py --profile-only --batch 1 --steps 1 --warmup 1 --no-baselines --no-cpu-baseline > /dev/null 2>&1; echo l1=$?
# selective-layer attention launches, full set: paired tiles at batch 32, single tiles at batch 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_attn_pair --launch-skip 5 --launch-count 1 -f -o gpurun_out/prof_attn_pair_b32 python bench.py --profile-only --steps 1 --warmup 1 --no-baselines --no-cpu-baseline > /dev/null 2>&1; echo a32=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_attn_tc --launch-skip 5 --launch-count 1 -f -o gpurun_out/prof_attn_tc_b1 python bench.py --profile-only --batch 1 --steps 1 --warmup 1 --no-baselines --no-cpu-baseline > /dev/null 2>&1; echo a1=$?
# one selective-layer gate/up GEMM (CTA pair) at batch 32, full set
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm_pair --launch-skip 7 --launch-count 1 -f -o gpurun_out/prof_gemm_pair_b32 python bench.py --profile-only --steps 1 --warmup 1 --no-baselines --no-cpu-baseline > /dev/null 2>&1; echo g=$?
