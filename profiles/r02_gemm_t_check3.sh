set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "residual_gemm or gemm_matches or selective_prefill_parity" > gpurun_out/t_gemm.log 2>&1; echo gemm=$?
tail -3 gpurun_out/t_gemm.log
timeout 300 python bench.py --batch 1 --steps 30 --no-baselines --no-cpu-baseline > gpurun_out/b1.log 2>&1; echo b1=$?
RC_GEMM_T=0 timeout 300 python bench.py --batch 1 --steps 30 --no-baselines --no-cpu-baseline > gpurun_out/b1_not.log 2>&1; echo b1n=$?
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
timeout 600 ncu --metrics $M --clock-control none -k "regex:^k_|k_gemm|k_attn" --csv --log-file gpurun_out/launches_b1.csv python bench.py --profile-only --batch 1 --steps 1 --warmup 1 --no-baselines --no-cpu-baseline > /dev/null 2>&1; echo l1=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm_t --launch-skip 40 --launch-count 3 -f -o gpurun_out/prof_gemm_t_b1 python bench.py --profile-only --batch 1 --steps 1 --warmup 1 --no-baselines --no-cpu-baseline > /dev/null 2>&1; echo pf=$?
