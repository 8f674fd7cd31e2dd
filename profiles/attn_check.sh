# attention change check: parity tests, b32/b1 bench, one ncu launch of the paired kernel (outputs in gpurun_out/)
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "attention or selective or full_prefill" > gpurun_out/t_attn.log 2>&1; echo tests=$?
tail -2 gpurun_out/t_attn.log
timeout 300 python bench.py --no-baselines --no-cpu-baseline --steps 3 > gpurun_out/ab32.log 2>&1
timeout 300 python bench.py --batch 1 --steps 20 --no-baselines --no-cpu-baseline > gpurun_out/ab1.log 2>&1
python profiles/summ.py gpurun_out/ab32.log gpurun_out/ab1.log
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second -k regex:k_attn --launch-skip 5 --launch-count 2 python bench.py --profile-only --steps 1 --warmup 1 --no-baselines --no-cpu-baseline 2>&1 | grep -E "k_attn|duration|tensor|issue|per_second"
