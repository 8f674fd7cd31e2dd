# batch-1 launch list (per-kernel ncu times, tensor activity) + tests + bench lines (outputs in gpurun_out/)
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu.log 2>&1; echo tests=$?; tail -2 gpurun_out/t_gpu.log
timeout 300 python bench.py --batch 1 --steps 30 --no-cpu-baseline > gpurun_out/b1.log 2>&1; echo b1=$?
timeout 400 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/b32.log 2>&1; echo b32=$?
python profiles/summ.py gpurun_out/b1.log gpurun_out/b32.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k "regex:^k_|k_gemm|k_attn" --csv --log-file gpurun_out/launches_b1.csv python bench.py --profile-only --batch 1 --steps 1 --warmup 1 --no-baselines --no-cpu-baseline > /dev/null 2>&1; echo l1=$?
python profiles/launch_table.py gpurun_out/launches_b1.csv
