# session-4 final evidence at HEAD: GPU suite, default bench lines (b32, b1), cfg5-mixed, ncu launch list b1
set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s4f_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/s4f_tests.log
timeout 900 python bench.py > gpurun_out/s4f_b32.log 2>&1; echo b32=$?
timeout 600 python bench.py --batch 1 --steps 30 > gpurun_out/s4f_b1.log 2>&1; echo b1=$?
timeout 900 python bench.py --config cfg5-mixed --steps 5 > gpurun_out/s4f_cfg5_mixed.log 2>&1; echo mixed=$?
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
B="python bench.py --profile-only --steps 1 --warmup 1 --no-baselines --no-cpu-baseline --pools random"
timeout 900 ncu --metrics $M --clock-control none -k "regex:^k_|k_gemm|k_attn" --csv --log-file gpurun_out/s4f_launches_b1.csv $B --batch 1 > /dev/null 2>&1; echo l1=$?
