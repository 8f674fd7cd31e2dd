# full GPU test suite + default bench lines (outputs in gpurun_out/)
set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/t_all.log 2>&1; echo tests=$?
tail -5 gpurun_out/t_all.log
timeout 600 python bench.py > gpurun_out/b32.log 2>&1; echo b32=$?
timeout 400 python bench.py --batch 1 --steps 30 > gpurun_out/b1.log 2>&1; echo b1=$?
timeout 400 python bench.py --batch 1 --steps 30 --pools random --no-baselines --no-cpu-baseline > gpurun_out/b1_rand.log 2>&1; echo b1r=$?
