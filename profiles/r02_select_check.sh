set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "deviation_and_selection or selective_prefill_parity or window or miss or ragged" > gpurun_out/t_sel.log 2>&1; echo t=$?
tail -3 gpurun_out/t_sel.log
timeout 300 python bench.py --batch 1 --steps 30 --no-cpu-baseline > gpurun_out/b1.log 2>&1; echo b1=$?
timeout 600 python bench.py --no-cpu-baseline --no-baselines > gpurun_out/b32.log 2>&1; echo b32=$?
