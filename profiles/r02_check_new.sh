set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests/test_gpu_fetch.py tests/test_gpu_pools.py -m gpu -q -s > gpurun_out/t_new.log 2>&1; echo new=$?
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -s > gpurun_out/t_par.log 2>&1; echo par=$?
