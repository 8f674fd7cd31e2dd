# NEXT-4 zero-copy V: tests, then a same-box A/B of step time at batch 32 and batch 1
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "zero_copy or gather_bitexact or selective_prefill_parity" > gpurun_out/t_zc.log 2>&1; echo t=$?
tail -5 gpurun_out/t_zc.log
timeout 600 python bench.py --no-baselines --no-cpu-baseline > gpurun_out/zc_b32_off.log 2>&1; echo off32=$?
RC_ZERO_COPY_V=1 timeout 600 python bench.py --no-baselines --no-cpu-baseline > gpurun_out/zc_b32_on.log 2>&1; echo on32=$?
timeout 300 python bench.py --batch 1 --steps 30 --no-baselines --no-cpu-baseline > gpurun_out/zc_b1_off.log 2>&1; echo off1=$?
RC_ZERO_COPY_V=1 timeout 300 python bench.py --batch 1 --steps 30 --no-baselines --no-cpu-baseline > gpurun_out/zc_b1_on.log 2>&1; echo on1=$?
