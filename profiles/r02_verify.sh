# verification at HEAD after removing the measured-negative GEMM experiments: full GPU suite, default
# bench lines, board power during batch 1 / r = 100 % / batch 32 (profiles/r02_power.sh)
set -x
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/verify_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/verify_tests.log
timeout 900 python bench.py > gpurun_out/verify_b32.log 2>&1; echo b32=$?
timeout 600 python bench.py --batch 1 --steps 30 > gpurun_out/verify_b1.log 2>&1; echo b1=$?
bash profiles/r02_power.sh
