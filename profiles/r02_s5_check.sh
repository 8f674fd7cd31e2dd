# session-5 re-entry check at HEAD: build, full GPU suite, default (b32) and b1 bench lines
set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s5_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/s5_tests.log
timeout 600 python bench.py > gpurun_out/s5_b32.log 2>&1; echo b32=$?
tail -1 gpurun_out/s5_b32.log
timeout 600 python bench.py --batch 1 --steps 30 > gpurun_out/s5_b1.log 2>&1; echo b1=$?
tail -1 gpurun_out/s5_b1.log
