# tests + bench lines used after each kernel change (outputs in gpurun_out/)
set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -x -q ${TESTSEL:-} > gpurun_out/t_gpu.log 2>&1; echo tests=$?
tail -3 gpurun_out/t_gpu.log
timeout 400 python bench.py ${BENCH32:-} > gpurun_out/b32.log 2>&1; echo b32=$?
timeout 300 python bench.py --batch 1 --steps 30 ${BENCH1:-} > gpurun_out/b1.log 2>&1; echo b1=$?
