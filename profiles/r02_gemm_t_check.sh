# transposed-GEMM / deterministic-reduction check: unit tests first (short timeout), then parity, then benches
set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "residual_gemm or gemm_matches" > gpurun_out/t_gemm.log 2>&1; echo gemm=$?
tail -15 gpurun_out/t_gemm.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/t_all.log 2>&1; echo all=$?
tail -15 gpurun_out/t_all.log
timeout 300 python bench.py --batch 1 --steps 30 > gpurun_out/b1.log 2>&1; echo b1=$?
timeout 400 python bench.py > gpurun_out/b32.log 2>&1; echo b32=$?
