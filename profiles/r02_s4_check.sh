# session-4 re-entry check at HEAD: build, full GPU suite, default b1 bench line, paired-attention phase timing
set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s4_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/s4_tests.log
timeout 600 python bench.py --batch 1 --steps 30 > gpurun_out/s4_b1.log 2>&1; echo b1=$?
tail -1 gpurun_out/s4_b1.log
bash profiles/r02_attn_phase.sh
