# round-2 re-run of the SURVEY §8(d) sweep at HEAD (profiles/sweep.sh) plus the default bench line;
# tables via profiles/sweep_table.py
set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py > gpurun_out/r02s_default.log 2>&1; echo default=$?
tail -1 gpurun_out/r02s_default.log > gpurun_out/r02s_default.json
bash profiles/sweep.sh
