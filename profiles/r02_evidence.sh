# round-2 evidence runs (outputs in gpurun_out/): config-5 mixed batch, flashinfer baseline,
# full ncu captures of the HBM-bound kernels (gather, select, gather_rows)
set -x
timeout 900 python bench.py --config cfg5-mixed --steps 5 > gpurun_out/b_cfg5_mixed.log 2>&1; echo mixed=$?
timeout 1200 python bench.py --batch 1 --steps 30 --flashinfer --no-cpu-baseline > gpurun_out/b1_fi.log 2>&1; echo fi=$?
B="python bench.py --profile-only --steps 1 --warmup 1 --no-baselines --no-cpu-baseline"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gather --launch-skip 2 --launch-count 1 -f -o gpurun_out/prof_gather_b32 $B > /dev/null 2>&1; echo g=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_select --launch-skip 1 --launch-count 1 -f -o gpurun_out/prof_select_b32 $B > /dev/null 2>&1; echo s=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gather_rows --launch-skip 1 --launch-count 1 -f -o gpurun_out/prof_gather_rows_b32 $B > /dev/null 2>&1; echo r=$?
