# batch-1 attention launch lists: single-tile (default) vs KV-chunked pairs (RC_ATTN_CHUNKED via
# --attn-kernel 5) at two chunk factors, and one full ncu capture of a chunked selective-layer launch
set -x
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size
B="python bench.py --profile-only --batch 1 --steps 1 --warmup 1 --no-baselines --no-cpu-baseline --pools random"
timeout 600 ncu --metrics $M --clock-control none -k "regex:k_attn" --csv --log-file gpurun_out/ac_tc.csv $B > /dev/null 2>&1; echo tc=$?
RC_ATTN_CHUNK_F=1 timeout 600 ncu --metrics $M --clock-control none -k "regex:k_attn" --csv --log-file gpurun_out/ac_f1.csv $B --attn-kernel 5 > /dev/null 2>&1; echo f1=$?
RC_ATTN_CHUNK_F=2 timeout 600 ncu --metrics $M --clock-control none -k "regex:k_attn" --csv --log-file gpurun_out/ac_f2.csv $B --attn-kernel 5 > /dev/null 2>&1; echo f2=$?
RC_ATTN_CHUNK_F=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_attn_pair --launch-skip 40 --launch-count 1 -f -o gpurun_out/prof_attn_chunk $B --attn-kernel 5 > /dev/null 2>&1; echo full=$?
