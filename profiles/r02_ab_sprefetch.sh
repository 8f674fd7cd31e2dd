# single-tile attention: S_{j+1} TMEM load issued before P_j is fenced/signalled (RC_ATTN_SPREFETCH)
# -- attention parity + batch-1 A/B + per-launch attention times
set -x
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "attention or selective_prefill_parity or window or ragged or spec" > gpurun_out/sp_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/sp_tests.log
for v in "p0:RC_ATTN_SPREFETCH=0" "p1:RC_ATTN_SPREFETCH=1" "p0b:RC_ATTN_SPREFETCH=0" "p1b:RC_ATTN_SPREFETCH=1" "p0c:RC_ATTN_SPREFETCH=0" "p1c:RC_ATTN_SPREFETCH=1"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 600 python bench.py --batch 1 --steps 20 --warmup 5 --no-cpu-baseline --no-baselines > gpurun_out/sp_b1_$n.log 2>&1
  python profiles/summ.py gpurun_out/sp_b1_$n.log 2>/dev/null | head -3
done
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size
B="python bench.py --profile-only --batch 1 --steps 1 --warmup 1 --no-baselines --no-cpu-baseline --pools random"
for v in "p0:RC_ATTN_SPREFETCH=0" "p1:RC_ATTN_SPREFETCH=1"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 600 ncu --metrics $M --clock-control none -k "regex:k_attn" --csv --log-file gpurun_out/sp_l_$n.csv $B > /dev/null 2>&1; echo l$n=$?
done
