# transposed GEMM with packed 128-token tails (RC_GEMM_T_PACK) and SwiGLU on it at M <= 1024
# (RC_GEMM_T=3): parity, batch-1 A/B, per-launch ncu times
set -x
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or transposed or selective_prefill_parity" > gpurun_out/tp_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/tp_tests.log
for v in "def:RC_GEMM_T=-1" "t3:RC_GEMM_T=3" "t3np:RC_GEMM_T=3 RC_GEMM_T_PACK=0" "defb:RC_GEMM_T=-1" "t3b:RC_GEMM_T=3" "t2:RC_GEMM_T=2" "t3c:RC_GEMM_T=3"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 600 python bench.py --batch 1 --steps 20 --warmup 5 --no-cpu-baseline --no-baselines > gpurun_out/tp_b1_$n.log 2>&1
  python profiles/summ.py gpurun_out/tp_b1_$n.log 2>/dev/null | head -2
done
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
B="python bench.py --profile-only --batch 1 --steps 1 --warmup 1 --no-baselines --no-cpu-baseline --pools random"
for v in "t3:RC_GEMM_T=3" "t2:RC_GEMM_T=2"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 600 ncu --metrics $M --clock-control none -k "regex:k_gemm" --csv --log-file gpurun_out/tp_l_$n.csv $B > /dev/null 2>&1; echo l$n=$?
done
