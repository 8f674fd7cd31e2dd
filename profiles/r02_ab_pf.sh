# weight L2 prefetch ahead of the TMA loads (RC_GEMM_PF k-blocks, first ones before the PDL wait):
# GEMM parity tests, batch-1 and batch-32 A/B over the distance, b1 GEMM launch list at the default
set -x
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or transposed or selective_prefill_parity or full_prefill" > gpurun_out/pf_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/pf_tests.log
for v in "pf0:RC_GEMM_PF=0" "pf8:RC_GEMM_PF=8" "pf16:RC_GEMM_PF=16" "pf4:RC_GEMM_PF=4" "pf0b:RC_GEMM_PF=0" "pf8b:RC_GEMM_PF=8" "pf16b:RC_GEMM_PF=16"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 600 python bench.py --batch 1 --steps 20 --warmup 5 --no-cpu-baseline --no-baselines > gpurun_out/pf_b1_$n.log 2>&1
  python profiles/summ.py gpurun_out/pf_b1_$n.log | head -3
done
for v in "pf0:RC_GEMM_PF=0" "pf8:RC_GEMM_PF=8"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/pf_b32_$n.log 2>&1
  python profiles/summ.py gpurun_out/pf_b32_$n.log | head -3
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
B="python bench.py --profile-only --batch 1 --steps 1 --warmup 1 --no-baselines --no-cpu-baseline --pools random"
for v in "pf0:RC_GEMM_PF=0" "pf8:RC_GEMM_PF=8"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 600 ncu --metrics $M --clock-control none -k "regex:k_gemm" --csv --log-file gpurun_out/pf_l_$n.csv $B > /dev/null 2>&1; echo l$n=$?
done
