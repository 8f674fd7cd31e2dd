# k-block rotation by weight tile for small-M GEMMs (RC_GEMM_KROT): parity, batch-1 A/B (default kernels
# and the transposed SwiGLU / QKV), batch 32 with rotation everywhere, per-launch ncu times at batch 1
set -x
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or transposed or selective_prefill_parity or full_prefill" > gpurun_out/kr_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/kr_tests.log
for v in "k0:RC_GEMM_KROT=0" "k1:RC_GEMM_KROT=1" "k0t2:RC_GEMM_KROT=0 RC_GEMM_T=2" "k1t2:RC_GEMM_KROT=1 RC_GEMM_T=2" "k0b:RC_GEMM_KROT=0" "k1b:RC_GEMM_KROT=1" "k1t2b:RC_GEMM_KROT=1 RC_GEMM_T=2"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 600 python bench.py --batch 1 --steps 20 --warmup 5 --no-cpu-baseline --no-baselines > gpurun_out/kr_b1_$n.log 2>&1
  python profiles/summ.py gpurun_out/kr_b1_$n.log 2>/dev/null | head -2
done
for v in "k0:RC_GEMM_KROT=0" "k2:RC_GEMM_KROT=2"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/kr_b32_$n.log 2>&1
  python profiles/summ.py gpurun_out/kr_b32_$n.log 2>/dev/null | head -2
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
B="python bench.py --profile-only --batch 1 --steps 1 --warmup 1 --no-baselines --no-cpu-baseline --pools random"
for v in "k1:RC_GEMM_KROT=1" "k1t2:RC_GEMM_KROT=1 RC_GEMM_T=2"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 600 ncu --metrics $M --clock-control none -k "regex:k_gemm" --csv --log-file gpurun_out/kr_l_$n.csv $B > /dev/null 2>&1; echo l$n=$?
done
