# batch 1: SwiGLU / QKV at M = 625 on CTA pairs (RC_GEMM_PAIR_MIN_M=512, 768 padded rows) vs the
# single-CTA 128 x 256 tiles: ncu launch lists per kernel class + bench A/B (outputs in gpurun_out/)
set -x
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
B="python bench.py --profile-only --batch 1 --steps 1 --warmup 1 --no-baselines --no-cpu-baseline --pools random"
for v in "def:RC_GEMM_PAIR_MIN_M=1024" "p512:RC_GEMM_PAIR_MIN_M=512"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 900 ncu --metrics $M --clock-control none -k "regex:k_gemm" --csv --log-file gpurun_out/pb_$n.csv $B > /dev/null 2>&1; echo l$n=$?

done
for v in "def:RC_GEMM_PAIR_MIN_M=1024" "p512:RC_GEMM_PAIR_MIN_M=512"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 600 python bench.py --batch 1 --steps 20 --warmup 5 --no-cpu-baseline --no-baselines > gpurun_out/pb_b1_$n.log 2>&1
  python profiles/summ.py gpurun_out/pb_b1_$n.log | head -3
done
