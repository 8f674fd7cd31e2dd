# batch 1: residual split-K partials as direct TMA reduce-adds (default) vs the deterministic mode
# (partials stored to the workspace, the last arrival sums them in K order and reduce-adds once);
# transposed split cap 3 / 4 / 6
set -x
for v in "d0:X=0" "d1:X=1" "d0b:X=0" "d1b:X=1" "d1s4:RC_GEMM_T_SPLITS=4" "d1s6:RC_GEMM_T_SPLITS=6" "d0s6:RC_GEMM_T_SPLITS=6"; do
  n=${v%%:*}; e=${v#*:}
  D=""; case $n in d1*) D="--deterministic";; esac
  env $e timeout 600 python bench.py --batch 1 --steps 20 --warmup 5 --no-cpu-baseline --no-baselines $D > gpurun_out/det_b1_$n.log 2>&1
  python profiles/summ.py gpurun_out/det_b1_$n.log | head -2
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-baselines --deterministic > gpurun_out/det_b32_d1.log 2>&1
python profiles/summ.py gpurun_out/det_b32_d1.log | head -2
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
B="python bench.py --profile-only --batch 1 --steps 1 --warmup 1 --no-baselines --no-cpu-baseline --pools random"
timeout 600 ncu --metrics $M --clock-control none -k "regex:k_gemm" --csv --log-file gpurun_out/det_l_d1.csv $B --deterministic > /dev/null 2>&1; echo l=$?
