# n-grouped GEMM raster without L2 eviction hints (RC_GEMM_RASTER=1 RC_GEMM_RASTER_HINT=0) vs the
# default m-groups at cfg3 batch 32: step time and per-class DRAM bytes (ncu)
set -x
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for v in "m:RC_GEMM_RASTER=0" "n:RC_GEMM_RASTER=1 RC_GEMM_RASTER_HINT=0" "mb:RC_GEMM_RASTER=0" "nb:RC_GEMM_RASTER=1 RC_GEMM_RASTER_HINT=0"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/r2_b32_$n.log 2>&1
  python profiles/summ.py gpurun_out/r2_b32_$n.log 2>/dev/null | head -2
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
B="python bench.py --profile-only --steps 1 --warmup 1 --no-baselines --no-cpu-baseline --pools random"
for v in "m:RC_GEMM_RASTER=0" "n:RC_GEMM_RASTER=1 RC_GEMM_RASTER_HINT=0"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 900 ncu --metrics $M --clock-control none -k "regex:k_gemm" --csv --log-file gpurun_out/r2_l_$n.csv $B > /dev/null 2>&1; echo l$n=$?
done
