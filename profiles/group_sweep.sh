# GEMM raster group sweep: DRAM bytes and time of the gate/up and down GEMMs of one selective layer (cfg3 batch 32)
for mb in 8 16 32 64 128; do
  RC_GROUP_A_MB=$mb timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_gemm --launch-skip 267 --launch-count 4 --csv --log-file gpurun_out/group_$mb.csv python bench.py --profile-only --steps 1 --warmup 1 --no-baselines --no-cpu-baseline > /dev/null 2>&1
  echo mb=$mb rc=$?
done
