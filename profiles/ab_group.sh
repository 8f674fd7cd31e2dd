# steady-state b32 bench lines for several GEMM raster-group L2 budgets (RC_GROUP_A_MB)
set -x
for rep in 1 2; do for v in 32 16 48 24; do
  timeout 300 env RC_GROUP_A_MB=$v python bench.py --no-baselines --no-cpu-baseline --steps 4 > gpurun_out/g32_${v}_$rep.log 2>&1
  python profiles/summ.py gpurun_out/g32_${v}_$rep.log | grep -E "ms/step|gemm"
done; done
