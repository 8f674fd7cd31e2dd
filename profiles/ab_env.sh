# A/B of one diagnostic environment knob on one box: AB_VAR=<name> AB_A=<value> AB_B=<value>
# runs the gpu tests (unless SKIP_TESTS=1), then b32 and b1 bench lines alternately for both values
set -x
if [ -z "$SKIP_TESTS" ]; then timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu.log 2>&1; echo tests=$?; tail -2 gpurun_out/t_gpu.log; fi
for rep in 1 2; do for v in "$AB_A" "$AB_B"; do
  timeout 300 env $AB_VAR=$v python bench.py --no-baselines --no-cpu-baseline --steps 3 > gpurun_out/ab32_${v}_$rep.log 2>&1
  timeout 300 env $AB_VAR=$v python bench.py --batch 1 --steps 20 --no-baselines --no-cpu-baseline > gpurun_out/ab1_${v}_$rep.log 2>&1
  python profiles/summ.py gpurun_out/ab32_${v}_$rep.log gpurun_out/ab1_${v}_$rep.log | grep -E "ms/step|attention|gather|gemm"
done; done
