# batch-1 A/B of one environment knob (AB_VAR, values AB_VALS), 3 repetitions interleaved
set -x
for rep in 1 2 3; do for v in $AB_VALS; do
  timeout 300 env $AB_VAR=$v python bench.py --batch 1 --steps 20 --no-baselines --no-cpu-baseline > gpurun_out/b1_${v}_$rep.log 2>&1
  python profiles/summ.py gpurun_out/b1_${v}_$rep.log | grep -E "ms/step|attention"
done; done
