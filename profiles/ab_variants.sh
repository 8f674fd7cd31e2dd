# A/B of compile-time variants built locally under build/variants/librc_<tag>.so (VARIANTS="tag ...")
set -x
for rep in 1 2; do for v in $VARIANTS; do
  cp build/variants/librc_$v.so paper_2605_07443_b200/librc.so
  timeout 300 python bench.py --no-baselines --no-cpu-baseline --steps 3 > gpurun_out/v32_${v}_$rep.log 2>&1
  timeout 300 python bench.py --batch 1 --steps 20 --no-baselines --no-cpu-baseline > gpurun_out/v1_${v}_$rep.log 2>&1
  python profiles/summ.py gpurun_out/v32_${v}_$rep.log gpurun_out/v1_${v}_$rep.log | grep -E "ms/step|attention"
done; done
