# A/B: single-tile attention with one 8-key chunk of 8 on the FMA pipe (RC_TC_POLY=0x01) vs SFU only (default)
set -x
for rep in 1 2; do for v in 0x00 0x01; do
  RC_BUILD_DEFS=-DRC_TC_POLY=$v python -m paper_2605_07443_b200.build --force > gpurun_out/build_$v.log 2>&1 || { tail -20 gpurun_out/build_$v.log; exit 1; }
  timeout 300 python bench.py --batch 1 --steps 20 --no-baselines --no-cpu-baseline > gpurun_out/abq1_${v}_$rep.log 2>&1
  python profiles/summ.py gpurun_out/abq1_${v}_$rep.log | grep -E "ms/step|attention|gemm"
done; done
