# A/B of the paired kernel's POLY_CHUNKS (build each variant first: set POLY_CHUNKS in k_attn_pair.cu, build,
# copy paper_2605_07443_b200/librc.so to build/variants/librc_<mask>.so), batch-32 bench lines per variant
set -x
for rep in 1 2; do for v in 0x44 0x10 0x11; do
  cp build/variants/librc_$v.so paper_2605_07443_b200/librc.so
  timeout 300 python bench.py --no-baselines --no-cpu-baseline --steps 4 > gpurun_out/p32_${v}_$rep.log 2>&1
  python profiles/summ.py gpurun_out/p32_${v}_$rep.log | grep -E "ms/step|attention"
done; done
