# A/B: paired-tile attention forced at batch 1 (RC_ATTN_PAIRS=1) and single-tile forced at batch 32 (=0) vs auto (-1)
set -x
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for rep in 1 2; do for v in -1 1; do
  timeout 300 env RC_ATTN_PAIRS=$v python bench.py --batch 1 --steps 20 --no-baselines --no-cpu-baseline > gpurun_out/abp1_${v}_$rep.log 2>&1
  python profiles/summ.py gpurun_out/abp1_${v}_$rep.log | grep -E "ms/step|attention|gemm"
done; done
for v in -1 0; do
  timeout 300 env RC_ATTN_PAIRS=$v python bench.py --no-baselines --no-cpu-baseline --steps 3 > gpurun_out/abp32_${v}.log 2>&1
  python profiles/summ.py gpurun_out/abp32_${v}.log | grep -E "ms/step|attention|gemm"
done
