# A/B of attention variants on one box: RC_ATTN_DEBUG=4 disables the speculative-base softmax path
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "attention or selective or full_prefill" > gpurun_out/t_attn.log 2>&1; echo tests=$?
tail -2 gpurun_out/t_attn.log
for v in 4 0 4 0; do
  timeout 300 env RC_ATTN_DEBUG=$v python bench.py --no-baselines --no-cpu-baseline --steps 3 > gpurun_out/ab32_$v.log 2>&1
  timeout 300 env RC_ATTN_DEBUG=$v python bench.py --batch 1 --steps 20 --no-baselines --no-cpu-baseline > gpurun_out/ab1_$v.log 2>&1
  python profiles/summ.py gpurun_out/ab32_$v.log gpurun_out/ab1_$v.log | grep -E "attention|ms/step"
done
