# head loads: the first k-blocks' weight boxes issued before griddepcontrol.wait (RC_GEMM_HEAD) -- parity + A/B
set -x
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or transposed or selective_prefill_parity or full_prefill or attention" > gpurun_out/hd_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/hd_tests.log
for v in "h0:RC_GEMM_HEAD=0" "h8:RC_GEMM_HEAD=8" "h0b:RC_GEMM_HEAD=0" "h8b:RC_GEMM_HEAD=8" "h2:RC_GEMM_HEAD=2" "h0c:RC_GEMM_HEAD=0" "h8c:RC_GEMM_HEAD=8"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 600 python bench.py --batch 1 --steps 20 --warmup 5 --no-cpu-baseline --no-baselines > gpurun_out/hd_b1_$n.log 2>&1
  python profiles/summ.py gpurun_out/hd_b1_$n.log | head -2
done
for v in "h0:RC_GEMM_HEAD=0" "h8:RC_GEMM_HEAD=8"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/hd_b32_$n.log 2>&1
  python profiles/summ.py gpurun_out/hd_b32_$n.log | head -2
done
