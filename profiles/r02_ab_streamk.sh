# single-CTA stream-K tail for SwiGLU / QKV (partials summed in K order into TMEM before the epilogue):
# GPU suite, then batch-1 A/B against RC_GEMM_STREAMK=0 at r = 10 / 15 / 20 %, two passes, alternating
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/sk_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/sk_tests.log
B="python bench.py --batch 1 --steps 20 --warmup 3 --no-baselines --no-cpu-baseline"
for pass in 1 2; do
for r in 1000 1500 2000; do
  for sk in 1 0; do
    out=$(RC_GEMM_STREAMK=$sk timeout 300 $B --r-bp $r 2>/dev/null | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print(f\"{d['ms_per_step']:.3f} gemm {k['gemm']['ms_per_step']:.3f} attn {k['attention']['ms_per_step']:.3f} mhz {d['clocks']['sm_mhz']}\")")
    echo "pass=$pass r=$r streamk=$sk $out"
  done
done
done
