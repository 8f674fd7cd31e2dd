# early O-projection at batch 1 (the transposed O-proj waits per 256-row token tile for the attention
# CTAs writing it, not for the whole attention grid): smoke, A/B against RC_OPROJ_EARLY=0, GPU suite
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
B="python bench.py --batch 1 --steps 20 --warmup 3 --no-baselines --no-cpu-baseline"
timeout 300 $B > gpurun_out/early_smoke.log 2>&1; echo smoke=$?
tail -3 gpurun_out/early_smoke.log | cut -c1-300
for pass in 1 2; do
for r in 1000 1500 2000; do
  for ea in 1 0; do
    out=$(RC_OPROJ_EARLY=$ea timeout 300 $B --r-bp $r 2>/dev/null | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print(f\"{d['ms_per_step']:.3f} ttft {d['ttft_ms']['p50']:.3f} gemm {k['gemm']['ms_per_step']:.3f} attn {k['attention']['ms_per_step']:.3f} mhz {d['clocks']['sm_mhz']}\")")
    echo "pass=$pass r=$r early=$ea $out"
  done
done
done
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/early_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/early_tests.log
