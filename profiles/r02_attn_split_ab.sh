# single-tile attention: KV split merged in-kernel by the last-arriving split CTA (no merge kernel),
# grid in longest-first order across KV heads; parity + batch-1 A/B of AUTO / SPLIT2 / ADAPTIVE
set -x
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "attention or selective_prefill_parity or window or ragged" > gpurun_out/as_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/as_tests.log
for ak in 0 3 4 0 3 4; do
  timeout 600 python bench.py --batch 1 --steps 20 --warmup 5 --no-cpu-baseline --attn-kernel $ak > gpurun_out/as_b1_$ak.log 2>&1
  grep -o '^{.*' gpurun_out/as_b1_$ak.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); b=d['baselines']; k=d['kernels']
print('ak=$ak', round(d['ms_per_step'],3), 'ttft', round(b['ttft_b1_ms']['selective_p50'],3), 'attn', round(k['attention']['ms_per_step'],3), k['attention']['launches_per_step'], 'x', round(b['ttft_b1_speedup_vs_full'],3), d['clocks']['sm_mhz'])"
done
