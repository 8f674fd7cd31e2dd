# bench lines of the gradual-filtering variant (R-GF: Sel 30% at layer 1 -> 15% at layer 3) next to the
# one-shot default, same box
set -x
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/gb_b32_base.log 2>&1; echo b32_base=$?
timeout 900 python bench.py --steps 5 --warmup 3 --gradual 2 --r-start 3000 > gpurun_out/gb_b32_g2.log 2>&1; echo b32_g2=$?
timeout 900 python bench.py --batch 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/gb_b1_base.log 2>&1; echo b1_base=$?
timeout 900 python bench.py --batch 1 --steps 20 --warmup 5 --gradual 2 --r-start 3000 > gpurun_out/gb_b1_g2.log 2>&1; echo b1_g2=$?
for f in gb_b32_base gb_b32_g2 gb_b1_base gb_b1_g2; do grep -o '^{.*' gpurun_out/$f.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); b=d.get('baselines',{})
print('$f', round(d['value']), round(d['ms_per_step'],3), d['config'].get('gradual'), b.get('ttft_b1_ms',{}).get('selective_p50'), d['clocks'])"; done
