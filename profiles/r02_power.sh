# board power and SM clock during the timed region (bench clocks sampler, 200 ms): batch-1 selective
# prefill over 300 steps, the same with r = 100 % (every non-prefix token recomputed, the FLOPs of a full
# prefill), and batch 32
set -x
timeout 600 python bench.py --batch 1 --steps 300 --warmup 5 --no-cpu-baseline --no-baselines > gpurun_out/pw_b1.log 2>&1; echo b1=$?
timeout 600 python bench.py --batch 1 --steps 60 --warmup 3 --r-bp 10000 --no-cpu-baseline --no-baselines > gpurun_out/pw_b1_r100.log 2>&1; echo b1r=$?
timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/pw_b32.log 2>&1; echo b32=$?
for f in pw_b1 pw_b1_r100 pw_b32; do grep -o '^{.*' gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['ms_per_step'],3), d['clocks'], round(d['kernels']['gemm']['tflops'],1))"; done
