# SURVEY §8(d) runs: r in {5,10,15,20,30}% x batch {1,32} on cfg3 (Llama-3-8B shape, 4K prompts),
# cfg2 (2.5K prompts) and cfg5 (Qwen2-7B shape, 8K prompts) at batch 1, r = 15%.
for b in 1 32; do
  for r in 500 1000 1500 2000 3000; do
    st=20; [ $b = 32 ] && st=5
    timeout 400 python bench.py --batch $b --r-bp $r --steps $st --no-baselines --no-cpu-baseline 2>/dev/null | grep '^{' > gpurun_out/sweep_cfg3_b${b}_r${r}.json
    echo cfg3 b=$b r=$r rc=$?
  done
done
timeout 400 python bench.py --config cfg2-llama-1k --batch 1 --steps 20 --no-cpu-baseline 2>/dev/null | grep '^{' > gpurun_out/sweep_cfg2_b1.json; echo cfg2 rc=$?
timeout 600 python bench.py --config cfg5-qwen-8k --batch 1 --steps 20 --no-cpu-baseline 2>/dev/null | grep '^{' > gpurun_out/sweep_cfg5_b1.json; echo cfg5 rc=$?
timeout 600 python bench.py --config cfg5-qwen-8k --batch 8 --steps 5 --no-baselines --no-cpu-baseline 2>/dev/null | grep '^{' > gpurun_out/sweep_cfg5_b8.json; echo cfg5b8 rc=$?
