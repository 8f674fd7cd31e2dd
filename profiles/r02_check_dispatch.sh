# SwiGLU on the transposed pair kernel at M <= 512 by default: GPU suite, batch-1 lines at r = 5 / 10 / 15 %
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/disp_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/disp_tests.log
B="python bench.py --batch 1 --steps 20 --warmup 3 --no-baselines --no-cpu-baseline"
for r in 500 1000 1500; do
  for mode in new old; do
    E=""; [ $mode = old ] && E="RC_GEMM_T=4"
    out=$(env $E timeout 300 $B --r-bp $r 2>/dev/null | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print(f\"{d['ms_per_step']:.3f} gemm {k['gemm']['ms_per_step']:.3f} attn {k['attention']['ms_per_step']:.3f} mhz {d['clocks']['sm_mhz']}\")")
    echo "r=$r dispatch=$mode $out"
  done
done
