# batch-1 GEMM dispatch A/B across r (M = |Sel| ~ 205 / 410 / 625 / 830): default (single-CTA SwiGLU/QKV
# below M 1024, transposed residual) vs SwiGLU transposed (RC_GEMM_T=3), SwiGLU+QKV transposed (=2),
# CTA pairs from M 512 (RC_GEMM_PAIR_MIN_M=512); two passes, alternating modes
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
B="python bench.py --batch 1 --steps 20 --warmup 3 --no-baselines --no-cpu-baseline"
for pass in 1 2; do
for r in 500 1000 1500 2000; do
  for mode in default T3 T2 P512; do
    case $mode in
      default) E="";; T3) E="RC_GEMM_T=3";; T2) E="RC_GEMM_T=2";; P512) E="RC_GEMM_PAIR_MIN_M=512";;
    esac
    out=$(env $E timeout 300 $B --r-bp $r 2>/dev/null | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print(f\"{d['ms_per_step']:.3f} gemm {k['gemm']['ms_per_step']:.3f} attn {k['attention']['ms_per_step']:.3f} mhz {d['clocks']['sm_mhz']}\")")
    echo "pass=$pass r=$r mode=$mode $out"
  done
done
done
