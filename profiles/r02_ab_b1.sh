# batch-1 A/B: CTA pairs for every 256-wide GEMM, and the paper-literal scoring (c = 0, lambda = 0.5)
set -x
timeout 300 python bench.py --batch 1 --steps 30 --no-cpu-baseline > gpurun_out/ab_base.log 2>&1; echo base=$?
RC_GEMM_PAIR=1 timeout 300 python bench.py --batch 1 --steps 30 --no-cpu-baseline --no-baselines > gpurun_out/ab_pair.log 2>&1; echo pair=$?
timeout 300 python bench.py --batch 1 --steps 30 --no-cpu-baseline --check-layer 0 --lam 0.5 > gpurun_out/ab_next1.log 2>&1; echo n1=$?
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
RC_GEMM_PAIR=1 timeout 600 ncu --metrics $M --clock-control none -k "regex:^k_|k_gemm|k_attn" --csv --log-file gpurun_out/launches_b1_pair.csv python bench.py --profile-only --batch 1 --steps 1 --warmup 1 --no-baselines --no-cpu-baseline > /dev/null 2>&1; echo l1=$?
