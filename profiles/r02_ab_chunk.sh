# KV-chunked persistent paired attention for small grids (RC_ATTN_CHUNKED / AUTO) and the n-grouped
# GEMM raster with L2 eviction hints: parity, batch-1 A/B over the chunk factor, batch-32 raster A/B
set -x
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "attention or selective_prefill_parity or window or ragged" > gpurun_out/ck_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/ck_tests.log
summ() {
  grep -o '^{.*' $1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); b=d.get('baselines') or {}; k=d['kernels']
print('$2', round(d['ms_per_step'],3), 'ttft', round(b.get('ttft_b1_ms',{}).get('selective_p50',0),3), 'attn', round(k['attention']['ms_per_step'],3), 'gemm', round(k['gemm']['ms_per_step'],3), 'x', round(b.get('ttft_b1_speedup_vs_full',0),3), d['clocks']['sm_mhz'])"
}
for v in "CK0:RC_ATTN_CHUNK_AUTO=0" "F2:RC_ATTN_CHUNK_F=2" "F1:RC_ATTN_CHUNK_F=1" "F3:RC_ATTN_CHUNK_F=3" "F1.5:RC_ATTN_CHUNK_F=1.5" "CK0b:RC_ATTN_CHUNK_AUTO=0" "F2b:RC_ATTN_CHUNK_F=2"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 600 python bench.py --batch 1 --steps 20 --warmup 5 --no-cpu-baseline --no-baselines > gpurun_out/ck_b1_$n.log 2>&1
  summ gpurun_out/ck_b1_$n.log $n
done
timeout 600 python bench.py --batch 1 --steps 30 --no-cpu-baseline > gpurun_out/ck_b1_full.log 2>&1; summ gpurun_out/ck_b1_full.log b1full
for v in "R0:RC_GEMM_RASTER=0" "Rauto:RC_GEMM_RASTER=-1" "R0b:RC_GEMM_RASTER=0" "Rautob:RC_GEMM_RASTER=-1"; do
  n=${v%%:*}; e=${v#*:}
  env $e timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/ck_b32_$n.log 2>&1
  summ gpurun_out/ck_b32_$n.log $n
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
B="python bench.py --profile-only --steps 1 --warmup 1 --no-baselines --no-cpu-baseline"
for r in 0 -1; do
  RC_GEMM_RASTER=$r timeout 900 ncu --metrics $M --clock-control none -k "regex:k_gemm" --csv --log-file gpurun_out/ck_gemm_r$r.csv $B > /dev/null 2>&1; echo ncu$r=$?
done
