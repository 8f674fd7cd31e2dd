# paired-attention phase timing (diagnostics build -DRC_ATTN_PROF; clock64 sums per role and phase,
# printed by rc_destroy): cfg3 batch 32, normal and with the MMAs skipped (RC_ATTN_DEBUG=2)
set -x
RC_BUILD_DEFS=-DRC_ATTN_PROF python -m paper_2605_07443_b200.build --force > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
RC_ATTN_PROF=1 timeout 600 python bench.py --profile-only --steps 2 --warmup 1 --no-baselines --no-cpu-baseline --pools random > gpurun_out/ph_b32.log 2>&1; echo a=$?
grep RC_ATTN_PROF gpurun_out/ph_b32.log
RC_ATTN_PROF=1 RC_ATTN_DEBUG=2 timeout 600 python bench.py --profile-only --steps 2 --warmup 1 --no-baselines --no-cpu-baseline --pools random > gpurun_out/ph_b32_nomma.log 2>&1; echo b=$?
grep RC_ATTN_PROF gpurun_out/ph_b32_nomma.log
RC_ATTN_PROF=1 RC_ATTN_DEBUG=1 timeout 600 python bench.py --profile-only --steps 2 --warmup 1 --no-baselines --no-cpu-baseline --pools random > gpurun_out/ph_b32_nosm.log 2>&1; echo c=$?
grep RC_ATTN_PROF gpurun_out/ph_b32_nosm.log
python -m paper_2605_07443_b200.build --force > gpurun_out/build2.log 2>&1; echo rebuilt=$?
