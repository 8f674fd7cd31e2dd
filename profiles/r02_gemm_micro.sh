# small-M GEMM micro-benchmark (profiles/micro/gemm_sweep.py): single-CTA vs CTA-pair, hot vs cold weights
set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
#TAG=default timeout 300 python profiles/micro/gemm_sweep.py > gpurun_out/gm_default.txt 2>&1; echo d=$?
#TAG=pair RC_GEMM_PAIR_MIN_M=256 timeout 300 python profiles/micro/gemm_sweep.py > gpurun_out/gm_pair.txt 2>&1; echo p=$?
#TAG=single RC_GEMM_PAIR=0 timeout 300 python profiles/micro/gemm_sweep.py > gpurun_out/gm_single.txt 2>&1; echo s=$?
#cat gpurun_out/gm_default.txt gpurun_out/gm_pair.txt gpurun_out/gm_single.txt
TAG=fixed timeout 300 python profiles/micro/gemm_fixed.py > gpurun_out/gf_default.txt 2>&1; echo f=$?
TAG=fixedP RC_GEMM_PAIR=1 timeout 300 python profiles/micro/gemm_fixed.py > gpurun_out/gf_pair.txt 2>&1; echo fp=$?
TAG=nopdl RC_PDL=0 timeout 300 python profiles/micro/gemm_fixed.py > gpurun_out/gf_nopdl.txt 2>&1; echo fn=$?
cat gpurun_out/gf_default.txt gpurun_out/gf_pair.txt gpurun_out/gf_nopdl.txt
