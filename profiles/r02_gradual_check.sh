# gradual filtering (R-GF): GPU tests + regression check of the one-shot path
set -x
python -m paper_2605_07443_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_gradual.py -x -q > gpurun_out/gradual_tests.log 2>&1; echo gradual=$?
tail -30 gpurun_out/gradual_tests.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/parity_tests.log 2>&1; echo parity=$?
tail -5 gpurun_out/parity_tests.log
