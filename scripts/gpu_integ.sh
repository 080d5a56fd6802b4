timeout 900 python -m pytest tests/test_integration.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3
timeout 2400 bash scripts/e2e_train.sh 2>&1 | tail -8
ls gpurun_out/e2e_*
