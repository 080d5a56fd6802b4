#!/bin/bash
# K8 (per-point decision values) and the device vote: parity on the B200.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_integration.py -q -m gpu -p no:cacheprovider \
  -k "model_decision or ovo_vote" > gpurun_out/k8_tests.log 2>&1; echo "rc=$?"; tail -30 gpurun_out/k8_tests.log
