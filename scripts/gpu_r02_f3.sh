#!/bin/bash
# f3 (q_diag from the device row norms, batched warm starts) + sanitizers over every kernel
# + drop-in phase trace + C2 train timing
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_integration.py tests/test_downstream_parity.py -q -m gpu -p no:cacheprovider > gpurun_out/f3_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/f3_tests.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 30 python scripts/sanitize_kernels.py > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitizer_$tool.txt
done
LPD_TRACE=1 timeout 600 python scripts/dropin_probe.py 581012 2 > gpurun_out/dropin_trace.log 2>&1; echo "probe rc=$?"; grep -v "^\[lpd\] compute" gpurun_out/dropin_trace.log | tail -40 | cut -c1-400
timeout 900 python integration/e2e_run.py b200 train c2 --n-test 20000 > gpurun_out/train_c2_b200.json 2> gpurun_out/train_c2_b200.err; echo "train rc=$?"; cat gpurun_out/train_c2_b200.json
