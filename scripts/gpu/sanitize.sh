#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel (scripts/sanitize_kernels.py)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 30 python scripts/sanitize_kernels.py > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitizer_$tool.txt
done
