#!/bin/bash
# drop-in phases at C2 (reference compute_G signature, fresh Matrix) + racecheck/synccheck of smoke()
mkdir -p gpurun_out
timeout 600 python scripts/dropin_probe.py > gpurun_out/dropin_probe.log 2>&1; echo "probe rc=$?"; cat gpurun_out/dropin_probe.log | cut -c1-1500
for tool in racecheck synccheck; do
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_$tool.txt 2>&1; echo "$tool rc=$?"; tail -5 gpurun_out/sanitizer_$tool.txt
done
