#!/bin/bash
# drop-in (reference compute_G signature, fresh Matrix) with and without the page-partitioned
# first touch; then the whole GPU suite
mkdir -p gpurun_out
for pf in 2 0 4; do
  LPD_PREFAULT=$pf timeout 600 python scripts/dropin_probe.py 581012 3 > gpurun_out/dropin_pf$pf.log 2>&1; echo "prefault=$pf rc=$?"; cut -c1-900 gpurun_out/dropin_pf$pf.log
done
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -s > gpurun_out/gputests_all.log 2>&1; echo "tests rc=$?"; grep -E "max row error|passed|failed|Error" gpurun_out/gputests_all.log | tail -20
