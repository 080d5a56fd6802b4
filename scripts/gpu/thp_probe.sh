#!/bin/bash
# Why does the drop-in's gmatrix (a fresh 19 GB Matrix) vary 0.7-2.8 s between boxes/runs?
# THP fault / fallback / direct-compaction counters around two lpdsvm.train runs at C2.
mkdir -p gpurun_out
snap() { grep -E "^(thp_fault_alloc|thp_fault_fallback|compact_stall|compact_fail|compact_success) " /proc/vmstat | tr '\n' ' '; echo; }
awk '{print $1,$2,$3,$4, "order9+:", $14, $15}' /proc/buddyinfo
for i in 1 2; do
  echo "== run $i"; snap
  timeout 600 python integration/e2e_run.py b200 train c2 --n-test 2000 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('gmatrix', j['gmatrix_seconds'], 'train', j['train_seconds'])"
  snap
  awk '{print $1,$2,$3,$4, "order9+:", $14, $15}' /proc/buddyinfo
done
