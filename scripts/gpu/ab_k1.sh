#!/bin/bash
# A/B of the factor kernel against an older commit built under scratch/oldtree (git worktree,
# git-ignored, shipped with the snapshot), alternating on one box: K1 ms, step ms, SM clock.
for i in 1 2 3; do
  for tree in scratch/oldtree .; do
    (cd $tree && timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-extras 2>/dev/null) | \
      python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$tree', round(j['roofline']['kernel_ms'],2), round(j['ms_per_step'],2), j['clocks']['sm_mhz'])"
  done
done
