#!/bin/bash
# Drop-in compute_G at C2, every call recorded (the first one included): where a
# process's first gmatrix call spends its time compared with the steady state.
set -e
mkdir -p gpurun_out
python - <<'PY'
import sys, numpy as np
sys.path.insert(0, ".")
import bench
from paper_2207_01016_b200 import synthetic
cfg = synthetic.CONFIGS["c2"]
X, _ = bench.synthetic_rows(cfg, 0, cfg.n, 1)
Y, L = bench.make_basis(X, cfg)
np.savez("/tmp/c2_basis.npz", Y=Y, L=L, gamma=cfg.gamma, workload=cfg.name)
PY
python integration/e2e_run.py b200 compute_g /tmp/c2_basis.npz --rows 581012 --warmup 0 --steps 4 --per-call \
    > gpurun_out/first_call.json
python - <<'PY'
import json
j = json.loads(open("gpurun_out/first_call.json").read().strip().splitlines()[-1])
for k, c in enumerate(j["per_call"]):
    p = c["phases"]
    print(k, round(c["gmatrix_seconds"], 3), {x: round(v, 3) for x, v in p.items()})
PY
