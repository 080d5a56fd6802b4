"""Probe: the reference-signature compute_G (adapter) at C2 with its phases.
  python scripts/dropin_probe.py [rows] [steps]"""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2207_01016_b200 import synthetic  # noqa: E402

cfg = synthetic.CONFIGS["c2"]
rows = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.n
steps = sys.argv[2] if len(sys.argv) > 2 else "3"
X, _ = synthetic.make(cfg, rows=slice(0, cfg.n), n=cfg.n)
Y, L = bench.make_basis(X, cfg)
with tempfile.TemporaryDirectory() as td:
    p = os.path.join(td, "basis.npz")
    np.savez(p, Y=Y, L=L, gamma=cfg.gamma, workload=cfg.name)
    for k in range(int(os.environ.get("PROBE_REPEAT", "1"))):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "integration", "e2e_run.py"), "b200", "compute_g", p,
                            "--rows", str(rows), "--steps", steps], capture_output=True, text=True)
        print(r.stdout.strip()[-2000:])
        if r.returncode or os.environ.get("LPD_TRACE"):
            print(r.stderr[-6000:])
