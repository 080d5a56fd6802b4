"""Probe: the high-precision path (fp64 Z + DMMA projection) at the C3 shape, γ = 2^-7.
  python scripts/hp_probe.py [rows]  -> kernel time, fp64 TFLOP/s of the projection"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import dataclasses  # noqa: E402
import paper_2207_01016_b200 as P  # noqa: E402
from paper_2207_01016_b200 import synthetic  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
cfg = dataclasses.replace(synthetic.CONFIGS["c3"], gamma=2.0 ** -7)
X, _ = synthetic.make(cfg, rows=slice(0, max(rows, 200000)))
dev = torch.device("cuda", 0)
t0 = time.perf_counter()
Y, L = bench.make_basis(X, cfg, device=dev)
basis_s = time.perf_counter() - t0
Xd = torch.from_numpy(X[:rows]).to(dev)
G = torch.empty((rows, L.shape[1]), dtype=torch.float32, device=dev)
out = {"rows": rows, "B": cfg.budget, "b_eff": int(L.shape[1]), "d": cfg.d, "gamma": cfg.gamma, "eigh_s": basis_s}
with P.Context(device_ids=[0]) as ctx:
    for mode in ("high", "fast"):
        ctx.set_precision(mode)
        ctx.set_basis_device(torch.from_numpy(Y).to(dev), torch.from_numpy(L).to(dev), cfg.gamma)
        for _ in range(2):
            ctx.compute_g_device(Xd, G)
        ctx.factor_kernel_stats(reset=True)
        for _ in range(3):
            ctx.compute_g_device(Xd, G)
        torch.cuda.synchronize()
        ms, k = ctx.factor_kernel_stats(reset=True)
        per = ms / k
        flops = 2.0 * rows * cfg.budget * L.shape[1]
        out[mode] = {"ms": per, "rows_per_s": rows / per * 1e3, "projection_tflops": flops / per / 1e9,
                     "estimate": ctx.basis_precision()[1], "high": ctx.basis_precision()[0]}
print(json.dumps(out))
