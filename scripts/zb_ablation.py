"""K1 Z·β mode (b_eff = 1) on C2-shaped rows through the device entry, CUDA-event timed:
run once per LPD_K1_DEBUG setting with LPD_LIBRARY=paper_2207_01016_b200/liblpd_nystrom_ablate.so
(`make variants`): 0 = production, 8 = GEMM1 MMAs skipped (epilogue-bound time),
32 = epilogue math skipped (GEMM1-bound time)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_01016_b200 as P  # noqa: E402
from paper_2207_01016_b200 import synthetic  # noqa: E402

cfg = synthetic.CONFIGS["c2"]
X, _ = synthetic.make(cfg, rows=slice(0, 581_012))
Y = X[: cfg.budget]
out = {"debug": os.environ.get("LPD_K1_DEBUG", "0"), "library": os.environ.get("LPD_LIBRARY", "default")}
with P.Context(1) as ctx:
    Xd = torch.from_numpy(X).cuda()
    for k in (1, 4):
        ctx.set_basis_dense(Y, np.random.default_rng(k).standard_normal((cfg.budget, k)) * 1e-2, cfg.gamma)
        G = torch.empty((X.shape[0], k), dtype=torch.float64, device="cuda")
        for _ in range(3):
            ctx.compute_g_device(Xd, G)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            ctx.compute_g_device(Xd, G)
        e1.record()
        torch.cuda.synchronize()
        out[f"b_eff_{k}_ms"] = e0.elapsed_time(e1) / 10
print(json.dumps(out))
