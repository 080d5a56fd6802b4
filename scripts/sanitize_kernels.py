"""Every device kernel of liblpd_nystrom.so once, at small sizes, for compute-sanitizer
(memcheck / racecheck / synccheck): K1 fused factor (dense + CSR), K1L panel path
(d >= 64), K2/K3 prep, K5 prediction + vote, K7 fp64 kernel block, K4/K6 decision values
and resident-G sweeps, K8 per-point decision values.
  compute-sanitizer --tool racecheck python scripts/sanitize_kernels.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2207_01016_b200 as P  # noqa: E402
from conftest import np_gaussian_L  # noqa: E402

rng = np.random.default_rng(0)
ctx = P.Context(1)
for n, d, B in ((300, 50, 100), (600, 100, 300)):  # fused K1, then the d >= 64 panel path
    X = rng.standard_normal((n, d)).astype(np.float32).astype(np.float64)
    Y = X[rng.choice(n, B, replace=False)]
    L = np_gaussian_L(Y, 1.0 / d)
    ctx.set_basis_dense(Y, L, 1.0 / d)
    ctx.set_keep_resident(True)
    G = ctx.compute_g_dense(X)
    ip = np.zeros(n + 1, np.int64)
    ip[1:] = np.cumsum(np.full(n, d))
    G2 = ctx.compute_g_csr(ip, np.tile(np.arange(d, dtype=np.int32), n), X.ravel())
    assert np.array_equal(G, G2)
    rows = np.arange(0, n, 3, dtype=np.int32)
    ctx.resident_gw(rows, rng.standard_normal((1, G.shape[1])))
    ctx.resident_gw(rows, rng.standard_normal((5, G.shape[1])))
    ctx.resident_gw(rows, rng.standard_normal((20, G.shape[1])))  # 8-row tile shape, 2 vectors per thread
    ctx.resident_gw(rows, rng.standard_normal((45, G.shape[1])))  # 8-row tile shape, 3 vectors per thread
    ctx.resident_gw(rows, rng.standard_normal((70, G.shape[1])))  # 4-row tile shape, P-tiles of 64
    ctx.resident_vote(rows, rng.standard_normal((3, G.shape[1])), 3)
    ctx.resident_gtv(rows, rng.standard_normal(rows.shape[0]))
    if hasattr(ctx, "resident_gtv_sets"):
        ctx.resident_gtv_sets(rows, rng.standard_normal((rows.shape[0], 11)))
        ctx.resident_row_sqnorms()
    ctx.decision_values(G, rng.standard_normal((3, G.shape[1])))
    ctx.set_keep_resident(False)
    ctx.kernel_block(X[:70], Y, 1.0 / d)
    betas = rng.standard_normal((3, B))
    ctx.set_basis_dense(Y, np.ascontiguousarray(betas.T), 1.0 / d)
    ctx.predict_ovo_dense(X, 3)
    ctx.set_model_dense(Y, betas, 1.0 / d)
    ctx.model_decision_values_dense(X[:50])
    ctx.ovo_vote(rng.standard_normal((100, 3)), 3)
# K9: rows far from every landmark at a large γ raise the probe flag, so row_shift and
# row_rescale run for real (fused path, then the d >= 64 panel path; fp32 and fp64 G)
import torch  # noqa: E402

for d in (32, 96):
    Y = rng.standard_normal((160, d))
    X = rng.standard_normal((600, d))
    X[:200] += 3.0 * np.sqrt(d)
    gamma = 16.0 / d
    ctx.set_precision("fast")
    ctx.set_basis_dense(Y, np_gaussian_L(Y, gamma, 1e-6), gamma)
    ctx.compute_g_dense(X)
    Gd = torch.empty((600, ctx.b_eff), dtype=torch.float64, device="cuda")
    ctx.compute_g_device(torch.from_numpy(X).cuda(), Gd)
    torch.cuda.synchronize()
    ctx.set_precision("auto")
# K1 Z·β mode (b_eff <= 4): 1- and 4-wide tables, host rows, device rows (fp64, pitched) and K5
for k in (1, 4):
    X = rng.standard_normal((700, 40))
    Y = X[:150]
    ctx.set_basis_dense(Y, rng.standard_normal((150, k)), 1.0 / 40)
    ctx.compute_g_dense(X)
    Gf = torch.zeros((700, k + 3), dtype=torch.float64, device="cuda")
    ctx.compute_g_device(torch.from_numpy(X).cuda(), Gf[:, :k])
    torch.cuda.synchronize()
    if k == 1:
        ctx.predict_ovo_dense(X, 2)
ctx.close()
print("sanitize_kernels: every kernel ran")
