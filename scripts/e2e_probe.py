"""e2e host-path breakdown (lpd_set_basis_dense + lpd_compute_g_dense into pageable fp64 G)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import bench
import paper_2207_01016_b200 as P
from paper_2207_01016_b200 import synthetic

cfg = synthetic.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
n = synthetic.rows_per_gpu(cfg)
X, _ = synthetic.make(cfg, rows=slice(0, n))
Y, L = bench.make_basis(X, cfg)
G = np.zeros((n, L.shape[1]))
import torch
Xp = torch.from_numpy(X).pin_memory().numpy()
with P.Context(1) as ctx:
    for i in range(3):
        t0 = time.perf_counter(); ctx.set_basis_dense(Y, L, cfg.gamma); print(f"set_basis (before compute) {time.perf_counter()-t0:.4f} s", flush=True)
    ctx.compute_g_dense(Xp, out=G)
    for _ in range(3):
        t0 = time.perf_counter(); ctx.set_basis_dense(Y, L, cfg.gamma); tb = time.perf_counter() - t0
        t = P.Timings()
        t0 = time.perf_counter()
        ctx.compute_g_dense(Xp, out=G, timings=t)
        dt = time.perf_counter() - t0
        print(f"set_basis {tb:.4f} s  compute wall {dt:.3f} s  {n/dt/1e6:.2f} M rows/s  {G.nbytes/dt/1e9:.1f} GB/s fp64 out  timings {t.as_dict()}", flush=True)
