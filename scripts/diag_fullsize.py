"""Per-row error diagnostics of a full one-GPU shard vs the reference compute_G."""
import json, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
import paper_2207_01016_b200 as P
from paper_2207_01016_b200 import synthetic
from oracle import oracle as O

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
nsamp = int(sys.argv[2]) if len(sys.argv) > 2 else 1500
cfg = synthetic.CONFIGS[wl]
n = synthetic.rows_per_gpu(cfg)
X, _ = synthetic.make(cfg, rows=slice(0, n))
dev = torch.device("cuda", 0)
Y, L, ids = bench.make_basis(X, cfg, device=dev, return_ids=True)
b_eff = L.shape[1]
X_dev = torch.from_numpy(X).to(dev)
G_dev = torch.empty((n, b_eff), dtype=torch.float32, device=dev)
ctx = P.Context(device_ids=[0])
ctx.set_basis_device(torch.from_numpy(Y).to(dev), torch.from_numpy(L).to(dev), cfg.gamma)
ctx.compute_g_device(X_dev, G_dev)
torch.cuda.synchronize()
rng = np.random.default_rng(1)
rows = np.unique(np.concatenate([rng.choice(n, nsamp, replace=False), ids[:16]]))
threads = O.ref_lib().ref_hardware_threads()
R = O.ref_compute_g(O.dense_to_csr(np.ascontiguousarray(X[rows])), O.dense_to_csr(Y), L, cfg.gamma,
                    max(1, -(-len(rows) // threads)), threads)
Gs = G_dev[torch.from_numpy(rows).to(dev)].double().cpu().numpy()
err = np.linalg.norm(Gs - R, axis=1) / np.linalg.norm(R, axis=1)
# same rows computed alone, as one small batch
G_alone = torch.empty((len(rows), b_eff), dtype=torch.float32, device=dev)
ctx.compute_g_device(X_dev[torch.from_numpy(rows).to(dev)].contiguous(), G_alone)
torch.cuda.synchronize()
Ga = G_alone.double().cpu().numpy()
err_alone = np.linalg.norm(Ga - R, axis=1) / np.linalg.norm(R, axis=1)
# fp64 device output for the same rows
G64 = torch.empty((len(rows), b_eff), dtype=torch.float64, device=dev)
ctx.compute_g_device(X_dev[torch.from_numpy(rows).to(dev)].contiguous(), G64)
torch.cuda.synchronize()
err64 = np.linalg.norm(G64.cpu().numpy() - R, axis=1) / np.linalg.norm(R, axis=1)
# column-wise error profile of the worst row
w = int(np.argmax(err))
colerr = np.abs(Gs[w] - R[w])
isl = np.isin(rows, ids)
out = {
    "workload": wl, "n": n, "b_eff": b_eff, "rows": len(rows),
    "max_err": float(err.max()), "median_err": float(np.median(err)), "p99_err": float(np.quantile(err, 0.99)),
    "max_err_alone": float(err_alone.max()), "max_err_f64_alone": float(err64.max()),
    "landmark_rows_max_err": float(err[isl].max()) if isl.any() else None,
    "nonlandmark_rows_max_err": float(err[~isl].max()),
    "worst": [{"row": int(rows[i]), "tile_row": int(rows[i] % 256), "err": float(err[i]),
               "err_alone": float(err_alone[i]), "norm": float(np.linalg.norm(R[i])),
               "landmark": bool(isl[i])} for i in np.argsort(-err)[:15]],
    "worst_row_top_cols": [[int(c), float(colerr[c]), float(R[w, c])] for c in np.argsort(-colerr)[:10]],
    "bitwise_alone_eq": bool(np.array_equal(Gs, Ga)),
}
print(json.dumps(out, indent=1))
