"""Every row of a one-GPU shard against the reference's own compute_G (oracle/_ref, all
host threads): max / quantiles of the row-normwise relative error over the whole shard,
not a sample. Test infrastructure (the reference runs on the host as the checker).

  python scripts/parity_full_shard.py c2 [out.json]     (C2: ~30 s of reference CPU time)
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench
import paper_2207_01016_b200 as P
from oracle import oracle as O
from paper_2207_01016_b200 import synthetic


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
    out_path = sys.argv[2] if len(sys.argv) > 2 else None
    cfg = synthetic.CONFIGS[wl]
    n = synthetic.rows_per_gpu(cfg)
    X, _ = synthetic.make(cfg, rows=slice(0, n))
    dev = torch.device("cuda", 0)
    Y, L = bench.make_basis(X, cfg, device=dev)
    b_eff = L.shape[1]
    G_dev = torch.empty((n, b_eff), dtype=torch.float32, device=dev)
    with P.Context(device_ids=[0]) as ctx:
        ctx.set_basis_device(torch.from_numpy(Y).to(dev), torch.from_numpy(L).to(dev), cfg.gamma)
        ctx.compute_g_device(torch.from_numpy(X).to(dev), G_dev)
        torch.cuda.synchronize()
    threads = O.ref_lib().ref_hardware_threads()
    ycsr = O.dense_to_csr(Y)
    errs = np.empty(n)
    t0 = time.perf_counter()
    blk = 32768
    for r0 in range(0, n, blk):
        r1 = min(n, r0 + blk)
        R = O.ref_compute_g(O.dense_to_csr(np.ascontiguousarray(X[r0:r1])), ycsr, L, cfg.gamma,
                            max(1, -(-(r1 - r0) // threads)), threads)
        Gb = G_dev[r0:r1].double().cpu().numpy()
        errs[r0:r1] = np.linalg.norm(Gb - R, axis=1) / np.linalg.norm(R, axis=1)
    secs = time.perf_counter() - t0
    w = int(np.argmax(errs))
    out = {"workload": cfg.name, "rows": n, "b_eff": b_eff, "reference_threads": threads,
           "reference_seconds": secs, "max_row_rel_err": float(errs.max()), "argmax_row": w,
           "p99_99": float(np.quantile(errs, 0.9999)), "p99": float(np.quantile(errs, 0.99)),
           "median": float(np.median(errs)), "rows_above_1e-4": int((errs > 1e-4).sum())}
    print(json.dumps(out))
    if out_path:
        with open(out_path, "w") as f:
            json.dump(out, f)


if __name__ == "__main__":
    main()
