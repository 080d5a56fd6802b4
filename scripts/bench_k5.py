"""K5 prediction (reference ovo_predict, multiclass.cpp:170-200: Z(points, landmarks)·βᵀ then
the one-vs-one vote) through the C ABI on C2-shaped data: n_test points, B = 4,096
landmarks, d = 54, binary (P = 1) and 10-class (P = 45) models with random β. Wall time of
lpd_set_basis_dense(landmarks, βᵀ) + lpd_predict_ovo_dense, median of the reps; kernel times
come from an ncu launch list of the same command.

  python scripts/bench_k5.py [--n-test 100000] [--reps 5]"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-test", type=int, default=100_000)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import paper_2207_01016_b200 as P
    from paper_2207_01016_b200 import synthetic

    cfg = synthetic.CONFIGS["c2"]
    X, _ = synthetic.make(cfg, rows=slice(0, args.n_test + cfg.budget))
    Y, Xt = X[: cfg.budget], np.ascontiguousarray(X[cfg.budget:])
    rng = np.random.default_rng(3)
    nnz = np.full(Xt.shape[0], cfg.d)
    ip = np.concatenate([[0], np.cumsum(nnz)]).astype(np.int64)
    ix = np.tile(np.arange(cfg.d, dtype=np.int32), Xt.shape[0])
    vv = Xt.ravel()
    out = {"n_test": int(Xt.shape[0]), "B": cfg.budget, "d": cfg.d, "gamma": cfg.gamma}
    with P.Context(1) as ctx:
        for classes in (2, 3, 10):
            Pp = classes * (classes - 1) // 2
            betas = rng.standard_normal((Pp, cfg.budget)) * 1e-2
            ts, tb = [], []
            bt = np.ascontiguousarray(betas.T)
            for _ in range(args.reps + 1):
                t0 = time.perf_counter()
                ctx.set_basis_dense(Y, bt, cfg.gamma)
                t1 = time.perf_counter()
                cls = ctx.predict_ovo_dense(Xt, classes)
                ts.append(time.perf_counter() - t0)
                tb.append(t1 - t0)
            t = float(np.median(ts[1:]))
            tc = []  # the same points as CSR (the adapter's ovo_predict path), basis already set
            for _ in range(args.reps + 1):
                t0 = time.perf_counter()
                cls_csr = ctx.predict_ovo_csr(ip, ix, vv, classes)
                tc.append(time.perf_counter() - t0)
            assert np.array_equal(cls_csr, cls)
            out[f"classes_{classes}"] = {"P": Pp, "seconds": t, "rows_per_s": Xt.shape[0] / t,
                                         "set_basis_seconds": float(np.median(tb[1:])),
                                         "csr_predict_seconds": float(np.median(tc[1:])),
                                         "high_precision_basis": bool(ctx.basis_precision()[0]),
                                         "class_histogram": np.bincount(cls, minlength=classes).tolist()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
