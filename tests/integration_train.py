"""Runs the reference's public Python API (`lpdsvm.train`, `Model.predict`,
`Model.decision_values`, `lpdsvm.cross_validate`) from one build of the
reference's `_core` module and saves the results, so two builds can be compared
in separate processes (two pybind11 modules registering the same C++ types cannot
share one interpreter).

  python tests/integration_train.py <module_dir> <out.npz> [--n N --d D --budget B ...]

<module_dir> is a directory holding `lpdsvm/_core*.so`:
  integration/_build  — the reference with compute_G served by the B200 library
  oracle/_ref         — the reference as is (CPU; test infrastructure)
"""
import argparse
import ctypes
import glob
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def libsvm_text(X, y, stride=1):
    # repr() of a float64 holding an fp32 value round-trips exactly through strtod;
    # feature j is written at index j·stride + 1 (stride > 1: a high-dimensional sparse set)
    lines = []
    for xi, yi in zip(X, y):
        feats = " ".join(f"{j * stride + 1}:{float(v)!r}" for j, v in enumerate(xi) if v != 0.0)
        lines.append(f"{int(yi)} {feats}")
    return "\n".join(lines) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("module_dir")
    ap.add_argument("out")
    ap.add_argument("--n", type=int, default=4000)
    ap.add_argument("--n-test", type=int, default=1000)
    ap.add_argument("--d", type=int, default=20)
    ap.add_argument("--budget", type=int, default=400)
    ap.add_argument("--gamma", type=float, default=0.05)
    ap.add_argument("--C", type=float, default=1.0)
    ap.add_argument("--classes", type=int, default=2)
    ap.add_argument("--threads", type=int, default=4, help="0 = all host threads")
    ap.add_argument("--tau", type=float, default=1e-6)
    ap.add_argument("--seed", type=int, default=11)
    ap.add_argument("--train-only", action="store_true", help="train + predict only (timing runs)")
    ap.add_argument("--index-stride", type=int, default=1,
                    help="feature j at index j*stride+1 (a sparse set of dimension ~d*stride)")
    args = ap.parse_args()

    mdir = args.module_dir if os.path.isabs(args.module_dir) else os.path.join(ROOT, args.module_dir)
    sys.path.insert(0, mdir)
    if os.path.isdir(os.path.join(mdir, "lpdsvm")):
        import lpdsvm  # the build under test (package layout of the reference)
    else:
        import _core as lpdsvm  # oracle/_ref ships the bare extension module

    sys.path.insert(0, ROOT)
    from paper_2207_01016_b200 import synthetic

    if args.classes == 2:
        X, y = synthetic.blobs(args.n + args.n_test, args.d, seed=args.seed)
    else:
        X, y = synthetic.imagenet_like(args.n + args.n_test, args.d, args.classes, seed=args.seed)
        X = X / 4.0  # keep γ·d² in a useful range for the small test
        X = X.astype(np.float32).astype(np.float64)
    t0 = time.perf_counter()
    train = lpdsvm.parse_dataset(libsvm_text(X[: args.n], y[: args.n], args.index_stride))
    test = lpdsvm.parse_dataset(libsvm_text(X[args.n :], y[args.n :], args.index_stride))
    parse_s = time.perf_counter() - t0

    t0 = time.perf_counter()
    model, stats = lpdsvm.train(train, budget=args.budget, C=args.C, gamma=args.gamma,
                                threads=args.threads, tau=args.tau)
    train_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    pred = model.predict(test, threads=args.threads)
    predict_s = time.perf_counter() - t0
    if args.train_only:
        import json

        # second, steady-state run in the same process (the first one also pays one-time
        # CUDA driver/context initialisation on the GPU build)
        t0 = time.perf_counter()
        model2, stats2 = lpdsvm.train(train, budget=args.budget, C=args.C, gamma=args.gamma,
                                      threads=args.threads, tau=args.tau)
        train2_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        pred2 = model2.predict(test, threads=args.threads)
        predict2_s = time.perf_counter() - t0
        extra = {}
        so = glob.glob(os.path.join(os.path.dirname(lpdsvm.__file__), "_core*.so"))[0]
        lib = ctypes.CDLL(so)
        if hasattr(lib, "lpd_adapter_phases"):
            ph = (ctypes.c_double * 4)()
            lib.lpd_adapter_phases(ph)
            tm = (ctypes.c_double * 10)()  # lpd_timings (64 bytes): total, h2d, kernel, d2h, host_copy, ...
            lib.lpd_adapter_last_timings(ctypes.cast(tm, ctypes.c_void_p))
            extra["compute_G_phases"] = {"flatten": ph[0], "basis": ph[1], "matrix_alloc_zero_fill": ph[2],
                                         "device_call": ph[3], "device_call_total": tm[0],
                                         "h2d_event_s": tm[1], "kernel_event_s": tm[2], "d2h_event_s": tm[3],
                                         "host_widen_s": tm[4]}
        out = {"build": args.module_dir, "n": args.n, "d": args.d, "budget": args.budget, **extra,
               "effective_rank": model.effective_rank, "threads": args.threads,
               "parse_seconds": parse_s,
               "cold": {"train_wall_seconds": train_s, "predict_seconds": predict_s,
                        **{k: stats[k] for k in ("preparation_seconds", "gmatrix_seconds", "training_seconds")}},
               "train_wall_seconds": train2_s, "predict_seconds": predict2_s,
               "test_error": float(np.mean(pred2 != y[args.n:])), **{k: stats2[k] for k in stats2}}
        with open(args.out, "w") as f:
            json.dump(out, f)
        np.save(args.out + ".pred.npy", pred2)
        print(json.dumps(out))
        return
    dv = model.decision_values(test)
    cv = lpdsvm.cross_validate(train, budget=args.budget, C=args.C, gamma=args.gamma, folds=3,
                               threads=args.threads, tau=args.tau)
    # warm-started (gamma, C) grid: exercises rebuild_w on the warm starts
    grid = lpdsvm.grid_search(train, gammas=[args.gamma], Cs=[0.5 * args.C, args.C], budget=args.budget,
                              folds=3, threads=args.threads, tau=args.tau)

    so = glob.glob(os.path.join(os.path.dirname(lpdsvm.__file__), "_core*.so"))[0]
    # (for the package layout, __file__ is lpdsvm/__init__.py next to _core*.so)
    lib = ctypes.CDLL(so)
    adapter_calls = predict_calls = block_calls = sweep_calls = score_calls = qdiag_calls = warm_batches = -1
    host_calls = -1
    if hasattr(lib, "lpd_adapter_calls"):
        lib.lpd_adapter_calls.restype = ctypes.c_longlong
        lib.lpd_adapter_predict_calls.restype = ctypes.c_longlong
        adapter_calls = int(lib.lpd_adapter_calls())
        predict_calls = int(lib.lpd_adapter_predict_calls())
        lib.lpd_adapter_block_calls.restype = ctypes.c_longlong
        block_calls = int(lib.lpd_adapter_block_calls())
        lib.lpd_adapter_sweep_calls.restype = ctypes.c_longlong
        lib.lpd_adapter_score_calls.restype = ctypes.c_longlong
        sweep_calls = int(lib.lpd_adapter_sweep_calls())
        score_calls = int(lib.lpd_adapter_score_calls())
        lib.lpd_adapter_qdiag_calls.restype = ctypes.c_longlong
        lib.lpd_adapter_warm_batches.restype = ctypes.c_longlong
        qdiag_calls = int(lib.lpd_adapter_qdiag_calls())
        warm_batches = int(lib.lpd_adapter_warm_batches())
        lib.lpd_adapter_host_calls.restype = ctypes.c_longlong
        host_calls = int(lib.lpd_adapter_host_calls())
    np.savez(
        args.out,
        pred=pred,
        dv=dv,
        y_test=y[args.n :],
        error_rate=model.error_rate(test),
        cv_mean_error=cv["mean_error"],
        cv_fold_errors=cv["fold_errors"],
        effective_rank=model.effective_rank,
        gmatrix_seconds=stats["gmatrix_seconds"],
        preparation_seconds=stats["preparation_seconds"],
        training_seconds=stats["training_seconds"],
        train_wall_seconds=train_s,
        epochs=stats["epochs"],
        adapter_calls=adapter_calls,
        predict_calls=predict_calls,
        block_calls=block_calls,
        sweep_calls=sweep_calls,
        score_calls=score_calls,
        qdiag_calls=qdiag_calls,
        warm_batches=warm_batches,
        host_calls=host_calls,
        cv_fold_epochs=np.array(cv["fold_epochs"]) if "fold_epochs" in cv else np.zeros(0),
        grid_errors=np.array([e["mean_error"] for e in grid["entries"]]),
        grid_warm=grid["warm_started_solves"],
        model_text=np.array(model.to_string()),
    )
    print(f"{args.module_dir}: error {model.error_rate(test):.4f} cv {cv['mean_error']:.4f} "
          f"gmatrix {stats['gmatrix_seconds']:.3f}s adapter_calls {adapter_calls}")


if __name__ == "__main__":
    main()
