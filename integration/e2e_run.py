#!/usr/bin/env python3
"""Drives integration/e2e_harness.cpp (the reference's public C++ API) over one build and
prints one JSON object. bench.py runs it in a subprocess per build, because the drop-in
build and the reference build define the same C++ symbols.

  python integration/e2e_run.py b200|ref compute_g <basis.npz> [--rows N] [--steps K]
      gmatrix stage (squared_norms + compute_G into a fresh Matrix, factor.cpp:129-133)
      for the first N rows of the bench workload, with the bench's landmarks and L
  python integration/e2e_run.py b200|ref train <c1|c2> [--n-test M]
      lpdsvm.train's train_impl (module.cpp:35-78) + error rate on held-out rows

Builds: b200 = integration/_build/libe2e_b200.so (compute_G, the landmark Gram, the
solver sweeps and ovo_predict on the B200); ref = oracle/_ref/libe2e_ref.so (the
unmodified reference on the host cores).
"""
import argparse
import ctypes
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

LIBS = {"b200": os.path.join(ROOT, "integration", "_build", "libe2e_b200.so"),
        "ref": os.path.join(ROOT, "oracle", "_ref", "libe2e_ref.so")}
_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)


def _p(a, t=ctypes.c_double):
    return a.ctypes.data_as(ctypes.POINTER(t))


def load(build):
    lib = ctypes.CDLL(LIBS[build])
    lib.e2e_last_error.restype = ctypes.c_char_p
    lib.e2e_hardware_threads.restype = ctypes.c_int
    lib.e2e_compute_g.argtypes = [ctypes.c_int64, _i64p, _i32p, _dp, ctypes.c_int64, _i64p, _i32p, _dp, _dp,
                                  ctypes.c_int64, ctypes.c_double, ctypes.c_int64, ctypes.c_int, ctypes.c_int64,
                                  _dp, _dp]
    lib.e2e_train.argtypes = [ctypes.c_int64, _i64p, _i32p, _dp, _dp, ctypes.c_int64, _i64p, _i32p, _dp, _dp,
                              ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                              ctypes.c_double, ctypes.c_int, ctypes.c_uint64, _dp]
    return lib


def csr(X):
    """Dense rows -> CSR without explicit zeros (a SparseVector never holds one,
    dataio.cpp:112-113)."""
    mask = X != 0.0
    indptr = np.zeros(X.shape[0] + 1, np.int64)
    np.cumsum(mask.sum(1), out=indptr[1:])
    cols = np.broadcast_to(np.arange(X.shape[1], dtype=np.int32), X.shape)
    return indptr, np.ascontiguousarray(cols[mask]), np.ascontiguousarray(X[mask])


def check(lib, rc):
    if rc != 0:
        raise RuntimeError(lib.e2e_last_error().decode())


def adapter_phases(lib):
    """The B200 build's breakdown of its last compute_G call (None for the reference build)."""
    if not hasattr(lib, "lpd_adapter_phases"):
        return None
    ph = (ctypes.c_double * 4)()
    lib.lpd_adapter_phases(ph)
    tm = (ctypes.c_double * 8)()  # lpd_timings: total, h2d, kernel, d2h, host_copy (s), ...
    lib.lpd_adapter_last_timings(ctypes.cast(tm, ctypes.c_void_p))
    return {"flatten": ph[0], "basis": ph[1], "matrix_alloc": ph[2], "device_call": ph[3],
            "h2d_event_s": tm[1], "kernel_event_s": tm[2], "d2h_event_s": tm[3], "host_widen_s": tm[4]}


def run_compute_g(lib, args):
    from paper_2207_01016_b200 import synthetic

    z = np.load(args.target)
    Y, L, gamma, workload = z["Y"], np.ascontiguousarray(z["L"]), float(z["gamma"]), str(z["workload"])
    cfg = {c.name: c for c in synthetic.CONFIGS.values()}[workload]
    n = args.rows
    X, _ = synthetic.make(cfg, rows=slice(0, n), n=max(n, cfg.n))
    xp, xi, xv = csr(X)
    lp, li, lv = csr(Y)
    threads = lib.e2e_hardware_threads()
    b, b_eff = L.shape
    k = min(256, n)
    sample = np.empty((k, b_eff))
    secs = np.zeros(3)

    per_call = []

    def call():
        check(lib, lib.e2e_compute_g(n, _p(xp, ctypes.c_int64), _p(xi, ctypes.c_int32), _p(xv), b,
                                     _p(lp, ctypes.c_int64), _p(li, ctypes.c_int32), _p(lv), _p(L), b_eff, gamma,
                                     4096, threads, k, _p(sample), _p(secs)))
        if args.per_call:
            per_call.append({"gmatrix_seconds": secs[0], "phases": adapter_phases(lib)})
        return secs.copy()

    for _ in range(args.warmup):
        call()
    runs = [call() for _ in range(args.steps)]
    stage = statistics.median(r[0] for r in runs)
    out = {"build": args.build, "workload": workload, "rows": n, "b_eff": int(b_eff), "threads": threads,
           "gmatrix_seconds": stage, "compute_G_seconds": statistics.median(r[1] for r in runs),
           "matrix_free_seconds": statistics.median(r[2] for r in runs), "rows_per_s": n / stage,
           "steps": args.steps, "warmup": args.warmup}
    if per_call:
        out["per_call"] = per_call
    if (ph := adapter_phases(lib)) is not None:  # the B200 build: where the last call's time went
        out["adapter_phases"] = ph
    if "G_sample" in z.files:  # spot check against the device-path rows bench.py produced
        ref = z["G_sample"][:k]
        out["sample_max_row_rel_diff"] = float(np.max(np.linalg.norm(sample - ref, axis=1)
                                                      / np.linalg.norm(ref, axis=1)))
    return out


def run_train(lib, args):
    from paper_2207_01016_b200 import synthetic

    cfg = synthetic.CONFIGS[args.target]
    n, n_test = cfg.n, args.n_test
    X, y = synthetic.blobs(n + n_test, cfg.d, seed=cfg.seed)
    threads = lib.e2e_hardware_threads()
    out = np.zeros(11)

    def train(Xa, ya, Xt, yt, budget):
        a, t = csr(Xa), csr(Xt)
        check(lib, lib.e2e_train(Xa.shape[0], _p(a[0], ctypes.c_int64), _p(a[1], ctypes.c_int32), _p(a[2]),
                                 _p(np.ascontiguousarray(ya)), Xt.shape[0], _p(t[0], ctypes.c_int64),
                                 _p(t[1], ctypes.c_int32), _p(t[2]), _p(np.ascontiguousarray(yt)), budget,
                                 cfg.C, cfg.gamma, 1e-3, 1e-12, threads, 1, _p(out)))
        return out.copy()

    # warm-up on a small problem: process-level one-time costs (CUDA context on the B200
    # build, thread pools, page cache) stay out of the timed train
    train(X[:2000], y[:2000], X[n:n + 100], y[n:n + 100], 100)
    vm0 = vmstat()
    o = train(X[:n], y[:n], X[n:], y[n:], cfg.budget)
    vm1 = vmstat()
    return {"build": args.build, "workload": cfg.name, "n": n, "n_test": n_test, "d": cfg.d, "B": cfg.budget,
            "gamma": cfg.gamma, "C": cfg.C, "eps": 1e-3, "tau": 1e-12, "threads": threads,
            "train_seconds": o[0], "preparation_seconds": o[1], "gmatrix_seconds": o[2],
            "training_seconds": o[3], "predict_seconds": o[4], "test_error": o[5], "epochs": int(o[6]),
            "b_eff": int(o[7]), "unconverged_pairs": int(o[8]), "dual_objective": o[9],
            "coordinate_visits": int(o[10]),
            # the host's huge-page faults during the train (the gmatrix stage's fresh 19 GB G is
            # first-touched on huge pages; fallbacks / direct compaction slow it down)
            "host_thp": {k: vm1.get(k, 0) - vm0.get(k, 0) for k in vm1},
            "adapter_phases": adapter_phases(lib)}


def vmstat():
    keys = ("thp_fault_alloc", "thp_fault_fallback", "compact_stall")
    try:
        with open("/proc/vmstat") as f:
            return {k: int(v) for k, v in (line.split() for line in f) if k in keys}
    except OSError:
        return {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("build", choices=sorted(LIBS))
    ap.add_argument("task", choices=["compute_g", "train"])
    ap.add_argument("target", help="basis .npz (compute_g) or config name (train)")
    ap.add_argument("--rows", type=int, default=0)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--n-test", type=int, default=10_000)
    ap.add_argument("--per-call", action="store_true", help="compute_g: record every call (warm-up included)")
    args = ap.parse_args()
    lib = load(args.build)
    t0 = time.perf_counter()
    res = run_compute_g(lib, args) if args.task == "compute_g" else run_train(lib, args)
    res["wall_seconds"] = time.perf_counter() - t0
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
