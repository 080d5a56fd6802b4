"""Seeded random sweep of the drop-in through the reference's Python API: for each seed,
tests/integration_train.py (train, predict, decision_values, cross_validate, a warm-started
grid) on the B200 build and on the unmodified reference build with the same random
settings (n, d, B, classes, γ, C, τ, sparsity via the index stride), compared the way
test_reference_api_on_gpu_matches_reference does.

  python scripts/fuzz_dropin.py [first] [count]"""
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUNNER = os.path.join(ROOT, "tests", "integration_train.py")


def run(build, out, args, env=None):
    r = subprocess.run([sys.executable, RUNNER, build, out, *args], capture_output=True, text=True, timeout=900,
                       env={**os.environ, **(env or {})})
    if r.returncode != 0:
        raise RuntimeError(r.stderr[-1500:])


first = int(sys.argv[1]) if len(sys.argv) > 1 else 0
count = int(sys.argv[2]) if len(sys.argv) > 2 else 10
bad = 0
for seed in range(first, first + count):
    rng = np.random.default_rng(7000 + seed)
    n = int(rng.integers(300, 5000)); d = int(rng.integers(2, 80)); B = int(rng.integers(20, min(n, 600)))
    classes = int(rng.integers(2, 6))
    gamma = float(np.exp(rng.uniform(np.log(0.3 / d), np.log(3.0 / d))))
    C = float(rng.choice([0.25, 1.0, 4.0]))
    tau = float(rng.choice([1e-12, 1e-6]))
    stride = int(rng.choice([1, 1, 3]))
    args = ["--n", str(n), "--n-test", "300", "--d", str(d), "--budget", str(B), "--classes", str(classes),
            "--gamma", str(gamma), "--C", str(C), "--tau", str(tau), "--index-stride", str(stride), "--threads", "8"]
    with tempfile.TemporaryDirectory() as tmp:
        try:
            run("integration/_build", f"{tmp}/g.npz", args, {"LPD_DEVICE_MIN_ELEMS": "0"})
            run("oracle/_ref", f"{tmp}/r.npz", args)
        except RuntimeError as e:
            bad += 1
            print(f"FAIL seed {seed} {args}: run error {e}", flush=True)
            continue
        g, r = np.load(f"{tmp}/g.npz"), np.load(f"{tmp}/r.npz")
        agree = float(np.mean(g["pred"] == r["pred"]))
        derr = abs(float(g["error_rate"]) - float(r["error_rate"]))
        dcv = abs(float(g["cv_mean_error"]) - float(r["cv_mean_error"]))
        dgrid = float(np.max(np.abs(g["grid_errors"] - r["grid_errors"])))
        dv = float(np.max(np.abs(g["dv"] - r["dv"])) / max(np.max(np.abs(r["dv"])), 1e-300))
        ok = agree >= 0.98 and derr <= 0.02 and dcv <= 0.02 and dgrid <= 0.02 and dv <= 5e-2 and \
            int(g["effective_rank"]) == int(r["effective_rank"])
        line = (f"seed {seed}: n {n} d {d} B {B} c {classes} gd {gamma * d:.2f} C {C} tau {tau} stride {stride} | "
                f"agree {agree:.4f} derr {derr:.4f} dcv {dcv:.4f} dgrid {dgrid:.4f} dv {dv:.2e} "
                f"rank {int(g['effective_rank'])}/{int(r['effective_rank'])}")
        if not ok:
            bad += 1
            print("FAIL " + line, flush=True)
        else:
            print("ok   " + line, flush=True)
print(f"seeds {first}..{first + count - 1}: {bad} failing")
