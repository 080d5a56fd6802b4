"""Seeded random sweep of K5 prediction (lpd_predict_ovo_dense) and K8 per-point decision
values against the oracle: classes must equal the oracle's vote on every row whose
smallest |decision| is clear of fp32-level rounding; K8 values within 1e-10 relative.

  python scripts/fuzz_predict.py [first] [count]"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2207_01016_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402

first = int(sys.argv[1]) if len(sys.argv) > 1 else 0
count = int(sys.argv[2]) if len(sys.argv) > 2 else 50
ctx = P.Context(1)
bad = 0
for seed in range(first, first + count):
    rng = np.random.default_rng(5000 + seed)
    n = int(rng.integers(1, 1200)); d = int(rng.integers(1, 140)); B = int(rng.integers(1, 300))
    c = int(rng.integers(2, 9)); Pp = c * (c - 1) // 2
    gamma = float(np.exp(rng.uniform(np.log(0.1 / d), np.log(5.0 / d))))
    X = rng.standard_normal((n, d)).astype(np.float32).astype(np.float64)
    Y = rng.standard_normal((B, d)).astype(np.float32).astype(np.float64)
    betas = rng.standard_normal((Pp, B))
    ctx.set_basis_dense(Y, np.ascontiguousarray(betas.T), gamma)
    cls = ctx.predict_ovo_dense(X, c)
    Z = O.ora_kernel_block(O.dense_to_csr(X), O.dense_to_csr(Y), gamma)
    D = Z @ betas.T
    ref = np.array([O.ora_vote(D[i], c) for i in range(n)])
    clear = np.min(np.abs(D), axis=1) > 1e-4 * np.max(np.abs(D), axis=1) + 1e-30
    mism = int(np.sum((cls != ref) & clear))
    ctx.set_model_dense(Y, betas, gamma)
    Dm = ctx.model_decision_values_dense(X[: min(n, 200)])
    e8 = float(np.max(np.abs(Dm - D[: min(n, 200)])) / max(np.max(np.abs(D)), 1e-300))
    if mism or e8 > 1e-10:
        bad += 1
        print(f"FAIL seed {seed}: n {n} d {d} B {B} c {c} gamma*d {gamma * d:.3g} mismatches {mism} "
              f"of {int(clear.sum())} clear rows; K8 rel {e8:.2e}", flush=True)
print(f"seeds {first}..{first + count - 1}: {bad} failing")
