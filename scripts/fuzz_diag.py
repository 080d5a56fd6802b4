"""Seeded random-problem sweep (the fuzz test's generator, many more seeds): for each seed,
the worst row of the host path (fp32 G, rows inside fp32's range) and of the device path
(fp64 G) against the oracle, relative to the conditioned bound; prints the seeds that fail.

  python scripts/fuzz_diag.py [first] [count]"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import torch  # noqa: E402

import paper_2207_01016_b200 as P  # noqa: E402
from conftest import np_gaussian_L  # noqa: E402
from oracle import oracle as O  # noqa: E402


BIG = os.environ.get("FUZZ_BIG") == "1"  # the panel path at large d and B


def case(seed):
    rng = np.random.default_rng((3000 if BIG else 1000) + seed)
    if BIG:
        n = int(rng.integers(1, 3001)); d = int(rng.integers(200, 2101)); B = int(rng.integers(256, 2049))
    else:
        n = int(rng.integers(1, 1501)); d = int(rng.integers(1, 161)); B = int(rng.integers(1, 401))
    gamma = float(np.exp(rng.uniform(np.log(0.1 / d), np.log(10.0 / d))))
    scale = float(rng.choice([1.0, 1.0, 7.0]))
    X = (rng.standard_normal((n, d)) * scale).astype(np.float32).astype(np.float64)
    if rng.random() < 0.5:
        X[rng.random(X.shape) < 0.7] = 0.0
    Y = X[rng.choice(n, B, replace=False)] if B <= n else \
        (rng.standard_normal((B, d)) * scale).astype(np.float32).astype(np.float64)
    L = np_gaussian_L(Y, gamma, float(rng.choice([1e-10, 1e-6, 1e-3])))
    return n, d, B, gamma, scale, X, Y, L


first = int(sys.argv[1]) if len(sys.argv) > 1 else 0
count = int(sys.argv[2]) if len(sys.argv) > 2 else 100
only = [int(x) for x in os.environ.get("FUZZ_SEEDS", "").split(",") if x]
ctx = P.Context(1)
ctx.set_precision(os.environ.get("FUZZ_PRECISION", "auto"))
worst = (0.0, None)
for seed in (only or range(first, first + count)):
    n, d, B, gamma, scale, X, Y, L = case(seed)
    ctx.set_basis_dense(Y, L, gamma)
    G = ctx.compute_g_dense(X)
    Gd = torch.empty((n, L.shape[1]), dtype=torch.float64, device="cuda")
    ctx.compute_g_device(torch.from_numpy(X).cuda(), Gd)
    G64 = Gd.cpu().numpy()
    R = O.ora_compute_g(O.dense_to_csr(X), O.dense_to_csr(Y), L, gamma, 4096)
    Z = O.ora_kernel_block(O.dense_to_csr(X), O.dense_to_csr(Y), gamma)
    bound = np.maximum(1e-4 * np.linalg.norm(R, axis=1), 1e-5 * np.linalg.norm(Z, axis=1) * np.linalg.norm(L, 2))
    live = np.abs(R).max(axis=1) >= 2.0 ** -100
    r32 = (np.linalg.norm(G - R, axis=1) / np.maximum(bound, 1e-300))[live]
    r64 = np.linalg.norm(G64 - R, axis=1) / np.maximum(bound, 1e-300)
    m = max(r32.max() if r32.size else 0.0, r64.max())
    if len(sys.argv) > 3:  # calibration dump: basis exponent magnitude, estimate, observed row error
        mu = Y.mean(0)
        rb = np.linalg.norm(Y - mu, axis=1).max()
        tb = 13 + gamma * 1.4426950408889634 * (2 * rb) ** 2
        rx = np.linalg.norm(X - mu, axis=1)
        tx = 13 + gamma * 1.4426950408889634 * (rx + rb) ** 2
        nr = np.linalg.norm(R, axis=1)
        ok = nr > 1e-300
        rel = np.linalg.norm(G64 - R, axis=1)[ok] / nr[ok]
        print(f"CAL {seed} tb {tb:.4g} txmax {tx.max():.4g} est {ctx.basis_precision()[1]:.3g} relerr {rel.max():.3g} ratio {m:.3g}", flush=True)
    if m > worst[0]:
        worst = (m, seed)
    if m > 1.0:
        print(f"FAIL seed {seed}: n {n} d {d} B {B} gamma*d {gamma * d:.3g} scale {scale} b_eff {L.shape[1]} "
              f"host {r32.max() if r32.size else 0:.3g} device {r64.max():.3g}", flush=True)
print(f"seeds {first}..{first + count - 1}: worst ratio to the bound {worst[0]:.3g} (seed {worst[1]})")
