"""Seeded random sweep of the resident-G products against host loops on the returned G:
scoring (bitwise, the reference's order), the device vote, rebuild_w (1e-12), the batched
warm starts (1e-12), row norms (bitwise), for one- and two-shard contexts on GPU 0.

  python scripts/fuzz_resident.py [first] [count]"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2207_01016_b200 as P  # noqa: E402
from conftest import np_gaussian_L  # noqa: E402
from oracle import oracle as O  # noqa: E402

first = int(sys.argv[1]) if len(sys.argv) > 1 else 0
count = int(sys.argv[2]) if len(sys.argv) > 2 else 40
bad = 0
for seed in range(first, first + count):
    rng = np.random.default_rng(9000 + seed)
    n = int(rng.integers(2, 5000)); d = int(rng.integers(1, 40)); B = int(rng.integers(1, min(n, 500) + 1))
    gamma = float(np.exp(rng.uniform(np.log(0.3 / d), np.log(3.0 / d))))
    X = rng.standard_normal((n, d)).astype(np.float32).astype(np.float64)
    Y = X[rng.choice(n, B, replace=False)]
    L = np_gaussian_L(Y, gamma, 1e-8)
    shards = 2 if seed % 2 else 1
    with P.Context(device_ids=[0] * shards) as ctx:
        ctx.set_basis_dense(Y, L, gamma)
        ctx.set_keep_resident(True)
        G = ctx.compute_g_dense(X)
        be = G.shape[1]
        rows = rng.choice(n, int(rng.integers(1, n + 1)), replace=True).astype(np.int32)
        msgs = []
        for Pp in (1, int(rng.integers(2, 5)), int(rng.integers(5, 80))):
            W = rng.standard_normal((Pp, be))
            D = ctx.resident_gw(rows, W)
            seq = np.add.accumulate(G[rows][:, None, :] * W[None, :, :], axis=2)[:, :, -1]
            if not np.array_equal(D, seq):
                msgs.append(f"gw P={Pp} max {np.max(np.abs(D - seq)):.2e}")
        c = int(rng.integers(2, 7))
        Wc = rng.standard_normal((c * (c - 1) // 2, be))
        cls = ctx.resident_vote(rows, Wc, c)
        Dc = ctx.resident_gw(rows, Wc)
        if not np.array_equal(cls, [O.ora_vote(x, c) for x in Dc]):
            msgs.append("vote")
        coef = rng.standard_normal(rows.size)
        w = ctx.resident_gtv(rows, coef)
        wr = coef @ G[rows]
        if np.max(np.abs(w - wr)) > 1e-12 * max(np.max(np.abs(wr)), 1e-300):
            msgs.append("gtv")
        S = int(rng.integers(1, 12))
        C = rng.standard_normal((rows.size, S))
        Ws = ctx.resident_gtv_sets(rows, C)
        Wr = C.T @ G[rows]
        if np.max(np.abs(Ws - Wr)) > 1e-12 * max(np.max(np.abs(Wr)), 1e-300):
            msgs.append("gtv_sets")
        q = ctx.resident_row_sqnorms()
        qr = np.array([np.add.accumulate(G[i] * G[i])[-1] for i in range(n)])
        if not np.array_equal(q, qr):
            msgs.append("sqnorms")
        ctx.set_keep_resident(False)
    if msgs:
        bad += 1
        print(f"FAIL seed {seed}: n {n} d {d} B {B} shards {shards}: {msgs}", flush=True)
print(f"seeds {first}..{first + count - 1}: {bad} failing")
