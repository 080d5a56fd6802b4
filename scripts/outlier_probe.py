import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); sys.path.insert(0, 'scripts')
import torch
import paper_2207_01016_b200 as P
from conftest import np_gaussian_L
from precision_probe import g64
rng = np.random.default_rng(3)
d, B, n = 32, 1024, 1536
ctx = P.Context(1)
base = rng.standard_normal((B + n, d)).astype(np.float32).astype(np.float64)
Y = base[:B]
for mult in (4.0, 8.0, 16.0):
    g = mult / d
    L = np_gaussian_L(Y, g, 1e-6)
    for shift in (4.0, 6.0, 8.0, 12.0):
        X = base[B:].copy(); u = rng.standard_normal(d); u /= np.linalg.norm(u)
        X[: n // 3] += shift * np.sqrt(d) * u
        X = X.astype(np.float32).astype(np.float64)
        ctx.set_basis_dense(Y, L, g)
        hp, est = ctx.basis_precision()
        Gd = torch.empty((n, L.shape[1]), dtype=torch.float64, device="cuda")
        ctx.compute_g_device(torch.from_numpy(X).cuda(), Gd)
        G = Gd.cpu().numpy(); R = g64(X, Y, L, g)
        nr = np.linalg.norm(R, axis=1); ok = nr > 0
        err = np.linalg.norm(G - R, axis=1)[ok] / nr[ok]
        mu = Y.mean(0); rb = np.linalg.norm(Y - mu, axis=1).max(); rx = np.linalg.norm(X - mu, axis=1)
        T = g * 1.4427 * (rx + rb) ** 2
        print(f"mult {mult} shift {shift} hp {hp} Tb {g*1.4427*4*rb*rb:.0f} Tmax {T.max():.0f} max err {err.max():.2e}", flush=True)
