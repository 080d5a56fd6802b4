import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2207_01016_b200 as P
from conftest import load_golden, row_rel_err
with P.Context(1) as ctx:
    for name in ["c1_mini.npz", "sparse_mini.npz", "susy_mini.npz"]:
        g = load_golden(name)
        X = g["X"].astype(np.float64); Y = X[g["ids"]]
        ctx.set_basis_dense(Y, g["L"], float(g["gamma"]))
        G = ctx.compute_g_dense(X)
        print(name, X.shape, g["L"].shape, "row err", row_rel_err(G, g["G"]))
