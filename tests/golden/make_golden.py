"""Generates the committed golden fixtures from the REFERENCE's own code.

Run in the build container (needs oracle/_ref, i.e. the reference sources
compiled unmodified by oracle/Makefile):  python tests/golden/make_golden.py

  spec_known_answers.json  SPEC.md known answers (analytic; SPEC line cited per entry)
  c1_mini.npz              C1 blobs, first 1024 rows, 128 landmarks chosen by the
                           reference select_landmarks(seed=1), L and G from the
                           reference build_factor_with_landmarks (factor.cpp:112-143)
  susy_mini.npz            SUSY-shaped d=18, gamma=2^-7 (ill-conditioned), n=512, B=256, tau=1e-6
  susy_mini_t12.npz        the same points and landmarks at the reference default tau=1e-12
                           (the high-precision path's fixture: lambda_min/lambda_max ~ 1e-12)
  sparse_mini.npz          random sparse CSR points incl. empty rows, n=300, d=40, B=64
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle import oracle as O  # noqa: E402
from paper_2207_01016_b200 import synthetic  # noqa: E402


def factor_fixture(X, budget, gamma, tau, seed=1):
    csr = O.dense_to_csr(X)
    ids = O.ref_select_landmarks(X.shape[0], budget, seed)
    Y = X[ids]
    f = O.ref_factor_with_landmarks(csr, O.dense_to_csr(Y), gamma, tau, 4096, 1)
    return ids, f


def main():
    spec = {
        "gaussian": [
            {"a": [[0, 1.0]], "b": [[0, 1.0]], "gamma": 3.7, "expect": 1.0, "spec": "SPEC.md:114 a=b -> 1"},
            {"a": [[0, 1.0]], "b": [[0, 2.0]], "gamma": float(np.log(2.0)), "expect": 0.5,
             "spec": "SPEC.md:115 ||a-b||^2=1, gamma=ln2 -> 0.5"},
            {"a": [[0, 1.0]], "b": [[1, 1.0]], "gamma": 0.5, "expect": float(np.exp(-1.0)),
             "spec": "SPEC.md:116 {1:1},{2:1}, gamma=0.5 -> exp(-1)"},
        ],
        "kernel_block_orthonormal": {"points": [[[0, 1.0]], [[1, 1.0]], [[2, 1.0]]], "gamma": 1.0,
                                     "diag": 1.0, "offdiag": float(np.exp(-2.0)),
                                     "spec": "SPEC.md:124 3 orthonormal unit points, gamma=1"},
        "build_L_scalar": {"K": 4.0, "L": 0.5, "spec": "SPEC.md:201 K=[4] -> L=[0.5]"},
        "compute_G_single_landmark": {"spec": "SPEC.md:211 B=1 -> G[i] = k(x_i, l)"},
    }
    with open(os.path.join(HERE, "spec_known_answers.json"), "w") as f:
        json.dump(spec, f, indent=1)

    X, y = synthetic.blobs(20_000, 50, 1, rows=slice(0, 1024))
    ids, f = factor_fixture(X, 128, 0.02, 1e-12)
    np.savez_compressed(os.path.join(HERE, "c1_mini.npz"), X=X.astype(np.float32), y=y, ids=ids,
                        L=f["L"], G=f["G"], gamma=0.02, tau=1e-12)

    rng = np.random.default_rng(7)
    Xs = rng.standard_normal((512, 18)).astype(np.float32).astype(np.float64)
    ids, f = factor_fixture(Xs, 256, 2.0 ** -7, 1e-6)
    np.savez_compressed(os.path.join(HERE, "susy_mini.npz"), X=Xs.astype(np.float32), ids=ids,
                        L=f["L"], G=f["G"], gamma=2.0 ** -7, tau=1e-6)
    ids, f = factor_fixture(Xs, 256, 2.0 ** -7, 1e-12)
    np.savez_compressed(os.path.join(HERE, "susy_mini_t12.npz"), X=Xs.astype(np.float32), ids=ids,
                        L=f["L"], G=f["G"], gamma=2.0 ** -7, tau=1e-12)

    rng = np.random.default_rng(11)
    Xp = rng.standard_normal((300, 40)).astype(np.float32).astype(np.float64)
    Xp[rng.random(Xp.shape) < 0.7] = 0.0
    Xp[[3, 17, 150]] = 0.0  # empty points
    ids, f = factor_fixture(Xp, 64, 0.1, 1e-12)
    np.savez_compressed(os.path.join(HERE, "sparse_mini.npz"), X=Xp.astype(np.float32), ids=ids,
                        L=f["L"], G=f["G"], gamma=0.1, tau=1e-12)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
