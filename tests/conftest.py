import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (driver runs `pytest -m gpu` on the GPU box)")


@pytest.fixture(scope="session")
def gpu_ctx():
    """A one-device context. GPU tests must fail loudly, never skip, when the
    CUDA library or the device is missing."""
    import paper_2207_01016_b200 as P

    ctx = P.Context(1)
    yield ctx
    ctx.close()


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name)) as z:
        return {k: z[k] for k in z.files}


def row_rel_err(G, R):
    """max_i ||G_i - R_i|| / ||R_i|| (elementwise relative error on
    G is ill-posed because of near-zero entries; the criterion is row-normwise)."""
    num = np.linalg.norm(G - R, axis=1)
    den = np.linalg.norm(R, axis=1)
    return float(np.max(num / np.maximum(den, 1e-300))) if len(R) else 0.0


def np_gaussian_L(Y, gamma, tau=1e-12):
    """L = U D^-1/2 on retained eigenvalues (reference factor.cpp:33-81), numpy eigh;
    used only to build test inputs — both paths under comparison get this same L."""
    ny = (Y * Y).sum(1)
    K = np.exp(-gamma * np.maximum(ny[:, None] + ny[None, :] - 2.0 * Y @ Y.T, 0.0))
    w, U = np.linalg.eigh(0.5 * (K + K.T))
    w, U = w[::-1], U[:, ::-1]
    keep = w > tau * w[0]
    return np.ascontiguousarray(U[:, keep] / np.sqrt(w[keep]))
