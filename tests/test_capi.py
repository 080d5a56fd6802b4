"""C-ABI library and host-side logic, no GPU needed (no compute calls)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2207_01016_b200 as P
from paper_2207_01016_b200 import sharding, synthetic

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "lpd_nystrom.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(lpd_\w+)\s*\(", text, re.M)))


def test_library_built_and_exports_header_symbols():
    assert os.path.exists(P.LIB_PATH), "liblpd_nystrom.so must be built in-tree"
    lib = ctypes.CDLL(P.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/lpd_nystrom.h but not exported"
    assert sorted(P.EXPORTED_SYMBOLS) == syms


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_device_count_without_compute():
    lib = P.load_library()
    assert lib.lpd_version() >= 10000
    assert lib.lpd_device_count() >= 0


def test_no_device_fails_loudly():
    if P.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(P.LpdError):
        P.Context(1)


def test_compute_G_argument_errors_match_reference():
    pts = np.zeros((3, 2))
    lms = np.zeros((2, 2))
    with pytest.raises(ValueError, match="chunk_size"):       # factor.cpp:87
        P.compute_G(pts, None, lms, None, np.eye(2), P.KernelParams(1.0), 0)
    with pytest.raises(ValueError, match="L row count"):      # factor.cpp:91
        P.compute_G(pts, None, lms, None, np.eye(3), P.KernelParams(1.0), 16)
    with pytest.raises(ValueError, match="gamma"):            # kernel.cpp:13-14
        P.compute_G(pts, None, lms, None, np.eye(2), P.KernelParams(-1.0), 16)
    with pytest.raises(ValueError, match="gamma"):
        P.compute_G(pts, None, lms, None, np.eye(2), P.KernelParams(float("inf")), 16)


def test_sparse_to_csr_reference_layout():
    pts = [[(0, 1.5), (3, -2.0)], [], [(1, 4.0)], np.array([0.0, 0.0, 7.0])]
    ip, ix, vv, dim = P.sparse_to_csr(pts)
    assert ip.tolist() == [0, 2, 2, 3, 4]
    assert ix.tolist() == [0, 3, 1, 2]
    assert vv.tolist() == [1.5, -2.0, 4.0, 7.0]
    assert dim == 4


@pytest.mark.parametrize("n,w", [(0, 1), (1, 1), (127, 2), (128, 2), (581_012, 8), (5_000_000, 8), (300, 7)])
def test_row_shard_partition(n, w):
    spans = [sharding.row_shard(n, w, r) for r in range(w)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c and a <= b
    for a, b in spans:
        assert a % sharding.ROW_ALIGN == 0 or a == n


def test_synthetic_row_ranges_consistent():
    X, y = synthetic.blobs(200_000, 6, 5)
    X2, y2 = synthetic.blobs(200_000, 6, 5, rows=slice(65_000, 140_000))
    assert np.array_equal(X[65_000:140_000], X2) and np.array_equal(y[65_000:140_000], y2)
    assert np.array_equal(X.astype(np.float32).astype(np.float64), X)  # fp32-representable
    assert abs(y.mean()) < 0.01
