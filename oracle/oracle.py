"""Oracle access — TEST INFRASTRUCTURE ONLY.

ctypes wrappers for
  * ``oracle/_build/liboracle.so``  — the plain-C restatement (lpd_oracle.c), and
  * ``oracle/_ref/liblpdsvm_ref.so`` — the reference's own sources compiled
    unmodified (oracle/Makefile) behind ref_harness.cpp,
plus the reference's pybind11 module ``_core`` (oracle/_ref).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg import
this module, and only as the checker / the timed reference arm. The B200
product path (paper_2207_01016_b200) never imports it.
"""
from __future__ import annotations

import ctypes
import os
import sys
from typing import Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(HERE, "_build", "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "liblpdsvm_ref.so")
REF_DIR = os.path.join(HERE, "_ref")

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_dp = ctypes.POINTER(ctypes.c_double)

_ora = None
_ref = None


def _p(a, t=ctypes.c_double):
    return a.ctypes.data_as(ctypes.POINTER(t))


def oracle_lib() -> ctypes.CDLL:
    global _ora
    if _ora is None:
        if not os.path.exists(ORACLE_LIB):
            raise RuntimeError(f"{ORACLE_LIB} missing: run `make -C oracle`")
        lib = ctypes.CDLL(ORACLE_LIB)
        lib.ora_squared_norms.argtypes = [ctypes.c_int64, _i64p, _dp, _dp]
        lib.ora_gaussian.argtypes = [_i32p, _dp, ctypes.c_int64, _i32p, _dp, ctypes.c_int64, ctypes.c_double]
        lib.ora_gaussian.restype = ctypes.c_double
        lib.ora_kernel_block.argtypes = [ctypes.c_int64, _i64p, _i32p, _dp, _dp, ctypes.c_int64, _i64p,
                                         _i32p, _dp, _dp, ctypes.c_double, _dp]
        lib.ora_compute_g.argtypes = [ctypes.c_int64, _i64p, _i32p, _dp, _dp, ctypes.c_int64, _i64p,
                                      _i32p, _dp, _dp, _dp, ctypes.c_int64, ctypes.c_double,
                                      ctypes.c_int64, _dp]
        lib.ora_compute_g.restype = ctypes.c_int
        lib.ora_decision_values.argtypes = [ctypes.c_int64, _i64p, _dp, ctypes.c_int64, ctypes.c_int64,
                                            _dp, ctypes.c_int64, _dp]
        lib.ora_vote.argtypes = [_dp, ctypes.c_int64]
        lib.ora_vote.restype = ctypes.c_int
        lib.ora_combine_seed.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        lib.ora_combine_seed.restype = ctypes.c_uint64
        lib.ora_select_landmarks.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, _i32p]
        lib.ora_select_landmarks.restype = ctypes.c_int64
        _ora = lib
    return _ora


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def ref_lib() -> ctypes.CDLL:
    global _ref
    if _ref is None:
        if not os.path.exists(REF_LIB):
            raise RuntimeError(f"{REF_LIB} missing: run `make -C oracle` where /root/reference exists")
        lib = ctypes.CDLL(REF_LIB)
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_hardware_threads.restype = ctypes.c_int
        lib.ref_gaussian.argtypes = [ctypes.c_int64, _i32p, _dp, ctypes.c_int64, _i32p, _dp, ctypes.c_double]
        lib.ref_gaussian.restype = ctypes.c_double
        lib.ref_kernel_block.argtypes = [ctypes.c_int64, _i64p, _i32p, _dp, ctypes.c_int64, _i64p, _i32p,
                                         _dp, ctypes.c_double, ctypes.c_int, _dp]
        lib.ref_squared_norms.argtypes = [ctypes.c_int64, _i64p, _i32p, _dp, _dp]
        lib.ref_compute_g.argtypes = [ctypes.c_int64, _i64p, _i32p, _dp, ctypes.c_int64, _i64p, _i32p, _dp,
                                      _dp, ctypes.c_int64, ctypes.c_double, ctypes.c_int64, ctypes.c_int,
                                      _dp, _dp]
        lib.ref_select_landmarks.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, _i32p]
        lib.ref_select_landmarks.restype = ctypes.c_int64
        lib.ref_factor_with_landmarks.argtypes = [ctypes.c_int64, _i64p, _i32p, _dp, ctypes.c_int64, _i64p,
                                                  _i32p, _dp, ctypes.c_double, ctypes.c_double,
                                                  ctypes.c_int64, ctypes.c_int, _i64p, _dp, _dp]
        lib.ref_factor_with_landmarks.restype = ctypes.c_void_p
        lib.ref_build_factor.argtypes = [ctypes.c_int64, _i64p, _i32p, _dp, ctypes.c_int64, ctypes.c_double,
                                         ctypes.c_double, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64,
                                         _i64p, _i64p, _dp, _dp]
        lib.ref_build_factor.restype = ctypes.c_void_p
        lib.ref_factor_copy.argtypes = [ctypes.c_void_p, _dp, _dp, _i32p]
        lib.ref_factor_free.argtypes = [ctypes.c_void_p]
        lib.ref_vote.argtypes = [_dp, ctypes.c_int64, ctypes.c_int64]
        lib.ref_vote.restype = ctypes.c_int
        lib.ref_solve_binary.argtypes = [ctypes.c_int64, ctypes.c_int64, _dp, _dp, ctypes.c_double,
                                         ctypes.c_double, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64,
                                         ctypes.c_uint64, _dp, _dp, _dp, _dp]
        _ref = lib
    return _ref


def ref_core():
    """The reference's pybind11 module (import name ``_core``)."""
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import _core  # noqa: E402

    return _core


# ----------------------------------------------------------------------------- CSR helpers
def dense_to_csr(X: np.ndarray) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Dense rows -> CSR with explicit zeros dropped (reference parse drops them,
    dataio.cpp:112-113)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    mask = X != 0.0
    counts = mask.sum(axis=1)
    indptr = np.zeros(X.shape[0] + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    rows, cols = np.nonzero(mask)
    return indptr, cols.astype(np.int32), X[rows, cols].astype(np.float64)


def _csr(a):
    ip, ix, vv = a
    return (np.ascontiguousarray(ip, np.int64), np.ascontiguousarray(ix, np.int32),
            np.ascontiguousarray(vv, np.float64))


# ----------------------------------------------------------------------------- restatement
def ora_squared_norms(csr) -> np.ndarray:
    ip, ix, vv = _csr(csr)
    out = np.empty(ip.shape[0] - 1)
    oracle_lib().ora_squared_norms(out.shape[0], _p(ip, ctypes.c_int64), _p(vv), _p(out))
    return out


def ora_kernel_block(a, b, gamma: float) -> np.ndarray:
    ap, ai, av = _csr(a)
    bp, bi, bv = _csr(b)
    na, nb = ap.shape[0] - 1, bp.shape[0] - 1
    norms_a, norms_b = ora_squared_norms((ap, ai, av)), ora_squared_norms((bp, bi, bv))
    out = np.empty((na, nb))
    oracle_lib().ora_kernel_block(na, _p(ap, ctypes.c_int64), _p(ai, ctypes.c_int32), _p(av), _p(norms_a),
                                  nb, _p(bp, ctypes.c_int64), _p(bi, ctypes.c_int32), _p(bv), _p(norms_b),
                                  float(gamma), _p(out))
    return out


def ora_gaussian(a_idx, a_val, b_idx, b_val, gamma: float) -> float:
    ai = np.ascontiguousarray(a_idx, np.int32); av = np.ascontiguousarray(a_val, np.float64)
    bi = np.ascontiguousarray(b_idx, np.int32); bv = np.ascontiguousarray(b_val, np.float64)
    return oracle_lib().ora_gaussian(_p(ai, ctypes.c_int32), _p(av), len(ai), _p(bi, ctypes.c_int32),
                                     _p(bv), len(bi), float(gamma))


def ora_compute_g(points, landmarks, L: np.ndarray, gamma: float, chunk_size: int = 4096) -> np.ndarray:
    xp, xi, xv = _csr(points)
    lp, li, lv = _csr(landmarks)
    n, b = xp.shape[0] - 1, lp.shape[0] - 1
    Lm = np.ascontiguousarray(L, np.float64)
    if Lm.shape[0] != b:
        raise ValueError("L row count must match landmark count")
    xn, ln = ora_squared_norms((xp, xi, xv)), ora_squared_norms((lp, li, lv))
    G = np.empty((n, Lm.shape[1]))
    rc = oracle_lib().ora_compute_g(n, _p(xp, ctypes.c_int64), _p(xi, ctypes.c_int32), _p(xv), _p(xn), b,
                                    _p(lp, ctypes.c_int64), _p(li, ctypes.c_int32), _p(lv), _p(ln), _p(Lm),
                                    Lm.shape[1], float(gamma), int(chunk_size), _p(G))
    if rc == -1:
        raise ValueError("invalid argument")
    if rc != 0:
        raise MemoryError("oracle allocation failed")
    return G


def ora_decision_values(G: np.ndarray, W: np.ndarray, rows: Optional[np.ndarray] = None) -> np.ndarray:
    G = np.ascontiguousarray(G, np.float64)
    W = np.ascontiguousarray(np.atleast_2d(W), np.float64)
    rid = None if rows is None else np.ascontiguousarray(rows, np.int64)
    nr = G.shape[0] if rid is None else rid.shape[0]
    D = np.empty((nr, W.shape[0]))
    oracle_lib().ora_decision_values(nr, None if rid is None else _p(rid, ctypes.c_int64), _p(G), G.shape[1],
                                     G.shape[1], _p(W), W.shape[0], _p(D))
    return D


def ora_vote(decisions: np.ndarray, num_classes: int) -> int:
    d = np.ascontiguousarray(decisions, np.float64)
    return int(oracle_lib().ora_vote(_p(d), int(num_classes)))


def ora_select_landmarks(n: int, budget: int, seed: int) -> np.ndarray:
    out = np.empty(min(n, budget), np.int32)
    k = oracle_lib().ora_select_landmarks(int(n), int(budget), int(seed), _p(out, ctypes.c_int32))
    if k < 0:
        raise ValueError("invalid landmark request")
    return out[:k]


# ----------------------------------------------------------------------------- reference build
def _ref_err() -> str:
    return (ref_lib().ref_last_error() or b"").decode()


def ref_kernel_block(a, b, gamma: float, threads: int = 1) -> np.ndarray:
    ap, ai, av = _csr(a)
    bp, bi, bv = _csr(b)
    na, nb = ap.shape[0] - 1, bp.shape[0] - 1
    out = np.empty((na, nb))
    rc = ref_lib().ref_kernel_block(na, _p(ap, ctypes.c_int64), _p(ai, ctypes.c_int32), _p(av), nb,
                                    _p(bp, ctypes.c_int64), _p(bi, ctypes.c_int32), _p(bv), float(gamma),
                                    int(threads), _p(out))
    if rc:
        raise (ValueError if rc == 1 else RuntimeError)(_ref_err())
    return out


def ref_squared_norms(csr) -> np.ndarray:
    ip, ix, vv = _csr(csr)
    out = np.empty(ip.shape[0] - 1)
    ref_lib().ref_squared_norms(out.shape[0], _p(ip, ctypes.c_int64), _p(ix, ctypes.c_int32), _p(vv), _p(out))
    return out


def ref_gaussian(a_idx, a_val, b_idx, b_val, gamma: float) -> float:
    ai = np.ascontiguousarray(a_idx, np.int32); av = np.ascontiguousarray(a_val, np.float64)
    bi = np.ascontiguousarray(b_idx, np.int32); bv = np.ascontiguousarray(b_val, np.float64)
    return ref_lib().ref_gaussian(len(ai), _p(ai, ctypes.c_int32), _p(av), len(bi), _p(bi, ctypes.c_int32),
                                  _p(bv), float(gamma))


def ref_compute_g(points, landmarks, L: np.ndarray, gamma: float, chunk_size: int = 4096,
                  threads: int = 1, return_seconds: bool = False):
    xp, xi, xv = _csr(points)
    lp, li, lv = _csr(landmarks)
    n, b = xp.shape[0] - 1, lp.shape[0] - 1
    Lm = np.ascontiguousarray(L, np.float64)
    G = np.empty((n, Lm.shape[1]))
    secs = ctypes.c_double(0.0)
    rc = ref_lib().ref_compute_g(n, _p(xp, ctypes.c_int64), _p(xi, ctypes.c_int32), _p(xv), b,
                                 _p(lp, ctypes.c_int64), _p(li, ctypes.c_int32), _p(lv), _p(Lm), Lm.shape[1],
                                 float(gamma), int(chunk_size), int(threads), _p(G), ctypes.byref(secs))
    if rc:
        raise (ValueError if rc == 1 else RuntimeError)(_ref_err())
    return (G, secs.value) if return_seconds else G


def ref_select_landmarks(n: int, budget: int, seed: int) -> np.ndarray:
    out = np.empty(min(n, budget), np.int32)
    k = ref_lib().ref_select_landmarks(int(n), int(budget), int(seed), _p(out, ctypes.c_int32))
    if k < 0:
        raise ValueError(_ref_err())
    return out[:k]


def ref_factor_with_landmarks(points, landmarks, gamma: float, tau: float = 1e-12, chunk_size: int = 4096,
                              threads: int = 1) -> dict:
    """Reference build_factor_with_landmarks (factor.cpp:112-143): L, G, b_eff, timings."""
    xp, xi, xv = _csr(points)
    lp, li, lv = _csr(landmarks)
    n, b = xp.shape[0] - 1, lp.shape[0] - 1
    b_eff = ctypes.c_int64(0)
    prep = ctypes.c_double(0.0)
    gm = ctypes.c_double(0.0)
    h = ref_lib().ref_factor_with_landmarks(n, _p(xp, ctypes.c_int64), _p(xi, ctypes.c_int32), _p(xv), b,
                                            _p(lp, ctypes.c_int64), _p(li, ctypes.c_int32), _p(lv),
                                            float(gamma), float(tau), int(chunk_size), int(threads),
                                            ctypes.byref(b_eff), ctypes.byref(prep), ctypes.byref(gm))
    if not h:
        raise RuntimeError(_ref_err())
    try:
        L = np.empty((b, b_eff.value))
        G = np.empty((n, b_eff.value))
        ref_lib().ref_factor_copy(h, _p(L), _p(G), None)
    finally:
        ref_lib().ref_factor_free(h)
    return {"L": L, "G": G, "b_eff": b_eff.value, "preparation_seconds": prep.value,
            "gmatrix_seconds": gm.value}


def ref_build_L(landmarks, gamma: float, tau: float = 1e-12, threads: int = 1) -> np.ndarray:
    """L exactly as the reference builds it (kernel_block -> eig_sym -> truncate -> build_L),
    via build_factor_with_landmarks on zero points."""
    lp, li, lv = _csr(landmarks)
    empty = (np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float64))
    return ref_factor_with_landmarks(empty, (lp, li, lv), gamma, tau, 4096, threads)["L"]


def ref_vote(decisions: np.ndarray, num_classes: int) -> int:
    d = np.ascontiguousarray(decisions, np.float64)
    return int(ref_lib().ref_vote(_p(d), d.shape[0], int(num_classes)))


def ref_solve_binary(G: np.ndarray, y: np.ndarray, C: float = 1.0, eps: float = 1e-3,
                     max_epochs: int = 1000, shrinking: bool = True, seed: int = 1,
                     problem_tag: int = 0, warm_alpha: Optional[np.ndarray] = None) -> dict:
    """The reference's make_binary_problem + solve_binary (dcd.cpp:60-89, 212-259) over all
    rows of G: alpha, w and the SolveReport (dual objective D(alpha) = sum(alpha) - |w|^2/2,
    dcd.cpp:104-108)."""
    G = np.ascontiguousarray(G, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    n, b = G.shape
    alpha = np.empty(n)
    w = np.empty(b)
    rep = np.empty(6)
    wa = None if warm_alpha is None else np.ascontiguousarray(warm_alpha, np.float64)
    rc = ref_lib().ref_solve_binary(n, b, _p(G), _p(y), float(C), float(eps), int(max_epochs),
                                    int(bool(shrinking)), int(seed), int(problem_tag),
                                    None if wa is None else _p(wa), _p(alpha), _p(w), _p(rep))
    if rc != 0:
        raise (ValueError if rc == 1 else RuntimeError)(_ref_err())
    return {"alpha": alpha, "w": w, "dual_objective": float(rep[0]), "epochs": int(rep[1]),
            "visits": int(rep[2]), "final_violation": float(rep[3]), "converged": bool(rep[4]),
            "shrunk_peak": int(rep[5])}
