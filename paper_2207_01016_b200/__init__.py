"""B200-native Nyström factor path of LPD-SVM (arXiv 2207.01016).

Python mirror of the reference's factor interface over the C ABI in
``include/lpd_nystrom.h`` (``liblpd_nystrom.so``, built in-tree). The reference
entry point this mirrors is ``lpdsvm::compute_G`` (reference
proj/include/lpdsvm/factor.hpp:50-55, proj/src/factor.cpp:83-110); argument
meaning and error behaviour follow it:

* ``chunk_size == 0``          -> ValueError  (factor.cpp:87, std::invalid_argument)
* ``L.rows != len(landmarks)`` -> ValueError  (factor.cpp:91)
* γ not positive and finite    -> ValueError  (kernel.cpp:10-15)
* device / driver failures     -> RuntimeError (std::runtime_error)

There is no CPU fallback: when the CUDA library cannot be loaded or no B200 is
visible, every compute call raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

__all__ = [
    "LIB_PATH",
    "LpdError",
    "Context",
    "Timings",
    "KernelParams",
    "load_library",
    "device_count",
    "compute_G",
    "sparse_to_csr",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# LPD_LIBRARY: an alternative in-tree build of the same library (profiling variants)
LIB_PATH = os.environ.get("LPD_LIBRARY") or os.path.join(_HERE, "liblpd_nystrom.so")

LPD_OK = 0
LPD_ERR_INVALID_ARGUMENT = 1
LPD_ERR_CUDA = 2
LPD_ERR_UNSUPPORTED = 3
LPD_ERR_OUT_OF_MEMORY = 4
LPD_ERR_NO_DEVICE = 5
LPD_FAULT_NONE = 0
LPD_FAULT_ALLOC = 1
LPD_FAULT_LAUNCH = 2
LPD_FAULT_D2H = 3
LPD_OUT_F64 = 0
LPD_OUT_F32 = 1
LPD_PRECISION_AUTO = 0
LPD_PRECISION_FAST = 1
LPD_PRECISION_HIGH = 2

# Every symbol include/lpd_nystrom.h declares (checked by the CPU test suite).
EXPORTED_SYMBOLS = (
    "lpd_last_error",
    "lpd_version",
    "lpd_device_count",
    "lpd_inject_fault",
    "lpd_context_create",
    "lpd_context_create_devices",
    "lpd_context_destroy",
    "lpd_context_num_devices",
    "lpd_set_basis_dense",
    "lpd_set_basis_csr",
    "lpd_compute_g_dense",
    "lpd_compute_g_csr",
    "lpd_compute_g_device",
    "lpd_decision_values_device",
    "lpd_decision_values",
    "lpd_last_factor_kernel_ms",
    "lpd_set_basis_device",
    "lpd_factor_kernel_stats",
    "lpd_predict_ovo_dense",
    "lpd_predict_ovo_csr",
    "lpd_kernel_block",
    "lpd_set_keep_resident",
    "lpd_resident_shape",
    "lpd_resident_gw",
    "lpd_resident_vote",
    "lpd_resident_gtv",
    "lpd_set_model_dense",
    "lpd_set_model_csr",
    "lpd_model_decision_values_dense",
    "lpd_model_decision_values_csr",
    "lpd_ovo_vote",
    "lpd_resident_gtv_sets",
    "lpd_resident_row_sqnorms",
    "lpd_set_precision",
    "lpd_basis_precision",
    "lpd_compute_g_rows",
)


class LpdError(RuntimeError):
    """Device-side failure (the reference's std::runtime_error)."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


class Timings(ctypes.Structure):
    _fields_ = [
        ("total_seconds", ctypes.c_double),
        ("h2d_seconds", ctypes.c_double),
        ("kernel_seconds", ctypes.c_double),
        ("d2h_seconds", ctypes.c_double),
        ("host_copy_seconds", ctypes.c_double),
        ("rows", ctypes.c_int64),
        ("launches", ctypes.c_int64),
        ("devices", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_ if name != "reserved"}


@dataclass(frozen=True)
class KernelParams:
    """reference proj/include/lpdsvm/kernel.hpp:11-19 (Gaussian only)."""

    gamma: float = 1.0


_lib = None

_c_dbl_p = ctypes.POINTER(ctypes.c_double)
_c_i64_p = ctypes.POINTER(ctypes.c_int64)
_c_i32_p = ctypes.POINTER(ctypes.c_int32)


def load_library(path: Optional[str] = None) -> ctypes.CDLL:
    """Load liblpd_nystrom.so (in-tree). Raises if it has not been built."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError(
            f"{p} is missing: build the CUDA library first (python -c 'import __graft_entry__ as g; g.build()' or make)"
        )
    lib = ctypes.CDLL(p)
    vp = ctypes.c_void_p
    i64 = ctypes.c_int64
    lib.lpd_last_error.restype = ctypes.c_char_p
    lib.lpd_version.restype = ctypes.c_int
    lib.lpd_device_count.restype = ctypes.c_int
    lib.lpd_context_create.argtypes = [ctypes.POINTER(vp), ctypes.c_int]
    lib.lpd_context_create_devices.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_int), ctypes.c_int]
    lib.lpd_context_destroy.argtypes = [vp]
    lib.lpd_context_num_devices.argtypes = [vp]
    lib.lpd_set_basis_dense.argtypes = [vp, _c_dbl_p, i64, i64, i64, _c_dbl_p, i64, ctypes.c_double]
    lib.lpd_set_basis_csr.argtypes = [vp, i64, i64, _c_i64_p, _c_i32_p, _c_dbl_p, _c_dbl_p, i64,
                                      ctypes.c_double]
    lib.lpd_compute_g_dense.argtypes = [vp, _c_dbl_p, i64, i64, i64, _c_dbl_p, i64,
                                        ctypes.POINTER(Timings)]
    lib.lpd_compute_g_csr.argtypes = [vp, i64, i64, _c_i64_p, _c_i32_p, _c_dbl_p, _c_dbl_p, i64,
                                      ctypes.POINTER(Timings)]
    lib.lpd_compute_g_device.argtypes = [vp, ctypes.c_int, vp, i64, i64, vp, i64, ctypes.c_int, vp]
    lib.lpd_decision_values_device.argtypes = [vp, ctypes.c_int, vp, ctypes.c_int, i64, i64, i64,
                                               vp, i64, vp, i64, vp]
    lib.lpd_decision_values.argtypes = [vp, _c_dbl_p, i64, i64, i64, _c_dbl_p, i64, _c_dbl_p, i64]
    lib.lpd_last_factor_kernel_ms.argtypes = [vp, ctypes.c_int]
    lib.lpd_last_factor_kernel_ms.restype = ctypes.c_double
    lib.lpd_set_basis_device.argtypes = [vp, ctypes.c_int, vp, i64, i64, i64, vp, i64, ctypes.c_double, vp]
    lib.lpd_factor_kernel_stats.argtypes = [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                            ctypes.POINTER(ctypes.c_int64), ctypes.c_int]
    lib.lpd_kernel_block.argtypes = [vp, i64, _c_i64_p, _c_i32_p, _c_dbl_p, _c_dbl_p, i64, _c_i64_p,
                                     _c_i32_p, _c_dbl_p, _c_dbl_p, i64, ctypes.c_double, _c_dbl_p, i64]
    lib.lpd_set_keep_resident.argtypes = [vp, ctypes.c_int]
    lib.lpd_resident_shape.argtypes = [vp, _c_i64_p, _c_i64_p]
    lib.lpd_resident_gw.argtypes = [vp, _c_i32_p, i64, _c_dbl_p, i64, _c_dbl_p]
    lib.lpd_resident_vote.argtypes = [vp, _c_i32_p, i64, _c_dbl_p, i64, _c_i32_p]
    lib.lpd_resident_gtv.argtypes = [vp, _c_i32_p, _c_dbl_p, i64, _c_dbl_p]
    lib.lpd_predict_ovo_dense.argtypes = [vp, _c_dbl_p, i64, i64, i64, i64, _c_i32_p]
    lib.lpd_predict_ovo_csr.argtypes = [vp, i64, i64, _c_i64_p, _c_i32_p, _c_dbl_p, i64, _c_i32_p]
    lib.lpd_set_model_dense.argtypes = [vp, _c_dbl_p, i64, i64, i64, _c_dbl_p, i64, ctypes.c_double]
    lib.lpd_set_model_csr.argtypes = [vp, i64, i64, _c_i64_p, _c_i32_p, _c_dbl_p, _c_dbl_p, i64,
                                      ctypes.c_double]
    lib.lpd_model_decision_values_dense.argtypes = [vp, _c_dbl_p, i64, i64, i64, _c_dbl_p, i64]
    lib.lpd_model_decision_values_csr.argtypes = [vp, i64, i64, _c_i64_p, _c_i32_p, _c_dbl_p, _c_dbl_p, i64]
    lib.lpd_ovo_vote.argtypes = [vp, _c_dbl_p, i64, i64, i64, _c_i32_p]
    lib.lpd_resident_gtv_sets.argtypes = [vp, _c_i32_p, _c_dbl_p, i64, i64, _c_dbl_p]
    lib.lpd_resident_row_sqnorms.argtypes = [vp, _c_dbl_p]
    lib.lpd_set_precision.argtypes = [vp, ctypes.c_int]
    lib.lpd_basis_precision.argtypes = [vp, ctypes.POINTER(ctypes.c_int), _c_dbl_p]
    if path is None:
        _lib = lib
    return lib


def _check(status: int) -> None:
    if status == LPD_OK:
        return
    msg = (_lib.lpd_last_error() or b"").decode(errors="replace")
    if status == LPD_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    raise LpdError(status, msg)


def device_count() -> int:
    return int(load_library().lpd_device_count())


def inject_fault(site: int, after: int = 0) -> None:
    """Test hook: the after-th next pass through `site` (LPD_FAULT_ALLOC / _LAUNCH / _D2H)
    fails like the real CUDA failure would; LPD_FAULT_NONE disarms."""
    lib = load_library()
    lib.lpd_inject_fault.argtypes = [ctypes.c_int, ctypes.c_int]
    _check(lib.lpd_inject_fault(int(site), int(after)))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray, ctype=ctypes.c_double):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def sparse_to_csr(points: Sequence) -> tuple:
    """Flatten a sequence of sparse points into (indptr, indices, values, dim).

    A point is either a dense 1-D array or a sequence of (index, value) pairs
    with strictly ascending 0-based indices, the reference's SparseVector
    (proj/include/lpdsvm/dataio.hpp:14-24). dim = 1 + max index (0 if empty).
    """
    indptr = np.zeros(len(points) + 1, dtype=np.int64)
    idx_parts, val_parts = [], []
    dim = 0
    for i, p in enumerate(points):
        if isinstance(p, np.ndarray) and p.ndim == 1 and p.dtype.kind == "f":
            nz = np.flatnonzero(p)
            idx = nz.astype(np.int32)
            val = p[nz].astype(np.float64)
            dim = max(dim, p.shape[0])
        else:
            if len(p):
                idx = np.fromiter((f[0] for f in p), dtype=np.int32, count=len(p))
                val = np.fromiter((f[1] for f in p), dtype=np.float64, count=len(p))
                dim = max(dim, int(idx.max()) + 1)
            else:
                idx = np.zeros(0, np.int32)
                val = np.zeros(0, np.float64)
        idx_parts.append(idx)
        val_parts.append(val)
        indptr[i + 1] = indptr[i] + len(idx)
    indices = np.concatenate(idx_parts) if idx_parts else np.zeros(0, np.int32)
    values = np.concatenate(val_parts) if val_parts else np.zeros(0, np.float64)
    return indptr, indices.astype(np.int32), values, dim


class Context:
    """A set of B200 devices holding one replicated basis (landmarks, L, γ)."""

    def __init__(self, num_devices: int = 0, device_ids: Optional[Sequence[int]] = None):
        self._lib = load_library()
        h = ctypes.c_void_p()
        if device_ids is not None:
            ids = (ctypes.c_int * len(device_ids))(*device_ids)
            _check(self._lib.lpd_context_create_devices(ctypes.byref(h), ids, len(device_ids)))
        else:
            _check(self._lib.lpd_context_create(ctypes.byref(h), int(num_devices)))
        self._h = h
        self.b_eff = 0
        self.dim = 0
        self.model_pairs = 0

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    @property
    def num_devices(self) -> int:
        return int(self._lib.lpd_context_num_devices(self._h))

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.lpd_context_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- basis
    def set_basis_dense(self, landmarks: np.ndarray, L: np.ndarray, gamma: float) -> None:
        lm = _f64(landmarks)
        if lm.ndim != 2:
            raise ValueError("landmarks must be a 2-D array")
        Lm = _f64(L)
        if Lm.ndim != 2 or Lm.shape[0] != lm.shape[0]:
            raise ValueError("L row count must match landmark count")
        _check(self._lib.lpd_set_basis_dense(self._h, _ptr(lm), lm.shape[0], lm.shape[1],
                                             lm.shape[1], _ptr(Lm), Lm.shape[1], float(gamma)))
        self.b_eff, self.dim = Lm.shape[1], lm.shape[1]

    def set_basis_csr(self, indptr, indices, values, dim: int, L: np.ndarray, gamma: float) -> None:
        ip = np.ascontiguousarray(indptr, dtype=np.int64)
        ix = np.ascontiguousarray(indices, dtype=np.int32)
        vv = _f64(values)
        Lm = _f64(L)
        B = ip.shape[0] - 1
        if Lm.ndim != 2 or Lm.shape[0] != B:
            raise ValueError("L row count must match landmark count")
        _check(self._lib.lpd_set_basis_csr(self._h, B, int(dim), _ptr(ip, ctypes.c_int64),
                                           _ptr(ix, ctypes.c_int32), _ptr(vv), _ptr(Lm),
                                           Lm.shape[1], float(gamma)))
        self.b_eff, self.dim = Lm.shape[1], int(dim)

    # ---------------------------------------------------------------- rows
    def compute_g_dense(self, X: np.ndarray, out: Optional[np.ndarray] = None,
                        timings: Optional[Timings] = None) -> np.ndarray:
        x = _f64(X)
        if x.ndim != 2:
            raise ValueError("X must be 2-D")
        n = x.shape[0]
        G = out if out is not None else np.empty((n, self.b_eff), dtype=np.float64)
        if G.dtype != np.float64 or not G.flags.c_contiguous or G.shape != (n, self.b_eff):
            raise ValueError("out must be a C-contiguous float64 (n, b_eff) array")
        t = timings if timings is not None else Timings()
        _check(self._lib.lpd_compute_g_dense(self._h, _ptr(x), n, x.shape[1], x.shape[1], _ptr(G),
                                             self.b_eff, ctypes.byref(t)))
        return G

    def compute_g_csr(self, indptr, indices, values, out: Optional[np.ndarray] = None,
                      timings: Optional[Timings] = None) -> np.ndarray:
        ip = np.ascontiguousarray(indptr, dtype=np.int64)
        ix = np.ascontiguousarray(indices, dtype=np.int32)
        vv = _f64(values)
        n = ip.shape[0] - 1
        G = out if out is not None else np.empty((n, self.b_eff), dtype=np.float64)
        if G.dtype != np.float64 or not G.flags.c_contiguous or G.shape != (n, self.b_eff):
            raise ValueError("out must be a C-contiguous float64 (n, b_eff) array")
        t = timings if timings is not None else Timings()
        _check(self._lib.lpd_compute_g_csr(self._h, n, self.dim, _ptr(ip, ctypes.c_int64),
                                           _ptr(ix, ctypes.c_int32), _ptr(vv), _ptr(G),
                                           self.b_eff, ctypes.byref(t)))
        return G

    def compute_g_device(self, X_dev, G_dev, device_index: int = 0, stream=None) -> None:
        """X_dev (n x d fp64) and G_dev (n x b_eff, fp64 or fp32) are torch CUDA tensors."""
        import torch

        if X_dev.dtype != torch.float64 or not X_dev.is_contiguous():
            raise ValueError("X_dev must be a contiguous float64 CUDA tensor")
        if G_dev.dtype not in (torch.float64, torch.float32):
            raise ValueError("G_dev must be float64 or float32")
        out_dtype = LPD_OUT_F64 if G_dev.dtype == torch.float64 else LPD_OUT_F32
        st = ctypes.c_void_p(stream.cuda_stream) if stream is not None else None
        _check(self._lib.lpd_compute_g_device(self._h, device_index, ctypes.c_void_p(X_dev.data_ptr()),
                                              X_dev.shape[0], X_dev.stride(0),
                                              ctypes.c_void_p(G_dev.data_ptr()), G_dev.stride(0),
                                              out_dtype, st))

    def set_basis_device(self, landmarks_dev, L_dev, gamma: float, device_index: int = 0, stream=None) -> None:
        """Basis from torch CUDA fp64 tensors (landmarks B x d, L B x b_eff), K2 on device."""
        import torch

        if landmarks_dev.dtype != torch.float64 or L_dev.dtype != torch.float64:
            raise ValueError("landmarks and L must be float64 CUDA tensors")
        if not L_dev.is_contiguous() or landmarks_dev.stride(1) != 1:
            raise ValueError("row-major tensors required")
        if L_dev.shape[0] != landmarks_dev.shape[0]:
            raise ValueError("L row count must match landmark count")
        st = ctypes.c_void_p(stream.cuda_stream) if stream is not None else None
        _check(self._lib.lpd_set_basis_device(self._h, device_index, ctypes.c_void_p(landmarks_dev.data_ptr()),
                                              landmarks_dev.shape[0], landmarks_dev.shape[1],
                                              landmarks_dev.stride(0), ctypes.c_void_p(L_dev.data_ptr()),
                                              L_dev.shape[1], float(gamma), st))
        self.b_eff, self.dim = L_dev.shape[1], landmarks_dev.shape[1]

    def factor_kernel_stats(self, device_index: int = 0, reset: bool = True):
        """(total_ms, launches) of the fused factor kernel since the last reset."""
        tot = ctypes.c_double(0.0)
        cnt = ctypes.c_int64(0)
        _check(self._lib.lpd_factor_kernel_stats(self._h, device_index, ctypes.byref(tot), ctypes.byref(cnt),
                                                 int(reset)))
        return tot.value, cnt.value

    def last_factor_kernel_ms(self, device_index: int = 0) -> float:
        return float(self._lib.lpd_last_factor_kernel_ms(self._h, device_index))

    # ---------------------------------------------------------------- decision values
    def predict_ovo_dense(self, X: np.ndarray, num_classes: int) -> np.ndarray:
        """Class indices of the one-vs-one vote for dense rows X; the basis must
        have been set with L := betas.T (reference ovo_predict, multiclass.cpp:170-200)."""
        x = _f64(X)
        out = np.empty(x.shape[0], dtype=np.int32)
        _check(self._lib.lpd_predict_ovo_dense(self._h, _ptr(x), x.shape[0], x.shape[1], x.shape[1],
                                               num_classes, _ptr(out, ctypes.c_int32)))
        return out

    def predict_ovo_csr(self, indptr, indices, values, num_classes: int) -> np.ndarray:
        ip = np.ascontiguousarray(indptr, dtype=np.int64)
        ix = np.ascontiguousarray(indices, dtype=np.int32)
        vv = _f64(values)
        n = ip.shape[0] - 1
        out = np.empty(n, dtype=np.int32)
        _check(self._lib.lpd_predict_ovo_csr(self._h, n, self.dim, _ptr(ip, ctypes.c_int64),
                                             _ptr(ix, ctypes.c_int32), _ptr(vv), num_classes,
                                             _ptr(out, ctypes.c_int32)))
        return out

    # ---------------------------------------------------------------- precision
    def set_precision(self, mode: str) -> None:
        """'auto' (default), 'fast' (tensor-core split-fp16) or 'high' (fp64 Z + fp64 DMMA
        projection); applies from the next set_basis_*."""
        modes = {"auto": LPD_PRECISION_AUTO, "fast": LPD_PRECISION_FAST, "high": LPD_PRECISION_HIGH}
        if mode not in modes:
            raise ValueError(f"precision mode must be one of {sorted(modes)}")
        _check(self._lib.lpd_set_precision(self._h, modes[mode]))

    def basis_precision(self) -> tuple:
        """(high: bool, estimate: float) for the current basis."""
        hi, est = ctypes.c_int(), ctypes.c_double()
        _check(self._lib.lpd_basis_precision(self._h, ctypes.byref(hi), ctypes.byref(est)))
        return bool(hi.value), est.value

    # ------------------------------------------------- per-point decision values (K8)
    def set_model_dense(self, landmarks: np.ndarray, betas: np.ndarray, gamma: float) -> None:
        """A trained OVO model (landmarks B × d, betas P × B — OvoModel::betas,
        multiclass.hpp:63) for model_decision_values_*."""
        lm = _f64(landmarks)
        bt = _f64(np.atleast_2d(betas))
        if lm.ndim != 2 or bt.shape[1] != lm.shape[0]:
            raise ValueError("betas must be P x B with B = landmark count")
        self.model_dim = lm.shape[1]
        _check(self._lib.lpd_set_model_dense(self._h, _ptr(lm), lm.shape[0], lm.shape[1], lm.shape[1],
                                             _ptr(bt), bt.shape[0], float(gamma)))
        self.model_pairs = bt.shape[0]

    def set_model_csr(self, indptr, indices, values, dim: int, betas: np.ndarray, gamma: float) -> None:
        ip = np.ascontiguousarray(indptr, dtype=np.int64)
        ix = np.ascontiguousarray(indices, dtype=np.int32)
        vv = _f64(values)
        bt = _f64(np.atleast_2d(betas))
        if bt.shape[1] != ip.shape[0] - 1:
            raise ValueError("betas must be P x B with B = landmark count")
        self.model_dim = int(dim)
        _check(self._lib.lpd_set_model_csr(self._h, ip.shape[0] - 1, int(dim), _ptr(ip, ctypes.c_int64),
                                           _ptr(ix, ctypes.c_int32), _ptr(vv), _ptr(bt), bt.shape[0],
                                           float(gamma)))
        self.model_pairs = bt.shape[0]

    def model_decision_values_dense(self, X: np.ndarray) -> np.ndarray:
        """Per-point decision values D (n × P) in fp64, the reference's
        decision_values (multiclass.cpp:137-151) for every row of X."""
        x = _f64(np.atleast_2d(X))
        D = np.empty((x.shape[0], self.model_pairs))
        _check(self._lib.lpd_model_decision_values_dense(self._h, _ptr(x), x.shape[0], x.shape[1], x.shape[1],
                                                         _ptr(D), self.model_pairs))
        return D

    def model_decision_values_csr(self, indptr, indices, values, dim: int) -> np.ndarray:
        ip = np.ascontiguousarray(indptr, dtype=np.int64)
        ix = np.ascontiguousarray(indices, dtype=np.int32)
        vv = _f64(values)
        D = np.empty((ip.shape[0] - 1, self.model_pairs))
        _check(self._lib.lpd_model_decision_values_csr(self._h, ip.shape[0] - 1, int(dim),
                                                       _ptr(ip, ctypes.c_int64), _ptr(ix, ctypes.c_int32),
                                                       _ptr(vv), _ptr(D), self.model_pairs))
        return D

    def ovo_vote(self, D: np.ndarray, num_classes: int) -> np.ndarray:
        """Class indices of the one-vs-one vote on given decision values
        (multiclass.cpp:153-168), on the device."""
        d = _f64(np.atleast_2d(D))
        out = np.empty(d.shape[0], dtype=np.int32)
        _check(self._lib.lpd_ovo_vote(self._h, _ptr(d), d.shape[0], d.shape[1], int(num_classes),
                                      _ptr(out, ctypes.c_int32)))
        return out

    # ------------------------------------------------------- resident G (K6)
    def set_keep_resident(self, enable: bool = True) -> None:
        """Keep the fp32 G of later compute_g_* calls on the devices (config 5)."""
        _check(self._lib.lpd_set_keep_resident(self._h, int(bool(enable))))

    def resident_shape(self) -> tuple:
        n, b = ctypes.c_int64(), ctypes.c_int64()
        _check(self._lib.lpd_resident_shape(self._h, ctypes.byref(n), ctypes.byref(b)))
        return n.value, b.value

    def resident_gw(self, rows, W: np.ndarray) -> np.ndarray:
        """D = G[rows] · Wᵀ on the resident G (held-out CV scoring, modelsel.cpp:123-140)."""
        r = np.ascontiguousarray(rows, dtype=np.int32)
        w = _f64(np.atleast_2d(W))
        D = np.empty((r.shape[0], w.shape[0]))
        _check(self._lib.lpd_resident_gw(self._h, _ptr(r, ctypes.c_int32), r.shape[0], _ptr(w), w.shape[0],
                                         _ptr(D)))
        return D

    def resident_vote(self, rows, W: np.ndarray, num_classes: int) -> np.ndarray:
        """Class index per listed row: D = G[rows]·Wᵀ for the c(c-1)/2 one-vs-one pair
        vectors, then the reference's vote (multiclass.cpp:153-168), all on the device."""
        r = np.ascontiguousarray(rows, dtype=np.int32)
        w = _f64(np.atleast_2d(W))
        if w.shape[0] != num_classes * (num_classes - 1) // 2:
            raise ValueError("W must hold num_classes*(num_classes-1)/2 pair vectors")
        out = np.empty(r.shape[0], dtype=np.int32)
        _check(self._lib.lpd_resident_vote(self._h, _ptr(r, ctypes.c_int32), r.shape[0], _ptr(w), num_classes,
                                           _ptr(out, ctypes.c_int32)))
        return out

    def resident_gtv(self, rows, coef) -> np.ndarray:
        """w = Σ_i coef_i · G[rows_i] on the resident G (rebuild_w, dcd.cpp:91-102)."""
        r = np.ascontiguousarray(rows, dtype=np.int32)
        c = _f64(coef)
        w = np.empty(self.resident_shape()[1])
        _check(self._lib.lpd_resident_gtv(self._h, _ptr(r, ctypes.c_int32), _ptr(c), r.shape[0], _ptr(w)))
        return w

    def resident_gtv_sets(self, rows, coef) -> np.ndarray:
        """W[s] = Σ_i coef[i, s] · G[rows_i] for every column s of coef at once (the warm
        starts of all (fold, pair) problems, dcd.cpp:91-102)."""
        r = np.ascontiguousarray(rows, dtype=np.int32)
        c = _f64(np.atleast_2d(np.asarray(coef).T).T if np.ndim(coef) == 1 else coef)
        W = np.empty((c.shape[1], self.resident_shape()[1]))
        _check(self._lib.lpd_resident_gtv_sets(self._h, _ptr(r, ctypes.c_int32), _ptr(c), r.shape[0], c.shape[1],
                                               _ptr(W)))
        return W

    def resident_row_sqnorms(self) -> np.ndarray:
        """q_i = Σ_j G_ij² for every resident row (make_binary_problem's q_diag, dcd.cpp:60-89)."""
        q = np.empty(self.resident_shape()[0])
        _check(self._lib.lpd_resident_row_sqnorms(self._h, _ptr(q)))
        return q

    def kernel_block(self, A: np.ndarray, B: np.ndarray, gamma: float, norms_a=None,
                     norms_b=None) -> np.ndarray:
        """fp64 kernel block of dense rows (reference kernel_block, kernel.cpp:31-57);
        norms default to the rows' squared norms (kernel.cpp:59-65)."""
        a, b = _f64(A), _f64(B)
        if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[1]:
            raise ValueError("A and B must be 2-D with the same number of columns")
        na = _f64((a * a).sum(1) if norms_a is None else norms_a)
        nb = _f64((b * b).sum(1) if norms_b is None else norms_b)
        out = np.zeros((a.shape[0], b.shape[0]))
        _check(self._lib.lpd_kernel_block(self._h, a.shape[0], None, None, _ptr(a), _ptr(na), b.shape[0],
                                          None, None, _ptr(b), _ptr(nb), a.shape[1], float(gamma),
                                          _ptr(out), b.shape[0]))
        return out

    def decision_values(self, G: np.ndarray, W: np.ndarray) -> np.ndarray:
        g = _f64(G)
        w = _f64(W)
        if w.ndim == 1:
            w = w[None, :]
        if g.shape[1] != w.shape[1]:
            raise ValueError("W column count must match G")
        D = np.empty((g.shape[0], w.shape[0]), dtype=np.float64)
        _check(self._lib.lpd_decision_values(self._h, _ptr(g), g.shape[0], g.shape[1], g.shape[1],
                                             _ptr(w), w.shape[0], _ptr(D), w.shape[0]))
        return D

    def decision_values_device(self, G_dev, W_dev, D_dev, device_index: int = 0, stream=None) -> None:
        import torch

        g_dtype = LPD_OUT_F64 if G_dev.dtype == torch.float64 else LPD_OUT_F32
        st = ctypes.c_void_p(stream.cuda_stream) if stream is not None else None
        _check(self._lib.lpd_decision_values_device(
            self._h, device_index, ctypes.c_void_p(G_dev.data_ptr()), g_dtype, G_dev.shape[0],
            G_dev.shape[1], G_dev.stride(0), ctypes.c_void_p(W_dev.data_ptr()), W_dev.shape[0],
            ctypes.c_void_p(D_dev.data_ptr()), D_dev.stride(0), st))


def compute_G(points, norms, landmarks, landmark_norms, L, params, chunk_size: int,
              num_threads: int = 1, context: Optional[Context] = None) -> np.ndarray:
    """Mirror of lpdsvm::compute_G (factor.hpp:52-55) on the B200 path.

    ``points``/``landmarks``: sequences of sparse points (see sparse_to_csr) or
    dense 2-D arrays. ``norms``/``landmark_norms`` are accepted for signature
    parity and ignored: the device recomputes them from the same values the
    tensor cores see. ``chunk_size`` is validated like the reference; the
    device pipeline chooses its own row chunking (results do not depend on
    it). ``num_threads`` is accepted and unused.
    """
    if chunk_size == 0:
        raise ValueError("chunk_size must be positive")
    gamma = params.gamma if hasattr(params, "gamma") else float(params)
    Lm = _f64(L)
    if isinstance(landmarks, np.ndarray) and landmarks.ndim == 2:
        B = landmarks.shape[0]
    else:
        B = len(landmarks)
    if Lm.ndim != 2 or Lm.shape[0] != B:
        raise ValueError("L row count must match landmark count")
    if not (gamma > 0.0) or not np.isfinite(gamma):
        raise ValueError("kernel gamma must be positive and finite")
    ctx = context or Context()
    try:
        dense_pts = isinstance(points, np.ndarray) and points.ndim == 2
        dense_lms = isinstance(landmarks, np.ndarray) and landmarks.ndim == 2
        if dense_pts and dense_lms:
            d = max(points.shape[1], landmarks.shape[1])
            X = np.zeros((points.shape[0], d)); X[:, : points.shape[1]] = points
            Y = np.zeros((B, d)); Y[:, : landmarks.shape[1]] = landmarks
            ctx.set_basis_dense(Y, Lm, gamma)
            return ctx.compute_g_dense(X)
        pip, pix, pvl, pdim = sparse_to_csr(list(points) if not dense_pts else list(points))
        lip, lix, lvl, ldim = sparse_to_csr(list(landmarks) if not dense_lms else list(landmarks))
        d = max(pdim, ldim)
        ctx.set_basis_csr(lip, lix, lvl, d, Lm, gamma)
        return ctx.compute_g_csr(pip, pix, pvl)
    finally:
        if context is None:
            ctx.close()
