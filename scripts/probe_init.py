"""Probe: CUDA context creation cost through the library, and first-call latencies."""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
t0 = time.perf_counter()
import paper_2207_01016_b200 as P  # noqa: E402

lib = P.load_library()
print("load", time.perf_counter() - t0)
t0 = time.perf_counter()
print("device_count", lib.lpd_device_count(), time.perf_counter() - t0)
t0 = time.perf_counter()
ctx = P.Context(1)
print("context_create", time.perf_counter() - t0)
import numpy as np  # noqa: E402

A = np.random.default_rng(0).standard_normal((1000, 50))
for i in range(3):
    t0 = time.perf_counter()
    ctx.kernel_block(A, A, 0.02)
    print("kernel_block", i, time.perf_counter() - t0)
L = np.eye(1000)
for i in range(3):
    t0 = time.perf_counter()
    ctx.set_basis_dense(A, L, 0.02)
    ctx.compute_g_dense(A)
    print("basis+G", i, time.perf_counter() - t0)
