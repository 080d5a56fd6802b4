"""e2e host-path breakdown (lpd_set_basis_dense + lpd_compute_g_dense into pageable fp64 G)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import bench
import paper_2207_01016_b200 as P
from paper_2207_01016_b200 import synthetic

cfg = synthetic.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
n = synthetic.rows_per_gpu(cfg)
X, _ = synthetic.make(cfg, rows=slice(0, n))
Y, L = bench.make_basis(X, cfg)
def thp_zeros(shape):
    # an mmap-backed buffer advised to use transparent huge pages before its first touch,
    # the way the adapter allocates the reference's Matrix
    import ctypes, mmap
    nbytes = int(np.prod(shape)) * 8
    buf = mmap.mmap(-1, nbytes + (2 << 20))
    addr = ctypes.addressof(ctypes.c_char.from_buffer(buf))
    a0 = (addr + (2 << 20) - 1) & ~((2 << 20) - 1)
    libc = ctypes.CDLL(None)
    libc.madvise(ctypes.c_void_p(a0), ctypes.c_size_t(nbytes), 14)  # MADV_HUGEPAGE
    arr = np.frombuffer(buf, dtype=np.uint8, count=nbytes, offset=a0 - addr).view(np.float64).reshape(shape)
    arr[:] = 0.0
    return arr, buf
import os
if os.environ.get("E2E_THP") == "1":
    G, _keep = thp_zeros((n, L.shape[1]))
else:
    G = np.zeros((n, L.shape[1]))
import torch
Xp = torch.from_numpy(X).pin_memory().numpy()
with P.Context(1) as ctx:
    for i in range(3):
        t0 = time.perf_counter(); ctx.set_basis_dense(Y, L, cfg.gamma); print(f"set_basis (before compute) {time.perf_counter()-t0:.4f} s", flush=True)
    ctx.compute_g_dense(Xp, out=G)
    for _ in range(3):
        t0 = time.perf_counter(); ctx.set_basis_dense(Y, L, cfg.gamma); tb = time.perf_counter() - t0
        t = P.Timings()
        t0 = time.perf_counter()
        ctx.compute_g_dense(Xp, out=G, timings=t)
        dt = time.perf_counter() - t0
        print(f"set_basis {tb:.4f} s  compute wall {dt:.3f} s  {n/dt/1e6:.2f} M rows/s  {G.nbytes/dt/1e9:.1f} GB/s fp64 out  timings {t.as_dict()}", flush=True)
