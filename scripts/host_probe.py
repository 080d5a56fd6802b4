"""Box probe: host fp32->fp64 widening throughput (torch CPU copy_, N threads) into a
pre-touched buffer, and pinned D2H bandwidth for fp32 / fp64 G chunks."""
import time

import torch

n_rows, cols = 65536, 4096
src = torch.randn(n_rows, cols, dtype=torch.float32).pin_memory()
dst = torch.zeros(n_rows, cols, dtype=torch.float64)
for th in (1, 4, 8, 16):
    torch.set_num_threads(th)
    dst.copy_(src)
    t = time.perf_counter()
    for _ in range(3):
        dst.copy_(src)
    dt = (time.perf_counter() - t) / 3
    print(f"widen fp32->fp64 threads={th}: {src.numel() * 4 / dt / 1e9:.1f} GB/s in, {dst.numel() * 8 / dt / 1e9:.1f} GB/s out")
dev = torch.empty(n_rows, cols, dtype=torch.float32, device="cuda")
for dt_, name in ((torch.float32, "fp32"), (torch.float64, "fp64")):
    g = torch.empty(n_rows // 2, cols, dtype=dt_, device="cuda")
    h = torch.empty(n_rows // 2, cols, dtype=dt_).pin_memory()
    h.copy_(g, non_blocking=True); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        h.copy_(g, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"D2H pinned {name}: {g.numel() * g.element_size() / ms / 1e6:.1f} GB/s")
    hp = torch.zeros(n_rows // 2, cols, dtype=dt_)
    t = time.perf_counter()
    hp.copy_(g); torch.cuda.synchronize()
    print(f"D2H pageable(pre-touched) {name}: {g.numel() * g.element_size() / (time.perf_counter() - t) / 1e9:.1f} GB/s")
