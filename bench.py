#!/usr/bin/env python3
"""Nyström factor benchmark (BASELINE.json metric: "Nyström factor rows/s &
TFLOP/s vs peak"), workload C2: covtype-shaped synthetic binary blobs,
n = 581,012 rows per GPU, d = 54, B = 4,096 landmarks, γ = 1/54.

One step = one pass of the hot path (reference lpdsvm::compute_G,
proj/src/factor.cpp:83-110) over the whole batch: basis prep of (landmarks, L)
(K2; with N > 1 preceded by the NCCL broadcast of the basis from rank 0, the
path's only collective), row prep (K3) and the fused factor kernel (K1)
writing G = Z·L (fp64) to HBM.

  value  rows/s over all ranks, inputs resident in HBM (max-over-ranks device time)
  e2e    the same metric through the C ABI host path (lpd_set_basis_dense +
         lpd_compute_g_dense): pinned host X in, fp64 G back into a host buffer
  roofline  K1 algorithmic TFLOP/s (F = 2nBd + 2nB·B_eff per launch, CUDA events
         on the launch stream) vs the measured dense bf16/fp16 peak
  cpu_baseline  the reference's own compute_G (oracle/_ref, all host threads) on a
         bounded row sample of the same workload

Weak scaling: rank r owns rows [r·n, (r+1)·n) of an N·n-row dataset.
`--impl reference` times the reference CPU implementation instead (rank 0).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Nyström factor rows/s"
UNIT = "rows/s"
# per step: K2 (column_sum_partial, column_mean_finalize, landmark_stats, basis_consts,
# prep_landmarks, col_stats, lt_split, col_norm_finalize) + K3 prep_rows + K9 row_shift and
# row_rescale + the factor: one fused K1 launch (d <= 63) or, on the panel path, a Z GEMM and
# a projection GEMM per <= 2 GB Z panel
def launches_per_step(n, d, B):
    if d <= 63:
        return 12
    bpad = -(-B // 256) * 256
    panel = max(256, (2 * 2**30 // (4 * bpad)) // 256 * 256)
    npad = -(-n // 256) * 256
    return 11 + 2 * (-(-npad // panel))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--rows", type=int, default=0, help="override rows per GPU (testing only)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the drop-in e2e, the train-seconds runs and the C4 shard record")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU-baseline sample time")
    return ap.parse_args()


def load_peaks():
    """Dense bf16 peaks from MEASURED_PEAKS.json (driver-written on this pool's B200s):
    the burst figure and the sustained one (back-to-back matmuls under the 1 kW cap)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        burst = float(p["bf16_tflops"])
        return {"burst": burst, "sustained": float(p.get("bf16_tflops_sustained", burst)),
                "hbm": float(p["hbm_gbs"]), "src": "measured"}
    except Exception:
        return {"burst": 1590.0, "sustained": 1590.0, "hbm": 6650.0, "src": "fallback (B200_PROFILING.md)"}


def load_traffic(workload):
    """dram read+write bytes per launch of this workload's dominant kernel, from the
    committed ncu --set full summaries (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)[workload]["bytes"]
    except Exception:
        return None


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled during the timed region: NVML
    polled every 10 ms from a thread (a C2 timed region is a few hundred ms), else
    `nvidia-smi -lms 100`."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.stop = threading.Event()
        self.t = None

    def _nvml_handle(self):
        import pynvml

        pynvml.nvmlInit()
        try:  # the CUDA device's own PCI address (CUDA and NVML orderings can differ)
            import torch

            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _poll(self, nv, h):
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while True:
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            act = ["Active" if r & bt else "Not Active" for bt in bits]
            self.lines.append(", ".join([str(sm), str(mx), hex(r)] + act))
            if self.stop.wait(0.01):
                break

    def __enter__(self):
        try:
            nv, h = self._nvml_handle()
            self.t = threading.Thread(target=self._poll, args=(nv, h), daemon=True)
            self.t.start()
            return self
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        elif self.t:
            self.t.join(timeout=5)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def make_basis(X0, cfg, seed=1, device=None, return_ids=False, host_max_b=8192):
    """Landmarks: B rows of rank 0's data drawn uniformly without replacement
    (as the reference's select_landmarks does, factor.cpp:27-31; numpy's seeded
    generator here); L from the eigendecomposition of K (factor.cpp:33-81).
    Setup only, outside the timed region: numpy LAPACK for B <= host_max_b, cuSOLVER
    through torch on the GPU for larger bases (C4: B = 16384)."""
    ids = np.random.default_rng(seed).choice(X0.shape[0], cfg.budget, replace=False)
    Y = np.ascontiguousarray(X0[ids])
    if cfg.budget <= host_max_b or device is None:
        ny = (Y * Y).sum(1)
        K = np.exp(-cfg.gamma * np.maximum(ny[:, None] + ny[None, :] - 2.0 * Y @ Y.T, 0.0))
        w, U = np.linalg.eigh(0.5 * (K + K.T))
        w, U = w[::-1], U[:, ::-1]
        keep = w > 1e-12 * w[0]
        L = np.ascontiguousarray(U[:, keep] / np.sqrt(w[keep]))
        return (Y, L, ids) if return_ids else (Y, L)
    import torch

    Yt = torch.from_numpy(Y).to(device)
    ny = (Yt * Yt).sum(1)
    K = torch.exp(-cfg.gamma * torch.clamp(ny[:, None] + ny[None, :] - 2.0 * Yt @ Yt.T, min=0.0))
    w, U = torch.linalg.eigh(0.5 * (K + K.T))
    w, U = torch.flip(w, [0]), torch.flip(U, [1])
    keep = w > 1e-12 * w[0]
    L = (U[:, keep] / torch.sqrt(w[keep])).contiguous().cpu().numpy()
    return (Y, L, ids) if return_ids else (Y, L)


def cpu_reference_rate(X, Y, L, gamma, target_s, threads, max_rows):
    """Reference compute_G (oracle/_ref, unmodified reference sources) on a bounded
    contiguous row sample with all host threads; returns (rows/s, rows, seconds)."""
    from oracle import oracle as O

    ycsr = O.dense_to_csr(Y)
    rows = min(max_rows, 2048)
    while True:
        xs = O.dense_to_csr(X[:rows])
        chunk = max(64, -(-rows // threads))
        _, secs = O.ref_compute_g(xs, ycsr, L, gamma, chunk, threads, return_seconds=True)
        if secs >= 0.5 * target_s or rows >= max_rows:
            return rows / secs, rows, secs
        rows = int(min(max_rows, max(rows * 2, rows * target_s / max(secs, 1e-3))))


def run_reference(args, cfg, rank):
    """--impl reference: the reference's own CPU compute_G on rank 0's host cores."""
    if rank != 0:
        return
    from oracle import oracle as O

    from paper_2207_01016_b200 import synthetic

    n = args.rows or synthetic.rows_per_gpu(cfg)
    X, _ = synthetic.make(cfg, rows=slice(0, n), n=max(n, cfg.n))
    import torch

    Y, L = make_basis(X, cfg, device="cuda" if torch.cuda.is_available() else None)
    threads = O.ref_lib().ref_hardware_threads()
    # size each step so warmup + steps stay within a few minutes
    per_step = max(2.0, min(20.0, 100.0 / max(1, args.steps + args.warmup)))
    rate, rows, secs = cpu_reference_rate(X, Y, L, cfg.gamma, per_step, threads, n)
    ycsr = O.dense_to_csr(Y)
    xs = O.dense_to_csr(X[:rows])
    chunk = max(64, -(-rows // threads))
    for _ in range(max(0, args.warmup - 1)):
        O.ref_compute_g(xs, ycsr, L, cfg.gamma, chunk, threads)
    ts = []
    for _ in range(args.steps):
        _, s = O.ref_compute_g(xs, ycsr, L, cfg.gamma, chunk, threads, return_seconds=True)
        ts.append(s)
    value = rows * len(ts) / sum(ts)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(ts) / len(ts),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "n": n, "d": cfg.d, "B": cfg.budget, "b_eff": int(L.shape[1]),
                   "gamma": cfg.gamma, "parallelism": f"host threads={threads}"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{rows} contiguous rows of the {n}-row workload per step, chunk_size={chunk}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        # the reference's compute_G above IS its drop-in API (squared_norms + compute_G into a
        # fresh Matrix, oracle/ref_harness.cpp ref_compute_g): same number
        "e2e_dropin": {"value": value, "unit": UNIT, "seconds_per_step": sum(ts) / len(ts), "rows": rows,
                       "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        # lpdsvm.train's train_impl (module.cpp:35-78) on the unmodified reference build
        "train_seconds": None if args.no_extras else {c: e2e_train("ref", c) for c in ("c1", "c2")},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test-only: every rank on GPU 0 with gloo collectives, to exercise the N > 1 code
    # path on a one-GPU machine (numbers meaningless; never used for measurements)
    one_gpu_test = os.environ.get("LPD_BENCH_ONE_GPU_TEST") == "1"
    if one_gpu_test:
        local = 0
    dist = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        if one_gpu_test:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2207_01016_b200 import synthetic

    cfg = synthetic.CONFIGS[args.workload]
    if args.impl == "reference":
        run_reference(args, cfg, rank)
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    import paper_2207_01016_b200 as P

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    n = args.rows or synthetic.rows_per_gpu(cfg)
    N = world
    res = measure(args, cfg, n, N, rank, local, dist, dev, P, args.steps, args.warmup, not args.no_e2e)

    cpu = dropin = trains = c3 = c4 = c5 = None
    if rank == 0 and N == 1:
        if not args.no_cpu_baseline:
            from oracle import oracle as O

            if O.ref_available():
                threads = O.ref_lib().ref_hardware_threads()
                rate, rows, secs = cpu_reference_rate(res["X"], res["Y"], res["L"], cfg.gamma, args.cpu_seconds,
                                                      threads, n)
                cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                       "sample": f"{rows} contiguous rows of the {n}-row workload, same landmarks/L, "
                                 f"{secs:.1f}s, chunk_size={max(64, -(-rows // threads))}"}
        if not args.no_extras:
            # end-to-end trains first, while the host's memory is least fragmented (their
            # gmatrix stage first-touches a fresh 19 GB G on huge pages)
            trains = {c: e2e_train("b200", c) for c in ("c1", "c2")}
            dropin = e2e_dropin("b200", cfg, res, n)
            c5 = c5_resident(res, cfg, P)
            if args.workload != "c4":
                c4cfg = synthetic.CONFIGS["c4"]
                r4 = measure(args, c4cfg, synthetic.rows_per_gpu(c4cfg), 1, 0, local, None, dev, P,
                             max(2, min(args.steps, 5)), 3, not args.no_e2e)
                c4 = {"workload": c4cfg.name, "value": r4["value"], "unit": UNIT, "n_per_gpu": r4["n"],
                      "d": c4cfg.d, "B": r4["B"], "b_eff": r4["b_eff"], "gamma": c4cfg.gamma,
                      "ms_per_step": r4["ms_per_step"], "steps": r4["steps"],
                      "path": "panel path: Z GEMM + projection GEMM (d >= 64)",
                      "roofline": r4["roofline"], "e2e": r4["e2e"], "clocks": r4["clocks"]}
                del r4
            if args.workload != "c3":  # device value only (its e2e needs an 82 GB host G)
                c3cfg = synthetic.CONFIGS["c3"]
                r3 = measure(args, c3cfg, synthetic.rows_per_gpu(c3cfg), 1, 0, local, None, dev, P,
                             max(2, min(args.steps, 5)), 3, False, host_max_b=0)
                c3 = {"workload": c3cfg.name, "value": r3["value"], "unit": UNIT, "n_per_gpu": r3["n"],
                      "d": c3cfg.d, "B": r3["B"], "b_eff": r3["b_eff"], "gamma": c3cfg.gamma,
                      "ms_per_step": r3["ms_per_step"], "steps": r3["steps"], "path": "fused K1 (d <= 63)",
                      "basis": "L from cuSOLVER eigh on the device (setup)",
                      "roofline": r3["roofline"], "clocks": r3["clocks"]}
                del r3

    if rank == 0:
        line = {
            "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f16x3 split operands, f32 accumulate, f64 G",
            "data": (f"synthetic ({'1000-class non-negative ImageNet-feature-shaped' if cfg.classes > 2 else 'two-class Gaussian blobs'}"
                     f", seed {cfg.seed}; landmarks drawn like the reference select_landmarks, L from eigh(K))"),
            "config": {"workload": cfg.name, "n_per_gpu": n, "d": cfg.d, "B": res["B"], "b_eff": res["b_eff"],
                       "gamma": cfg.gamma, "parallelism": f"rows sharded over {N} GPU(s), basis broadcast",
                       "path": "fused K1 (d <= 63)" if cfg.d <= 63 else "panel path: Z GEMM + projection GEMM (d >= 64)",
                       "l2": f"inputs larger than L2 (G {n * res['b_eff'] * 8 / 1e9:.1f} GB/step per GPU written, "
                             f"X {res['X'].nbytes / 1e9:.2f} GB read)"},
            "roofline": res["roofline"],
            "cpu_baseline": cpu,
            "e2e": res["e2e"],
            # the reference's own C++ API (compute_G with SparseVector rows into a fresh
            # Matrix, the gmatrix stage of factor.cpp:129-133) on the drop-in build
            "e2e_dropin": dropin,
            # lpdsvm.train's train_impl (module.cpp:35-78) end to end on the drop-in build
            "train_seconds": trains,
            "c3_shard": c3,
            "c4_shard": c4,
            # config 5: the products cross_validate / the solver run on the resident G
            "c5_resident": c5,
            "gpu_launches": launches_per_step(n, cfg.d, res["B"]) * args.steps,
            "clocks": res["clocks"],
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def c5_resident(res, cfg, P, reps=5):
    """BASELINE config 5's device products on this workload's factor kept resident in HBM
    (lpd_set_keep_resident): a 5-fold split's held-out scoring — binary (P = 1, the
    reference's loop order bit for bit, lpd_resident_gw) and a 10-class fold (45 pair
    vectors + the one-vs-one vote on the device, lpd_resident_vote) — and the warm-start
    rebuild w = Σ coef_i·G_i over the training rows (lpd_resident_gtv). Wall time through
    the C ABI (row list and W up, results down), median of `reps`; roofline = HBM time of
    the G rows read vs fp64 time of the (product, add) pairs at half the DGEMM rate."""
    import torch

    X, Y, L = res["X"], res["Y"], res["L"]
    n, b_eff = X.shape[0], L.shape[1]
    a = torch.randn(4096, 4096, dtype=torch.float64, device="cuda")
    a @ a
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(4):
        a @ a
    torch.cuda.synchronize()
    dgemm = 4 * 2 * 4096.0 ** 3 / (time.perf_counter() - t0) / 1e12
    del a
    peaks = load_peaks()
    rng = np.random.default_rng(5)
    fold = rng.permutation(n) % 5
    held = np.flatnonzero(fold == 0).astype(np.int32)
    train = np.flatnonzero(fold != 0).astype(np.int32)
    out = {"n": n, "b_eff": b_eff, "held_out_rows": int(held.size), "train_rows": int(train.size),
           "fp64_dgemm_tflops": dgemm, "hbm_peak_gbs": peaks["hbm"]}
    G = np.empty((n, b_eff))
    with P.Context(1) as ctx:
        ctx.set_basis_dense(Y, L, cfg.gamma)
        ctx.set_keep_resident(True)
        ctx.compute_g_dense(X, out=G)
        if ctx.resident_shape() != (n, b_eff):
            return {"skipped": "resident G did not fit"}

        def timed(f):
            f()
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter()
                f()
                ts.append(time.perf_counter() - t0)
            return statistics.median(ts)

        def roof(t, rows, pairs):
            t_hbm = rows * b_eff * 4 / (peaks["hbm"] * 1e9)
            t_f64 = 2.0 * rows * pairs * b_eff / (dgemm * 0.5e12)
            return {"seconds": t, "rows_per_s": rows / t, "bound": "hbm" if t_hbm >= t_f64 else "fp64",
                    "frac_of_roofline_c_abi": max(t_hbm, t_f64) / t}

        w1 = rng.standard_normal((1, b_eff))
        D = ctx.resident_gw(held, w1)
        k = min(2000, held.size)
        seq = np.add.accumulate(G[held[:k]] * w1[0], axis=1)[:, -1]
        out["score_binary"] = {**roof(timed(lambda: ctx.resident_gw(held, w1)), held.size, 1),
                               "bitwise_equal_to_reference_loop_sample": bool(np.array_equal(D[:k, 0], seq))}
        w45 = rng.standard_normal((45, b_eff))
        out["score_vote_10class"] = roof(timed(lambda: ctx.resident_vote(held, w45, 10)), held.size, 45)
        coef = rng.standard_normal(train.size)
        t = timed(lambda: ctx.resident_gtv(train, coef))
        out["rebuild_w"] = {"seconds": t, "rows": int(train.size),
                            "frac_of_hbm_c_abi": train.size * b_eff * 4 / (peaks["hbm"] * 1e9) / t}
        ctx.set_keep_resident(False)
    del G
    return out


def _run_e2e_subprocess(argv, timeout):
    """integration/e2e_run.py in its own process (the two builds define the same C++
    symbols); returns its JSON or an error record."""
    cmd = [sys.executable, os.path.join(ROOT, "integration", "e2e_run.py"), *argv]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    except subprocess.TimeoutExpired:
        return {"error": f"timeout after {timeout}s"}
    if r.returncode != 0:
        return {"error": (r.stderr or r.stdout).strip().splitlines()[-1:] or ["rc != 0"]}
    return json.loads(r.stdout.strip().splitlines()[-1])


def e2e_dropin(build, cfg, res, rows):
    """The gmatrix stage through the reference's compute_G signature (SparseVector rows,
    a fresh Matrix per call) on `build`, with the bench's landmarks and L."""
    import tempfile

    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "basis.npz")
        np.savez(path, Y=res["Y"], L=res["L"], gamma=cfg.gamma, workload=cfg.name,
                 **({"G_sample": res["G_sample"]} if res.get("G_sample") is not None else {}))
        out = _run_e2e_subprocess([build, "compute_g", path, "--rows", str(rows)], 900)
    if "error" in out:
        return out
    b_eff = out["b_eff"]
    return {"value": out["rows_per_s"], "unit": UNIT, "seconds_per_step": out["gmatrix_seconds"],
            "compute_G_seconds": out["compute_G_seconds"], "rows": out["rows"], "steps": out["steps"],
            "h2d_bytes_per_step": int(rows * cfg.d * 12 + res["B"] * cfg.d * 12 + res["B"] * b_eff * 8),
            "d2h_bytes_per_step": int(rows * (-(-b_eff // 4) * 4) * 4),
            "sample_max_row_rel_diff_vs_device_path": out.get("sample_max_row_rel_diff"),
            "phases": out.get("adapter_phases"),
            "path": "lpdsvm::squared_norms + lpdsvm::compute_G (factor.hpp:52-55) with std::vector<Feature> rows "
                    "into a fresh lpdsvm::Matrix (adapter -> C ABI -> B200), median of the steps"}


def e2e_train(build, config):
    return _run_e2e_subprocess([build, "train", config, "--n-test", "10000" if config == "c1" else "20000"], 1500)


def measure(args, cfg, n, N, rank, local, dist, dev, P, steps, warmup, want_e2e, host_max_b=8192):
    """Device value (inputs resident in HBM), the factor kernel's roofline and the C-ABI
    e2e for one workload; rank r owns rows [r·n, (r+1)·n) of an N·n-row dataset."""
    import torch

    X, _ = synthetic_rows(cfg, rank, n, N)
    if rank == 0:
        Y, L = make_basis(X, cfg, device=dev, host_max_b=host_max_b)
        meta = torch.tensor([Y.shape[0], L.shape[1]], dtype=torch.int64, device=dev)
    else:
        meta = torch.zeros(2, dtype=torch.int64, device=dev)
    if dist:
        dist.broadcast(meta, 0)
    B, b_eff = int(meta[0]), int(meta[1])
    lm_dev = torch.empty((B, cfg.d), dtype=torch.float64, device=dev)
    L_dev = torch.empty((B, b_eff), dtype=torch.float64, device=dev)
    if rank == 0:
        lm_dev.copy_(torch.from_numpy(Y))
        L_dev.copy_(torch.from_numpy(L))
    X_dev = torch.from_numpy(X).to(dev)
    G_dev = torch.empty((n, b_eff), dtype=torch.float64, device=dev)

    ctx = P.Context(device_ids=[local])  # one device per process
    stream = torch.cuda.current_stream(dev)

    def step():
        if dist:
            dist.broadcast(lm_dev, 0)
            dist.broadcast(L_dev, 0)
        ctx.set_basis_device(lm_dev, L_dev, cfg.gamma, stream=stream)
        ctx.compute_g_device(X_dev, G_dev, stream=stream)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize(dev)
    ctx.factor_kernel_stats(reset=True)

    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        e0.record(stream)
        for _ in range(steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    elapsed_ms = e0.elapsed_time(e1)
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t.item())
    k_total_ms, k_launches = ctx.factor_kernel_stats(reset=True)
    k_ms = k_total_ms / max(1, k_launches)

    value = N * n * steps / (elapsed_ms / 1e3)
    F = 2.0 * n * B * cfg.d + 2.0 * n * B * b_eff
    peaks = load_peaks()
    achieved = F / (k_ms / 1e3) / 1e12
    # The factor kernel runs back to back for the whole timed region (tens of ms per
    # launch, sw_power_cap engaged): the sustained peak is its roof; a short region
    # would be judged against the burst figure.
    sustained = elapsed_ms >= 100.0 and k_ms >= 10.0
    peak = peaks["sustained"] if sustained else peaks["burst"]
    peak_src = (f"MEASURED_PEAKS.json bf16_tflops{'_sustained' if sustained else ''} ({peaks['src']}; "
                f"kind::f16 runs at the bf16 rate; {'kernel timed inside a long step' if sustained else 'short timed region'})")
    traffic = load_traffic(cfg.name)
    # issued tensor work (3-term split, padded shapes, GEMM1 recomputed per 256-column block)
    npad, epad = -(-n // 256) * 256, -(-b_eff // 256) * 256
    if cfg.d <= 63:  # fused kernel: GEMM1 (d + norm column, 16-wide K steps) per 256-column block
        bpad = -(-B // 64) * 64
        k1 = -(-(cfg.d + 1) // 16) * 16
        issued = 3 * (2.0 * npad * bpad * k1 * (epad // 256) + 2.0 * npad * bpad * epad)
    else:  # panel path: Z GEMM once (K = d + norm column, 64-wide chunks), then the projection
        bpad = -(-B // 256) * 256
        kd = -(-(cfg.d + 1) // 64) * 64
        issued = 3 * (2.0 * npad * bpad * kd + 2.0 * npad * bpad * epad)
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel_ms": k_ms, "flops_per_launch": F, "issued_tensor_flops_per_launch": issued,
                "issued_frac": issued / (k_ms / 1e3) / 1e12 / peak,
                "peak_source": peak_src, "peak_burst": peaks["burst"],
                "frac_of_burst": achieved / peaks["burst"]}

    # ---------------- end to end through the C ABI with host buffers ----------------
    e2e = None
    G_sample = G_dev[: min(256, n)].cpu().numpy()
    if want_e2e:
        import psutil

        # every local rank holds its own fp64 G in host RAM: at N > 1 on one host the
        # e2e rows per GPU shrink to what fits (stated in the line), never skipped
        local_ranks = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
        budget = psutil.virtual_memory().available / (2.5 * max(1, local_ranks))
        n_fit = int(budget // (8 * b_eff))
        n_e2e = n if n_fit >= n else n_fit // 256 * 256
        if dist:
            t_n = torch.tensor([n_e2e], dtype=torch.int64, device=dev)
            dist.all_reduce(t_n, op=dist.ReduceOp.MIN)
            n_e2e = int(t_n.item())
        if n_e2e >= 256:
            Xh = torch.from_numpy(np.ascontiguousarray(X[:n_e2e])).pin_memory()
            Yh = lm_dev.cpu().numpy()
            Lh = L_dev.cpu().numpy()
            Xn = Xh.numpy()

            def run_e2e(Gout):
                ctx.set_basis_dense(Yh, Lh, cfg.gamma)
                ctx.compute_g_dense(Xn, out=Gout)  # warm-up (also first-touches Gout)
                ts, tb, tm = [], [], []
                for _ in range(args.e2e_steps):
                    if dist:
                        dist.barrier()
                    t0 = time.perf_counter()
                    ctx.set_basis_dense(Yh, Lh, cfg.gamma)
                    t1 = time.perf_counter()
                    tmg = P.Timings()
                    ctx.compute_g_dense(Xn, out=Gout, timings=tmg)
                    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
                    tm.append(tmg.as_dict())
                    if dist:
                        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
                    ts.append(float(dt.item()))
                    tb.append(t1 - t0)
                # spot-check the host result against the device-path result
                k = min(1000, Gout.shape[0])
                assert np.array_equal(Gout[:k], G_dev[:k].cpu().numpy())
                mid = sorted(range(len(ts)), key=lambda i: ts[i])[len(ts) // 2]
                return statistics.median(ts), statistics.median(tb), tm[mid]

            # the caller's G is ordinary pageable, pre-touched memory, like the
            # reference's zero-filled Matrix (matrix.hpp:15-16)
            Gn = np.zeros((n_e2e, b_eff), dtype=np.float64)
            t_e2e, t_basis, phases = run_e2e(Gn)
            e2e = {"value": N * n_e2e / t_e2e, "unit": UNIT,
                   "h2d_bytes_per_step": int(Xn.nbytes + Yh.nbytes + Lh.nbytes),
                   "d2h_bytes_per_step": int(n_e2e * (-(-b_eff // 4) * 4) * 4),
                   "seconds_per_step": t_e2e, "basis_seconds_per_step": t_basis,
                   "rows_per_gpu": n_e2e,
                   # the median step's library timings: D2H stream busy time, the host team's
                   # widening time, the factor launches (CUDA events) — they overlap
                   "phases": {"d2h_seconds": phases["d2h_seconds"], "d2h_gbs": n_e2e * (-(-b_eff // 4) * 4) * 4 / max(phases["d2h_seconds"], 1e-9) / 1e9,
                              "host_widen_seconds": phases["host_copy_seconds"], "kernel_seconds": phases["kernel_seconds"],
                              "library_seconds": phases["total_seconds"],
                              # share of the serial sum (D2H + widen + kernels) hidden by overlap
                              "overlap": 1.0 - phases["total_seconds"] / max(1e-9, phases["d2h_seconds"] + phases["host_copy_seconds"] + phases["kernel_seconds"])},
                   "path": "lpd_set_basis_dense + lpd_compute_g_dense: pinned host X -> device; fp32 G -> "
                           "8 MB pinned ring -> host threads widen each buffer (AVX-512 streaming stores) "
                           "into the caller's pageable fp64 G; median of the steps"}
            del Xh, Gn
        else:
            e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                   "skipped": "host RAM too small for a pinned fp64 G of this workload"}
    out = {"value": value, "ms_per_step": elapsed_ms / steps, "steps": steps, "n": n, "B": B, "b_eff": b_eff,
           "roofline": roofline, "e2e": e2e, "clocks": clocks.summary(), "X": X,
           "Y": lm_dev.cpu().numpy(), "L": L_dev.cpu().numpy(), "G_sample": G_sample}
    ctx.close()
    del X_dev, G_dev, lm_dev, L_dev
    torch.cuda.empty_cache()
    return out


def synthetic_rows(cfg, rank, n, N):
    from paper_2207_01016_b200 import synthetic

    return synthetic.make(cfg, rows=slice(rank * n, (rank + 1) * n), n=N * n)


if __name__ == "__main__":
    main()
