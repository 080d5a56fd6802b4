"""Synthetic inputs for the BASELINE.json configs.

No datasets are reachable (no network), so every workload is generated here
from a seed. Values are generated in fp32 and widened to fp64 so that the
reference (fp64 SparseVector values) and this library see identical inputs.

  C1 blobs      n=20,000   d=50   B=1,000   γ=0.02          seed 1
  C2 covtype    n=581,012  d=54   B=4,096   γ=1/d           seed 2
  C3 SUSY       n=5,000,000 d=18  B=8,192   γ=1/d           seed 3
  C4 ImageNet   n=1,281,167 d=2048 B=16,384 γ=1/d, 1000 classes, non-negative  seed 4

Two-class blobs: y = ±1 with p = 1/2, x ~ N(y·μ, I_d), ‖μ‖ = 1 along a seeded
random unit vector (Bayes error Φ(−1) ≈ 15.9%).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["Config", "CONFIGS", "blobs", "imagenet_like", "make", "rows_per_gpu"]


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    d: int
    budget: int
    gamma: float
    C: float
    seed: int
    classes: int = 2
    rows_per_gpu: int = 0  # bench: rows per GPU (weak scaling); 0 = n


def rows_per_gpu(cfg: "Config") -> int:
    return cfg.rows_per_gpu or cfg.n


CONFIGS = {
    "c1": Config("c1_blobs", 20_000, 50, 1_000, 0.02, 1.0, 1),
    "c2": Config("c2_covtype_shaped", 581_012, 54, 4_096, 1.0 / 54, 1.0, 2),
    # C3/C4 are row-sharded over 8 GPUs in BASELINE.json: a GPU owns n/8 rows
    "c3": Config("c3_susy_shaped", 5_000_000, 18, 8_192, 1.0 / 18, 1.0, 3, rows_per_gpu=625_000),
    "c4": Config("c4_imagenet_shaped", 1_281_167, 2048, 16_384, 1.0 / 2048, 1.0, 4, classes=1000,
                 rows_per_gpu=160_146),
}


def blobs(n: int, d: int, seed: int, rows: slice | None = None):
    """(X fp64 [n×d] with fp32-representable values, y in {+1, −1}).

    Rows are generated in independent 65,536-row blocks from (seed, block) so a
    row range can be produced without materialising the rest.
    """
    root = np.random.default_rng(seed)
    mu = root.standard_normal(d).astype(np.float32)
    mu /= np.float32(np.linalg.norm(mu))
    r0, r1 = (0, n) if rows is None else (rows.start or 0, min(n, rows.stop))
    X = np.empty((max(0, r1 - r0), d), dtype=np.float64)
    y = np.empty(max(0, r1 - r0), dtype=np.float64)
    blk = 65_536
    for b in range(r0 // blk, (r1 + blk - 1) // blk if r1 > r0 else r0 // blk):
        g = np.random.default_rng([seed, b])
        lo, hi = b * blk, min(n, (b + 1) * blk)
        yy = np.where(g.random(hi - lo) < 0.5, 1.0, -1.0).astype(np.float32)
        xx = g.standard_normal((hi - lo, d), dtype=np.float32) + yy[:, None] * mu[None, :]
        s0, s1 = max(lo, r0), min(hi, r1)
        X[s0 - r0 : s1 - r0] = xx[s0 - lo : s1 - lo].astype(np.float64)
        y[s0 - r0 : s1 - r0] = yy[s0 - lo : s1 - lo]
    return X, y


def imagenet_like(n: int, d: int, classes: int, seed: int, rows: slice | None = None):
    """Non-negative, non-centred features x = max(0, c_y + ε), c_y, ε ~ N(0, I)
    (exercises the ‖x‖²+‖b‖²−2x·b cancellation)."""
    root = np.random.default_rng(seed)
    centres = root.standard_normal((classes, d), dtype=np.float32)
    r0, r1 = (0, n) if rows is None else (rows.start or 0, min(n, rows.stop))
    X = np.empty((max(0, r1 - r0), d), dtype=np.float64)
    y = np.empty(max(0, r1 - r0), dtype=np.float64)
    blk = 16_384
    for b in range(r0 // blk, (r1 + blk - 1) // blk if r1 > r0 else r0 // blk):
        g = np.random.default_rng([seed, b])
        lo, hi = b * blk, min(n, (b + 1) * blk)
        yy = g.integers(0, classes, hi - lo)
        xx = np.maximum(0.0, centres[yy] + g.standard_normal((hi - lo, d), dtype=np.float32))
        s0, s1 = max(lo, r0), min(hi, r1)
        X[s0 - r0 : s1 - r0] = xx[s0 - lo : s1 - lo].astype(np.float64)
        y[s0 - r0 : s1 - r0] = yy[s0 - lo : s1 - lo]
    return X, y


def make(cfg: Config, rows: slice | None = None, n: int | None = None):
    """Rows `rows` of the config's n-row (or `n`-row) dataset."""
    n = cfg.n if n is None else n
    if cfg.classes > 2:
        return imagenet_like(n, cfg.d, cfg.classes, cfg.seed, rows)
    return blobs(n, cfg.d, cfg.seed, rows)
