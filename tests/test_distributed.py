"""Multi-process (world_size 2, gloo, CPU) coverage of the row-sharded path:
basis broadcast from rank 0 and disjoint contiguous row shards whose union,
computed independently per rank, equals the single-process result. The CPU
oracle stands in for the device kernel here (CPU-only test); the device path is
covered by the GPU parity tests, which check batch invariance bitwise."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import load_golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2207_01016_b200 import sharding

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = load_golden("c1_mini.npz")
        X = g["X"].astype(np.float64)
        if rank == 0:
            lm, L, gamma = sharding.broadcast_basis(X[g["ids"]], g["L"], float(g["gamma"]))
        else:
            lm, L, gamma = sharding.broadcast_basis(None, None, None)
        b, e = sharding.row_shard(X.shape[0], world, rank)
        G = O.ora_compute_g(O.dense_to_csr(X[b:e]), O.dense_to_csr(lm), L, gamma, 4096)
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), G)
        np.save(os.path.join(out_dir, f"span{rank}.npy"), np.array([b, e]))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_factor(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    g = load_golden("c1_mini.npz")
    parts = [np.load(tmp_path / f"rank{r}.npy") for r in range(world)]
    spans = [np.load(tmp_path / f"span{r}.npy") for r in range(world)]
    assert spans[0][0] == 0 and spans[0][1] == spans[1][0] and spans[1][1] == g["G"].shape[0]
    G = np.concatenate(parts)
    assert np.abs(G - g["G"]).max() <= 1e-12 * np.abs(g["G"]).max()


def _gpu_worker(rank, world, port, out_dir):
    """Each rank: its own B200 context (all on device 0 on a one-GPU box), the library
    computing its shard (sharding.compute_g_sharded), basis broadcast over gloo."""
    import torch.distributed as dist

    import paper_2207_01016_b200 as P
    from paper_2207_01016_b200 import sharding

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = load_golden("c1_mini.npz")
        X = np.tile(g["X"].astype(np.float64), (7, 1))  # 3,584 rows: ragged shards of the 256-row tile
        with P.Context(device_ids=[0]) as ctx:
            if rank == 0:
                b, e, G = sharding.compute_g_sharded(ctx, X, X[g["ids"]], g["L"], float(g["gamma"]))
            else:
                b, e, G = sharding.compute_g_sharded(ctx, X, None, None, None)
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), G)
        np.save(os.path.join(out_dir, f"span{rank}.npy"), np.array([b, e]))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_multiprocess_library_shards_bitwise(tmp_path, gpu_ctx, world):
    """One process per rank calling the LIBRARY (not the oracle): the concatenated shards
    equal the single-process G bit for bit (fixed per-row reduction order, no split-K),
    as the reference promises worker-count invariance."""
    mp.spawn(_gpu_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    g = load_golden("c1_mini.npz")
    X = np.tile(g["X"].astype(np.float64), (7, 1))
    gpu_ctx.set_basis_dense(X[g["ids"]], g["L"], float(g["gamma"]))
    full = gpu_ctx.compute_g_dense(X)
    spans = [np.load(tmp_path / f"span{r}.npy") for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == X.shape[0]
    assert all(spans[r][1] == spans[r + 1][0] for r in range(world - 1))
    G = np.concatenate([np.load(tmp_path / f"rank{r}.npy") for r in range(world)])
    assert np.array_equal(G, full)
