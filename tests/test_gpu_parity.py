"""Parity of the B200 path (through the C ABI) against the oracle and the
reference build. Run on a B200 with `pytest -m gpu`.

Tolerances (north star: "G must match the reference's CPU factor within a
stated relative tolerance"): row-normwise relative error
    max_i ||G_i - G_ref,i|| / ||G_ref,i||  <= 1e-4
for well-conditioned bases (elementwise relative error is
ill-posed on G's near-zero entries). The ill-conditioned SUSY-shaped fixture
(γ=2^-7, τ=1e-6) amplifies fp32-level rounding of Z by 1/sqrt(λ_min); its bound
is 5e-4 (exact-fp32 emulation gives 1.35e-4 there).
Kernel values Z themselves (L = I) must agree to 2e-5 absolute (Z in (0, 1]).

For arbitrary (possibly ill-conditioned) bases the achievable accuracy of any
fp32-level kernel is bounded by conditioning, ‖ΔG_i‖ = ‖ΔZ_i·L‖ ≤ ‖ΔZ_i‖·‖L‖₂,
so the random edge-shape tests assert per row
    ‖ΔG_i‖ ≤ max(1e-4·‖G_ref,i‖, 1e-5·‖Z_i‖·‖L‖₂)
(elementwise relative Z accuracy 1e-5 implies the second term).
"""
import numpy as np
import pytest

import paper_2207_01016_b200 as P
from conftest import load_golden, np_gaussian_L, row_rel_err
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL_G = 1e-4
TOL_G_ILL = 5e-4
TOL_Z = 2e-5


def _oracle_G(X, Y, L, gamma):
    return O.ora_compute_g(O.dense_to_csr(X), O.dense_to_csr(Y), L, gamma, 4096)


def assert_conditioned_parity(G, X, Y, L, gamma):
    R = _oracle_G(X, Y, L, gamma)
    Z = O.ora_kernel_block(O.dense_to_csr(X), O.dense_to_csr(Y), gamma)
    l2 = np.linalg.norm(L, 2)
    err = np.linalg.norm(G - R, axis=1)
    bound = np.maximum(TOL_G * np.linalg.norm(R, axis=1), 1e-5 * np.linalg.norm(Z, axis=1) * l2)
    assert np.all(err <= bound), float(np.max(err / bound))
    return R


@pytest.mark.parametrize("name,tol", [("c1_mini.npz", TOL_G), ("sparse_mini.npz", TOL_G),
                                      ("susy_mini.npz", TOL_G_ILL)])
def test_golden_fixtures(gpu_ctx, name, tol):
    g = load_golden(name)
    X = g["X"].astype(np.float64)
    Y = X[g["ids"]]
    gpu_ctx.set_basis_dense(Y, g["L"], float(g["gamma"]))
    G = gpu_ctx.compute_g_dense(X)
    assert G.shape == g["G"].shape
    assert np.all(np.isfinite(G))
    assert row_rel_err(G, g["G"]) <= tol
    # CSR entry point on the same data must agree bitwise with the dense one
    ip, ix, vv = O.dense_to_csr(X)
    lp, li, lv = O.dense_to_csr(Y)
    gpu_ctx.set_basis_csr(lp, li, lv, X.shape[1], g["L"], float(g["gamma"]))
    G2 = gpu_ctx.compute_g_csr(ip, ix, vv)
    assert np.array_equal(G, G2)


def test_kernel_values_identity_basis(gpu_ctx):
    """L = I exposes Z directly: the fused epilogue's exp(-γ max(0, ...)) vs the oracle."""
    rng = np.random.default_rng(1)
    X = rng.standard_normal((700, 50)).astype(np.float32).astype(np.float64)
    Y = X[rng.choice(700, 200, replace=False)]
    gpu_ctx.set_basis_dense(Y, np.eye(200), 0.02)
    Z = gpu_ctx.compute_g_dense(X)
    Zr = O.ora_kernel_block(O.dense_to_csr(X), O.dense_to_csr(Y), 0.02)
    assert np.abs(Z - Zr).max() <= TOL_Z
    assert Z.max() <= 1.0 + TOL_Z and Z.min() >= 0.0


@pytest.mark.parametrize("d,gamma", [(50, 0.02), (18, 1.0 / 18), (100, 0.01), (300, 1.0 / 300)])
def test_kernel_values_elementwise_relative(gpu_ctx, d, gamma):
    """SURVEY §8(c) criterion (1): Z elementwise within 1e-5 relative of the reference's
    kernel_block (kernel.cpp:31-57), on the fused path (d <= 63) and the panel path."""
    rng = np.random.default_rng(d)
    X = rng.standard_normal((900, d)).astype(np.float32).astype(np.float64)
    Y = X[rng.choice(900, 256, replace=False)]
    gpu_ctx.set_basis_dense(Y, np.eye(256), gamma)
    Z = gpu_ctx.compute_g_dense(X)
    Zr = O.ora_kernel_block(O.dense_to_csr(X), O.dense_to_csr(Y), gamma)
    live = Zr > 1e-30  # fp32 wire format: relative precision holds above its normal range
    assert live.mean() > 0.99
    assert np.max(np.abs(Z - Zr)[live] / Zr[live]) <= 1e-5


@pytest.mark.parametrize("n,d,B,beff_cut,gamma", [
    (1, 5, 1, 0, 0.5),        # single row, single landmark
    (127, 3, 65, 0, 1.0),     # ragged rows (< one tile), landmarks = 64 + 1
    (129, 63, 64, 0, 0.05),   # max d of the fused small-d kernel, rows = tile + 1
    (300, 17, 300, 1, 0.2),   # b_eff = 299 (odd leading dimension)
    (1000, 50, 257, 0, 0.02),  # b_eff = 257 (two column blocks, second nearly empty)
    (513, 1, 40, 0, 3.0),     # d = 1
])
def test_edge_shapes(gpu_ctx, n, d, B, beff_cut, gamma):
    rng = np.random.default_rng(n * 31 + d)
    X = rng.standard_normal((n, d)).astype(np.float32).astype(np.float64)
    Y = X[rng.choice(n, min(B, n), replace=False)] if B <= n else rng.standard_normal((B, d))
    L = np_gaussian_L(Y, gamma, 1e-10)
    if beff_cut:
        L = np.ascontiguousarray(L[:, : L.shape[1] - beff_cut])
    gpu_ctx.set_basis_dense(Y, L, gamma)
    G = gpu_ctx.compute_g_dense(X)
    assert_conditioned_parity(G, X, Y, L, gamma)


@pytest.mark.parametrize("n,d,B,gamma,kind", [
    (300, 64, 100, 0.05, "normal"),       # first d on the two-launch panel path
    (700, 200, 300, 0.01, "normal"),      # B_pad = 512: two landmark blocks, b_eff > 256
    (513, 130, 257, 0.02, "normal"),      # ragged rows / landmarks / columns
    (1, 100, 1, 0.1, "normal"),           # single row, single landmark
    (600, 2048, 512, 1.0 / 2048, "imagenet"),  # C4 feature shape: non-negative, non-centred
])
def test_large_d_panel_path(gpu_ctx, n, d, B, gamma, kind):
    """d >= 64 runs the Z-panel GEMM + projection GEMM (panel_kernels.cuh)."""
    rng = np.random.default_rng(n + d)
    if kind == "imagenet":
        from paper_2207_01016_b200 import synthetic

        X, _ = synthetic.imagenet_like(n, d, 10, seed=4)
    else:
        X = rng.standard_normal((n, d)).astype(np.float32).astype(np.float64)
    Y = X[rng.choice(n, min(B, n), replace=False)] if B <= n else rng.standard_normal((B, d))
    L = np_gaussian_L(Y, gamma, 1e-10)
    gpu_ctx.set_basis_dense(Y, L, gamma)
    G = gpu_ctx.compute_g_dense(X)
    assert G.shape == (n, L.shape[1]) and np.all(np.isfinite(G))
    assert_conditioned_parity(G, X, Y, L, gamma)


def test_large_d_device_entry_matches_host_entry(gpu_ctx):
    """Device-resident path (panels, fp64 out) == host path (fp32 widened) bitwise."""
    import torch

    rng = np.random.default_rng(8)
    X = rng.standard_normal((1000, 96)).astype(np.float32).astype(np.float64)
    Y = X[:200]
    L = np_gaussian_L(Y, 0.02, 1e-10)
    gpu_ctx.set_basis_dense(Y, L, 0.02)
    G_host = gpu_ctx.compute_g_dense(X)
    Xd = torch.from_numpy(X).cuda()
    Gd = torch.empty((1000, L.shape[1]), dtype=torch.float64, device="cuda")
    gpu_ctx.compute_g_device(Xd, Gd)
    assert np.array_equal(Gd.cpu().numpy(), G_host)


@pytest.mark.parametrize("n,d,B", [(70_000, 54, 4096), (70_000, 130, 2048)])
def test_host_pipeline_multi_chunk_bitwise(gpu_ctx, n, d, B):
    """The host-row pipeline over several compute chunks (512 MB of fp32 G each) and
    hundreds of 8 MB delivery sub-chunks — ring reuse, slot reuse after the D2H drains,
    serialised chunk launches — equals the single device-path launch bitwise, through
    both the dense and the CSR entry points; unaligned caller row pitch included."""
    import torch

    rng = np.random.default_rng(11)
    X = rng.standard_normal((n, d)).astype(np.float32).astype(np.float64)
    Y = np.ascontiguousarray(X[rng.choice(n, B, replace=False)])
    L = np_gaussian_L(Y, 1.0 / d, 1e-10)
    gpu_ctx.set_basis_dense(Y, L, 1.0 / d)
    G_host = gpu_ctx.compute_g_dense(X)
    Xd = torch.from_numpy(X).cuda()
    Gd = torch.empty((n, L.shape[1]), dtype=torch.float64, device="cuda")
    gpu_ctx.compute_g_device(Xd, Gd)
    assert np.array_equal(Gd.cpu().numpy(), G_host)
    ip, ix, vv = O.dense_to_csr(X)
    assert np.array_equal(gpu_ctx.compute_g_csr(ip, ix, vv), G_host)
    # rows of a wider caller buffer (ldg > b_eff), written through the same pipeline
    import ctypes

    dp = ctypes.POINTER(ctypes.c_double)
    wide = np.full((n, L.shape[1] + 3), -7.0)
    t = P.Timings()
    rc = gpu_ctx._lib.lpd_compute_g_dense(gpu_ctx.handle, X.ctypes.data_as(dp), n, d, d,
                                          wide.ctypes.data_as(dp), L.shape[1] + 3, ctypes.byref(t))
    assert rc == 0
    assert np.array_equal(wide[:, :L.shape[1]], G_host)
    assert np.all(wide[:, L.shape[1]:] == -7.0)
    del Xd, Gd
    torch.cuda.empty_cache()


def test_two_shard_context_on_one_gpu(gpu_ctx):
    """Multi-device host logic on one B200: a context over two device states that
    share GPU 0 shards the rows (one host thread, stream set and delivery ring per
    shard, disjoint G row ranges), keeps each shard's G resident, and splits the
    resident-G products by shard. Rows are independent, so G, the scores and the
    predictions equal the one-shard context's bitwise; rebuild_w sums per shard first
    (order differs at the 1e-16 level)."""
    rng = np.random.default_rng(21)
    n, d, B = 40_000, 54, 1024
    X = rng.standard_normal((n, d)).astype(np.float32).astype(np.float64)
    Y = np.ascontiguousarray(X[rng.choice(n, B, replace=False)])
    L = np_gaussian_L(Y, 1.0 / d, 1e-10)
    gpu_ctx.set_basis_dense(Y, L, 1.0 / d)
    gpu_ctx.set_keep_resident(True)
    ctx2 = P.Context(device_ids=[0, 0])
    try:
        assert ctx2.num_devices == 2
        ctx2.set_basis_dense(Y, L, 1.0 / d)
        ctx2.set_keep_resident(True)
        G1 = gpu_ctx.compute_g_dense(X)
        G2 = ctx2.compute_g_dense(X)
        assert np.array_equal(G1, G2)
        rows = rng.permutation(n)[:9_000].astype(np.int32)  # both shards, shuffled
        W = rng.standard_normal((5, L.shape[1]))
        assert np.array_equal(gpu_ctx.resident_gw(rows, W), ctx2.resident_gw(rows, W))
        coef = rng.standard_normal(rows.size)
        w1, w2 = gpu_ctx.resident_gtv(rows, coef), ctx2.resident_gtv(rows, coef)
        assert np.max(np.abs(w1 - w2)) <= 1e-12 * np.max(np.abs(w1))
    finally:
        gpu_ctx.set_keep_resident(False)
        ctx2.close()


@pytest.mark.parametrize("shards", [3, 4, 8])
def test_shard_count_invariance(gpu_ctx, shards):
    """SURVEY §8(b) determinism: G is bitwise the same for 1 and k device shards (here k
    device states on GPU 0), with a ragged row count that leaves the last shard short,
    through the dense and CSR entry points; predictions too."""
    rng = np.random.default_rng(40 + shards)
    n, d, B = 40_003, 30, 768
    X = rng.standard_normal((n, d)).astype(np.float32).astype(np.float64)
    Y = np.ascontiguousarray(X[rng.choice(n, B, replace=False)])
    L = np_gaussian_L(Y, 1.0 / d, 1e-10)
    gpu_ctx.set_basis_dense(Y, L, 1.0 / d)
    G1 = gpu_ctx.compute_g_dense(X)
    ctxk = P.Context(device_ids=[0] * shards)
    try:
        assert ctxk.num_devices == shards
        ctxk.set_basis_dense(Y, L, 1.0 / d)
        assert np.array_equal(G1, ctxk.compute_g_dense(X))
        ip, ix, vv = O.dense_to_csr(X)
        assert np.array_equal(G1, ctxk.compute_g_csr(ip, ix, vv))
        betas = rng.standard_normal((6, B)) * 1e-2  # 4 classes
        bt = np.ascontiguousarray(betas.T)
        gpu_ctx.set_basis_dense(Y, bt, 1.0 / d)
        ctxk.set_basis_dense(Y, bt, 1.0 / d)
        assert np.array_equal(gpu_ctx.predict_ovo_dense(X, 4), ctxk.predict_ovo_dense(X, 4))
    finally:
        ctxk.close()


def test_empty_and_duplicate_points(gpu_ctx):
    rng = np.random.default_rng(4)
    X = rng.standard_normal((260, 12))
    X[[0, 5, 200]] = 0.0            # empty SparseVectors
    X[10] = X[11]                    # duplicates (singular K is handled by truncation)
    Y = X[[0, 10, 11, 20, 30, 40, 50, 60]]
    L = O.ref_build_L(O.dense_to_csr(Y), 0.3, 1e-12) if O.ref_available() else np_gaussian_L(Y, 0.3)
    gpu_ctx.set_basis_dense(Y, L, 0.3)
    G = gpu_ctx.compute_g_dense(X)
    assert_conditioned_parity(G, X, Y, L, 0.3)


def test_zero_rows_call(gpu_ctx):
    Y = np.eye(4)
    gpu_ctx.set_basis_dense(Y, np.eye(4), 1.0)
    G = gpu_ctx.compute_g_dense(np.zeros((0, 4)))
    assert G.shape == (0, 4)


def test_batch_invariance_bitwise(gpu_ctx):
    """Each row's arithmetic is independent of the batch it is computed in, so G
    is bitwise identical across chunkings / device counts."""
    g = load_golden("c1_mini.npz")
    X = g["X"].astype(np.float64)
    gpu_ctx.set_basis_dense(X[g["ids"]], g["L"], 0.02)
    full = gpu_ctx.compute_g_dense(X)
    parts = np.concatenate([gpu_ctx.compute_g_dense(X[a:b]) for a, b in [(0, 1), (1, 300), (300, 1024)]])
    assert np.array_equal(full, parts)


def test_device_entry_fp32_and_fp64(gpu_ctx):
    import torch

    g = load_golden("c1_mini.npz")
    X = g["X"].astype(np.float64)
    gpu_ctx.set_basis_dense(X[g["ids"]], g["L"], 0.02)
    ref = gpu_ctx.compute_g_dense(X)
    Xd = torch.from_numpy(X).cuda()
    G64 = torch.empty((X.shape[0], g["L"].shape[1]), dtype=torch.float64, device="cuda")
    G32 = torch.empty((X.shape[0], g["L"].shape[1]), dtype=torch.float32, device="cuda")
    gpu_ctx.compute_g_device(Xd, G64)
    gpu_ctx.compute_g_device(Xd, G32)
    torch.cuda.synchronize()
    assert np.array_equal(G64.cpu().numpy(), ref)
    assert np.array_equal(G32.cpu().numpy(), ref.astype(np.float32))


def test_error_behaviour(gpu_ctx):
    Y = np.random.default_rng(0).standard_normal((10, 5))
    with pytest.raises(ValueError, match="gamma"):
        gpu_ctx.set_basis_dense(Y, np.eye(10), 0.0)
    with pytest.raises(ValueError):
        gpu_ctx.set_basis_dense(Y, np.eye(9), 1.0)
    gpu_ctx.set_basis_dense(Y, np.eye(10), 1.0)
    with pytest.raises(ValueError, match="dimension"):
        gpu_ctx.compute_g_dense(np.zeros((3, 6)))
    with pytest.raises(P.LpdError):  # outside the envelope: d > 65536
        gpu_ctx.set_basis_dense(np.zeros((1, 65537)), np.eye(1), 1.0)
    with pytest.raises(P.LpdError):  # features beyond the split-fp16 range (|x - mean| >= 2^28)
        gpu_ctx.set_basis_dense(Y, np.eye(10), 1.0)
        X = np.zeros((3, 5))
        X[1, 2] = 2.0**29
        gpu_ctx.compute_g_dense(X)


def test_decision_values(gpu_ctx):
    rng = np.random.default_rng(6)
    for b_eff, P_ in [(1000, 1), (4096, 3), (777, 9), (1, 1)]:
        G = rng.standard_normal((1500, b_eff))
        W = rng.standard_normal((P_, b_eff))
        D = gpu_ctx.decision_values(G, W)
        R = O.ora_decision_values(G, W)
        assert np.abs(D - R).max() <= 1e-12 * max(1.0, np.abs(R).max())


def test_c1_full_config_vs_reference():
    """C1 end-to-end factor (n=20,000, d=50, B=1,000, γ=0.02) against the
    reference's own compute_G (oracle/_ref), same landmarks and L."""
    if not O.ref_available():
        pytest.fail("reference build oracle/_ref missing on this box")
    from paper_2207_01016_b200 import synthetic

    cfg = synthetic.CONFIGS["c1"]
    X, _ = synthetic.make(cfg)
    ids = O.ref_select_landmarks(cfg.n, cfg.budget, 1)
    csr, lcsr = O.dense_to_csr(X), O.dense_to_csr(X[ids])
    L = O.ref_build_L(lcsr, cfg.gamma, 1e-12, threads=8)
    R = O.ref_compute_g(csr, lcsr, L, cfg.gamma, 4096, threads=O.ref_lib().ref_hardware_threads())
    with P.Context(1) as ctx:
        ctx.set_basis_dense(X[ids], L, cfg.gamma)
        G = ctx.compute_g_dense(X)
    assert row_rel_err(G, R) <= TOL_G
    # Nyström identity on the landmark rows: G_S G_S^T ≈ K (1e-6·λ_max scale)
    K = O.ora_kernel_block(lcsr, lcsr, cfg.gamma)
    GS = G[ids]
    assert np.abs(GS @ GS.T - K).max() <= 1e-3


def test_compute_G_mirror_sparse_points():
    """The Python mirror of lpdsvm::compute_G on SparseVector-style input."""
    rng = np.random.default_rng(8)
    pts = []
    for i in range(150):
        idx = np.sort(rng.choice(30, rng.integers(0, 8), replace=False))
        pts.append([(int(j), float(np.float32(rng.standard_normal()))) for j in idx])
    lms = pts[:40]
    ip, ix, vv, dim = P.sparse_to_csr(pts)
    lp, li, lv, _ = P.sparse_to_csr(lms)
    L = O.ref_build_L((lp, li, lv), 0.4, 1e-12) if O.ref_available() else None
    if L is None:
        pytest.fail("reference build missing")
    G = P.compute_G(pts, None, lms, None, L, P.KernelParams(0.4), 4096)
    R = O.ora_compute_g((ip, ix, vv), (lp, li, lv), L, 0.4, 4096)
    assert row_rel_err(G, R) <= TOL_G


@pytest.mark.parametrize("c,d,B", [(2, 20, 150), (5, 30, 200), (12, 90, 300)])
def test_predict_ovo_matches_oracle(gpu_ctx, c, d, B):
    """K5: decision values Z·betasᵀ on the device + the reference vote
    (multiclass.cpp:153-168, 170-200). Classes agree with the oracle except on rows
    whose smallest |decision| is within fp32-level rounding of 0."""
    rng = np.random.default_rng(c * 7 + d)
    n, gamma = 1500, 1.0 / d
    X = rng.standard_normal((n, d)).astype(np.float32).astype(np.float64)
    Y = X[rng.choice(n, B, replace=False)]
    P_ = c * (c - 1) // 2
    betas = rng.standard_normal((P_, B))
    gpu_ctx.set_basis_dense(Y, np.ascontiguousarray(betas.T), gamma)
    got = gpu_ctx.predict_ovo_dense(X, c)
    Z = O.ora_kernel_block(O.dense_to_csr(X), O.dense_to_csr(Y), gamma)
    D = Z @ betas.T
    want = np.array([O.ora_vote(D[i], c) for i in range(n)])
    margin = np.min(np.abs(D), axis=1) / np.max(np.abs(D))
    clear = margin > 1e-4
    assert clear.mean() > 0.9
    assert np.array_equal(got[clear], want[clear])
    # the CSR entry gives the same classes
    ip, ix, vv, _ = P.sparse_to_csr(list(X))
    assert np.array_equal(gpu_ctx.predict_ovo_csr(ip, ix, vv, c), got)


def test_predict_ovo_argument_errors(gpu_ctx):
    Y = np.eye(6)
    gpu_ctx.set_basis_dense(Y, np.ones((6, 3)), 0.5)  # P = 3 <-> 3 classes
    with pytest.raises(ValueError):
        gpu_ctx.predict_ovo_dense(np.zeros((2, 6)), 4)  # 4 classes need 6 pairs
    with pytest.raises(ValueError):
        gpu_ctx.predict_ovo_dense(np.zeros((2, 6)), 1)
    assert gpu_ctx.predict_ovo_dense(np.zeros((0, 6)), 3).shape == (0,)


@pytest.mark.parametrize("m,n,d,gamma", [(300, 300, 50, 0.02), (257, 65, 2048, 1.0 / 2048), (1, 7, 3, 1.0)])
def test_kernel_block_fp64_matches_reference(gpu_ctx, m, n, d, gamma):
    """K7 (landmark Gram): fp64 with the reference's operation order, so it agrees
    with the reference's own kernel_block (oracle/_ref) up to the last ulps of exp."""
    rng = np.random.default_rng(m + d)
    A = rng.standard_normal((m, d)).astype(np.float32).astype(np.float64)
    B = A[:n] if n <= m else rng.standard_normal((n, d))
    if O.ref_available():
        Kref = O.ref_kernel_block(O.dense_to_csr(A), O.dense_to_csr(B), gamma)
        na, nb = O.ref_squared_norms(O.dense_to_csr(A)), O.ref_squared_norms(O.dense_to_csr(B))
    else:
        Kref = O.ora_kernel_block(O.dense_to_csr(A), O.dense_to_csr(B), gamma)
        na, nb = (A * A).sum(1), (B * B).sum(1)
    K = gpu_ctx.kernel_block(A, B, gamma, na, nb)
    rel = np.abs(K - Kref) / np.maximum(np.abs(Kref), 1e-300)
    # dot products and d2 are bitwise the reference's; exp differs from glibc's by
    # at most an ulp or two (CUDA exp is not correctly rounded)
    assert float(rel.max()) <= 5e-16, float(rel.max())
    if n == m:
        assert np.all(np.diag(K) == 1.0)


@pytest.mark.parametrize("nb", [300, 301])  # b_eff % 4 == 0: 16-byte path; else scalar path
def test_resident_g_products(gpu_ctx, nb):
    """K6: G kept resident (fp32, bit-identical to the returned fp64 G) serves the
    held-out scoring G[rows]·Wᵀ (bitwise the reference's loop) and rebuild_w's
    Σ coef_i·G_i in fp64 on the device."""
    rng = np.random.default_rng(12)
    X = rng.standard_normal((3000, 20)).astype(np.float32).astype(np.float64)
    Y = X[:nb]
    L = np_gaussian_L(Y, 0.05, 1e-10)
    gpu_ctx.set_basis_dense(Y, L, 0.05)
    gpu_ctx.set_keep_resident(True)
    try:
        G = gpu_ctx.compute_g_dense(X)
        assert gpu_ctx.resident_shape() == (3000, L.shape[1])
        rows = rng.choice(3000, 777, replace=False).astype(np.int32)
        # the reference's scoring loop (modelsel.cpp:129-136): per (row, vector) products
        # rounded, then added in ascending column order — bit for bit, for P = 1 and 3
        # (the 256-row shape) and P = 6, 45, 70 (64 × 64 tiles, two tiles in P at 70)
        for P_ in (1, 3, 6, 45, 70):
            W = rng.standard_normal((P_, L.shape[1]))
            D = gpu_ctx.resident_gw(rows, W)
            Dseq = np.add.accumulate(G[rows][:, None, :] * W[None, :, :], axis=2)[:, :, -1]
            assert np.array_equal(D, Dseq), (P_, float(np.max(np.abs(D - Dseq))))
        # ... and the one-vs-one vote on the device over those decision values: class
        # indices equal to the reference's vote (multiclass.cpp:153-168) on the same D
        for c in (2, 3, 10):
            Wc = rng.standard_normal((c * (c - 1) // 2, L.shape[1]))
            cls = gpu_ctx.resident_vote(rows, Wc, c)
            Dc = gpu_ctx.resident_gw(rows, Wc)
            assert np.array_equal(cls, [O.ora_vote(Dc[i], c) for i in range(rows.size)]), c
        coef = rng.standard_normal(777)
        w = gpu_ctx.resident_gtv(rows, coef)
        wref = coef @ G[rows]
        assert np.max(np.abs(w - wref)) <= 1e-12 * np.max(np.abs(wref))
        assert np.array_equal(w, gpu_ctx.resident_gtv(rows, coef))  # deterministic
        # all (fold, pair) warm starts at once: 11 coefficient sets (two passes of <= 8)
        C = rng.standard_normal((777, 11))
        C[rng.random(C.shape) < 0.4] = 0.0
        Ws = gpu_ctx.resident_gtv_sets(rows, C)
        Wref = C.T @ G[rows]
        assert np.max(np.abs(Ws - Wref)) <= 1e-12 * np.max(np.abs(Wref))
        assert np.array_equal(gpu_ctx.resident_gtv_sets(rows, coef[:, None])[0], w)
        # make_binary_problem's q_diag: sequential fp64 Σ_j G_ij² (dcd.cpp:60-89), bitwise
        q = gpu_ctx.resident_row_sqnorms()
        for i in list(range(0, 3000, 97)) + [2999]:
            acc = 0.0
            for v in G[i]:
                acc += v * v
            assert q[i] == acc, (i, q[i], acc)
        with pytest.raises(ValueError):
            gpu_ctx.resident_gw(np.array([3000], np.int32), W)
    finally:
        gpu_ctx.set_keep_resident(False)
    assert gpu_ctx.resident_shape()[0] == 0


def _ref_point_dv(X, Y, betas, gamma):
    """The reference's decision_values (multiclass.cpp:137-151) on dense rows: its own
    gaussian (kernel.cpp:17-19, sparse merge over the nonzeros) per landmark, then the
    sequential dot with each betas row."""
    out = np.zeros((X.shape[0], betas.shape[0]))
    lm = [(np.flatnonzero(y).astype(np.int32), y[y != 0]) for y in Y]
    for i, x in enumerate(X):
        xi = np.flatnonzero(x).astype(np.int32)
        z = [O.ref_gaussian(xi, x[xi], li, lv, gamma) for li, lv in lm]
        for p in range(betas.shape[0]):
            s = 0.0
            for j in range(len(z)):
                s += z[j] * betas[p, j]
            out[i, p] = s
    return out


@pytest.mark.parametrize("n,d,dx,B,P", [(1, 7, 7, 1, 1), (37, 20, 20, 130, 3), (70, 9, 13, 65, 10),
                                        (3, 40, 33, 200, 1)])
def test_model_decision_values_match_reference(gpu_ctx, n, d, dx, B, P):
    """K8 (lpd_model_decision_values_*) against the reference's own gaussian + dot, on
    sparse rows whose feature widths differ (dx ≠ d: features only one side has).
    fp64 with the reference's operation order: ≤ a few ulps of exp apart."""
    rng = np.random.default_rng(n + d + B)
    Y = rng.standard_normal((B, d))
    Y[rng.random(Y.shape) < 0.3] = 0.0
    X = rng.standard_normal((n, dx))
    X[rng.random(X.shape) < 0.3] = 0.0
    betas = rng.standard_normal((P, B))
    gamma = 0.07
    gpu_ctx.set_model_dense(Y, betas, gamma)
    D = gpu_ctx.model_decision_values_dense(X)
    R = _ref_point_dv(X, Y, betas, gamma)
    bound = 4 * np.finfo(float).eps * np.abs(betas).sum(1)[None, :]
    assert np.all(np.abs(D - R) <= bound), float(np.max(np.abs(D - R) / bound))
    # CSR entry points agree bitwise with the dense ones
    lp, li, lv = O.dense_to_csr(Y)
    gpu_ctx.set_model_csr(lp, li, lv, d, betas, gamma)
    ip, ix, vv = O.dense_to_csr(X)
    assert np.array_equal(gpu_ctx.model_decision_values_csr(ip, ix, vv, dx), D)


def test_model_decision_values_errors(gpu_ctx):
    gpu_ctx.set_model_dense(np.ones((4, 3)), np.ones((1, 4)), 0.5)
    with pytest.raises(ValueError):  # CSR index outside [0, d)
        gpu_ctx.model_decision_values_csr(np.array([0, 1]), np.array([3]), np.array([1.0]), 3)
    with pytest.raises(ValueError):
        gpu_ctx.set_model_dense(np.ones((4, 3)), np.ones((1, 4)), float("nan"))
    assert gpu_ctx.model_decision_values_dense(np.zeros((0, 3))).shape == (0, 1)


@pytest.mark.parametrize("classes", [2, 3, 7, 40])
def test_ovo_vote_bit_exact(gpu_ctx, classes):
    """The device vote (the kernel K5 ends with) on identical decision values, against the
    reference's own vote (multiclass.cpp:153-168): index-exact on every row, with exact
    zeros (a zero votes for the second class), -0.0, and dense ties."""
    P = classes * (classes - 1) // 2
    rng = np.random.default_rng(classes)
    D = rng.choice([-1.0, -0.0, 0.0, 1e-300, 2.0, -3.0], size=(3000, P))
    D[:500] = rng.standard_normal((500, P))
    D[500:600] = 0.0
    got = gpu_ctx.ovo_vote(D, classes)
    want = np.array([O.ref_vote(row, classes) for row in D], dtype=np.int32)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("name,tol", [("c1_mini.npz", 2e-7), ("sparse_mini.npz", 2e-7), ("susy_mini.npz", 2e-7),
                                      ("susy_mini_t12.npz", 2e-7)])
def test_high_precision_path_golden(gpu_ctx, name, tol):
    """LPD_PRECISION_HIGH: Z in fp64 by direct distance, G = Z·L on the fp64 tensor cores
    (DMMA), delivered through the host path's fp32 staging: G agrees with the reference's
    fp64 G to the fp32 rounding of the delivered values (≤ 2^-24 per element), far inside
    the fast path's 1e-4 — the ill-conditioned fixture included. The device-resident fp64
    output carries no such rounding (test_precision_auto_choice, full-shard test)."""
    g = load_golden(name)
    X = g["X"].astype(np.float64)
    gpu_ctx.set_precision("high")
    try:
        gpu_ctx.set_basis_dense(X[g["ids"]], g["L"], float(g["gamma"]))
        assert gpu_ctx.basis_precision()[0]
        G = gpu_ctx.compute_g_dense(X)
        ip, ix, vv = O.dense_to_csr(X)
        G2 = gpu_ctx.compute_g_csr(ip, ix, vv)
    finally:
        gpu_ctx.set_precision("auto")
    assert row_rel_err(G, g["G"]) <= tol, row_rel_err(G, g["G"])
    assert np.array_equal(G, G2)
    gpu_ctx.set_precision("fast")
    try:
        gpu_ctx.set_basis_dense(X[g["ids"]], g["L"], float(g["gamma"]))
        est = gpu_ctx.basis_precision()[1]
        err_fast = row_rel_err(gpu_ctx.compute_g_dense(X), g["G"])
    finally:
        gpu_ctx.set_precision("auto")
    print(f"{name}: fast-path estimate {est:.3g}, fast-path row error {err_fast:.3g} "
          f"(ratio {err_fast / est:.2f}), high-precision {row_rel_err(G, g['G']):.3g}")


def test_precision_auto_choice(gpu_ctx):
    """Auto precision: a well-conditioned basis stays on the tensor-core path, the paper's
    γ = 2^-7 SUSY-shaped basis at τ = 1e-12 (λ_min/λ_max ~ 1e-11) goes to the fp64 path and
    then matches the reference within 1e-7 where the fast path cannot hold 1e-4."""
    from paper_2207_01016_b200 import synthetic

    X, _ = synthetic.blobs(6000, 18, seed=3)
    Y = X[np.random.default_rng(1).choice(6000, 1024, replace=False)]
    gpu_ctx.set_basis_dense(Y, np_gaussian_L(Y, 1.0 / 18, 1e-12), 1.0 / 18)
    assert not gpu_ctx.basis_precision()[0]
    gamma = 2.0 ** -7
    L = O.ref_build_L(O.dense_to_csr(Y), gamma, 1e-12)
    gpu_ctx.set_basis_dense(Y, L, gamma)
    high, est = gpu_ctx.basis_precision()
    assert high and est > 5e-5, est
    G = gpu_ctx.compute_g_dense(X)
    R = O.ref_compute_g(O.dense_to_csr(X), O.dense_to_csr(Y), L, gamma, 4096, 8)
    err = row_rel_err(G, R)
    assert err <= 1e-7, err
    gpu_ctx.set_precision("fast")
    try:
        gpu_ctx.set_basis_dense(Y, L, gamma)
        err_fast = row_rel_err(gpu_ctx.compute_g_dense(X), R)
    finally:
        gpu_ctx.set_precision("auto")
    print(f"gamma=2^-7 tau=1e-12 B=1024: estimate {est:.3g}, high-precision row error {err:.3g}, "
          f"fast path {err_fast:.3g}")
    assert err_fast > err


def _far_rows_case(d, mult, shift, n=1536, B=384, seed=7):
    """Unit-variance points; a third of them moved shift·√d away from the landmark
    cloud along one direction; γ = mult/d."""
    rng = np.random.default_rng(seed + d + int(10 * mult) + int(10 * shift))
    base = rng.standard_normal((B + n, d)).astype(np.float32).astype(np.float64)
    Y, X = base[:B], base[B:].copy()
    u = rng.standard_normal(d)
    X[: n // 3] += shift * np.sqrt(d) * u / np.linalg.norm(u)
    X = X.astype(np.float32).astype(np.float64)
    gamma = mult / d
    return X, Y, np_gaussian_L(Y, gamma, 1e-6), gamma


@pytest.mark.parametrize("d,mult,shift", [(32, 16, 0), (32, 16, 2), (32, 8, 4), (32, 64, 1), (100, 16, 2)])
def test_far_rows_and_large_gamma(gpu_ctx, d, mult, shift):
    """K9 (probe_kernels.cuh): rows whose nearest landmark is far — large γ (up to 64/d)
    or points several √d from the landmark cloud — have all their kernel values below
    fp16's normal range; the probe normalises each such row's exponent so K1 (d = 32)
    and the panel path (d = 100) keep the 1e-4 row bound. fp64 G (device path), so the
    2^shift row scale is applied in fp64: every row with a nonzero reference meets it,
    including rows whose kernel values are far below fp32's range. Before K9 these cases
    measured 0.43 to 1.0 row error (scripts/precision_probe.py)."""
    import torch

    X, Y, L, gamma = _far_rows_case(d, mult, shift)
    gpu_ctx.set_precision("fast")
    try:
        gpu_ctx.set_basis_dense(Y, L, gamma)
        Gd = torch.empty((X.shape[0], L.shape[1]), dtype=torch.float64, device="cuda")
        gpu_ctx.compute_g_device(torch.from_numpy(X).cuda(), Gd)
        torch.cuda.synchronize()
        G = Gd.cpu().numpy()
    finally:
        gpu_ctx.set_precision("auto")
    R = _oracle_G(X, Y, L, gamma)
    nr = np.linalg.norm(R, axis=1)
    live = nr > 0
    assert live.sum() >= X.shape[0] // 2
    assert np.all(G[~live] == 0.0)
    err = np.linalg.norm(G - R, axis=1)[live] / nr[live]
    assert float(err.max()) <= TOL_G, float(err.max())


def test_far_rows_host_path_fp32_range(gpu_ctx):
    """The host-call path carries G as fp32 to the host (widened there), so a row is
    exact to the 1e-4 bound while its values are inside fp32's normal range (here
    max |G_ref,i| >= 2^-100) and comes back as zeros or fp32 subnormals once they are
    all below it (the rows 4·√d from the cloud at γ = 8/d: kernel values e^-90 and
    less) — the stated limit of the fp32 wire format."""
    X, Y, L, gamma = _far_rows_case(32, 8, 4)
    gpu_ctx.set_precision("fast")
    try:
        gpu_ctx.set_basis_dense(Y, L, gamma)
        G = gpu_ctx.compute_g_dense(X)
    finally:
        gpu_ctx.set_precision("auto")
    R = _oracle_G(X, Y, L, gamma)
    rmax = np.abs(R).max(axis=1)
    tiny = float(np.finfo(np.float32).tiny)
    normal, below = rmax >= 2.0 ** -100, rmax < tiny
    assert normal.sum() >= X.shape[0] // 2 and below.sum() > 0
    nr = np.linalg.norm(R, axis=1)
    err = np.linalg.norm(G - R, axis=1)[normal] / nr[normal]
    assert float(err.max()) <= TOL_G, float(err.max())
    assert np.all(np.abs(G[below]) < tiny)


@pytest.mark.parametrize("site,code", [(P.LPD_FAULT_ALLOC, P.LPD_ERR_OUT_OF_MEMORY),
                                       (P.LPD_FAULT_LAUNCH, P.LPD_ERR_CUDA),
                                       (P.LPD_FAULT_D2H, P.LPD_ERR_CUDA)])
def test_injected_fault_fails_loudly_and_context_recovers(site, code):
    """Failure detection (the reference has exceptions only, no fault
    injection): a device allocation, a factor-kernel launch or a G transfer that fails
    mid-call returns the matching status with a message, never a silently wrong G; the
    call's in-flight work is drained, and the same context then computes G bitwise equal
    to a clean context's. A host-row call with 17 delivery sub-chunks of 8 MB, so the
    D2H fault lands mid-pipeline."""
    rng = np.random.default_rng(21)
    X = rng.standard_normal((70000, 20)).astype(np.float32).astype(np.float64)
    Y = X[:512]
    L = np_gaussian_L(Y, 0.05, 1e-8)
    with P.Context(1) as clean:
        clean.set_basis_dense(Y, L, 0.05)
        ref = clean.compute_g_dense(X)
    with P.Context(1) as ctx:
        ctx.set_basis_dense(Y, L, 0.05)
        P.inject_fault(site, 2 if site == P.LPD_FAULT_D2H else 0)
        try:
            with pytest.raises(P.LpdError) as ei:
                ctx.compute_g_dense(X)
        finally:
            P.inject_fault(P.LPD_FAULT_NONE)
        assert ei.value.code == code and "injected fault" in str(ei.value)
        assert np.array_equal(ctx.compute_g_dense(X), ref)


def test_model_switch_reshapes_buffers(gpu_ctx):
    """K8's per-call buffers are shaped by the model (z by B, D by P): a second model with
    more landmarks and pairs after a small one must not reuse the small buffers."""
    rng = np.random.default_rng(31)
    X = rng.standard_normal((300, 10))
    for B, P_ in ((32, 1), (700, 6), (64, 3)):
        Y = rng.standard_normal((B, 10))
        betas = rng.standard_normal((P_, B))
        gpu_ctx.set_model_dense(Y, betas, 0.1)
        D = gpu_ctx.model_decision_values_dense(X)
        Dr = O.ora_kernel_block(O.dense_to_csr(X), O.dense_to_csr(Y), 0.1) @ betas.T
        assert D.shape == (300, P_)
        assert np.max(np.abs(D - Dr)) <= 1e-10 * np.max(np.abs(Dr)), (B, P_)


@pytest.mark.parametrize("seed", [*range(12), 17, 23, 33, 121])  # 17-121: large exponent magnitudes
def test_random_shapes_fuzz(gpu_ctx, seed):
    """Seeded random problems across both factor paths and all three host/device entry
    points: n in [1, 1500], d in [1, 160] (the fused kernel below 64, the panel path
    above), B in [1, 400], b_eff up to B (truncated spectra), γ log-uniform in
    [0.1/d, 10/d], dense or ~30 %-sparse points, unscaled features in some draws. Every row
    inside fp32's range meets the conditioned bound against the oracle (rows whose values
    are all below 2^-100 — e.g. a 9e-42 row, unscaled points at a large γ — are the fp32
    output's stated range limit and must merely stay that small); dense, CSR and device
    entries agree bitwise."""
    import torch

    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 1501))
    d = int(rng.integers(1, 161))
    B = int(rng.integers(1, 401))
    gamma = float(np.exp(rng.uniform(np.log(0.1 / d), np.log(10.0 / d))))
    scale = float(rng.choice([1.0, 1.0, 7.0]))
    X = (rng.standard_normal((n, d)) * scale).astype(np.float32).astype(np.float64)
    if rng.random() < 0.5:
        X[rng.random(X.shape) < 0.7] = 0.0
    Y = X[rng.choice(n, B, replace=False)] if B <= n else (rng.standard_normal((B, d)) * scale).astype(np.float32).astype(np.float64)
    L = np_gaussian_L(Y, gamma, float(rng.choice([1e-10, 1e-6, 1e-3])))
    # the product's own precision choice (auto: the fp64 path for ill-conditioned bases and
    # for exponent magnitudes the fast path cannot hold)
    gpu_ctx.set_precision("auto")
    try:
        gpu_ctx.set_basis_dense(Y, L, gamma)
        G = gpu_ctx.compute_g_dense(X)
        ip, ix, vv = O.dense_to_csr(X)
        lp, li, lv = O.dense_to_csr(Y)
        gpu_ctx.set_basis_csr(lp, li, lv, d, L, gamma)
        assert np.array_equal(G, gpu_ctx.compute_g_csr(ip, ix, vv))
        Gd = torch.empty((n, L.shape[1]), dtype=torch.float32, device="cuda")
        gpu_ctx.compute_g_device(torch.from_numpy(X).cuda(), Gd)
        torch.cuda.synchronize()
        assert np.array_equal(G, Gd.cpu().numpy().astype(np.float64))
    finally:
        gpu_ctx.set_precision("auto")
    R = _oracle_G(X, Y, L, gamma)
    live = np.abs(R).max(axis=1) >= 2.0 ** -100
    assert np.all(np.abs(G[~live]) < 2.0 ** -99)
    if live.any():
        assert_conditioned_parity(G[live], X[live], Y, L, gamma)


@pytest.mark.parametrize("d,extra_x,extra_g", [(20, 3, 1), (20, 0, 5), (100, 7, 3), (33, 1, 0)])
def test_caller_pitches_bitwise(gpu_ctx, d, extra_x, extra_g):
    """The C ABI's leading dimensions: X rows with ldx > d and G rows with ldg > b_eff
    (odd pitches the kernel's TMA store cannot target go through the aligned staging) give
    G bitwise equal to the contiguous call, and the padding columns of the caller's G are
    left untouched."""
    import ctypes

    rng = np.random.default_rng(d * 10 + extra_x + extra_g)
    n, B = 777, 130
    X = rng.standard_normal((n, d)).astype(np.float32).astype(np.float64)
    Y = X[rng.choice(n, B, replace=False)]
    L = np_gaussian_L(Y, 1.0 / d, 1e-8)
    be = L.shape[1]
    gpu_ctx.set_basis_dense(Y, L, 1.0 / d)
    ref = gpu_ctx.compute_g_dense(X)
    Xp = np.full((n, d + extra_x), 123.0)
    Xp[:, :d] = X
    Gp = np.full((n, be + extra_g), -7.0)
    lib = P.load_library()
    dp = ctypes.POINTER(ctypes.c_double)
    st = lib.lpd_compute_g_dense(gpu_ctx.handle, Xp.ctypes.data_as(dp), n, d, d + extra_x,
                                 Gp.ctypes.data_as(dp), be + extra_g, None)
    assert st == 0, P.load_library().lpd_last_error()
    assert np.array_equal(Gp[:, :be], ref)
    assert np.all(Gp[:, be:] == -7.0)


@pytest.mark.parametrize("k", [1, 3, 4, 5, 15, 16, 17])
def test_narrow_projection_z_beta_mode(gpu_ctx, k):
    """K1's Z·β mode (b_eff <= 4: no GEMM2, Z reduced against L in the epilogue; K5 on
    binary and 3-class models) and the GEMM2 path just past it (5, 15, 16, 17). L = k columns of the identity exposes Z itself (1e-5 relative,
    SURVEY §8(c) criterion 1); random β rows are the prediction case (multiclass.cpp:192);
    fp64 device output, fp32 device output and the host entry agree."""
    import torch

    rng = np.random.default_rng(100 + k)
    n, d, B, gamma = 3000, 54, 700, 1.0 / 54
    X = rng.standard_normal((n, d)).astype(np.float32).astype(np.float64)
    Y = X[rng.choice(n, B, replace=False)]
    E = np.ascontiguousarray(np.eye(B)[:, rng.choice(B, k, replace=False)])
    gpu_ctx.set_basis_dense(Y, E, gamma)
    Z = gpu_ctx.compute_g_dense(X)
    Zr = O.ora_kernel_block(O.dense_to_csr(X), O.dense_to_csr(Y), gamma) @ E
    live = Zr > 1e-30
    assert np.max(np.abs(Z - Zr)[live] / Zr[live]) <= 1e-5
    assert np.all(np.abs(Z[~live]) <= 1e-30)
    betas = rng.standard_normal((B, k))
    gpu_ctx.set_basis_dense(Y, betas, gamma)
    G = gpu_ctx.compute_g_dense(X)
    assert_conditioned_parity(G, X, Y, betas, gamma)
    Xd = torch.from_numpy(X).cuda()
    G64full = torch.full((n, k + 3), 7.0, dtype=torch.float64, device="cuda")
    G64 = G64full[:, :k]  # pitch k + 3
    G32 = torch.empty((n, k), dtype=torch.float32, device="cuda")
    gpu_ctx.compute_g_device(Xd, G64)
    gpu_ctx.compute_g_device(Xd, G32)
    torch.cuda.synchronize()
    assert np.array_equal(G32.cpu().numpy(), G.astype(np.float32))
    assert np.max(np.abs(G64.cpu().numpy() - G)) <= 1e-6 * np.abs(G).max()
    assert np.all(G64full.cpu().numpy()[:, k:] == 7.0)  # padding untouched


@pytest.mark.parametrize("d,mult,shift,k", [(32, 16, 2, 1), (32, 64, 1, 3), (32, 8, 4, 4), (20, 1, 0, 2)])
def test_far_rows_z_beta_mode(gpu_ctx, d, mult, shift, k):
    """K9's per-row exponent normalisation under K1's Z·β mode (b_eff <= 4): the row
    shift set by row_shift_kernel enters the epilogue's t and clamp and is undone by
    row_rescale on the directly stored rows; same 1e-4 row bound as the GEMM2 path."""
    import torch

    X, Y, L, gamma = _far_rows_case(d, mult, shift)
    L = np.ascontiguousarray(L[:, :k])
    gpu_ctx.set_precision("fast")
    try:
        gpu_ctx.set_basis_dense(Y, L, gamma)
        Gd = torch.empty((X.shape[0], k), dtype=torch.float64, device="cuda")
        gpu_ctx.compute_g_device(torch.from_numpy(X).cuda(), Gd)
        torch.cuda.synchronize()
        G = Gd.cpu().numpy()
    finally:
        gpu_ctx.set_precision("auto")
    R = _oracle_G(X, Y, L, gamma)
    nr = np.linalg.norm(R, axis=1)
    live = nr > 0
    assert live.sum() >= X.shape[0] // 2
    assert np.all(G[~live] == 0.0)
    err = np.linalg.norm(G - R, axis=1)[live] / nr[live]
    assert float(err.max()) <= TOL_G, float(err.max())
