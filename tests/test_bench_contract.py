"""bench.py's JSON contract, checked on CPU through the reference arm (`--impl
reference`: the reference's own compute_G from oracle/_ref on the host cores) at a
tiny size. The GPU arm prints the same keys (plus roofline / clocks / gpu_launches);
it is exercised on the B200 by the driver."""
import json
import os
import subprocess
import sys

import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref is built where /root/reference exists")
def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "c1",
                          "--rows", "2048", "--steps", "1", "--warmup", "1", "--no-extras"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in j, k
    assert j["impl"] == "reference" and j["unit"] == "rows/s" and j["higher_is_better"] is True
    assert j["value"] > 0 and j["steps"] == 1 and j["warmup"] == 1
    assert j["config"]["workload"] == "c1_blobs"
    cb = j["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == j["value"]
    assert j["e2e"]["value"] == j["value"] and j["e2e"]["h2d_bytes_per_step"] == 0


def test_issued_work_and_launch_counts():
    """Bookkeeping the bench line reports: launches per step for both paths."""
    sys.path.insert(0, ROOT)
    import bench

    # K2 (8) + K3 + K9 probe + K1 + K9 rescale (profiles/r02 launch lists: 11 before the
    # sliced column statistics split col_absmax/col_norm_range/column_mean into 5)
    assert bench.launches_per_step(581_012, 54, 4096) == 12
    # C4 panel path: 11 prep/probe launches + Z and projection GEMMs per <= 2 GB Z panel
    assert bench.launches_per_step(160_146, 2048, 16_384) == 11 + 2 * 5


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref is built where /root/reference exists")
def test_e2e_harness_reference_train_c1():
    """integration/e2e_run.py (bench.py's train_seconds) over the reference build at C1."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "integration", "e2e_run.py"), "ref", "train", "c1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    j = json.loads(out.stdout.strip().splitlines()[-1])
    assert j["b_eff"] == 1000 and j["unconverged_pairs"] == 0
    assert 0.14 < j["test_error"] < 0.18  # Bayes error of the C1 blobs is Φ(−1) ≈ 15.9 %
    assert j["train_seconds"] >= j["gmatrix_seconds"] + j["training_seconds"]


def test_e2e_harness_b200_build_links_the_adapter():
    so = os.path.join(ROOT, "integration", "_build", "libe2e_b200.so")
    if not os.path.exists(so):
        pytest.skip("integration build needs /root/reference at build time")
    syms = subprocess.run(["nm", "-D", so], capture_output=True, text=True).stdout
    assert "T e2e_train" in syms and "T e2e_compute_g" in syms
    assert "U lpd_compute_g_rows" in syms  # compute_G is the adapter's, over the C ABI
