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
                          "--rows", "2048", "--steps", "1", "--warmup", "1"],
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

    assert bench.launches_per_step(581_012, 54, 4096) == 8          # K2 (6) + K3 + K1
    # C4 panel path: 7 prep launches + Z and projection GEMMs per <= 2 GB Z panel
    assert bench.launches_per_step(160_146, 2048, 16_384) == 7 + 2 * 5
