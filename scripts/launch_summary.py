"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel
launches, total ms and share of this library's device time (cold-cache, serialised
ncu replays: compare shares, not absolute times)."""
import csv
import subprocess
import sys
from collections import defaultdict

OURS = ("nystrom_factor_kernel", "panel_gemm_kernel", "prep_rows_kernel", "column_sum_partial_kernel",
        "column_mean_finalize_kernel", "col_stats_kernel", "col_norm_finalize_kernel", "landmark_stats_kernel",
        "basis_consts_kernel", "prep_landmarks_kernel", "lt_split_kernel", "row_shift_kernel",
        "row_rescale_kernel", "csr_to_dense_kernel", "ovo_vote_kernel", "gram_", "gather_g", "decision_", "hp_",
        "pointdv_", "lpd::")
UNIT_MS = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def demangle(names):
    """c++filt over mangled names (launch lists taken with --kernel-name-base mangled)."""
    mangled = sorted({n for n in names if n.startswith("_Z")})
    if not mangled:
        return {}
    out = subprocess.run(["c++filt"], input="\n".join(mangled), capture_output=True, text=True).stdout.splitlines()
    return dict(zip(mangled, out))


def main(path, title):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    all_ms = 0.0
    dm = demangle(r["Kernel Name"] for r in rows)
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        ms = float(r["Metric Value"].replace(",", "")) * UNIT_MS[r["Metric Unit"]]
        all_ms += ms
        name = dm.get(r["Kernel Name"], r["Kernel Name"]).split("(")[0].strip()
        if any(k in name for k in OURS):
            tot[name] += ms
            cnt[name] += 1
    lib = sum(tot.values())
    print(f"# {title}")
    print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare shares)")
    print(f"# all launches {all_ms:.1f} ms, this library's kernels {lib:.1f} ms")
    for name in sorted(tot, key=lambda k: -tot[k]):
        print(f"{name[:60]:60s} launches {cnt[name]:5d} total_ms {tot[name]:10.3f} share_of_library {100 * tot[name] / lib:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
