"""Per-kernel launch durations from an `ncu --csv --metrics gpu__time_duration.sum` log:
  python scripts/ncu_durations.py launches.csv   -> name, count, mean/min/max (us)"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
acc = defaultdict(list)
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6}
for r in rows[1:]:
    try:
        acc[r[ki]].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
    except ValueError:
        pass
for k, v in acc.items():
    print(f"{len(v):5d}  mean {sum(v) / len(v):10.1f} us  min {min(v):10.1f}  max {max(v):10.1f}  {k[:110]}")
