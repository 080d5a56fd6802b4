"""SASS instruction histogram of every kernel in liblpd_nystrom.so (cuobjdump -sass): proves
which units each kernel drives (UTC*MMA = tcgen05.mma, UTMALDG/UTMASTG = TMA, LDTM/STTM =
TMEM loads/stores, DMMA = fp64 tensor core, HMMA = legacy mma.sync, MUFU = SFU).

  python scripts/sass_histogram.py [lib.so] > profiles/r02/sass_histogram.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2207_01016_b200", "liblpd_nystrom.so")
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
KEYS = ["UTCHMMA", "UTCQMMA", "UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "LDTM", "STTM", "UTCBAR", "DMMA", "HMMA",
        "MUFU", "DFMA", "DMUL", "DADD", "FFMA2", "FFMA", "SYNCS", "LDS", "STS", "LDG", "STG", "F2FP", "F2F"]
kern, counts, order = None, {}, []
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        order.append(kern)
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if kern and m:
        op = m.group(1)
        counts[kern]["total"] += 1
        for k in KEYS:
            if op == k or (k in ("UTCHMMA", "UTCQMMA") and op.startswith(k)):
                counts[kern][k] += 1
                break
print(f"# {os.path.relpath(lib, ROOT)}: {len(order)} kernels; static SASS instruction counts per kernel")
for k in order:
    c = counts[k]
    name = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
    tags = " ".join(f"{key}={c[key]}" for key in KEYS if c[key])
    print(f"{name[:100]}\n    total={c['total']} {tags}")
