timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "resident" 2>&1 | tail -2
timeout 900 python scripts/bench_c5.py > gpurun_out/c5_resident_v7.json 2> gpurun_out/c5.err; tail -2 gpurun_out/c5.err; cat gpurun_out/c5_resident_v7.json
ncu --kernel-name-base mangled -k regex:_ZN3lpd.*gather --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/launches_c5_v7.csv python scripts/bench_c5.py --reps 2 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[l for l in open('gpurun_out/launches_c5_v7.csv')]
start=[i for i,l in enumerate(rows) if l.startswith('"ID"')][0]
from collections import defaultdict
d=defaultdict(list)
for r in csv.DictReader(rows[start:]):
    d[(r['Kernel Name'][:60], r['Metric Name'])].append(float(r['Metric Value'].replace(',','')))
for k,v in sorted(d.items()): print(k, len(v), 'median', sorted(v)[len(v)//2], v[0] if v else None)
PY
