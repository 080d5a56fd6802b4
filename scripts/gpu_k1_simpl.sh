timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for w in c2 c3; do timeout 300 python bench.py --workload $w --steps 6 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$w kernel_ms', round(j['roofline']['kernel_ms'],2), round(j['roofline']['issued_frac'],3), j['clocks']['sm_mhz'])"; done
