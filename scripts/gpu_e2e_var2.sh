uptime
run() { echo "== $*"; env "$@" timeout 300 python scripts/e2e_probe.py c2 2>&1 | grep "compute wall" | sed 's/timings.*host_copy_seconds/host_copy/' | cut -c1-150; }
run LPD_SPIN_US=200
run LPD_SPIN_US=2000
run LPD_SPIN_US=20
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('bench e2e', round(j['e2e']['seconds_per_step'],3), 'basis', round(j['e2e']['basis_seconds_per_step'],4))"; done
