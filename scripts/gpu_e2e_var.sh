cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag; nproc; uptime; free -g | head -2
run() { echo "== $*"; env "$@" timeout 300 python scripts/e2e_probe.py c2 2>&1 | grep "compute wall" | sed 's/timings.*host_copy_seconds/host_copy/' | cut -c1-200; }
run LPD_RING_MB=8
run LPD_SPIN_LIMIT=100000000
run LPD_WIDEN_THREADS=8
run LPD_RING_MB=8
