run() { echo "== $*"; env "$@" timeout 300 python scripts/e2e_probe.py c2 2>&1 | grep "compute wall" | awk '{print $5, $6, $12, $13, $14}' | tr '\n' ' '; echo; }
run LPD_RING_MB=8
run LPD_RING_MB=8 LPD_SPIN_LIMIT=2000000
run LPD_RING_MB=16 LPD_RING_SLOTS=6
run LPD_RING_MB=8 LPD_RING_SLOTS=12
run LPD_RING_MB=8 LPD_WIDEN_THREADS=12
run LPD_RING_MB=4 LPD_RING_SLOTS=12 LPD_SPIN_LIMIT=2000000
run LPD_RING_MB=8
