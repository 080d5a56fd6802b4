run() { echo "== $*"; env "$@" timeout 300 python scripts/e2e_probe.py c2 2>&1 | grep "compute wall" | awk '{print $5, $6}' | tr '\n' ' '; echo; }
run LPD_RING_MB=8 LPD_RING_SLOTS=6
run LPD_RING_MB=8 LPD_RING_SLOTS=4
run LPD_RING_MB=8 LPD_RING_SLOTS=3
run LPD_RING_MB=4 LPD_RING_SLOTS=6
run LPD_RING_MB=16 LPD_RING_SLOTS=4
run LPD_RING_MB=8 LPD_RING_SLOTS=6 LPD_WIDEN_THREADS=12
run LPD_RING_MB=8 LPD_RING_SLOTS=6 LPD_WIDEN_THREADS=8
run LPD_RING_MB=8 LPD_RING_SLOTS=6
