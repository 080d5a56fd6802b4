run() { echo "== $*"; env "$@" timeout 300 python scripts/e2e_probe.py c2 2>&1 | grep "compute wall" | awk '{print $5, $6}' | tr '\n' ' '; echo; }
for r in "8 6" "8 8" "16 4" "16 6" "12 6" "32 3" "8 6"; do set -- $r; run LPD_RING_MB=$1 LPD_RING_SLOTS=$2; done
