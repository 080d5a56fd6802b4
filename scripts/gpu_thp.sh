run() { echo "== $*"; env "$@" timeout 300 python scripts/e2e_probe.py c2 2>&1 | grep -E "compute wall|Error|error" | awk '{print $5, $6, $7}' | tr '\n' ' '; echo; }
run E2E_THP=0
run E2E_THP=1
run E2E_THP=0
run E2E_THP=1
