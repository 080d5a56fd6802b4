run() { echo "== $*"; env "$@" timeout 300 python scripts/e2e_probe.py c2 2>&1 | grep "compute wall" | awk '{print $5, $6}' | tr '\n' ' '; echo; }
run LPD_D2H_STREAMS=1
run LPD_D2H_STREAMS=2
run LPD_D2H_STREAMS=2 LPD_RING_SLOTS=8
run LPD_D2H_STREAMS=1
run LPD_D2H_STREAMS=2
LPD_D2H_STREAMS=2 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "multi_chunk or two_shard or golden" 2>&1 | tail -1
