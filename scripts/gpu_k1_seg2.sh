# K1: one N=256 MMA + synchronous segment flush (default) vs split halves; ring delivery e2e.
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for cfg in "0 4" "0 8" "0 64" "1 4"; do set -- $cfg; for w in c2 c3; do
  LPD_K1_SPLIT=$1 LPD_SEG_CHUNKS=$2 timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$w split $1 seg $2', 'kernel_ms', round(j['roofline']['kernel_ms'],2), 'value', round(j['value']), 'issued_frac', round(j['roofline']['issued_frac'],3), 'clk', j['clocks']['sm_mhz'])"
done; done
for w in c2 c3; do LPD_SEG_CHUNKS=4 timeout 900 python scripts/diag_fullsize.py $w 400 > gpurun_out/diag_${w}_s0seg4.json 2>/dev/null; echo "$w split0 seg4"; head -9 gpurun_out/diag_${w}_s0seg4.json | grep -E "max_err\"|median"; done
timeout 900 python bench.py > gpurun_out/bench_c2_ring.json 2> gpurun_out/bench_c2_ring.err; tail -2 gpurun_out/bench_c2_ring.err; cat gpurun_out/bench_c2_ring.json
