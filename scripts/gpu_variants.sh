# K1 compile variants (register reallocation / segment flushes) and e2e ring geometry.
for v in "" _noseg _nosegnoreg _noreg; do
  LPD_LIBRARY=$PWD/paper_2207_01016_b200/liblpd_nystrom$v.so timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('variant [$v]', 'kernel_ms', round(j['roofline']['kernel_ms'],2), 'issued_frac', round(j['roofline']['issued_frac'],3), 'clk', j['clocks']['sm_mhz'])"
done
for r in "8 6" "32 4" "128 3" "4 8"; do set -- $r; echo "ring $1 MB x $2"; LPD_RING_MB=$1 LPD_RING_SLOTS=$2 timeout 300 python scripts/e2e_probe.py c2 2>&1 | tail -2; done
