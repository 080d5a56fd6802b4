for v in _old "" _old ""; do
  LPD_LIBRARY=$PWD/paper_2207_01016_b200/liblpd_nystrom$v.so timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('lib [$v]', 'kernel_ms', round(j['roofline']['kernel_ms'],2), 'issued_frac', round(j['roofline']['issued_frac'],3), 'clk', j['clocks']['sm_mhz'], 'e2e_s', round(j['e2e']['seconds_per_step'],3))"
done
timeout 300 python scripts/e2e_probe.py c2 2>&1 | tail -2
