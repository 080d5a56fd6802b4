for v in "" _old; do
  LPD_LIBRARY=$PWD/paper_2207_01016_b200/liblpd_nystrom$v.so timeout 600 python bench.py --no-cpu-baseline --e2e-steps 4 2>/dev/null | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('lib [$v]', 'kernel_ms', round(j['roofline']['kernel_ms'],2), 'issued_frac', round(j['roofline']['issued_frac'],3), 'clk', j['clocks']['sm_mhz'], 'e2e', j['e2e'])"
done
LPD_K1_SPLIT=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('split1 kernel_ms', round(j['roofline']['kernel_ms'],2))"
