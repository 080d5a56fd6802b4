for rep in 1 2; do for v in "" _lt8 _lt7 _stg1; do
  LPD_LIBRARY=$PWD/paper_2207_01016_b200/liblpd_nystrom$v.so timeout 300 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('[$v] c2 kernel_ms', round(j['roofline']['kernel_ms'],2), 'issued', round(j['roofline']['issued_frac'],3), j['clocks']['sm_mhz'])"
done; done
