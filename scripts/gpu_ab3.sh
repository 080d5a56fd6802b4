timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
for rep in 1 2; do for v in "" _prev; do for w in c2 c3; do
  LPD_LIBRARY=$PWD/paper_2207_01016_b200/liblpd_nystrom$v.so timeout 300 python bench.py --workload $w --steps 6 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('[$v] $w kernel_ms', round(j['roofline']['kernel_ms'],2), round(j['roofline']['issued_frac'],3), j['clocks']['sm_mhz'])"
done; done; done
