for v in "" _noseg _nosegnoreg; do
  LPD_SEG_CHUNKS=64 LPD_LIBRARY=$PWD/paper_2207_01016_b200/liblpd_nystrom$v.so timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('variant [$v] seg64', 'kernel_ms', round(j['roofline']['kernel_ms'],2), 'issued_frac', round(j['roofline']['issued_frac'],3), 'clk', j['clocks']['sm_mhz'])"
done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c2_ring2.json 2> gpurun_out/bench_c2_ring2.err; tail -2 gpurun_out/bench_c2_ring2.err; cut -c 1-200 gpurun_out/bench_c2_ring2.json; python -c "import json; j=json.load(open('gpurun_out/bench_c2_ring2.json')); print(j['e2e'], j['roofline']['kernel_ms'])"
