for sy in 0 256 32 8; do
  LPD_PANEL_SYNC=$sy timeout 600 python bench.py --workload c4 --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_c4_sync$sy.json 2>/dev/null; python -c "import json; j=json.load(open('gpurun_out/bench_c4_sync$sy.json')); print('sync $sy', round(j['value']), round(j['roofline']['kernel_ms'],1), round(j['roofline']['issued_frac'],3), 'e2e', round(j['e2e']['seconds_per_step'],3), 'basis', round(j['e2e']['basis_seconds_per_step'],3), j['clocks']['sm_mhz'])"
done
LPD_PANEL_SYNC=32 ncu --set full --clock-control none -k regex:panel_gemm -s 10 -c 2 -o gpurun_out/prof_panel_sync32 python bench.py --workload c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/prof_panel_sync32.ncu-rep | grep -E "##|dram__bytes_read|duration|tensor_cycles|hit_rate|per_second"
