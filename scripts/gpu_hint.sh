for rep in 1 2; do for v in "" _nohint; do for w in c2 c3; do
  LPD_LIBRARY=$PWD/paper_2207_01016_b200/liblpd_nystrom$v.so timeout 300 python bench.py --workload $w --steps 6 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('[$v] $w kernel_ms', round(j['roofline']['kernel_ms'],2), j['clocks']['sm_mhz'])"
done; done; done
ncu --set full --clock-control none -k regex:nystrom_factor -s 1 -c 1 -o gpurun_out/prof_k1_hint python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/prof_k1_hint.ncu-rep | grep -E "dram|duration|tensor_cycles|hit_rate|per_second"
