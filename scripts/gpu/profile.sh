#!/bin/bash
# Evidence run (tag = $1, default r02): bench lines C2/C3/C4, ncu --set full captures of K1 (C2)
# and the panel GEMMs (C4), launch lists of the timed command (C2, C4), SASS histogram.
T=${1:-r02}
mkdir -p gpurun_out
for w in c2 c3 c4; do
  timeout 900 python bench.py --workload $w --no-extras > gpurun_out/bench_${w}_$T.json 2> gpurun_out/bench_${w}_$T.err; echo "== $w rc=$?"
  python -c "import json; j=json.load(open('gpurun_out/bench_${w}_$T.json')); r=j['roofline']; print('$w', round(j['value']), round(r['kernel_ms'],2), round(r['achieved']), round(r['frac'],3), round(r['issued_frac'],3), 'e2e', round(j['e2e']['value']), round(j['e2e']['seconds_per_step'],3), 'cpu', round(j['cpu_baseline']['value'],1), j['clocks'])"
done
ncu --set full --clock-control none --import-source on -k regex:nystrom_factor -s 1 -c 1 -o gpurun_out/prof_k1_c2_$T python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extras > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:panel_gemm -s 10 -c 2 -o gpurun_out/prof_panel_c4_$T python bench.py --workload c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extras > /dev/null 2>&1
ncu --kernel-name-base mangled -k regex:_ZN3lpd --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_$T.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-extras > /dev/null 2>&1
ncu --kernel-name-base mangled -k regex:_ZN3lpd --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_$T.csv python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-extras > /dev/null 2>&1
ls gpurun_out | grep $T
