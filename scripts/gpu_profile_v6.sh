# v6 (segmented accumulation + ring delivery): bench lines C2/C3/C4, ncu captures, launch lists.
for w in c2 c3 c4; do
  timeout 1200 python bench.py --workload $w > gpurun_out/bench_${w}_v6.json 2> gpurun_out/bench_${w}_v6.err; echo "== $w rc=$?"; tail -1 gpurun_out/bench_${w}_v6.err; cut -c 1-300 gpurun_out/bench_${w}_v6.json
done
ncu --set full --clock-control none --import-source on -k regex:nystrom_factor -s 1 -c 1 -o gpurun_out/prof_k1v6_c2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k1v6.log 2>&1; tail -2 gpurun_out/ncu_k1v6.log
ncu --set full --clock-control none --import-source on -k regex:panel_gemm -s 10 -c 2 -o gpurun_out/prof_panel_v6_c4 python bench.py --workload c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_panel_v6.log 2>&1; tail -2 gpurun_out/ncu_panel_v6.log
ncu --kernel-name-base mangled -k regex:_ZN3lpd --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_v6.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ncu --kernel-name-base mangled -k regex:_ZN3lpd --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_v6.csv python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out | tail -12
