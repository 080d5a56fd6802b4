# Full-size parity + K1/panel ncu captures + launch lists for the current kernels (one B200).
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q 2>&1 | tail -15
set -x
ncu --set full --clock-control none --import-source on -k regex:nystrom_factor -s 1 -c 1 -o gpurun_out/prof_k1v5_c2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k1v5.log 2>&1
tail -3 gpurun_out/ncu_k1v5.log
ncu --set full --clock-control none --import-source on -k regex:panel_gemm -s 10 -c 2 -o gpurun_out/prof_panel_v5_c4 python bench.py --workload c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_panel_v5.log 2>&1
tail -3 gpurun_out/ncu_panel_v5.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_v5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_v5.csv python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out
