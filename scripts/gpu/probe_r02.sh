#!/bin/bash
# Round-2 probes: K1 ablations (upper bound of removing GEMM1 work), K5 prediction timing +
# launch list, host-path phase trace of set_basis / compute_g (LPD_TRACE), box topology.
mkdir -p gpurun_out
{ lscpu | grep -iE "numa|model name|^cpu\(s\)|socket"; nvidia-smi topo -m | head -4; free -g | head -2; } > gpurun_out/topology.txt 2>&1
VARIANTS="0 8 4 12" bash scripts/k1_ablation.sh > gpurun_out/k1_ablation.txt 2>&1; cat gpurun_out/k1_ablation.txt
timeout 600 python scripts/bench_k5.py > gpurun_out/k5.json 2> gpurun_out/k5.err; cat gpurun_out/k5.json; tail -2 gpurun_out/k5.err
ncu --clock-control none -k regex:"nystrom|prep|vote|row_shift" --metrics gpu__time_duration.sum --csv --log-file gpurun_out/k5_launches.csv python scripts/bench_k5.py --reps 1 > /dev/null 2>&1
python scripts/ncu_durations.py gpurun_out/k5_launches.csv
LPD_TRACE=1 timeout 600 python scripts/e2e_probe.py c2 > gpurun_out/e2e_trace.log 2>&1; grep -v "compute_g" gpurun_out/e2e_trace.log | tail -30
