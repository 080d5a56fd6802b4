# K1 Z·β mode (b_eff <= 16): parity subset, K5 bench with and without it (LPD_ZBETA=0),
# launch lists of both, one ncu --set full capture of the Z·β kernel (binary model).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "narrow or predict or edge or fuzz or golden or pitches or vote or device_entry or batch" 2>&1 | grep -E "Error|assert|passed|failed" | head -30
timeout 300 python scripts/bench_k5.py --n-test 1000000 > gpurun_out/k5_zb.json 2> gpurun_out/k5_zb.err; echo "zb rc=$?"; cat gpurun_out/k5_zb.json
LPD_ZBETA=0 timeout 300 python scripts/bench_k5.py --n-test 1000000 > gpurun_out/k5_nozb.json 2> gpurun_out/k5_nozb.err; echo "nozb rc=$?"; cat gpurun_out/k5_nozb.json
ncu --kernel-name-base mangled -k regex:_ZN3lpd --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k5_zb_launches.csv python scripts/bench_k5.py --n-test 1000000 --reps 1 > /dev/null 2>&1
LPD_ZBETA=0 ncu --kernel-name-base mangled -k regex:_ZN3lpd --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k5_nozb_launches.csv python scripts/bench_k5.py --n-test 1000000 --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:nystrom_factor -s 0 -c 1 -o gpurun_out/prof_k5_zb_p1 python scripts/bench_k5.py --n-test 1000000 --reps 0 > /dev/null 2>&1
ls gpurun_out | grep k5
