#!/bin/bash
# high-precision path: parity (golden fixtures, auto choice, C3 shard at γ = 2^-7) + perf probe
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "high_precision or precision_auto" -s > gpurun_out/hp_tests.log 2>&1; echo "tests rc=$?"; tail -12 gpurun_out/hp_tests.log
timeout 600 python scripts/hp_probe.py 131072 > gpurun_out/hp_probe.json 2> gpurun_out/hp_probe.err; echo "probe rc=$?"; cat gpurun_out/hp_probe.json; tail -3 gpurun_out/hp_probe.err
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -p no:cacheprovider -k "c3_ill" > gpurun_out/hp_full.log 2>&1; echo "full rc=$?"; tail -12 gpurun_out/hp_full.log
