#!/bin/bash
# Round 2: downstream parity (alpha, w, D(alpha), test accuracy) at C1 and C2-shaped 200k,
# plus C1 through the reference API in both builds.
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
python tests/downstream.py c1 gpurun_out/downstream_c1.json > gpurun_out/downstream_c1.log 2>&1
python tests/downstream.py c2_200k gpurun_out/downstream_c2_200k.json > gpurun_out/downstream_c2.log 2>&1
python -m pytest tests/test_integration.py -m gpu -x -q -k c1 2>&1 | tail -5
