#!/bin/bash
# Round 2 re-entry: full GPU suite + default bench line (validates the restored tree).
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt; nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cut -c1-600 gpurun_out/bench.json
