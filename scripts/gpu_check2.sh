# Full GPU suite, smoke, default bench line.
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_c2_v7.json 2> gpurun_out/bench_c2_v7.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_c2_v7.err; cat gpurun_out/bench_c2_v7.json
