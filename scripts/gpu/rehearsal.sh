# What the driver runs at round end, in order (one B200).
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --impl reference > gpurun_out/rehearsal_ref.json 2> gpurun_out/rehearsal_ref.err; echo "ref rc=$?"; cut -c1-200 gpurun_out/rehearsal_ref.json
timeout 900 python bench.py > gpurun_out/rehearsal.json 2> gpurun_out/rehearsal.err; echo "bench rc=$?"; python -c "import json; j=json.load(open('gpurun_out/rehearsal.json')); print(j['value'], j['e2e']['value'], j['roofline']['frac'], j['roofline']['issued_frac'], j['cpu_baseline']['value'], j['clocks'])"
