# Smoke, then e2e (C2, C ABI into pageable fp64 G) with 8 / 12 / 16 host widen threads, twice each,
# alternating, on one box (the host side is what differs between boxes).
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for rep in 1 2; do
  for w in 8 12 16; do
    LPD_WIDEN_THREADS=$w timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/widen_${w}_${rep}.json 2>/dev/null
    python -c "import json; j=json.load(open('gpurun_out/widen_${w}_${rep}.json')); e=j['e2e']; print('widen', $w, 'rep', $rep, round(e['value']), round(e['seconds_per_step'],3), {k: round(v,3) for k,v in e['phases'].items()})"
  done
done
