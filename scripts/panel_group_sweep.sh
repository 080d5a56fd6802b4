# C4 panel path: raster group size (row pairs per group) vs projection time, clocks and DRAM traffic.
for g in ${GROUPS_R:-2 4 8 16 32}; do
  LPD_PANEL_GROUP=$g timeout 600 python bench.py --workload c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('group', $g, 'kernel_ms', round(j['roofline']['kernel_ms'],2), 'value', round(j['value']), 'clk', j['clocks'])"
done
