# Panel path with segmented accumulation: parity suite, C4 error vs segment length, C4 bench.
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "large_d or golden or edge" 2>&1 | tail -3
for sg in 4 2 8; do
  LPD_SEG_CHUNKS=$sg timeout 900 python scripts/diag_fullsize.py c4 48 > gpurun_out/diag_c4_seg$sg.json 2> gpurun_out/diag_c4_seg$sg.err
  echo "seg $sg"; head -8 gpurun_out/diag_c4_seg$sg.json | grep err; tail -1 gpurun_out/diag_c4_seg$sg.err
done
for g in 8 16 32; do
  LPD_PANEL_GROUP=$g timeout 600 python bench.py --workload c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('group', $g, 'kernel_ms', round(j['roofline']['kernel_ms'],2), 'value', round(j['value']), 'clk', j['clocks'])"
done
