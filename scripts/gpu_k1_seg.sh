# K1 with segmented G accumulation: parity suite, C2/C3 error vs segment length, C2/C3 bench.
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for sg in 4 2; do for w in c2 c3; do
  LPD_SEG_CHUNKS=$sg timeout 900 python scripts/diag_fullsize.py $w 400 > gpurun_out/diag_${w}_seg$sg.json 2> gpurun_out/diag_${w}_seg$sg.err
  echo "$w seg $sg"; head -9 gpurun_out/diag_${w}_seg$sg.json | grep err; tail -1 gpurun_out/diag_${w}_seg$sg.err
done; done
for sg in 2 4 8 64; do for w in c2 c3; do
  LPD_SEG_CHUNKS=$sg timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$w seg', $sg, 'kernel_ms', round(j['roofline']['kernel_ms'],2), 'value', round(j['value']), 'issued_frac', round(j['roofline']['issued_frac'],3), 'clk', j['clocks']['sm_mhz'])"
done; done
