for fp in 0 1; do for w in c2 c3; do
  LPD_FORCE_PANEL=$fp timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('panel=$fp $w', round(j['value']), 'kernel_ms', round(j['roofline']['kernel_ms'],2), j['clocks']['sm_mhz'])"
done; done
for w in c2 c3; do LPD_FORCE_PANEL=1 timeout 600 python scripts/diag_fullsize.py $w 300 > gpurun_out/diag_${w}_panel.json 2>/dev/null; echo "$w panel"; head -8 gpurun_out/diag_${w}_panel.json | grep -E "max_err\"|median"; done
