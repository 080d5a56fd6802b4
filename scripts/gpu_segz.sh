for sz in 2 8 33; do
  LPD_SEG_Z=$sz timeout 600 python scripts/diag_fullsize.py c4 48 > gpurun_out/diag_c4_segz$sz.json 2>/dev/null; echo "segz $sz"; head -8 gpurun_out/diag_c4_segz$sz.json | grep -E "max_err\"|median"
  LPD_SEG_Z=$sz timeout 600 python bench.py --workload c4 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('segz $sz kernel_ms', round(j['roofline']['kernel_ms'],1), j['clocks']['sm_mhz'])"
done
