#!/bin/bash
# Design studies recorded in DESIGN.md, one function each: `bash scripts/gpu/studies.sh <name>`.
#   force_panel  fused K1 vs the two-GEMM panel path on C2/C3 (LPD_FORCE_PANEL)
#   panel_sync   projection GEMM K-progress rendezvous period (LPD_PANEL_SYNC)
#   e2e_matrix   delivery-ring geometries (LPD_RING_MB / LPD_RING_SLOTS / LPD_WIDEN_THREADS)
#   segz         panel Z GEMM segment length vs row error (LPD_SEG_Z)
mkdir -p gpurun_out
force_panel() {
for fp in 0 1; do for w in c2 c3; do
  LPD_FORCE_PANEL=$fp timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('panel=$fp $w', round(j['value']), 'kernel_ms', round(j['roofline']['kernel_ms'],2), j['clocks']['sm_mhz'])"
done; done
for w in c2 c3; do LPD_FORCE_PANEL=1 timeout 600 python scripts/diag_fullsize.py $w 300 > gpurun_out/diag_${w}_panel.json 2>/dev/null; echo "$w panel"; head -8 gpurun_out/diag_${w}_panel.json | grep -E "max_err\"|median"; done
}
panel_sync() {
for sy in 0 256 32 8; do
  LPD_PANEL_SYNC=$sy timeout 600 python bench.py --workload c4 --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_c4_sync$sy.json 2>/dev/null; python -c "import json; j=json.load(open('gpurun_out/bench_c4_sync$sy.json')); print('sync $sy', round(j['value']), round(j['roofline']['kernel_ms'],1), round(j['roofline']['issued_frac'],3), 'e2e', round(j['e2e']['seconds_per_step'],3), 'basis', round(j['e2e']['basis_seconds_per_step'],3), j['clocks']['sm_mhz'])"
done
LPD_PANEL_SYNC=32 ncu --set full --clock-control none -k regex:panel_gemm -s 10 -c 2 -o gpurun_out/prof_panel_sync32 python bench.py --workload c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/prof_panel_sync32.ncu-rep | grep -E "##|dram__bytes_read|duration|tensor_cycles|hit_rate|per_second"
}
e2e_matrix() {
run() { echo "== $*"; env "$@" timeout 300 python scripts/e2e_probe.py c2 2>&1 | grep "compute wall" | awk '{print $5, $6, $12, $13, $14}' | tr '\n' ' '; echo; }
run LPD_RING_MB=8
run LPD_RING_MB=8 LPD_SPIN_LIMIT=2000000
run LPD_RING_MB=16 LPD_RING_SLOTS=6
run LPD_RING_MB=8 LPD_RING_SLOTS=12
run LPD_RING_MB=8 LPD_WIDEN_THREADS=12
run LPD_RING_MB=4 LPD_RING_SLOTS=12 LPD_SPIN_LIMIT=2000000
run LPD_RING_MB=8
}
segz() {
for sz in 2 8 33; do
  LPD_SEG_Z=$sz timeout 600 python scripts/diag_fullsize.py c4 48 > gpurun_out/diag_c4_segz$sz.json 2>/dev/null; echo "segz $sz"; head -8 gpurun_out/diag_c4_segz$sz.json | grep -E "max_err\"|median"
  LPD_SEG_Z=$sz timeout 600 python bench.py --workload c4 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('segz $sz kernel_ms', round(j['roofline']['kernel_ms'],1), j['clocks']['sm_mhz'])"
done
}
"${1:?study name}"
