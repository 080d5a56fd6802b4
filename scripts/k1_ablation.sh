# Times the fused factor kernel (C2 shape) under profiling ablations (LPD_K1_DEBUG bits:
# needs the ablation build: nvcc ... -DLPD_K1_ABLATIONS=1 -o paper_2207_01016_b200/liblpd_nystrom_ablate.so (see Makefile target ablate)
# 1 = no exp/split math in the Z epilogue, 2 = no G stores, 4 = no GEMM2 MMAs, 8 = no GEMM1 MMAs).
for v in ${VARIANTS:-0 1 2 3 4 8 12}; do
  LPD_LIBRARY=$PWD/paper_2207_01016_b200/liblpd_nystrom_ablate.so LPD_K1_DEBUG=$v python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} 2>/dev/null | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('variant', $v, 'kernel_ms', round(j['roofline']['kernel_ms'],3), 'clk', j['clocks']['sm_mhz'])"
done
