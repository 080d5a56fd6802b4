# One bench line per workload (C2 default, C3 SUSY-shaped, C4 ImageNet-shaped) into gpurun_out/.
for w in ${WORKLOADS:-c2 c3 c4}; do
  timeout 900 python bench.py --workload $w ${BENCH_ARGS:-} > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  echo "== $w rc=$?"; tail -2 gpurun_out/bench_$w.err; cut -c1-400 gpurun_out/bench_$w.json
done
