# End-to-end training through the reference's own Python API (lpdsvm.train + predict):
# the integration build (compute_G / Gram / predict on the B200) vs the unmodified
# reference build on all host cores, same data. One JSON line per build and size.
T=$(nproc)
run() {  # n d budget gamma
  for b in integration/_build oracle/_ref; do
    timeout 1800 python tests/integration_train.py $b gpurun_out/e2e_${1}_$(basename $(dirname $b)).json \
      --n $1 --d $2 --budget $3 --gamma $4 --n-test 20000 --threads $T --tau 1e-12 --train-only --seed 1 \
      2>&1 | tail -1
  done
}
run ${N1:-20000} 50 1000 0.02
run ${N2:-200000} 54 2048 0.0185
run ${N3:-581012} 54 4096 0.0185
