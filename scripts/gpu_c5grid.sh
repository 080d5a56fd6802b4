for b in integration/_build oracle/_ref; do timeout 1500 python scripts/c5_grid.py $b gpurun_out/c5_grid_$(basename $(dirname $b)).json --n 200000 --budget 2048 2>&1 | tail -1; done
