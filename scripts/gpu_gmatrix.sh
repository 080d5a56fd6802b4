# gmatrix of the reference API's train through the integration build at C2 size (GPU build only).
timeout 900 python tests/integration_train.py integration/_build gpurun_out/e2e_gm.json --n 581012 --d 54 --budget 4096 --gamma 0.0185 --n-test 20000 --threads $(nproc) --tau 1e-12 --train-only --seed 1 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('gmatrix', j['gmatrix_seconds'], 'cold', j['cold']['gmatrix_seconds'], j['compute_G_phases'])"
timeout 600 python -m pytest tests/test_integration.py -q -x 2>&1 | tail -1
