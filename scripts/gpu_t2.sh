timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "two_shard or multi_chunk or resident" 2>&1 | tail -15
