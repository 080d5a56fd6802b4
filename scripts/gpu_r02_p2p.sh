#!/bin/bash
# peer-copy basis broadcast (two-shard context on one GPU), multi-process library shards,
# drop-in with the balanced first touch (+ phase trace), then the default bench line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_distributed.py tests/test_integration.py -q -m gpu -p no:cacheprovider > gpurun_out/p2p_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/p2p_tests.log
for pf in 4 8; do
  LPD_TRACE=1 LPD_PREFAULT=$pf timeout 600 python scripts/dropin_probe.py 581012 3 > gpurun_out/dropin2_pf$pf.log 2>&1; echo "prefault=$pf rc=$?"; head -1 gpurun_out/dropin2_pf$pf.log | cut -c1-900; grep "set_basis" gpurun_out/dropin2_pf$pf.log | tail -8
done
timeout 1200 python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench rc=$?"; python -c "
import json; j=json.load(open('gpurun_out/bench2.json'))
print(j['value'], j['e2e']['value'], j['roofline']['frac'], j['e2e_dropin'].get('seconds_per_step'), j['e2e_dropin'].get('phases'), j['clocks'])"
