#!/bin/bash
# LOMO host-span path keeping its resident gradient between calls: the host-path tests,
# the per-phase trace, then the default bench line (e2e is its headline).
mkdir -p gpurun_out
timeout 600 python -m pytest -x -q tests/test_gpu_fused.py -k "host" 2>&1 | tail -3
MCO_HOST_TRACE=1 timeout 300 python tools/e2e_trace.py 2>&1 | tail -12
timeout 900 python bench.py > gpurun_out/bench_hostcache.json 2> gpurun_out/bench_hostcache.log
echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_hostcache.json'))
print('value', d['value'], 'e2e', d['e2e']['value'], d['e2e']['roofline']['frac'])
print({k: v['ms'] for k, v in d['e2e']['per_optimizer'].items()})
print('clocks', d['clocks'])"
