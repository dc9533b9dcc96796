#!/bin/bash
# GPU call: end-of-round check of the committed code -- smoke, the GPU suite, then the
# reference arm and the bench line back to back (the driver's order).
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log; echo ref_rc=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.log; echo bench_rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); r=json.load(open('gpurun_out/bench_ref.json'))
print('value', d['value'], 'e2e', d['e2e']['value'], 'ref', r['value'], 'clocks', d['clocks'])"
