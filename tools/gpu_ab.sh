#!/bin/bash
# A/B of the stored-state kernel variants on one B200 (+ the variant parity tests).
# usage: bash tools/gpu_ab.sh "tma tma_ds" [extra bench args]
VARIANTS=${1:-"ldg tma"}
timeout 900 python -m pytest tests/test_gpu_flat.py -q -x -k variants > gpurun_out/pytest_variants.txt 2>&1; tail -2 gpurun_out/pytest_variants.txt
for rep in 1 2; do
for v in $VARIANTS; do
  MCO_FLAT_VARIANT=$v timeout 300 python bench.py --optimizers adamw,lion,adan,sophia --no-e2e --no-cpu-baseline --no-extra --steps 10 --warmup 3 --repeats 3 $2 > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.log
  python -c "
import json; d=json.load(open('gpurun_out/ab_$v.json'))
print('$v', {k:(v['ms'],v['frac_of_measured_hbm']) for k,v in d['per_optimizer'].items()}, d['clocks']['sm_mhz'])"
done
done
