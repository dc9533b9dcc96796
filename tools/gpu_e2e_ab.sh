#!/bin/bash
# A/B of the host-span (e2e) pipeline between library builds, interleaved.
# usage: bash tools/gpu_e2e_ab.sh "tagA=/path/libmco.so tagB=/path/libmco.so"
for round in 1 2; do
  for pair in $1; do
    tag=${pair%%=*}; lib=${pair#*=}
    MCO_LIB_PATH=$lib timeout 600 python bench.py --optimizers adamw,lomo,adalomo --no-cpu-baseline --steps 3 --warmup 3 --e2e-steps 2 > gpurun_out/e2e_$tag.json 2> gpurun_out/e2e_$tag.log
    python -c "
import json; d=json.load(open('gpurun_out/e2e_$tag.json'))
print('$tag', {k:v['ms'] for k,v in d['e2e']['per_optimizer'].items()}, d['e2e']['roofline']['frac'], d['e2e']['roofline']['peak'])"
  done
done
