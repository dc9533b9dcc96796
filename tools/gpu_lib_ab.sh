#!/bin/bash
# A/B two builds of libmco.so on one B200 (same box, interleaved runs).
# usage: bash tools/gpu_lib_ab.sh "tagA=/path/libmco.so tagB=/path/libmco.so" [bench args]
PAIRS=${1}
ARGS=${2:-"--optimizers adamw,lion,adan,sophia"}
for round in 1 2; do
  for pair in $PAIRS; do
    tag=${pair%%=*}; lib=${pair#*=}
    MCO_LIB_PATH=$lib timeout 300 python bench.py $ARGS --no-e2e --no-cpu-baseline --no-collectives --steps 10 --warmup 3 > gpurun_out/lab_$tag.json 2> gpurun_out/lab_$tag.log
    python -c "
import json; d=json.load(open('gpurun_out/lab_$tag.json'))
print('$tag', {k:(v['ms'],v['frac_of_measured_hbm']) for k,v in d['per_optimizer'].items()}, d['clocks']['sm_mhz'])"
  done
done
