#!/bin/bash
# A/B of library builds on the hook-form (per-tensor) and multi-tensor AdaLomo / LOMO.
for round in 1 2; do
  for pair in $1; do
    tag=${pair%%=*}; lib=${pair#*=}
    echo "== $tag"; MCO_LIB_PATH=$lib timeout 600 python tools/bench_configs.py hooks | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print(' ', d['config'], d['ms'], d['frac'])"
  done
done
