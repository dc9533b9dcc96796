#!/bin/bash
# A/B of libmco.so builds on AdaLomo forms (same box, interleaved): hook / list /
# multi-tensor / bf16 (tools/bench_configs.py hooks bf16) and the hook-form breakdown.
# usage: bash tools/gpu_ada_lib_ab.sh "tagA=/path/libmco.so tagB=..."
mkdir -p gpurun_out
for round in 1 2; do
  for pair in $1; do
    tag=${pair%%=*}; lib=${pair#*=}
    echo "== $tag round $round"
    MCO_LIB_PATH=$lib timeout 300 python tools/bench_configs.py hooks bf16 2>&1 | \
      python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print('  ', d['config'][:60], d['ms'], d.get('frac'))"
    MCO_LIB_PATH=$lib timeout 300 python tools/hook_parts.py 2>&1 | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print('   parts', round(d['all_ms'], 3), {k: v['us_per_call'] for k, v in d.items() if isinstance(v, dict) and 'us_per_call' in v})"
  done
done
