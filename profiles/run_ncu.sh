#!/bin/bash
# Profiling recipe (run under gpurun on ONE B200).  Outputs land in gpurun_out/;
# summaries are copied into profiles/ and committed.
set -x
TAG=${1:-r01}
# (1) every launch with its device time (cold-cache, serialised: compare SHARES)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --repeats 1 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench_${TAG}.json
# (2) the hot kernels once each, full set, on a 4-layer subset of the 7B shapes
ncu --set full --clock-control none --import-source on \
    -k regex:"flat_tma_kernel|flat_step_kernel|lomo_kernel|lomo_tma_kernel|k1_stats|k4_usq|k6_update" -c 8 \
    -o gpurun_out/prof_${TAG} -f \
    python bench.py --layers 4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null
