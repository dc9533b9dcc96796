#!/bin/bash
# Round-2 profiling recipe (run under gpurun on ONE B200).  Outputs land in gpurun_out/;
# the summaries are copied into profiles/ and committed.
#   (1) the launch list of the bench command itself (every launch, device time + DRAM
#       bytes; cold-cache and serialised, so compare SHARES of the step);
#   (2) `ncu --set full` of every hot kernel family, each launched once or twice by
#       tools/profile_kernels.py (no repeats crowding out kernels, unlike round 1's -c 8).
# The full report (~90 MB) stays on the box (/tmp); its summaries (key metrics, raw CSV
# page, source hot spots of the AdaLomo passes) come back.
set -x
TAG=${1:-r02}
REP=/tmp/prof_${TAG}
[ "${SKIP_LAUNCHES:-0}" = 1 ] || ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --repeats 1 --no-e2e --no-cpu-baseline --no-extra \
    > gpurun_out/launches_bench_${TAG}.json
ncu --set full --clock-control none --import-source on \
    -k regex:"flat_tma_kernel|flat_step_kernel|sophia_m64|lomo_kernel|lomo_tma_kernel|sumsq_kernel|k1_stats|kr_stats|k2_scalars|k3_moments|k4_usq|k5_damp|k6_update|k_small_vec|peer_step_kernel" \
    -c 60 -o ${REP} -f python tools/profile_kernels.py ${ONLY:+--only $ONLY} > gpurun_out/prof_${TAG}.log 2>&1
echo ncu_rc=$?
python profiles/summarize_full_r02.py ${REP}.ncu-rep > gpurun_out/ncu_full_${TAG}.md
ncu -i ${REP}.ncu-rep --page raw --csv > gpurun_out/ncu_raw_${TAG}.csv
gzip -f gpurun_out/ncu_raw_${TAG}.csv

