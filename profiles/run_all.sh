#!/bin/bash
# Round-end evidence run (ONE B200, under gpurun).  Everything lands in gpurun_out/.
TAG=${1:-r01}
set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; tail -3 gpurun_out/pytest_gpu_${TAG}.txt
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; tail -2 gpurun_out/smoke_${TAG}.txt
# clocks during the bench, sampled by nvidia-smi independently of bench.py's own sampler
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/clocks_${TAG}.csv &
SMI=$!
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.log
kill $SMI
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.log
timeout 900 python tools/bench_configs.py > gpurun_out/configs_${TAG}.jsonl 2> gpurun_out/configs_${TAG}.log
timeout 900 bash profiles/run_ncu.sh ${TAG} > gpurun_out/ncu_${TAG}.log 2>&1
ls -la gpurun_out/
