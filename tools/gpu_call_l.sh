# GPU call: list-form TMA kernel with shifted streams: tests, speed, sanitizers.
set -x
timeout 1500 python -m pytest -q -p no:cacheprovider tests/test_gpu_flat_list.py tests/test_gpu_graph.py tests/test_gpu_flat.py tests/test_gpu_overlap.py tests/test_gpu_fused.py -m gpu > gpurun_out/pytest_l.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_l.log
MCO_LIST_CASES=300 timeout 1500 python -m pytest -q -p no:cacheprovider tests/test_gpu_flat_list.py -m gpu -k random > gpurun_out/pytest_l_wide.log 2>&1; echo wide_rc=$?
tail -2 gpurun_out/pytest_l_wide.log
timeout 600 python tools/bench_configs.py phases > gpurun_out/phases_l.jsonl 2>&1
cat gpurun_out/phases_l.jsonl | cut -c1-140
for tool in memcheck racecheck synccheck; do
timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_flat_list.py -q -x -k "not random" 2>&1 | grep -E "passed|failed|SUMMARY|rror|azard" | head -5
done
