# GPU call: shifted-gradient TMA read path (flat + LOMO): tests and speed.
set -x
timeout 1500 python -m pytest -q -p no:cacheprovider tests/test_gpu_flat.py tests/test_gpu_fused.py tests/test_gpu_randomized.py tests/test_gpu_flat_list.py tests/test_gpu_graph.py tests/test_gpu_zero.py tests/test_gpu_overlap.py -m gpu > gpurun_out/pytest_j.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_j.log
timeout 600 python tools/bench_configs.py phases > gpurun_out/phases_j.jsonl 2>&1
cat gpurun_out/phases_j.jsonl
