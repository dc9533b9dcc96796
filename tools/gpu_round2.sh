# GPU call: the GPU test files from test_gpu_memory on, then the r02 ncu recipe
set -x
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_memory.py tests/test_gpu_overlap.py tests/test_gpu_randomized.py tests/test_gpu_shim.py tests/test_gpu_zero.py tests/test_gpu_zero_buckets.py tests/test_multigpu.py -m gpu > gpurun_out/pytest_gpu2.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu2.log
timeout 1500 bash profiles/run_ncu_r02.sh r02; echo ncu_rc=$?
ls -la gpurun_out
