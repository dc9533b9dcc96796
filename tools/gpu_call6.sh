set -x
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_fused.py tests/test_gpu_fused_backward.py tests/test_gpu_configs_parity.py tests/test_gpu_dp_processes.py tests/test_gpu_randomized.py tests/test_gpu_fullsize.py tests/test_gpu_graph.py tests/test_gpu_zero.py -m gpu > gpurun_out/pytest_c6.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_c6.log
for v in tma tiles chunks; do
  MCO_ADALOMO_K6=$v timeout 600 python tools/bench_configs.py hooks bf16 > gpurun_out/cfg_k6_$v.jsonl 2>&1
done
ONLY=adalomo SKIP_LAUNCHES=1 timeout 900 bash profiles/run_ncu_r02.sh r02c > /dev/null 2>&1
ls -la gpurun_out
