# GPU call: cooperative K4 + K5 + K6 (k46_coop): AdaLomo tests, A/B against separate launches.
set -x
timeout 1200 python -m pytest -q -p no:cacheprovider -x tests/test_gpu_fused.py tests/test_gpu_fused_backward.py tests/test_gpu_configs_parity.py tests/test_gpu_randomized.py -m gpu > gpurun_out/pytest_aa.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_aa.log
for rep in 1 2; do
  for k in 1 0; do
    MCO_ADALOMO_K46=$k timeout 600 python tools/bench_configs.py hooks c3 bf16 2>&1 | grep config | grep -v "hook-form lomo" | sed "s/^/k46=$k /"
  done
done
