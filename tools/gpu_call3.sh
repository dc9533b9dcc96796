set -x
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_fused.py tests/test_gpu_fused_backward.py tests/test_gpu_zero.py -m gpu > gpurun_out/pytest_c3.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_c3.log
MCO_ADALOMO_HOOK_OVERLAP=0 timeout 600 python tools/bench_configs.py hooks bf16 > gpurun_out/cfg_hooks_off.jsonl 2>&1
timeout 600 python tools/bench_configs.py hooks bf16 > gpurun_out/cfg_hooks_on.jsonl 2>&1
timeout 900 python bench.py --optimizers lomo,adalomo --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo bench_rc=$?
timeout 1500 bash profiles/run_ncu_r02.sh r02
ls -la gpurun_out
