# GPU call: AdaLomo packed-pair (FFMA2/FMUL2) K1/K4/K6, hoisted a_i loads: tests, configs, ncu.
set -x
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_gpu_fused.py tests/test_gpu_fused_backward.py tests/test_gpu_configs_parity.py tests/test_gpu_dp_processes.py tests/test_gpu_graph.py tests/test_gpu_randomized.py tests/test_gpu_fullsize.py -m gpu > gpurun_out/pytest_g.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_g.log
timeout 900 python tools/bench_configs.py hooks bf16 c3 > gpurun_out/cfg_g.jsonl 2>&1
ONLY=adalomo SKIP_LAUNCHES=1 timeout 1200 bash profiles/run_ncu_r02.sh r02g > /dev/null 2>&1
cat gpurun_out/ncu_full_r02g.md
