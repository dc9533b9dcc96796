# GPU call: AdaLomo strided scalar-path tile layout: tests + cliff bench.
set -x
timeout 1500 python -m pytest -q -p no:cacheprovider tests/test_gpu_fused.py tests/test_gpu_fused_backward.py tests/test_gpu_configs_parity.py tests/test_gpu_dp_processes.py tests/test_gpu_zero.py tests/test_gpu_graph.py -m gpu > gpurun_out/pytest_o.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_o.log
MCO_RANDOM_ADA_CASES=60 timeout 1500 python -m pytest -q -p no:cacheprovider tests/test_gpu_randomized.py -m gpu -k ada > gpurun_out/pytest_o_ada.log 2>&1; echo ada_rc=$?
tail -2 gpurun_out/pytest_o_ada.log
timeout 600 python tools/bench_configs.py cliff bf16 > gpurun_out/cfg_o.jsonl 2>&1
cat gpurun_out/cfg_o.jsonl | cut -c1-150
