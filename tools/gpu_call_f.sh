set -x
for sm in 1 0; do MCO_ADALOMO_SMALL=$sm python tools/small_vec_prof.py; done
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_fused.py tests/test_gpu_fused_backward.py tests/test_gpu_graph.py tests/test_gpu_randomized.py -m gpu > gpurun_out/pytest_f.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_f.log
timeout 600 python tools/bench_configs.py hooks > gpurun_out/cfg_f.jsonl 2>&1
cat gpurun_out/cfg_f.jsonl
