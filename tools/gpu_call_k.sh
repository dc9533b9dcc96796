# GPU call: A/B of the AdaLomo tile loops with 32-bit row indices (this tree) against the
# previous commit's library (gpurun_lib/base), interleaved.
set -x
for rep in 1 2; do
  MCO_LIB_PATH=gpurun_lib/base/libmco.so timeout 600 python tools/bench_configs.py bf16 hooks c3 > gpurun_out/abk_base_$rep.jsonl 2>&1
  timeout 600 python tools/bench_configs.py bf16 hooks c3 > gpurun_out/abk_new_$rep.jsonl 2>&1
done
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_fused.py tests/test_gpu_configs_parity.py -m gpu > gpurun_out/pytest_k.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_k.log
