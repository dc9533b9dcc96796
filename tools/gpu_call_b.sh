# GPU call: AdaLomo after the K6 default change / per-tensor vector split: tests, configs,
# hook-form breakdown, ncu launch list of the hook form on the 4096^2 shape.
set -x
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_fused.py tests/test_gpu_zero_buckets.py tests/test_gpu_configs_parity.py -m gpu > gpurun_out/pytest_b.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_b.log
timeout 600 python tools/bench_configs.py hooks bf16 cliff > gpurun_out/cfg_b.jsonl 2>&1
timeout 600 python tools/hook_breakdown.py > gpurun_out/hook_breakdown.jsonl 2>&1
HB_R=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/hook_launches.csv python tools/hook_breakdown.py > /dev/null 2>&1
echo done
