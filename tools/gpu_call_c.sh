# GPU call: AdaLomo tile plan A/B (whole-wave tiles vs round-1 power-of-2 heights) and the
# unrolled tile-partial reductions; AdaLomo GPU tests.
set -x
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_fused.py tests/test_gpu_fused_backward.py tests/test_gpu_configs_parity.py tests/test_gpu_dp_processes.py -m gpu > gpurun_out/pytest_c.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_c.log
for t in waves pow2; do
  MCO_ADALOMO_TILES=$t timeout 600 python tools/hook_breakdown.py > gpurun_out/hb_$t.jsonl 2>&1
  MCO_ADALOMO_TILES=$t timeout 900 python tools/bench_configs.py hooks bf16 c3 > gpurun_out/cfg_$t.jsonl 2>&1
done
MCO_ADALOMO_TILES=waves timeout 600 python tools/hook_breakdown.py > gpurun_out/hb_waves2.jsonl 2>&1
HB_R=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/hook_launches_c.csv python tools/hook_breakdown.py > /dev/null 2>&1
echo done
