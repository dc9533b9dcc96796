# GPU call: AdaLomo one-launch small-vector hook path + per-tensor KR blocks: tests, A/B.
set -x
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_gpu_fused.py tests/test_gpu_fused_backward.py tests/test_gpu_configs_parity.py tests/test_gpu_dp_processes.py tests/test_gpu_graph.py tests/test_gpu_randomized.py tests/test_gpu_fullsize.py tests/test_gpu_zero.py -m gpu > gpurun_out/pytest_d.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_d.log
for sm in 1 0; do
  MCO_ADALOMO_SMALL=$sm timeout 600 python tools/hook_breakdown.py > gpurun_out/hb_small$sm.jsonl 2>&1
  MCO_ADALOMO_SMALL=$sm timeout 900 python tools/bench_configs.py hooks bf16 > gpurun_out/cfg_small$sm.jsonl 2>&1
done
HB_R=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/hook_launches_d.csv python tools/hook_breakdown.py > /dev/null 2>&1
echo done
