# GPU call: AdaLomo A/B of the tree in gpurun_lib/old (built from an earlier commit) against
# this tree, per K6 traversal; then the whole GPU test suite (no -x: every failure listed).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
(cd gpurun_lib/old && timeout 600 python tools/bench_configs.py hooks bf16 > ../../gpurun_out/cfg_old.jsonl 2>&1)
for v in default tma tiles chunks; do
  MCO_ADALOMO_K6=$v timeout 600 python tools/bench_configs.py hooks bf16 cliff > gpurun_out/cfg_new_$v.jsonl 2>&1
done
(cd gpurun_lib/old && timeout 600 python tools/bench_configs.py hooks bf16 > ../../gpurun_out/cfg_old2.jsonl 2>&1)
timeout ${PYTEST_TIMEOUT:-2700} python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_gpu.log
