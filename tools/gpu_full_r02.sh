# GPU call: the round-2 evidence set on the current code -- smoke, the GPU test suite,
# bench.py (both arms), configs 3-5 + hook / bf16 / cliff lines, the ncu recipe.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
timeout 1200 python tools/bench_configs.py > gpurun_out/configs.jsonl 2>&1; echo cfg_rc=$?
timeout 600 python tools/hook_breakdown.py > gpurun_out/hook_breakdown.jsonl 2>&1
timeout 1800 bash profiles/run_ncu_r02.sh r02 > gpurun_out/ncu_recipe.log 2>&1; echo ncu_rc=$?
ls -la gpurun_out
