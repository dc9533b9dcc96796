# GPU call: final check of the committed code -- the GPU suite, smoke, configs, list forms.
set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 1200 python tools/bench_configs.py > gpurun_out/configs.jsonl 2>&1; echo cfg_rc=$?
timeout 600 python tools/bench_list_kinds.py > gpurun_out/list_kinds.json 2>&1
timeout 600 python tools/bench_lomo_list.py > gpurun_out/lomo_list.jsonl 2>&1
