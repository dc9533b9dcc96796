set -x
for rep in 1 2; do
python tools/bench_configs.py hooks > gpurun_out/k3_base_$rep.jsonl 2>&1
MCO_LIB_PATH=gpurun_lib/nok3/libmco.so python tools/bench_configs.py hooks > gpurun_out/k3_skip_$rep.jsonl 2>&1
done
MCO_HOST_TRACE=1 python tools/e2e_trace.py > gpurun_out/e2e_trace.log 2>&1
python tools/malloc_cost.py >> gpurun_out/e2e_trace.log 2>&1
