# GPU call: sumsq with four fp64 partials: A/B (C5 LOMO + clip lines, bench LOMO leg) + tests.
for rep in 1 2; do
  for v in base new; do
    if [ $v = base ]; then L=gpurun_lib/base/libmco.so; else L=paper_2312_00407_b200/_build/libmco.so; fi
    MCO_LIB_PATH=$L timeout 600 python tools/bench_configs.py c5 2>&1 | grep config | sed "s/^/$v /"
    MCO_LIB_PATH=$L timeout 600 python bench.py --optimizers lomo --no-e2e --no-cpu-baseline --no-extra --steps 10 --warmup 3 --repeats 2 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['per_optimizer']['lomo']; print('$v bench-lomo', e['ms'], e['frac_of_measured_hbm'])"
  done
done
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_gpu_fused.py tests/test_gpu_fused_backward.py tests/test_gpu_dp_processes.py tests/test_gpu_zero.py tests/test_gpu_flat_list.py -m gpu 2>&1 | tail -1
