# GPU call: Adan stage count (default now 3; tma_s5 = 5, tma = 4 for Adan via tma_hint-free
# cfg... compare tma (Adan 3 stages), tma_s2, tma_s5) on fp32, bf16-grad and mixed Adan.
set -x
for rep in 1 2; do
for v in tma tma_s2 tma_s5; do
  MCO_FLAT_VARIANT=$v timeout 300 python bench.py --optimizers adan --no-e2e --no-cpu-baseline --no-extra --steps 10 --warmup 3 --repeats 2 > gpurun_out/v_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/v_$v.json'))
print('$v', {k:(v['ms'],v['frac_of_measured_hbm']) for k,v in d['per_optimizer'].items()}, d['clocks']['sm_mhz'])"
  MCO_FLAT_VARIANT=$v timeout 300 python tools/bench_configs.py c4 2>&1 | grep adan | sed "s/^/$v /" | cut -c1-140
done
done
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_flat.py tests/test_gpu_graph.py tests/test_gpu_randomized.py -m gpu > gpurun_out/pytest_t.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_t.log
