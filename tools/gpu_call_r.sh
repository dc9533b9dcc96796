# GPU call: Sophia precise-m on the bulk-copy pipeline: tests and an A/B against the LDG kernel.
set -x
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_flat.py -m gpu -k "precise_m or sophia_m64" > gpurun_out/pytest_r.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_r.log
for rep in 1 2; do
  for v in tma ldg; do
    MCO_SOPHIA_M64=$v timeout 600 python bench.py --optimizers sophia --no-e2e --no-cpu-baseline --steps 10 --warmup 3 --repeats 1 > gpurun_out/m64_$v.json 2>gpurun_out/m64_$v.err
    python -c "
import json; d=json.load(open('gpurun_out/m64_$v.json')); e=d['extra_not_in_value']['sophia_precise_m']; print('$v', e['ms'], e['frac_of_measured_hbm'], d['clocks']['sm_mhz'])"
  done
done
timeout 900 compute-sanitizer --tool memcheck python -m pytest -q -p no:cacheprovider tests/test_gpu_flat.py -m gpu -k "precise_m" 2>&1 | grep -E "passed|failed|SUMMARY" | head -3
timeout 900 compute-sanitizer --tool racecheck python -m pytest -q -p no:cacheprovider tests/test_gpu_flat.py -m gpu -k "precise_m and 10317" 2>&1 | grep -E "passed|failed|SUMMARY" | head -3
