# GPU call: Adan over TMA configurations (MCO_TMA_CFG = flat_tma.cu MCO_TMA_CONFIGS id)
for rep in 1 2; do
for c in 1 10 11 12 13 4; do
  MCO_TMA_CFG=$c timeout 300 python bench.py --optimizers adan --no-e2e --no-cpu-baseline --no-extra --steps 10 --warmup 3 --repeats 2 > gpurun_out/c_$c.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/c_$c.json'))
print('cfg$c', {k:(v['ms'],v['frac_of_measured_hbm']) for k,v in d['per_optimizer'].items()}, d['clocks']['sm_mhz'])"
done
done
