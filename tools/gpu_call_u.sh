# GPU call: stage count A/B for Lion / Sophia / LOMO (tma = default, tma_s3, tma_s5)
for rep in 1 2; do
for v in tma tma_s3 tma_s5; do
  MCO_FLAT_VARIANT=$v timeout 300 python bench.py --optimizers lion,sophia,lomo --no-e2e --no-cpu-baseline --no-extra --steps 10 --warmup 3 --repeats 2 > gpurun_out/v_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/v_$v.json'))
print('$v', {k:(v['ms'],v['frac_of_measured_hbm']) for k,v in d['per_optimizer'].items()}, d['clocks']['sm_mhz'])"
done
done
