# GPU call: AdaLomo tile-wave A/B (MCO_ADALOMO_WAVE = tile-kernel CTAs per SM of a wave)
# and the LOMO e2e leg after freeing the device-timed buffers.
for rep in 1 2; do
  for w in 3 2 4 6; do
    MCO_ADALOMO_WAVE=$w python tools/bench_configs.py hooks c3 bf16 2>&1 | grep config | grep -v "hook-form lomo" | sed "s/^/w$w /"
  done
done
timeout 600 python bench.py --optimizers lomo,adalomo --no-cpu-baseline --no-extra --steps 3 --warmup 1 --repeats 1 2>&1 | grep "e2e\]"
