# GPU call: same-box A/B of the flat / LOMO TMA kernels before the shifted-gradient
# change (gpurun_lib/base) and now, aligned and shifted gradients, interleaved.
for rep in 1 2 3; do
  MCO_LIB_PATH=gpurun_lib/base/libmco.so python tools/bench_configs.py phases 2>&1 | grep -v "list form" | sed 's/^/base /'
  python tools/bench_configs.py phases 2>&1 | grep -v "list form" | sed 's/^/new  /'
done
