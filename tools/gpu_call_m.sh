# GPU call: same-box A/B of the list form (gpurun_lib/base = previous commit) on aligned
# and shifted tensor lists, interleaved.
for rep in 1 2 3; do
  MCO_LIB_PATH=gpurun_lib/base/libmco.so python tools/bench_configs.py phases 2>&1 | grep "list form" | sed 's/^/base /'
  python tools/bench_configs.py phases 2>&1 | grep "list form" | sed 's/^/new  /'
done
