# GPU call: same-box A/B of this tree's library against gpurun_lib/base on the AdaLomo
# forms, plus the AdaLomo tests on this tree.
for rep in 1 2; do
  for v in base new; do
    if [ $v = base ]; then L=gpurun_lib/base/libmco.so; else L=paper_2312_00407_b200/_build/libmco.so; fi
    MCO_LIB_PATH=$L timeout 600 python tools/bench_configs.py hooks c3 bf16 2>&1 | grep config | grep -v "hook-form lomo" | sed "s/^/$v /"
  done
done
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_gpu_fused.py tests/test_gpu_fused_backward.py tests/test_gpu_configs_parity.py -m gpu 2>&1 | tail -1
