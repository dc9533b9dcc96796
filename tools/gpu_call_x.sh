# GPU call: K4 rows-in-flight / register-cap A/B on bf16 AdaLomo (libs in gpurun_lib/<v>)
for rep in 1 2; do
  for v in base k4r16m2 k4r16m3 k4r12m2; do
    if [ $v = base ]; then L=paper_2312_00407_b200/_build/libmco.so; else L=gpurun_lib/$v/libmco.so; fi
    MCO_LIB_PATH=$L python tools/bench_configs.py bf16 2>&1 | grep config | sed "s/^/$v /"
  done
done
MCO_LIB_PATH=paper_2312_00407_b200/_build/libmco.so python -m pytest -q -p no:cacheprovider tests/test_gpu_fused.py -m gpu -k "bf16" 2>&1 | tail -1
