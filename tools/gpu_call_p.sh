# GPU call: register-cap A/B of the bf16 AdaLomo tile kernels (libs in gpurun_lib/<v>).
for rep in 1 2; do
  for v in base k4m4 k1m4 k6m3 k4m2; do
    if [ $v = base ]; then L=paper_2312_00407_b200/_build/libmco.so; else L=gpurun_lib/$v/libmco.so; fi
    MCO_LIB_PATH=$L python tools/bench_configs.py bf16 2>&1 | grep config | sed "s/^/$v /"
  done
done
