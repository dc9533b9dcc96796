# GPU call: A/B of KR / K3 triggering their dependents early (gpurun_lib/early).
for rep in 1 2; do
  for v in base early; do
    if [ $v = base ]; then L=paper_2312_00407_b200/_build/libmco.so; else L=gpurun_lib/$v/libmco.so; fi
    MCO_LIB_PATH=$L python tools/bench_configs.py hooks c3 2>&1 | grep config | grep -v "hook-form lomo" | sed "s/^/$v /"
  done
done
