# GPU call: K4 / K6 fp32 rows-in-flight / register-cap A/B (libs in gpurun_lib/<v>)
for rep in 1 2; do
  for v in base k6r4m2 k4r8m2 both; do
    if [ $v = base ]; then L=paper_2312_00407_b200/_build/libmco.so; else L=gpurun_lib/$v/libmco.so; fi
    MCO_LIB_PATH=$L python tools/bench_configs.py hooks c3 2>&1 | grep config | grep -v "hook-form lomo" | sed "s/^/$v /"
  done
done
