# GPU call: K1 rows-in-flight / register-cap A/B on bf16 AdaLomo (libs in gpurun_lib/<v>)
for rep in 1 2; do
  for v in base rb8m3 rb8m2 rb2m4; do
    if [ $v = base ]; then L=paper_2312_00407_b200/_build/libmco.so; else L=gpurun_lib/$v/libmco.so; fi
    MCO_LIB_PATH=$L python tools/bench_configs.py bf16 2>&1 | grep config | sed "s/^/$v /"
  done
done
