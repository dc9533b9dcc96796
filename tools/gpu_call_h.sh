# GPU call: A/B of AdaLomo kernel variants (libs built with -D knobs into gpurun_lib/<v>)
set -x
for rep in 1 2; do
for v in B A C D; do
  if [ $v = B ]; then L=paper_2312_00407_b200/_build/libmco.so; else L=gpurun_lib/$v/libmco.so; fi
  MCO_LIB_PATH=$L timeout 600 python tools/bench_configs.py bf16 hooks > gpurun_out/ab_${v}_$rep.jsonl 2>&1
done
done
